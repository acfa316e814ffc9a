set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err; tail -3 gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json
timeout 300 python bench.py --workload resnet18_int4_b16 --no-cpu-baseline --layers-out gpurun_out/layers_r18_int4.json > gpurun_out/bench_r18i4.json 2> gpurun_out/bench_r18i4.err
timeout 300 python bench.py --workload resnet18_int8_b1 --no-cpu-baseline --layers-out gpurun_out/layers_r18_int8.json > gpurun_out/bench_r18i8.json 2> gpurun_out/bench_r18i8.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50.csv python bench.py --steps 2 --warmup 3 --no-tune --no-e2e --no-stem --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l3c2 python scripts/prof_layer.py --layer l3.b1.c2 > gpurun_out/ncu_l3c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l1c3 python scripts/prof_layer.py --layer l1.b0.c3 > gpurun_out/ncu_l1c3.log 2>&1
ls -la gpurun_out
