# quick iteration: parity + bench + ncu captures
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --no-cpu-baseline --layers-out gpurun_out/layers_r50_int8.json > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
cat gpurun_out/bench_r50.json; cat gpurun_out/bench_r50.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l1c3 python scripts/prof_layer.py --layer l1.b0.c3 > gpurun_out/ncu_l1c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o gpurun_out/prof_l2c2 python scripts/prof_layer.py --layer l2.b1.c2 > gpurun_out/ncu_l2c2.log 2>&1
