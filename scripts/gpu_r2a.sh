#!/bin/bash
# round-2 evidence pass: full GPU suite, default bench (as the driver runs it), INT4/b1/residual benches, ncu launch list
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $O/gputest.log 2>&1; echo "pytest=$?" >> $O/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?" >> $O/smoke.log
CONV_Q_CACHE=$O/cache_r50.json timeout 900 python bench.py --steps 20 --warmup 5 --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err; echo bench=$? >> $O/bench_r50.err
for w in resnet18_int4_b16 resnet18_int8_b1 resnet50_int8_b256_res; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 600 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
CONV_Q_CACHE=$O/cache_r50.json timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
   --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-tune --no-graph --no-e2e --no-parity --no-cpu-baseline --no-k7 > $O/ncu_bench.log 2>&1
tail -3 $O/gputest.log
