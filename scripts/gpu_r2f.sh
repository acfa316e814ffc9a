#!/bin/bash
# round-2 session: GPU tests, A/B of the all-warps epilogue, INT4 bench, ncu launch list
O=gpurun_out/r2f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -k "not sanitizer" -x > $O/gputest.log 2>&1
for lib in libconvq.so libconvq_allw0.so; do
  CONV_Q_LIB=paper_2202_06819_b200/$lib CONV_Q_CACHE=$O/cache_$lib.json timeout 600 python bench.py --steps 200 --warmup 10 \
    --no-cpu-baseline --no-parity --no-k7 --layers-out $O/layers_$lib.json > $O/bench_$lib.json 2> $O/bench_$lib.err
done
timeout 600 python bench.py --workload resnet18_int4_b16 --steps 200 --warmup 10 --no-cpu-baseline --no-k7 \
   --layers-out $O/layers_int4.json > $O/bench_int4.json 2> $O/bench_int4.err
CONV_Q_CACHE=$O/cache_libconvq.so.json timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active \
   --clock-control none -k regex:"conv_igemm|quantize|maxpool" -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-tune --no-graph --no-e2e --no-parity --no-cpu-baseline --no-k7 > $O/ncu_bench.log 2>&1
tail -3 $O/gputest.log
