#!/bin/bash
# round 2: unsigned-format parity + the full GPU suite, unsigned bench lines
O=gpurun_out/r2c; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_unsigned.py -q -x -rf > $O/gpu_unsigned.log 2>&1; echo "rc=$?" >> $O/gpu_unsigned.log
timeout 1800 python -m pytest tests -m gpu -q -rf > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
for w in resnet50_int8_b256_uns resnet18_int4_b16_uns resnet18_int4_b16 resnet50_int8_b256_res_uns; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/gpu_unsigned.log; tail -3 $O/gputest.log
