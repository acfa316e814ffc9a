#!/bin/bash
# round 2: INT4 weight-stationary / MT2 -- full GPU suite, INT4 bench, ResNet-50 bench
O=gpurun_out/r2i; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf -x > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
for w in resnet18_int4_b16 resnet50_int8_b256; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
tail -3 $O/gputest.log
