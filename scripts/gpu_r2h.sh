#!/bin/bash
# round 2: cross-launch row flags -- dataflow parity, benches with / without
O=gpurun_out/r2h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dataflow.py -q -x -rf > $O/dataflow_tests.log 2>&1; echo "rc=$?" >> $O/dataflow_tests.log
for w in resnet18_int8_b1 resnet18_int4_b16 resnet50_int8_b256; do
  for df in "--dataflow=on" "--dataflow=off"; do
    CONV_Q_CACHE=$O/cache_$w.json timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e $df --layers-out $O/layers_$w$df.json > $O/bench_$w$df.json 2> $O/bench_$w$df.err
  done
done
tail -3 $O/dataflow_tests.log
