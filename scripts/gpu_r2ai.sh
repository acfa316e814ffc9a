#!/bin/bash
# dataflow counters at batch 16 (INT4 / INT8 ResNet-18): on vs off
O=gpurun_out/r2ai; mkdir -p $O
for i in 1 2; do for df in on off; do
  timeout 600 python bench.py --workload resnet18_int4_b16 --dataflow $df --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_i4_${df}_$i.json 2> $O/bench_i4_${df}_$i.err
  timeout 600 python bench.py --workload resnet18_int8_b1 --batch 16 --dataflow $df --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_i8_${df}_$i.json 2> $O/bench_i8_${df}_$i.err
done; done
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'])"; done
