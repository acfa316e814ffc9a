#!/bin/bash
# the per-rank workload of an 8-GPU strong-scaling run: ResNet-50 INT8 at 32 images (and 64, 128)
O=gpurun_out/r2aa; mkdir -p $O
for b in 32 64 128; do
  timeout 900 python bench.py --batch $b --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_b$b.json > $O/bench_b$b.json 2> $O/bench_b$b.err
  timeout 900 python bench.py --batch $b --dataflow on --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_b${b}_df.json 2> $O/bench_b${b}_df.err
done
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['parity_ok'], d.get('graph_layers_sum_ms'), d['stem'])"; done
