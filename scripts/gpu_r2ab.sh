#!/bin/bash
# small per-rank batches: exhaustive TileConfig tuning vs the learned search over the enlarged space
O=gpurun_out/r2ab; mkdir -p $O
for b in 32 64; do for i in 1 2; do
  timeout 900 python bench.py --batch $b --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e > $O/bench_b${b}_ex$i.json 2> $O/bench_b${b}_ex$i.err
  timeout 1200 python bench.py --batch $b --search 128 --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_b${b}_se$i.json > $O/bench_b${b}_se$i.json 2> $O/bench_b${b}_se$i.err
done; done
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['parity_ok'], d.get('graph_layers_sum_ms'), d.get('tuning'))"; done
