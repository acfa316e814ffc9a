#!/bin/bash
# session-3 final evidence after the INT4 epilogue change: ablation (INT4/INT8 column), benches
O=gpurun_out/r2w; mkdir -p $O
timeout 2400 python scripts/ablation.py --out $O/r02s3_ablation.json > $O/r02s3_ablation.md 2> $O/ablation.err
for w in resnet18_int4_b16 resnet18_int4_b16_uns; do
  CONV_Q_CACHE=$O/cache_$w.json timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_$w.json > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --steps 20 --warmup 5 --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
cat $O/r02s3_ablation.md | tail -12
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity_ok'], d['e2e'])"; done
