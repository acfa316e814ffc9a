#!/bin/bash
# graph-timed per-layer tables; INT8 vs INT4 ResNet-18 at b16
O=gpurun_out/r2n; mkdir -p $O
CONV_Q_CACHE=$O/cache_r50.json timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
for w in "resnet18_int4_b16" "resnet18_int8_b1 --batch 16" "resnet18_int8_b1" "resnet50_int8_b256_res"; do
  t=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-k7 --no-e2e --layers-out $O/layers_$t.json > $O/bench_$t.json 2> $O/bench_$t.err
done
for f in $O/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d.get('graph_layers_sum_ms'), d['roofline']['kernel_ms_per_step'], d.get('graph_step_roofline_frac'))"; done
