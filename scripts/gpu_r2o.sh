#!/bin/bash
# e2e with two copy streams; probe modes (instrumented build) for the stem, l1 3x3, l3 c3
O=gpurun_out/r2o; mkdir -p $O
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-k7 --layers-out $O/layers_r50.json > $O/bench_r50.json 2> $O/bench_r50.err
python -c "import json; d=json.loads(open('$O/bench_r50.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
PROBE_CFG=bm256_bn64_kc64x1_c2_st_h_w_m2,bm256_bn64_kc64x1_c2_st_h_w,bm128_bn64_kc64x1_c1_st_h_w_m2 timeout 600 python scripts/probe.py stem l1.b0.c2 > $O/probe_a.txt 2>&1
PROBE_CFG=bm128_bn128_kc128x2_c1_w,bm128_bn256_kc128x2_c1_w,bm256_bn128_kc128x2_c2 timeout 600 python scripts/probe.py l3.b1.c3 > $O/probe_b.txt 2>&1
cat $O/probe_a.txt $O/probe_b.txt
