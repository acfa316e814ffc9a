#!/bin/bash
# round 2: NEXT-3 ablation table, bench with the conv-chain window, source-level ncu of the epilogue-bound 1x1
O=gpurun_out/r2b; mkdir -p $O
timeout 1200 python scripts/ablation.py --out $O/r02_ablation.json > $O/ablation.md 2> $O/ablation.err
CONV_Q_CACHE=gpurun_out/r2a/cache_r50.json timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-tune > $O/bench_r50.json 2> $O/bench_r50.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_igemm -s 2 -c 1 -o $O/l3c3 \
    python scripts/prof_layer.py --layer l3.b1.c3 --config bm128_bn128_kc128x2_c1_w > $O/l3c3.log 2>&1
ncu -i $O/l3c3.ncu-rep --page source --csv > $O/l3c3_src.csv 2>/dev/null
ncu -i $O/l3c3.ncu-rep --page raw --csv > $O/l3c3_raw.csv 2>/dev/null
rm -f $O/l3c3.ncu-rep
