#!/bin/bash
# round 2: residual candidate timings, CTA-0 timelines of the epilogue-bound 1x1 layers
O=gpurun_out/r2e; mkdir -p $O
for l in l1.b0.c3 l3.b1.c3 l2.b1.c3; do timeout 300 python scripts/res_cands.py $l 256 > $O/res_$l.txt 2>&1; done
for lc in "l3.b1.c3 bm128_bn128_kc128x2_c1_w" "l3.b1.c3 bm128_bn256_kc128x2_c1_w" "l3.b1.c3 bm256_bn256_kc128x1_c2_w" "l2.b1.c3 bm128_bn128_kc128x1_c1_w" "l3.b1.c2 bm256_bn256_kc128x2_c2_st"; do
  set -- $lc
  for m in 0 7; do echo "=== $1 $2 probe $m"; CONV_Q_PROBE=$m timeout 120 python scripts/timeline.py $1 $2 256 6 2>&1 | tail -12; done
done > $O/timelines.txt 2>&1
