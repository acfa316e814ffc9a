#!/bin/bash
# CTA-0 timelines (instrumented build): l3.b1.c3 bn256 WS and the stem MT2 pair, probe 0 / 7
O=gpurun_out/r2p; mkdir -p $O
for pr in 0 7; do
  CONV_Q_PROBE=$pr timeout 300 python scripts/timeline.py l3.b1.c3 bm128_bn256_kc128x2_c1_w 256 12 > $O/tl_l3c3_p$pr.txt 2>&1
  CONV_Q_PROBE=$pr timeout 300 python scripts/timeline.py l3.b1.c3 bm128_bn128_kc128x2_c1_w 256 12 > $O/tl_l3c3bn128_p$pr.txt 2>&1
  CONV_Q_PROBE=$pr timeout 300 python scripts/timeline.py stem bm128_bn64_kc64x1_c1_st_h_w_m2 256 12 > $O/tl_stem_p$pr.txt 2>&1
done
tail -n 30 $O/*.txt
