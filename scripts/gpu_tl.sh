for lc in "l1.b0.c1 bm128_bn64_kc64x1_c1_w" "l1.b0.c2 bm128_bn64_kc64x1_c1_st_h_w" "l3.b1.c3 bm128_bn256_kc128x2_c1_w" "l1.b0.c3 bm128_bn128_kc64x1_c1_w" "stem bm128_bn64_kc64x1_c1_st_h_w"; do
  set -- $lc
  for m in 0 7; do echo "=== $1 $2 probe $m"; CONV_Q_PROBE=$m timeout 120 python scripts/timeline.py $1 $2 256 10 2>&1 | tail -30; done
done
