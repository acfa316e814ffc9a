timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for a in "l1.b0.c1 bm128_bn64_kc64x1_c1_w_m2" "l2.b0.c3 bm128_bn128_kc128x1_c1_w_m2" "l1.b0.c3 bm128_bn128_kc64x1_c1_w_m2"; do
  for n in 8 256; do timeout 60 python scripts/check_cfg.py $a $n 2>&1 | tail -1; done
done
export PROBE_MODES=0
PROBE_CFG=bm128_bn64_kc64x1_c1_w,bm128_bn64_kc64x1_c1_w_m2,bm128_bn64_kc64x1_c1_st_w_m2 timeout 300 python scripts/probe.py l1.b0.c1
PROBE_CFG=bm128_bn128_kc64x1_c1_w,bm128_bn128_kc64x1_c1_w_m2 timeout 300 python scripts/probe.py l1.b0.c3
PROBE_CFG=bm128_bn128_kc128x1_c1_w,bm128_bn128_kc128x1_c1_w_m2 timeout 300 python scripts/probe.py l2.b0.c3 l2.b1.c1
PROBE_CFG=bm128_bn64_kc128x2_c1_st_w,bm128_bn64_kc128x1_c1_w_m2,bm128_bn64_kc128x2_c1_w timeout 300 python scripts/probe.py l1.b1.c1
