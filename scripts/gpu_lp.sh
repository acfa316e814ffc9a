timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
export PROBE_CFG=bm128_bn64_kc64x2_c1_w,bm128_bn64_kc64x1_c1_w,bm128_bn64_kc64x4_c1,bm256_bn64_kc64x4_c2,bm128_bn256_kc64x2_c1_w,bm128_bn128_kc128x1_c1_st,bm128_bn256_kc128x1_c1,bm256_bn256_kc128x2_c2_st
export PROBE_MODES=0,7
timeout 600 python scripts/probe.py stem l1.b0.c1 l1.b0.c3 l2.b0.c2 l3.b1.c2 l4.b0.c3
