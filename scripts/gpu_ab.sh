# A/B: 4 vs 6 INT8 epilogue warpgroups (BN <= 128), probe.py normal mode, then parity of the wg6 build
export PROBE_CFG=bm128_bn64_kc64x2_c1_w,bm128_bn64_kc64x1_c1_w,bm128_bn64_kc64x1_c1,bm128_bn128_kc64x1_c1_w,bm128_bn128_kc64x2_c1_w,bm128_bn256_kc64x2_c1_w,bm128_bn128_kc128x1_c1_st,bm128_bn128_kc128x1_c1,bm128_bn128_kc128x1_c1_w,bm256_bn128_kc128x2_c2_st,bm256_bn128_kc128x3_c2_st_h,bm256_bn64_kc64x1_c2_st_h_w,bm128_bn128_kc128x2_c1_st,bm128_bn64_kc128x2_c1,bm256_bn128_kc128x2_c2
export PROBE_MODES=0
for lib in libconvq.so libconvq_wg6.so; do echo "== $lib"; CONV_Q_LIB=$PWD/paper_2202_06819_b200/$lib timeout 600 python scripts/probe.py stem l1.b0.c1 l1.b0.c2 l1.b0.c3 l1.b1.c1 l2.b0.c1 l2.b0.c3 l2.b1.c1 l2.b1.c2 l2.b0.c2 l4.b1.c1; done
CONV_Q_LIB=$PWD/paper_2202_06819_b200/libconvq_wg6.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
