export PROBE_CFG=bm128_bn256_kc128x2_c1_w,bm128_bn256_kc128x1_c1,bm256_bn256_kc128x1_c2,bm128_bn128_kc128x1_c1_w
export PROBE_MODES=0,1,2,3,4,7
timeout 600 python scripts/probe.py l3.b1.c3 l3.b1.c1 l4.b0.c3
timeout 300 python scripts/trace.py l3.b1.c3 bm128_bn256_kc128x2_c1_w bm128_bn256_kc128x1_c1 bm256_bn256_kc128x1_c2
