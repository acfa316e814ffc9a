timeout 300 python scripts/trace.py stem 2>&1 | tail -20
timeout 300 python scripts/trace.py l1.b0.c1 2>&1 | tail -20
timeout 300 python scripts/trace.py l1.b0.c3 bm128_bn256_kc64x2_c1_w bm128_bn256_kc64x1_c1 bm128_bn128_kc64x1_c1 bm128_bn64_kc64x1_c1 2>&1 | tail -20
timeout 300 python scripts/trace.py l4.b0.c3 2>&1 | tail -30
