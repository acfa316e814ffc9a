for n in 16 32 64 128 256; do timeout 60 python scripts/check_cfg.py l1.b1.c1 bm128_bn64_kc128x2_c1 $n 2>&1 | tail -1; done
for n in 32 128; do timeout 60 python scripts/check_cfg.py l2.b0.c3 bm128_bn128_kc128x1_c1 $n 2>&1 | tail -1; done
for n in 64 256; do timeout 60 python scripts/check_cfg.py l1.b0.c1 bm128_bn64_kc64x1_c1 $n 2>&1 | tail -1; done
