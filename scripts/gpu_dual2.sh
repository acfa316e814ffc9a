export CONV_Q_LIB=$PWD/paper_2202_06819_b200/libconvq_dual.so
CONV_Q_OUT_POLICY=0 timeout 60 python scripts/check_cfg.py l1.b1.c1 bm128_bn64_kc128x2_c1 256 2>&1 | tail -1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python scripts/check_cfg.py l1.b1.c1 bm128_bn64_kc128x2_c1 256 2>&1 | grep -v "^=========     " | head -40
