export NVCC_APPEND_FLAGS="-DCONVQ_HANG_CHECK"
python paper_2202_06819_b200/_build.py > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
unset NVCC_APPEND_FLAGS
python paper_2202_06819_b200/_build.py > /dev/null 2>&1
timeout 300 python scripts/trace.py l1.b0.c2 bm128_bn64_kc64x3_c1_st_h bm128_bn64_kc64x1_c1_st_h bm256_bn64_kc64x3_c2_st_h bm256_bn64_kc64x1_c2_st_h 2>&1
timeout 300 python scripts/trace.py l2.b1.c2 bm128_bn128_kc128x3_c1_st_h bm128_bn128_kc128x1_c1_st_h bm256_bn128_kc128x3_c2_st_h bm256_bn128_kc128x1_c2_st_h bm128_bn128_kc128x2_c1_st 2>&1
