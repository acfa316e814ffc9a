timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "4" 2>&1 | tail -2
export TRACE_NET=resnet18 TRACE_N=16 TRACE_BITS=4
timeout 200 python scripts/trace.py l1.b0.c1 bm128_bn64_kc64x1_c1_st bm128_bn64_kc64x4_c1_st 
timeout 200 python scripts/trace.py l3.b1.c2 bm128_bn64_kc128x2_c1_st bm128_bn128_kc128x2_c1_st
