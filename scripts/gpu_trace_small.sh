set -x
export TRACE_NET=resnet18
TRACE_N=16 TRACE_BITS=4 timeout 200 python scripts/trace.py l1.b0.c1 bm128_bn64_kc64x4_c1_st bm128_bn64_kc64x1_c1
TRACE_N=16 TRACE_BITS=4 timeout 200 python scripts/trace.py l2.b0.ds bm128_bn64_kc64x1_c1_st
TRACE_N=16 TRACE_BITS=8 timeout 200 python scripts/trace.py l1.b0.c1 bm128_bn64_kc64x4_c1_st
TRACE_N=1 TRACE_BITS=8 timeout 200 python scripts/trace.py l4.b1.c2 
