// kern_b8_o8.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_TMA | OUT_RES: the fused residual-add epilogue
// (DESIGN reading 15).  Separate translation unit only to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_8(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 8>(p, scale, y);
}
}  // namespace convq
