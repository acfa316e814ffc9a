// kern_b4_o4.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=4, output path OUT_TMA | OUT_RELU (smem staging + TMA store): the INT4 ReLU
// epilogue (F2I.U8 conversion, runtime top code 7 / 15 for signed / unsigned
// codes, DESIGN reading 16).  Separate translation unit only to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_4_4(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<4, 4>(p, scale, y);
}
}  // namespace convq
