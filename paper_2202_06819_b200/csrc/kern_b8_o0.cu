// kern_b8_o0.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_TMA (packed, TMA store).
// Split into separate translation units only to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_0(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 0>(p, scale, y);
}
}  // namespace convq
