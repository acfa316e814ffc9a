// kern_b4_o1.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=4, output path OUT_S32 (raw accumulators).
// Split into separate translation units only to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_4_1(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<4, 1>(p, scale, y);
}
}  // namespace convq
