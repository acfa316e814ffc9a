// kern_b8_o2.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_DIRECT (packed, direct stores).
// Split into separate translation units only to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_2(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 2>(p, scale, y);
}
}  // namespace convq
