// kern_b8_o6.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_DIRECT (packed, direct stores) with the
// ReLU-specialised epilogue (OUT_RELU).  Separate translation unit only to
// compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_6(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 6>(p, scale, y);
}
}  // namespace convq
