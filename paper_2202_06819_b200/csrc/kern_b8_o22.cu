// kern_b8_o22.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_DIRECT | OUT_RELU | OUT_U (direct stores): the ReLU epilogue
// writing unsigned u8 codes (DESIGN reading 16).  Separate translation unit only
// to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_22(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 22>(p, scale, y);
}
}  // namespace convq
