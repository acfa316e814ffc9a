// kern_b8_o20.cu -- instantiates the implicit-GEMM conv kernels for
// BITS=8, output path OUT_TMA | OUT_RELU | OUT_U (smem staging + TMA store): the ReLU epilogue
// writing unsigned u8 codes (DESIGN reading 16).  Separate translation unit only
// to compile in parallel.
#include "plan.cuh"

namespace convq {
int dispatch_conv_8_20(conv_q_plan_s *p, const float *scale, void *y) {
    return dispatch_bn_kch<8, 20>(p, scale, y);
}
}  // namespace convq
