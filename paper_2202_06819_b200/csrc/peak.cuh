// peak.cuh -- K7: dense INT8 tensor-core rate microbenchmark (measurement only).
// Each CTA keeps one M=128 x N=256 x K=32 tcgen05.mma kind::i8 stream busy on
// operands resident in shared memory (no HBM traffic); the achieved ops/s is
// the measured roofline denominator for the conv kernel.
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace convq {

__global__ void __launch_bounds__(128, 1) int8_peak_kernel(int iters, int *sink) {
    constexpr int PM = 128, PN = 256, KB = 128;  // A 128x128 B, B 256x128 B, SW128 K-major
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *a = smem;
    uint8_t *b = smem + PM * KB;
    uint64_t *done = reinterpret_cast<uint64_t *>(b + PN * KB);
    uint32_t *holder = reinterpret_cast<uint32_t *>(done + 1);
    for (int i = threadIdx.x; i < (PM + PN) * KB / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<256>(holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    if (threadIdx.x == 32) {
        const uint32_t idesc = idesc_i8(PM, PN);
        const uint32_t aa = smem_u32(a), ba = smem_u32(b);
        for (int i = 0; i < iters; ++i) {
            const int k = i & 3;
            mma_i8(tmem, umma_desc_kmajor(aa + 32 * k, KB), umma_desc_kmajor(ba + 32 * k, KB), idesc, i != 0);
        }
        mma_commit(done);
        mbar_wait(done, 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {  // read one accumulator so the work is observable
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)32 << 16), v);
        if (threadIdx.x == 32 && blockIdx.x == 0) *sink = (int)v[0];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

}  // namespace convq
