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
    if (warp == 1) {
        const uint32_t idesc = idesc_i8(PM, PN);
        const uint64_t ad = umma_desc_kmajor(smem_u32(a), KB), bd = umma_desc_kmajor(smem_u32(b), KB);
        if (elect_one()) {
            for (int i = 0; i < iters; ++i) {
                const int k = i & 3;
                mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, i != 0);
            }
            mma_commit(done);
        }
        __syncwarp();
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

namespace convq {
// Pipeline probe (measurement only): groups of G MMAs (M=128, N=n, K=32,
// SW128 K-major operands in smem) committed to a ring of S mbarriers; before
// issuing group g the thread waits for the commit of group g-(S-1), i.e. at
// most S-1 groups are in flight -- the handshake pattern of the conv
// mainloop without any TMA traffic.  S = 1 means no waits at all.
__global__ void __launch_bounds__(128, 1) mma_pipe_probe_kernel(int groups, int G, int S, int n, int *sink) {
    constexpr int PM = 128, PN = 256, KB = 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *a = smem;
    uint8_t *b = smem + PM * KB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(b + PN * KB);   // 16 barriers
    uint32_t *holder = reinterpret_cast<uint32_t *>(bars + 16);
    for (int i = threadIdx.x; i < (PM + PN) * KB / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<256>(holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    if (warp == 1) {   // whole warp converged; elected lane issues
        const uint32_t idesc = idesc_i8(PM, n);
        const uint64_t ad = umma_desc_kmajor(smem_u32(a), KB), bd = umma_desc_kmajor(smem_u32(b), KB);
        for (int g = 0; g < groups; ++g) {
            if (S > 1 && g >= S - 1) {
                const int w = g - (S - 1);
                mbar_wait(&bars[w % S], (w / S) & 1);
                tc_fence_after();
            }
            if (elect_one()) {
                for (int i = 0; i < G; ++i) {
                    const int k = i & 3;
                    mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, (g | i) != 0);
                }
                mma_commit(&bars[g % (S > 1 ? S : 16)]);
            }
            __syncwarp();
        }
        // drain
        const int last = groups - 1;
        const int ring = S > 1 ? S : 16;
        mbar_wait(&bars[last % ring], (last / ring) & 1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
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

namespace convq {
// CTA-pair variant of the pipeline probe: the leader of each cluster of 2
// issues tcgen05.mma.cta_group::2 (M=256, N=n) groups and multicasts each
// commit to both CTAs' barrier ring; waits as in mma_pipe_probe_kernel.
__global__ void __launch_bounds__(128, 1) mma_pipe_probe2_kernel(int groups, int G, int S, int n, int *sink) {
    constexpr int PM = 128, PN = 256, KB = 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *a = smem;
    uint8_t *b = smem + PM * KB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(b + PN * KB);
    uint32_t *holder = reinterpret_cast<uint32_t *>(bars + 16);
    for (int i = threadIdx.x; i < (PM + PN) * KB / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (warp == 0) tmem_alloc_cg2<256>(holder);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *holder;
    const int ring = S > 1 ? S : 16;
    if (warp == 1 && rank == 0) {
        const uint32_t idesc = idesc_i8(2 * PM, n);
        const uint64_t ad = umma_desc_kmajor(smem_u32(a), KB), bd = umma_desc_kmajor(smem_u32(b), KB);
        for (int g = 0; g < groups; ++g) {
            if (S > 1 && g >= S - 1) {
                const int w = g - (S - 1);
                mbar_wait(&bars[w % S], (w / S) & 1);
                tc_fence_after();
            }
            if (elect_one()) {
                for (int i = 0; i < G; ++i) {
                    const int k = i & 3;
                    mma_i8_cg2(tmem, ad + 2 * k, bd + 2 * k, idesc, (g | i) != 0);
                }
                mma_commit_cg2_mc(&bars[g % ring], 0x3);
            }
            __syncwarp();
        }
    }
    if (warp == 1) {   // both CTAs: wait for the last group's commit
        const int last = groups - 1;
        mbar_wait(&bars[last % ring], (last / ring) & 1);
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1 && rank == 0 && blockIdx.x == 0) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + ((uint32_t)32 << 16), v);
        if (threadIdx.x == 32) *sink = (int)v[0];
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_cg2<256>(tmem);
    }
}
}  // namespace convq
