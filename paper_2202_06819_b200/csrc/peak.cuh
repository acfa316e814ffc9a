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
// Measurement only: single-thread cost of the MMA warp's primitives, in SM
// cycles per iteration (clock64), one CTA.  mode:
//   0  mbarrier.try_wait on an already-completed phase (result consumed)
//   1  mbarrier.test_wait on an already-completed phase
//   2  tcgen05.mma M=128 N=n K=32, back to back (no commit)
//   3  tcgen05.mma + tcgen05.commit (arrive on a barrier nobody waits for)
//   4  tcgen05.commit alone
//   5  G=4 x tcgen05.mma + commit + try_wait(completed barrier), as one stage
//   6  like 5, but the try_wait of the *next* stage is issued before the MMAs
template <int mode>
__global__ void __launch_bounds__(128, 1) micro_probe_kernel(int iters, int n, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *a = smem, *b = smem + 128 * 128;
    uint64_t *bars = reinterpret_cast<uint64_t *>(b + 256 * 128);
    uint32_t *holder = reinterpret_cast<uint32_t *>(bars + 4);
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
        mbar_arrive(&bars[0]);   // phase 0 of bars[0] complete
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<256>(holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    long long t = 0;
    if (warp == 1) {
        const uint32_t idesc = idesc_i8(128, n);
        const uint64_t ad = umma_desc_kmajor(smem_u32(a), 128), bd = umma_desc_kmajor(smem_u32(b), 128);
        uint32_t acc = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if constexpr (mode == 7) {
                acc += (uint32_t)it * 3u;
            } else if constexpr (mode == 8) {
                if (elect_one()) acc += 1u;
                __syncwarp();
            } else if constexpr (mode == 9) {
                asm volatile("" ::: "memory");
                acc += 1u;
            } else if constexpr (mode == 0) {
                acc += mbar_try_wait(&bars[0], 0) ? 1u : 0u;
            } else if constexpr (mode == 1) {
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bars[0])), "r"(0u) : "memory");
                acc += ok;
            } else if constexpr (mode == 2) {
                if (elect_one()) mma_i8(tmem, ad, bd, idesc, it != 0);
                __syncwarp();
            } else if constexpr (mode == 3) {
                if (elect_one()) { mma_i8(tmem, ad, bd, idesc, it != 0); mma_commit(&bars[1]); }
                __syncwarp();
            } else if constexpr (mode == 4) {
                if (elect_one()) mma_commit(&bars[1]);
                __syncwarp();
            } else if constexpr (mode == 5) {
                mbar_wait(&bars[0], 0);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
                    mma_commit(&bars[1]);
                }
                __syncwarp();
            } else {
                const bool ready = mbar_try_wait(&bars[0], 0);
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
                    mma_commit(&bars[1]);
                }
                __syncwarp();
                if (!ready) mbar_wait(&bars[0], 0);
            }
        }
        t = clock64() - t0;
        if (threadIdx.x == 32) out[0] = t + (acc == 12345 ? 1 : 0);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

}  // namespace convq
