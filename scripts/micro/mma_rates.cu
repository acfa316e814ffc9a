// tcgen05.mma kind::i8 issue rate with smem-resident operands (measurement only):
// 1-CTA M=128 and CTA-pair (cta_group::2) M=256, N in {64,128,256}, K=32 per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2202_06819_b200/csrc -o mma_rates mma_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace convq;

template <int CG, int N, int KB = 128, int AOFF = 0, int RND = 0>
__global__ void __launch_bounds__(128, 1) kern(int iters, int *sink, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *a = smem;
    uint8_t *b = smem + 128 * KB;
    uint64_t *done = reinterpret_cast<uint64_t *>(b + 256 * KB);
    uint32_t *holder = reinterpret_cast<uint32_t *>(done + 1);
    for (int i = threadIdx.x; i < (128 + 256) * KB / 16; i += blockDim.x)
    {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
        auto nx = [&]() { h ^= h << 13; h ^= h >> 17; h ^= h << 5; return RND ? h : 0x01010101u; };
        uint32_t a0 = nx(), a1 = nx(), a2 = nx(), a3 = nx();
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(a0, a1, a2, a3);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        if constexpr (CG == 2) tmem_alloc_cg2<256>(holder);
        else tmem_alloc<256>(holder);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    long long t0 = clock64();
    if (warp == 1 && rank == 0) {
        const uint32_t idesc = idesc_i8(128 * CG, N);
        const uint64_t ad = umma_desc_kmajor(smem_u32(a), KB) + (AOFF >> 4), bd = umma_desc_kmajor(smem_u32(b), KB);
        if (elect_one()) {
            for (int i = 0; i < iters; ++i) {
                const int k = i & (KB / 32 - 1);
                if constexpr (CG == 2) mma_i8_cg2(tmem, ad + 2 * k, bd + 2 * k, idesc, i != 0);
                else mma_i8(tmem, ad + 2 * k, bd + 2 * k, idesc, i != 0);
            }
            if constexpr (CG == 2) mma_commit_cg2_mc(done, 0x3);
            else mma_commit(done);
        }
        __syncwarp();
    }
    if (warp == 1) mbar_wait(done, 0);
    long long t1 = clock64();
    if (warp == 1 && threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) {
        uint32_t v[32];
        tc_fence_after();
        tmem_ld_32x32b_x32(tmem + ((uint32_t)32 << 16), v);
        if (threadIdx.x == 32 && blockIdx.x == 0) *sink = (int)v[0];
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_cg2<256>(tmem);
        else tmem_dealloc<256>(tmem);
    }
}

template <int CG, int N, int KB = 128, int AOFF = 0, int RND = 0>
void run() {
    int *sink; long long *cyc;
    cudaMalloc(&sink, 4); cudaMalloc(&cyc, 148 * 8);
    const int smem = (128 + 256) * 128 + 8192;
    cudaFuncSetAttribute(kern<CG, N, KB, AOFF, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 20000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, kern<CG, N, KB, AOFF, RND>, iters, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double macs_per_sm = (double)iters * 128 * N * 32;   // per CTA (each CTA of a pair owns 128 rows)
    printf("RND=%d KB=%3d AOFF=%4d CG=%d M=%3d N=%3d: %6.1f cyc/MMA  %7.0f MAC/clk/SM  (%s)\n", RND, KB, AOFF, CG, 128 * CG, N,
           (double)c / iters, macs_per_sm / c, cudaGetErrorString(e));
}
int main() {
    run<1, 64>(); run<1, 128>(); run<1, 256>();
    run<2, 64>(); run<2, 128>(); run<2, 256>();
    run<1, 64, 128, 0, 1>(); run<1, 128, 128, 0, 1>(); run<1, 256, 128, 0, 1>();
    run<2, 64, 128, 0, 1>(); run<2, 128, 128, 0, 1>(); run<2, 256, 128, 0, 1>();
    run<1, 64, 64, 64, 1>(); run<2, 64, 64, 64, 1>();
    return 0;
}
