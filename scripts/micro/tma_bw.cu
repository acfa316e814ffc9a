// TMA load throughput per SM vs bytes in flight (measurement only).
// One producer lane issues 2-D tiled TMA loads (128-byte rows, SWIZZLE_128B,
// box = ROWS x 128 B) of an L2-resident matrix into an S-stage ring; one
// consumer lane waits on each stage's full barrier and frees it at once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu -lcuda && ./tma_bw
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                 ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap tm, int rows, int stages, int iters,
                                              int total_rows, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *buf = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(buf + stages * rows * 128);
    uint64_t *empty = full + 16;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_tx(&full[s], rows * 128);
            const int r0 = ((blockIdx.x * 977 + i * 131) * rows) % (total_rows - rows);
            tma2d(buf + s * rows * 128, &tm, &full[s], 0, r0);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r));
    return d;
}
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// CTA pair: both CTAs load their own tile, the bytes of both count on the leader's barrier
// (cp.async.bulk.tensor.cta_group::2); the leader's consumer frees the stage in both CTAs.
__global__ void __launch_bounds__(64, 1) kern_pair(const __grid_constant__ CUtensorMap tm, int rows, int stages,
                                                   int iters, int total_rows, long long *cyc, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *buf = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(buf + stages * rows * 128);
    uint64_t *empty = full + 16;
    uint64_t *ready = full + 32;
    const uint32_t rank = ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); mbar_init(&ready[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const long long t0 = clock64();
    // mode 0: cta_group::2 loads, bytes of both CTAs on the leader's barrier, leader frees both
    // mode 1: cta_group::2 loads on the CTA's own barrier, each CTA consumes its own
    // mode 2: plain loads on the own barrier inside the cluster, each CTA consumes its own
    if (threadIdx.x == 0) {
        int s = 0; uint32_t ph = 0;
        const uint32_t full0 = mode == 0 ? mapa(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            if (mode != 0) mbar_arrive_tx(&full[s], rows * 128);
            else if (rank == 0) mbar_arrive_tx(&full[s], 2 * rows * 128);
            const int r0 = ((blockIdx.x * 977 + i * 131) * rows) % (total_rows - rows);
            if (mode >= 2)
                tma2d(buf + s * rows * 128, &tm, &full[s], 0, r0);
            else
                asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(smem_u32(buf + s * rows * 128)), "l"(&tm), "r"(full0 + 8u * s), "r"(0), "r"(r0) : "memory");
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32 && mode == 3) {
        // relay design: follower relays its filled stage to the leader's ready barrier;
        // the leader waits both, then frees the stage in both CTAs
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[s], ph);
            if (rank == 1) {
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&ready[s]), 0)) : "memory");
            } else {
                mbar_wait(&ready[s], ph);
                mbar_arrive(&empty[s]);
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&empty[s]), 1)) : "memory");
            }
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32 && (rank == 0 || mode != 0)) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (mode == 0)
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(&empty[s]), 1)) : "memory");
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    const int total_rows = 1 << 19;  // 64 MB of 128-byte rows (L2-resident after the first pass)
    void *mat;
    cudaMalloc(&mat, (size_t)total_rows * 128);
    cudaMemset(mat, 1, (size_t)total_rows * 128);
    long long *cyc;
    cudaMalloc(&cyc, 148 * 8);
    typedef CUresult (*enc_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                              const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    enc_t enc = (enc_t)fn;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    cudaFuncSetAttribute(kern_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    for (int rows : {64, 128, 256}) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, (cuuint64_t)total_rows};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {128, (cuuint32_t)rows};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, mat, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int stages : {1, 2, 4, 6, 8, 12, 16}) {
            const int bytes = stages * rows * 128;
            if (bytes + 4096 > 232448) continue;
            const int iters = 4000 * 128 / rows;
            for (int rep = 0; rep < 2; ++rep) kern<<<148, 64, bytes + 4096>>>(tm, rows, stages, iters, total_rows, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c[148];
            cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
            const double bpc = (double)iters * rows * 128 / mx;
            {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(148); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = bytes + 4096;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                for (int mode = 0; mode < 4; ++mode) {
                for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, kern_pair, tm, rows, stages, iters, total_rows, cyc, mode);
                cudaError_t e2 = cudaDeviceSynchronize();
                long long c2[148];
                cudaMemcpy(c2, cyc, sizeof c2, cudaMemcpyDeviceToHost);
                long long mx2 = 0;
                for (int i = 0; i < 148; ++i) mx2 = c2[i] > mx2 ? c2[i] : mx2;
                printf("PAIR mode%d rows=%3d stages=%2d  %6.1f B/clk/SM (%s)\n", mode, rows, stages, (double)iters * rows * 128 / mx2, cudaGetErrorString(e2));
                }
            }
            printf("rows=%3d stages=%2d inflight=%6d B  %6.1f B/clk/SM  chip %.1f TB/s @%d MHz  (%s)\n", rows, stages,
                   bytes, bpc, bpc * 148 * clk_khz * 1e3 / 1e12, clk_khz / 1000, cudaGetErrorString(e));
        }
    }
    return 0;
}
