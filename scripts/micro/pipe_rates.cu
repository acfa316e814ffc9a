// Issue rates of the epilogue's instruction classes and TMEM read bandwidth (measurement only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu && ./pipe_rates
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// OP: 0 I2FP, 1 F2I.rni.s32, 2 F2I.rni.sat.s8, 3 FFMA, 4 FMNMX, 5 IADD, 6 PRMT, 7 I2IP(s8 pack), 8 FADD,
//     9 IMNMX, 10 F2I.rni.sat.u8
template <int OP>
__global__ void __launch_bounds__(1024, 1) ops(int iters, uint32_t *out, long long *cyc) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 7919u + i * 104729u;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            uint32_t x = r[i], d;
            if (OP == 0) asm volatile("cvt.rn.f32.s32 %0, %1;" : "=r"(d) : "r"(x));
            if (OP == 1) asm volatile("cvt.rni.s32.f32 %0, %1;" : "=r"(d) : "r"(x));
            if (OP == 2) asm volatile("cvt.rni.sat.s8.f32 %0, %1;" : "=r"(d) : "r"(x));
            if (OP == 3) asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]), "r"(r[(i + 2) & 15]));
            if (OP == 4) asm volatile("max.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]));
            if (OP == 5) asm volatile("add.s32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]));
            if (OP == 6) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]));
            if (OP == 7) asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]), "r"(r[(i + 2) & 15]));
            if (OP == 8) asm volatile("add.rn.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]));
            if (OP == 9) asm volatile("max.s32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(r[(i + 1) & 15]));
            if (OP == 10) asm volatile("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(d) : "r"(x));
            r[i] = d;
        }
    }
    const long long t1 = clock64();
    uint32_t a = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) a ^= r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// TMEM read: W warps, each loads its lane quadrant with 32x32b.xX (+ wait::ld)
template <int X>
__device__ __forceinline__ void tld(uint32_t a, uint32_t *v) {
    if constexpr (X == 16)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(a));
    if constexpr (X == 32)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                       "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                       "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                     : "r"(a));
}
template <int X, int PIPE>
__global__ void __launch_bounds__(512, 1) tmem_bw(int iters, uint32_t *out, long long *cyc) {
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = holder;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 3) * 128;
    uint32_t acc = 0;
    const long long t0 = clock64();
    if constexpr (PIPE) {
        uint32_t va[X], vb[X];
        tld<X>(base, va);
        for (int it = 0; it < iters; it += 2) {
            tld<X>(base + ((it + 1) & 3) * X % 128, vb);
#pragma unroll
            for (int i = 0; i < X; ++i) acc += va[i];
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tld<X>(base + ((it + 2) & 3) * X % 128, va);
#pragma unroll
            for (int i = 0; i < X; ++i) acc += vb[i];
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
    } else {
        for (int it = 0; it < iters; ++it) {
            uint32_t v[X];
            tld<X>(base + (it & 3) * X % 128, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < X; ++i) acc += v[i];
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const char *names[] = {"I2FP.s32", "F2I.rni.s32", "F2I.rni.sat.s8", "FFMA", "FMNMX", "IADD", "PRMT", "I2IP.s8",
                           "FADD", "IMNMX", "F2I.rni.sat.u8"};
    void (*kk[])(int, uint32_t *, long long *) = {ops<0>, ops<1>, ops<2>, ops<3>, ops<4>, ops<5>, ops<6>, ops<7>,
                                                  ops<8>, ops<9>, ops<10>};
    const int iters = 4096;
    for (int o = 0; o < 11; ++o) {
        for (int warps : {16, 32}) {
            kk[o]<<<148, warps * 32>>>(iters, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double lane_ops = (double)iters * 16 * warps * 32;
            printf("%-16s warps=%2d  %6.1f lane-ops/clk/SM  (%s)\n", names[o], warps, lane_ops / c, cudaGetErrorString(e));
        }
    }
    for (int warps : {4, 8, 16}) {
        {
            tmem_bw<16, 0><<<148, warps * 32>>>(4096, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("tmem x16 serial warps=%2d %6.1f B/clk/SM (%s)\n", warps, 4096.0 * warps * 32 * 16 * 4 / c, cudaGetErrorString(e));
        }
        {
            tmem_bw<16, 1><<<148, warps * 32>>>(4096, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("tmem x16 pipelined warps=%2d %6.1f B/clk/SM (%s)\n", warps, 4096.0 * warps * 32 * 16 * 4 / c, cudaGetErrorString(e));
        }
        {
            tmem_bw<32, 0><<<148, warps * 32>>>(4096, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("tmem x32 serial warps=%2d %6.1f B/clk/SM (%s)\n", warps, 4096.0 * warps * 32 * 32 * 4 / c, cudaGetErrorString(e));
        }
        {
            tmem_bw<32, 1><<<148, warps * 32>>>(4096, out, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("tmem x32 pipelined warps=%2d %6.1f B/clk/SM (%s)\n", warps, 4096.0 * warps * 32 * 32 * 4 / c, cudaGetErrorString(e));
        }
    }
    return 0;
}
