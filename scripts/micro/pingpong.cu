// Producer/consumer mbarrier ping-pong through a ring of S stages (no TMA, no
// MMA): cycles per stage for try_wait vs test_wait polling, and with the
// consumer's release done by tcgen05.commit (the conv kernel's path) instead of
// a plain arrive.  nvcc -gencode arch=compute_100a,code=sm_100a -o pingpong pingpong.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ bool test_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph, int mode) {
    if (mode == 0) { while (!try_wait(b, ph)) {} }
    else { while (!test_wait(b, ph)) {} }
}
__device__ __forceinline__ void commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(b)) : "memory");
}
template <int S, int mode, int use_commit>
__global__ void k(int iters, long long *out) {
    __shared__ uint64_t full[16], empty[16];
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { for (int i = 0; i < S; ++i) { init(&full[i], 1); init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (warp == 1) asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&holder)));
    __syncthreads();
    long long t0 = clock64();
    int st = 0; uint32_t ph = 0;
    if (warp == 0) {          // producer
        for (int i = 0; i < iters; ++i) {
            wait(&empty[st], ph ^ 1, mode);
            if (lane == 0) arrive(&full[st]);
            __syncwarp();
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1) {   // consumer
        for (int i = 0; i < iters; ++i) {
            wait(&full[st], ph, mode);
            if (lane == 0) { if (use_commit) commit(&empty[st]); else arrive(&empty[st]); }
            __syncwarp();
            if (++st == S) { st = 0; ph ^= 1; }
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(holder));
    }
    if (threadIdx.x == 32 && blockIdx.x == 0) *out = t1 - t0;
}
int main() {
    long long *d; cudaMalloc(&d, 8);
    void (*ks[20])(int, long long *) = {k<1,0,0>, k<2,0,0>, k<3,0,0>, k<4,0,0>, k<8,0,0>,
                                        k<1,1,0>, k<2,1,0>, k<3,1,0>, k<4,1,0>, k<8,1,0>,
                                        k<1,0,1>, k<2,0,1>, k<3,0,1>, k<4,0,1>, k<8,0,1>,
                                        k<1,1,1>, k<2,1,1>, k<3,1,1>, k<4,1,1>, k<8,1,1>};
    const int Ss[5] = {1, 2, 3, 4, 8};
    for (int j = 0; j < 20; ++j) {
        const int uc = j / 10, mode = (j / 5) % 2, S = Ss[j % 5];
        const int iters = 20000;
        ks[j]<<<148, 64>>>(iters, d);
        cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%s %s S=%d: %.1f cycles/stage (%s)\n", uc ? "commit " : "arrive ", mode ? "test_wait" : "try_wait ", S,
               (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
