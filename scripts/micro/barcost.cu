// Cost of single mbarrier / sync operations in a one-warp loop (no partner):
// cycles per iteration of {op} for: try_wait on a completed phase, test_wait on a
// completed phase, arrive (lane 0), arrive by all lanes to a 32-count barrier,
// elect.sync + __syncwarp, tcgen05.commit (lane 0) with no MMAs outstanding,
// and an arrive followed by a try_wait on the phase it completes (1-count).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t *b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ bool test_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok; asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory"); return ok; }
__device__ __forceinline__ bool elect() { uint32_t p; asm volatile("{.reg .pred P; elect.sync _|P, 0xffffffff; selp.u32 %0,1,0,P;}" : "=r"(p)); return p; }
__device__ __forceinline__ void commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(b)) : "memory"); }
template <int mode>
__global__ void k(int iters, long long *out) {
    __shared__ uint64_t bar[4];
    __shared__ uint32_t holder;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { init(&bar[0], 1); init(&bar[1], 1); init(&bar[2], 32); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(su32(&holder)));
    __syncwarp();
    if (lane == 0) arrive(&bar[0]);      // phase 0 of bar[0] complete: try_wait(bar0, 0) always succeeds
    __syncwarp();
    while (!try_wait(&bar[0], 0)) {}
    long long t0 = clock64();
    uint32_t ph = 0; int acc = 0;
    for (int i = 0; i < iters; ++i) {
        if constexpr (mode == 0) acc += try_wait(&bar[0], 0);
        if constexpr (mode == 1) acc += test_wait(&bar[0], 0);
        if constexpr (mode == 2) { if (lane == 0) arrive(&bar[1]); __syncwarp(); }
        if constexpr (mode == 3) arrive(&bar[2]);
        if constexpr (mode == 4) { acc += elect(); __syncwarp(); }
        if constexpr (mode == 5) { if (lane == 0) commit(&bar[1]); __syncwarp(); }
        if constexpr (mode == 6) { if (lane == 0) arrive(&bar[1]); __syncwarp(); while (!try_wait(&bar[1], ph)) {} ph ^= 1; }
        if constexpr (mode == 7) { if (elect()) commit(&bar[1]); __syncwarp(); while (!try_wait(&bar[1], ph)) {} ph ^= 1; }
        if constexpr (mode == 8) { acc += i; }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(holder));
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0, out[1] = acc;
}
int main() {
    long long *d; cudaMalloc(&d, 16);
    const char *nm[] = {"try_wait (completed)", "test_wait (completed)", "arrive lane0 + syncwarp", "arrive x32 lanes",
                        "elect + syncwarp", "tcgen05.commit lane0 (idle)", "arrive -> try_wait own phase",
                        "commit -> try_wait own phase", "empty loop"};
    void (*ks[9])(int, long long *) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>};
    for (int m = 0; m < 9; ++m) {
        const int iters = 10000;
        ks[m]<<<148, 32>>>(iters, d);
        cudaDeviceSynchronize();
        long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-32s %7.1f cycles/iter (%s)\n", nm[m], (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
