// Semantics check of cvt.pack.sat (measurement/dev only)
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t *o) {
    int a = 0x11, b = 0x22;
    uint32_t c = 0xA1B2C3D4u, d;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); o[0] = d;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(300), "r"(-300), "r"(0)); o[1] = d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(300), "r"(-300), "r"(0)); o[2] = d;
    asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(3), "r"(-2), "r"(c)); o[3] = d;
    asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(30), "r"(-30), "r"(0)); o[4] = d;
    int r; float nan = __int_as_float(0x7fc00000);
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(nan)); o[5] = r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(3e10f)); o[6] = r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(-3e10f)); o[7] = r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(2.5f)); o[8] = r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(-2.5f)); o[9] = r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(3.5f)); o[10] = r;
}
int main() {
    uint32_t *o, h[12] = {0};
    cudaMalloc(&o, sizeof h);
    k<<<1, 1>>>(o);
    cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    const char *n[12] = {"s8 (0x11,0x22,c)", "s8 sat(300,-300,0)", "u8 sat(300,-300,0)", "s4 (3,-2,c)", "s4 sat(30,-30,0)",
                         "rni NaN", "rni 3e10", "rni -3e10", "rni 2.5", "rni -2.5", "rni 3.5", "s16 (0x11,0x22,c)"};
    for (int i = 0; i < 12; ++i) printf("%-22s 0x%08x\n", n[i], h[i]);
}
