// pack.cuh -- a1 activation quantize + pack (fp16 NHWC -> packed s8/s4 NHWC)
// and a2 weight pack (int8 KRSC codes -> packed KRSC).
//
// PAPER.md:42 (section 1): "In the case of INT4 MMA, the packing includes
// quantization of 8 consecutive values (in 32-bit) into a packed vector of
// 4-bit elements. This low-level data alignment incurs noticeable overhead with
// additional memory accesses."  The kernel is HBM-bound (2 + b/8 bytes per
// element): every thread moves whole 16-byte vectors, loads first, grid sized
// to a multiple of the SM count.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

#include "ptx.cuh"   // FastDiv

namespace convq {

// q = clamp(rne(fp32(x) * inv_scale), lo, hi); NaN -> lo (max.f32 returns the
// non-NaN operand), +-inf saturate.  One binary32 multiply (no FMA).  The
// rounding uses the 1.5*2^23 add after the clamp (integer bounds, so
// clamp-then-round == round-then-clamp): the code is left in the low bits of
// the returned word, which the packers below read as a byte / nibble.
__device__ __forceinline__ int quant1(__half h, float inv_scale, float lo, float hi) {
    float f = __half2float(h);
    float v = __fmul_rn(f, inv_scale);
    float c = fminf(fmaxf(v, lo), hi);
    return __float_as_int(__fadd_rn(c, 12582912.0f));
}

// 4 codes (low byte of each word) -> 4 bytes, code i in byte i.
__device__ __forceinline__ uint32_t pack4_s8(int a, int b, int c, int d) {
    uint32_t ab = __byte_perm((uint32_t)a, (uint32_t)b, 0x0040);
    uint32_t cd = __byte_perm((uint32_t)c, (uint32_t)d, 0x0040);
    return __byte_perm(ab, cd, 0x5410);
}
// 8 codes (low nibble of each word) -> one 32-bit word, code i in bits [4i, 4i+4)
// (little-nibble-first).
__device__ __forceinline__ uint32_t pack8_s4(const int (&q)[8]) {
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= ((uint32_t)q[i] & 0xFu) << (4 * i);
    return w;
}

// Fast path: C == C' (no channel padding), so the packed tensor is the flat
// element stream.  Each work item produces one 16-byte output vector:
// 16 codes (s8, reads 32 B) or 32 codes (s4, reads 64 B).
template <int BITS, int UNROLL>
__global__ void __launch_bounds__(256) quantize_flat_kernel(const uint4 *__restrict__ x, uint4 *__restrict__ y,
                                                           int64_t n_out_vec, float inv_scale) {
    constexpr int IN_VEC = BITS == 8 ? 2 : 4;  // 16-byte fp16 vectors per output vector
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const float lo = -(float)(1 << (BITS - 1)), hi = (float)((1 << (BITS - 1)) - 1);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n_out_vec;
         base += stride * UNROLL) {
        uint4 in[UNROLL][IN_VEC];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            int64_t o = base + u * stride;
            if (o < n_out_vec) {
#pragma unroll
                for (int v = 0; v < IN_VEC; ++v) in[u][v] = __ldcs(x + o * IN_VEC + v);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            int64_t o = base + u * stride;
            if (o >= n_out_vec) break;
            // the 8 (s8) or 16 (s4) input words hold 2 fp16 values each, low half first
            uint32_t w[IN_VEC * 4];
#pragma unroll
            for (int v = 0; v < IN_VEC; ++v) {
                w[4 * v] = in[u][v].x; w[4 * v + 1] = in[u][v].y; w[4 * v + 2] = in[u][v].z; w[4 * v + 3] = in[u][v].w;
            }
            int q[IN_VEC * 8];
#pragma unroll
            for (int i = 0; i < IN_VEC * 4; ++i) {
                q[2 * i] = quant1(__ushort_as_half((unsigned short)(w[i] & 0xFFFFu)), inv_scale, lo, hi);
                q[2 * i + 1] = quant1(__ushort_as_half((unsigned short)(w[i] >> 16)), inv_scale, lo, hi);
            }
            uint32_t out[4];
            if constexpr (BITS == 8) {
#pragma unroll
                for (int k = 0; k < 4; ++k) out[k] = pack4_s8(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    int t[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) t[i] = q[8 * k + i];
                    out[k] = pack8_s4(t);
                }
            }
            __stcs(y + o, make_uint4(out[0], out[1], out[2], out[3]));
        }
    }
}

// General path (C' > C, e.g. conv1's C=3 -> 16/32): one 16-byte output vector
// per work item, scalar fp16 loads, padded channels written as code 0.
template <int BITS>
__global__ void __launch_bounds__(256) quantize_padded_kernel(const __half *__restrict__ x, uint4 *__restrict__ y,
                                                             int64_t npix, int C, int vec_per_pix,
                                                             float inv_scale) {
    constexpr int CH = BITS == 8 ? 16 : 32;  // channels per output vector
    const float lo = -(float)(1 << (BITS - 1)), hi = (float)((1 << (BITS - 1)) - 1);
    const int64_t total = npix * vec_per_pix;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        int64_t pix = o / vec_per_pix;
        int c0 = (int)(o - pix * vec_per_pix) * CH;
        int q[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            int c = c0 + i;
            q[i] = c < C ? quant1(x[pix * C + c], inv_scale, lo, hi) : 0;
        }
        uint32_t out[4];
        if constexpr (BITS == 8) {
#pragma unroll
            for (int k = 0; k < 4; ++k) out[k] = pack4_s8(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int t[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) t[i] = q[8 * k + i];
                out[k] = pack8_s4(t);
            }
        }
        y[o] = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

// a2: int8 codes [rows][C] -> packed [rows][C*BITS/8]; one 16-byte output
// vector per work item (C*BITS % 128 == 0 is required by the caller).
template <int BITS>
__global__ void __launch_bounds__(256) pack_weights_kernel(const int8_t *__restrict__ w, uint4 *__restrict__ y,
                                                          int64_t n_out_vec) {
    constexpr int CH = BITS == 8 ? 16 : 32;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n_out_vec;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int8_t *src = w + o * CH;
        uint32_t out[4];
        if constexpr (BITS == 8) {
            uint4 v = *reinterpret_cast<const uint4 *>(src);
            out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
        } else {
            uint4 v0 = *reinterpret_cast<const uint4 *>(src);
            uint4 v1 = *reinterpret_cast<const uint4 *>(src + 16);
            const int8_t *b0 = reinterpret_cast<const int8_t *>(&v0);
            const int8_t *b1 = reinterpret_cast<const int8_t *>(&v1);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int t[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    int c = 8 * k + i;
                    t[i] = c < 16 ? b0[c] : b1[c - 16];
                }
                out[k] = pack8_s4(t);
            }
        }
        y[o] = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

// ---------------------------------------------------------------- s2d stem
// ResNet-style stem (a stride-2 R x S conv over an image with C <= 4 (s8) /
// 8 (s4) channels) run as a stride-1 conv over a space-to-depth(2) view
// (conv_q_plan_s2d, "stem").  One s2d pixel (h2, w2) is
// 16 bytes: the 2x2 input pixels (2*h2+dh, 2*w2+dw) x CP channels, code index
// (2*dh + dw)*CP + c, zero where the pixel or channel does not exist.
// Stored column xc holds s2d column xc - PL (zero outside [0, ceil(W/2))), so
// the S2P-pixel windows the conv reads never leave the row.
// C3 = true: the RGB fast path (C == 3): the two pixels of a row are 12
// contiguous, 4-byte aligned bytes -> three 32-bit read-only loads per row.
template <int BITS, bool C3>
__global__ void __launch_bounds__(256) s2d_quantize_kernel(const __half *__restrict__ x, uint4 *__restrict__ y,
                                                          int N, int H, int W, int C, int H2, int XW, int PL,
                                                          float inv_scale, FastDiv fd_xw, FastDiv fd_h2) {
    constexpr int CP = BITS == 8 ? 4 : 8;      // channels per phase (16 bytes = 4 phases)
    const float lo = -(float)(1 << (BITS - 1)), hi = (float)((1 << (BITS - 1)) - 1);
    const int total = N * H2 * XW;              // < 2^31 (checked on the host)
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int t = fd_xw.div(o);
        const int xc = o - t * XW;
        const int n = fd_h2.div(t);
        const int h2 = t - n * H2;
        const int w2 = xc - PL;
        int q[4 * CP];
#pragma unroll
        for (int i = 0; i < 4 * CP; ++i) q[i] = 0;
        if (C3 && w2 >= 0 && 2 * w2 + 1 < W) {
#pragma unroll
            for (int dh = 0; dh < 2; ++dh) {
                const int h = 2 * h2 + dh;
                if (h >= H) continue;
                const uint32_t *src = reinterpret_cast<const uint32_t *>(x + (((int64_t)n * H + h) * W + 2 * w2) * 3);
                const uint32_t a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
                const uint32_t hv[3] = {a, b, c};   // halves: (p0c0 p0c1) (p0c2 p1c0) (p1c1 p1c2)
#pragma unroll
                for (int e = 0; e < 6; ++e) {
                    const unsigned short bits = (unsigned short)(e & 1 ? hv[e >> 1] >> 16 : hv[e >> 1] & 0xFFFFu);
                    q[(2 * dh + e / 3) * CP + e % 3] = quant1(__ushort_as_half(bits), inv_scale, lo, hi);
                }
            }
        } else if (w2 >= 0 && 2 * w2 < W) {
#pragma unroll
            for (int dh = 0; dh < 2; ++dh) {
                const int h = 2 * h2 + dh;
                if (h >= H) continue;
#pragma unroll
                for (int dw = 0; dw < 2; ++dw) {
                    const int w = 2 * w2 + dw;
                    if (w >= W) continue;
                    const __half *src = x + (((int64_t)n * H + h) * W + w) * C;
#pragma unroll
                    for (int c = 0; c < CP; ++c)
                        if (c < C) q[(2 * dh + dw) * CP + c] = quant1(src[c], inv_scale, lo, hi);
                }
            }
        }
        uint32_t out[4];
        if constexpr (BITS == 8) {
#pragma unroll
            for (int k = 0; k < 4; ++k) out[k] = pack4_s8(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int u[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) u[i] = q[8 * k + i];
                out[k] = pack8_s4(u);
            }
        }
        y[o] = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

// RGB fast path with 16-byte loads (C == 3, W % 8 == 0, x 16-byte aligned): one
// thread per 4 consecutive s2d columns of a row -- 8 input pixels x 3 halves =
// 48 contiguous bytes per input row = three 16-byte loads (instead of a thread
// per s2d column with three 4-byte loads per row) -- and 4 stored 16-byte
// pixels; the remaining threads of the row write its zero border columns.
// Codes exactly as s2d_quantize_kernel (same quant1, same layout).
template <int BITS>
__global__ void __launch_bounds__(256) s2d_quantize_c3v_kernel(const __half *__restrict__ x, uint4 *__restrict__ y,
                                                              int N, int H, int W, int H2, int XW, int PL, int G,
                                                              int TR, float inv_scale, FastDiv fd_tr, FastDiv fd_h2) {
    constexpr int CP = BITS == 8 ? 4 : 8;
    const float lo = -(float)(1 << (BITS - 1)), hi = (float)((1 << (BITS - 1)) - 1);
    const int total = N * H2 * TR;              // TR = G groups + border columns per row (< 2^31, host-checked)
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= total) return;
    const int t = fd_tr.div(o);
    const int k = o - t * TR;
    const int n = fd_h2.div(t);
    const int h2 = t - n * H2;
    uint4 *row = y + ((int64_t)n * H2 + h2) * XW;
    auto pack_pixel = [&](const int (&q)[4 * CP]) -> uint4 {
        uint32_t out[4];
        if constexpr (BITS == 8) {
#pragma unroll
            for (int i = 0; i < 4; ++i) out[i] = pack4_s8(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                int u[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) u[e] = q[8 * i + e];
                out[i] = pack8_s4(u);
            }
        }
        return make_uint4(out[0], out[1], out[2], out[3]);
    };
    if (k >= G) {   // a zero border column: left [0, PL) or right [PL + W/2, XW)
        const int b = k - G;
        row[b < PL ? b : PL + W / 2 + (b - PL)] = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    int q[4][4 * CP];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4 * CP; ++i) q[j][i] = 0;
#pragma unroll
    for (int dh = 0; dh < 2; ++dh) {
        const int h = 2 * h2 + dh;
        if (h >= H) continue;
        const uint4 *src = reinterpret_cast<const uint4 *>(x + (((int64_t)n * H + h) * W + 8 * k) * 3);
        const uint4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
        const uint32_t hw[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 24; ++e) {   // half e = pixel e / 3, channel e % 3
            const unsigned short bits = (unsigned short)(e & 1 ? hw[e >> 1] >> 16 : hw[e >> 1] & 0xFFFFu);
            const int px = e / 3, ch = e % 3;
            q[px >> 1][(2 * dh + (px & 1)) * CP + ch] = quant1(__ushort_as_half(bits), inv_scale, lo, hi);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) row[PL + 4 * k + j] = pack_pixel(q[j]);
}

// Stem weights (once per model): int8 codes [K][R][S][C] -> [K][R2][S2P*16 bytes].
// Window tap (jr, js), phase (dh, dw), channel c holds w[k, r, s, c] with
// r = 2*(jr - PL) + dh + pad, s = 2*(js - PL) + dw + pad (0 outside the filter),
// so sum over the window of x_s2d * w_s2d == the stride-2 conv's sum.
template <int BITS>
__global__ void __launch_bounds__(256) s2d_weights_kernel(const int8_t *__restrict__ w, uint4 *__restrict__ y,
                                                         int K, int R, int S, int C, int R2, int S2P, int PL,
                                                         int pad) {
    constexpr int CP = BITS == 8 ? 4 : 8;
    const int64_t total = (int64_t)K * R2 * S2P;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int js = (int)(o % S2P);
        const int64_t t = o / S2P;
        const int jr = (int)(t % R2);
        const int k = (int)(t / R2);
        int q[4 * CP];
#pragma unroll
        for (int e = 0; e < 4 * CP; ++e) {
            const int ph = e / CP, c = e % CP;
            const int r = 2 * (jr - PL) + (ph >> 1) + pad, s = 2 * (js - PL) + (ph & 1) + pad;
            q[e] = (c < C && r >= 0 && r < R && s >= 0 && s < S) ? (int)w[(((int64_t)k * R + r) * S + s) * C + c] : 0;
        }
        uint32_t out[4];
        if constexpr (BITS == 8) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) out[kk] = pack4_s8(q[4 * kk], q[4 * kk + 1], q[4 * kk + 2], q[4 * kk + 3]);
        } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                int u[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) u[i] = q[8 * kk + i];
                out[kk] = pack8_s4(u);
            }
        }
        y[o] = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

// ---------------------------------------------------------------- max pool
// R x R max pooling of packed NHWC codes (the ResNet stem's 3x3/2 pool between
// conv1 and layer1): one thread per 16-byte output vector
// (16 s8 / 32 s4 channels of one output pixel), consecutive threads along the
// channel vectors of a pixel, then along pixels (coalesced 16-byte loads and
// stores; the R*R-fold tap re-reads hit L1/L2).  Out-of-range taps are
// skipped (padding never wins); quantization is monotone, so the max of the
// codes is the code of the max.  s8: byte-wise signed max (VIMNMX.S8); s4: the
// even / odd nibbles expanded to 16*v bytes, byte max, repacked.
__device__ __forceinline__ uint32_t vmax_s8x4(uint32_t a, uint32_t b) { return __vmaxs4(a, b); }
// unsigned codes (DESIGN reading 16): byte-wise unsigned max; u4 nibbles as 16*v bytes
__device__ __forceinline__ uint32_t vmax_u8x4(uint32_t a, uint32_t b) { return __vmaxu4(a, b); }
__device__ __forceinline__ uint32_t vmax_u4x8(uint32_t a, uint32_t b) {
    const uint32_t ae = (a << 4) & 0xF0F0F0F0u, ao = a & 0xF0F0F0F0u;
    const uint32_t be = (b << 4) & 0xF0F0F0F0u, bo = b & 0xF0F0F0F0u;
    const uint32_t me = __vmaxu4(ae, be), mo = __vmaxu4(ao, bo);
    return ((me >> 4) & 0x0F0F0F0Fu) | (mo & 0xF0F0F0F0u);
}
__device__ __forceinline__ uint32_t vmax_s4x8(uint32_t a, uint32_t b) {
    const uint32_t ae = (a << 4) & 0xF0F0F0F0u, ao = a & 0xF0F0F0F0u;   // 16 * even / odd nibbles as s8
    const uint32_t be = (b << 4) & 0xF0F0F0F0u, bo = b & 0xF0F0F0F0u;
    const uint32_t me = __vmaxs4(ae, be), mo = __vmaxs4(ao, bo);
    return ((me >> 4) & 0x0F0F0F0Fu) | (mo & 0xF0F0F0F0u);
}
template <int BITS, int R, bool UNS = false>
__global__ void __launch_bounds__(256) maxpool_kernel(const uint4 *__restrict__ x, uint4 *__restrict__ y, int N,
                                                     int H, int W, int P, int Q, int vpp, int stride, int pad,
                                                     FastDiv fd_vpp, FastDiv fd_q, FastDiv fd_p) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");   // x is the previous kernel's output
    // identity of the max: the most negative code in every lane (out-of-range
    // taps read as it, so the padding never wins: every window has an in-range tap)
    constexpr uint32_t MINV = UNS ? 0u : BITS == 8 ? 0x80808080u : 0x88888888u;
    const int total = N * P * Q * vpp;          // < 2^31 (checked on the host)
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int pix = fd_vpp.div(o);
        const int v = o - pix * vpp;
        const int t = fd_q.div(pix);
        const int q = pix - t * Q;
        const int n = fd_p.div(t);
        const int p = t - n * P;
        const int h0 = p * stride - pad, w0 = q * stride - pad;
        const uint4 *base = x + ((int64_t)n * H * W) * vpp + v;
        uint4 a[R * R];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int s = 0; s < R; ++s) {   // all R*R loads in flight before the first max
                const int h = h0 + r, w = w0 + s;
                a[r * R + s] = (h >= 0 && h < H && w >= 0 && w < W) ? __ldg(base + ((int64_t)h * W + w) * vpp)
                                                                    : make_uint4(MINV, MINV, MINV, MINV);
            }
        uint4 m = a[0];
#pragma unroll
        for (int i = 1; i < R * R; ++i) {
            if constexpr (BITS == 8 && UNS)
                m = make_uint4(vmax_u8x4(m.x, a[i].x), vmax_u8x4(m.y, a[i].y), vmax_u8x4(m.z, a[i].z),
                               vmax_u8x4(m.w, a[i].w));
            else if constexpr (UNS)
                m = make_uint4(vmax_u4x8(m.x, a[i].x), vmax_u4x8(m.y, a[i].y), vmax_u4x8(m.z, a[i].z),
                               vmax_u4x8(m.w, a[i].w));
            else if constexpr (BITS == 8)
                m = make_uint4(vmax_s8x4(m.x, a[i].x), vmax_s8x4(m.y, a[i].y), vmax_s8x4(m.z, a[i].z),
                               vmax_s8x4(m.w, a[i].w));
            else
                m = make_uint4(vmax_s4x8(m.x, a[i].x), vmax_s4x8(m.y, a[i].y), vmax_s4x8(m.z, a[i].z),
                               vmax_s4x8(m.w, a[i].w));
        }
        y[o] = m;
    }
}


// 3x3 / stride-2 max pool (the ResNet stem's), T output rows per thread: the
// horizontal 3-tap max of each input row is computed once and shared by the two
// output rows it belongs to (input row 2p+1 is row 2p+1 of output p and row -1 of
// output p+1): 3(2T+1) loads per T outputs instead of 9T.  One thread per
// (image, T-row group, output column, 16-byte channel vector); consecutive
// threads walk the channel vectors, then the columns (coalesced).
template <int BITS, bool UNS, int T>
__global__ void __launch_bounds__(256) maxpool3s2_rows_kernel(const uint4 *__restrict__ x, uint4 *__restrict__ y,
                                                              int N, int H, int W, int P, int Q, int vpp, int pad,
                                                              int groups, FastDiv fd_vpp, FastDiv fd_q,
                                                              FastDiv fd_g) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr uint32_t MINV = UNS ? 0u : BITS == 8 ? 0x80808080u : 0x88888888u;
    auto vmax = [](uint32_t a, uint32_t b) -> uint32_t {
        if constexpr (BITS == 8 && UNS) return vmax_u8x4(a, b);
        else if constexpr (BITS == 8) return vmax_s8x4(a, b);
        else if constexpr (UNS) return vmax_u4x8(a, b);
        else return vmax_s4x8(a, b);
    };
    auto vmax4 = [&](uint4 a, uint4 b) { return make_uint4(vmax(a.x, b.x), vmax(a.y, b.y), vmax(a.z, b.z), vmax(a.w, b.w)); };
    const int total = N * groups * Q * vpp;     // < 2^31 (checked on the host)
    // s8 / u8 codes: bytes widened to 16-bit lanes (sign- or zero-extended, two
    // PRMT per word) so every max is ONE native VIMNMX.{S,U}16x2 per two codes
    // instead of the 6-instruction byte-SIMD emulation of __vmax{s,u}4; one PRMT
    // per output word packs the low bytes back
    if constexpr (BITS == 8) {
        constexpr uint32_t SEL_E = UNS ? 0x4240u : 0xA280u;   // bytes 0, 2 -> 16-bit lanes
        constexpr uint32_t SEL_O = UNS ? 0x4341u : 0xB391u;   // bytes 1, 3 -> 16-bit lanes
        auto mx = [](uint32_t a, uint32_t b) -> uint32_t { return UNS ? __vmaxu2(a, b) : __vmaxs2(a, b); };
        for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
            const int pix = fd_vpp.div(o);
            const int v = o - pix * vpp;
            const int t = fd_q.div(pix);
            const int q = pix - t * Q;
            const int n = fd_g.div(t);
            const int p0 = (t - n * groups) * T;
            const int w0 = 2 * q - pad;
            const uint4 *base = x + (int64_t)n * H * W * vpp + v;
            constexpr int NR = 2 * T + 1;
            uint4 a[NR][3];
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                const int h = 2 * p0 - pad + i;
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    const int w = w0 + s;
                    a[i][s] = (h >= 0 && h < H && w >= 0 && w < W) ? __ldg(base + ((int64_t)h * W + w) * vpp)
                                                                    : make_uint4(MINV, MINV, MINV, MINV);
                }
            }
            // row maxima in widened form: hm[i][2k] = even bytes of word k, hm[i][2k+1] = odd bytes
            uint32_t hm[NR][8];
#pragma unroll
            for (int i = 0; i < NR; ++i)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t w_0 = (&a[i][0].x)[k], w_1 = (&a[i][1].x)[k], w_2 = (&a[i][2].x)[k];
                    hm[i][2 * k] = mx(mx(__byte_perm(w_0, 0u, SEL_E), __byte_perm(w_1, 0u, SEL_E)),
                                      __byte_perm(w_2, 0u, SEL_E));
                    hm[i][2 * k + 1] = mx(mx(__byte_perm(w_0, 0u, SEL_O), __byte_perm(w_1, 0u, SEL_O)),
                                          __byte_perm(w_2, 0u, SEL_O));
                }
#pragma unroll
            for (int kk = 0; kk < T; ++kk) {
                const int p = p0 + kk;
                if (p < P) {
                    uint32_t r[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t e = mx(mx(hm[2 * kk][2 * k], hm[2 * kk + 1][2 * k]), hm[2 * kk + 2][2 * k]);
                        const uint32_t od = mx(mx(hm[2 * kk][2 * k + 1], hm[2 * kk + 1][2 * k + 1]),
                                               hm[2 * kk + 2][2 * k + 1]);
                        r[k] = __byte_perm(e, od, 0x6240);   // bytes: e0, od0, e2, od2
                    }
                    y[(((int64_t)n * P + p) * Q + q) * vpp + v] = make_uint4(r[0], r[1], r[2], r[3]);
                }
            }
        }
        return;
    }
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int pix = fd_vpp.div(o);
        const int v = o - pix * vpp;
        const int t = fd_q.div(pix);
        const int q = pix - t * Q;
        const int n = fd_g.div(t);
        const int p0 = (t - n * groups) * T;
        const int w0 = 2 * q - pad;
        const uint4 *base = x + (int64_t)n * H * W * vpp + v;
        // horizontal maxima of input rows 2 p0 - pad .. 2 (p0 + T - 1) - pad + 2, all loads first
        constexpr int NR = 2 * T + 1;
        uint4 a[NR][3];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int h = 2 * p0 - pad + i;
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const int w = w0 + s;
                a[i][s] = (h >= 0 && h < H && w >= 0 && w < W) ? __ldg(base + ((int64_t)h * W + w) * vpp)
                                                                : make_uint4(MINV, MINV, MINV, MINV);
            }
        }
        uint4 hm[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) hm[i] = vmax4(vmax4(a[i][0], a[i][1]), a[i][2]);
#pragma unroll
        for (int k = 0; k < T; ++k) {
            const int p = p0 + k;
            if (p < P)
                y[(((int64_t)n * P + p) * Q + q) * vpp + v] = vmax4(vmax4(hm[2 * k], hm[2 * k + 1]), hm[2 * k + 2]);
        }
    }
}

}  // namespace convq
