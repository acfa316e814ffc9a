/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the quantized
 * convolution path of arXiv 2202.06819 ("Learning from Distinctive Candidates
 * to Optimize Reduced-Precision Convolution Program on Tensor Cores").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2202_06819_b200/csrc); neither side includes or links the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (no FMA contraction: every float operation below rounds exactly
 *         once, as written; fmaf() is the one explicitly fused step).
 *
 * Citations are PAPER.md / SPEC.md line numbers under /root/reference plus
 * the section they fall in; "reading N" refers to the numbered readings of
 * the paper listed in DESIGN.md section 3 (taken from SURVEY.md section 8(c)).
 *
 * Functions and their pins (tests/test_oracle_*.py):
 *   oracle_half_to_float   pinned: all 65536 fp16 codes vs numpy's IEEE decode
 *   oracle_quantize_value  pinned: closed forms (exact multiples, RNE ties,
 *                          +-65504, +-inf, -0, NaN)
 *   oracle_pack/unpack     pinned: SPEC.md:226,235-237 words (0x87654321 ...)
 *                          and 10^4 random round trips
 *   oracle_conv_s32        pinned: pure-python brute force on tiny shapes,
 *                          torch float64 conv2d (exact for |acc| < 2^53),
 *                          explicit GEMM for 1x1, all-ones tap counts
 *                          (SPEC.md:76 -> 4C/6C/9C), identity 1x1, zero in
 *   oracle_requant_value   pinned: closed forms (scale 1 -> saturating cast,
 *                          scale 0.5 ties -> even, ReLU, 2^-k shifts) and
 *                          40 000 adversarial near-tie (acc, scale, shift)
 *                          triples vs an exact-rational single-rounding
 *                          evaluation (separates fmaf from mul-then-add)
 *   oracle_maxpool         pinned: torch max_pool2d (float64, library) on the
 *                          unpacked codes; all-equal / one-hot windows
 *   oracle_requant_res_value  pinned: res_scale 0 == oracle_requant_value;
 *                          unit scales == clamp(acc + skip) (exact integers);
 *                          exact-rational evaluation with the two single
 *                          roundings of reading 15 on random / near-tie cases
 *   *_fmt variants (unsigned post-ReLU codes, reading 16): unpack_fmt pinned by
 *                          all 256 bytes / the SPEC.md:226 word read unsigned;
 *                          conv_s32_fmt by torch float64 conv2d on the unsigned
 *                          values and by the identity u = s + 2^b [s < 0]
 *                          (acc_u = acc_s + 2^b conv(neg-mask, w)); requant_fmt
 *                          by closed forms (scale 1 -> clamp(acc, 0, 2^b - 1))
 *                          and exact rationals; maxpool_fmt by torch max_pool2d
 *                          on the unsigned values
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#define ORACLE_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------
 * fp16 -> fp32, written out from the IEEE 754 binary16 definition
 * (1 sign, 5 exponent bits with bias 15, 10 fraction bits).  Every binary16
 * value is exactly representable in binary32, so this is exact.
 * Input of the quantizer: PAPER.md:42 (section 1) "the packing includes
 * quantization of 8 consecutive values".
 * ---------------------------------------------------------------------- */
ORACLE_API float oracle_half_to_float(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    float mag;
    if (e == 0)            /* zero / subnormal: m * 2^-24 */
        mag = ldexpf((float)m, -24);
    else if (e == 31)      /* inf / NaN */
        mag = m ? NAN : INFINITY;
    else                   /* normal: (1024 + m) * 2^(e - 15 - 10) */
        mag = ldexpf((float)(1024 + m), e - 25);
    return sign ? -mag : mag;
}

/* Signed range of a b-bit two's-complement code: [-2^(b-1), 2^(b-1)-1].
 * SPEC.md:274 ("two's-complement nibbles clipped to [-8,7]"); reading 3. */
static float lo_of(int bits) { return -(float)(1 << (bits - 1)); }
static float hi_of(int bits) { return (float)((1 << (bits - 1)) - 1); }

/* ------------------------------------------------------------------------
 * Quantize one value (reading 1: symmetric, zero point 0, per-tensor
 * inv_scale; one binary32 multiply, round half to even, saturate).
 *   v = f * inv_scale ; r = nearbyint(v) ; q = clamp(r, lo, hi)
 * The clamp is done in float with fmaxf first so that NaN -> lo
 * (fmaxf returns the non-NaN operand), and +-inf saturate.
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_quantize_value(float f, float inv_scale, int bits)
{
    float v = f * inv_scale;
    float r = nearbyintf(v);              /* default rounding mode: ties to even */
    float c = fminf(fmaxf(r, lo_of(bits)), hi_of(bits));
    return (int)c;
}

/* ------------------------------------------------------------------------
 * Channel packing ("8 consecutive values (in 32-bit) into a packed
 * vector of 4-bit elements"; SPEC.md:220-228 pack_int4 "nibble i at bit 4i",
 * little-nibble-first, reading 2).
 *   bits = 8: byte c = (uint8) q[c]
 *   bits = 4: 32-bit word c/8 holds q[c] & 0xF at bits 4*(c mod 8).  On
 *             little-endian memory that is byte c/2, low nibble = even c.
 * count = number of channel values (must make whole bytes).
 * ---------------------------------------------------------------------- */
ORACLE_API void oracle_pack(const int8_t *q, int64_t count, int bits, uint8_t *out)
{
    if (bits == 8) {
        for (int64_t c = 0; c < count; ++c) out[c] = (uint8_t)q[c];
        return;
    }
    memset(out, 0, (size_t)(count / 2));
    for (int64_t c = 0; c < count; ++c) {
        uint32_t word_shift = 4u * (uint32_t)(c % 8);          /* bit offset in the u32 word */
        uint32_t nib = (uint32_t)(q[c] & 0xF);
        /* word c/8 = bytes 4*(c/8) .. 4*(c/8)+3, little endian */
        int64_t byte = 4 * (c / 8) + word_shift / 8;
        out[byte] |= (uint8_t)(nib << (word_shift % 8));
    }
}

/* Inverse of oracle_pack; nibbles are sign-extended. */
ORACLE_API void oracle_unpack(const uint8_t *p, int64_t count, int bits, int8_t *q)
{
    if (bits == 8) {
        for (int64_t c = 0; c < count; ++c) q[c] = (int8_t)p[c];
        return;
    }
    for (int64_t c = 0; c < count; ++c) {
        uint32_t word_shift = 4u * (uint32_t)(c % 8);
        int64_t byte = 4 * (c / 8) + word_shift / 8;
        int nib = (p[byte] >> (word_shift % 8)) & 0xF;
        q[c] = (int8_t)(nib >= 8 ? nib - 16 : nib);
    }
}

/* ------------------------------------------------------------------------
 * Code formats (reading 16, SURVEY 8(f) NEXT-2 "unsigned u8/u4 post-ReLU
 * activations"): a packed tensor holds either signed two's-complement codes
 * (reading 3) or unsigned codes [0, 2^b - 1] -- the same b bits per value, the
 * same little-nibble-first layout (reading 2); only their meaning differs.
 * Weights are always signed.
 * ---------------------------------------------------------------------- */
static int code_lo(int bits, int uns) { return uns ? 0 : -(1 << (bits - 1)); }
static int code_hi(int bits, int uns) { return uns ? (1 << bits) - 1 : (1 << (bits - 1)) - 1; }

/* Unpack count codes of format uns (0 signed, 1 unsigned) into int16 values. */
ORACLE_API void oracle_unpack_fmt(const uint8_t *p, int64_t count, int bits, int uns, int16_t *q)
{
    for (int64_t c = 0; c < count; ++c) {
        int v;
        if (bits == 8) {
            v = p[c];                                   /* the byte as 0..255 */
        } else {
            uint32_t word_shift = 4u * (uint32_t)(c % 8);
            int64_t byte = 4 * (c / 8) + word_shift / 8;
            v = (p[byte] >> (word_shift % 8)) & 0xF;    /* the nibble as 0..15 */
        }
        if (!uns && v >= (1 << (bits - 1))) v -= 1 << bits;   /* two's complement */
        q[c] = (int16_t)v;
    }
}

/* Pack int16 codes (each within its format's range): the low b bits of each
 * value at the position oracle_pack uses (reading 2). */
ORACLE_API void oracle_pack_fmt(const int16_t *q, int64_t count, int bits, uint8_t *out)
{
    if (bits == 8) {
        for (int64_t c = 0; c < count; ++c) out[c] = (uint8_t)(q[c] & 0xFF);
        return;
    }
    memset(out, 0, (size_t)(count / 2));
    for (int64_t c = 0; c < count; ++c) {
        uint32_t word_shift = 4u * (uint32_t)(c % 8);
        int64_t byte = 4 * (c / 8) + word_shift / 8;
        out[byte] |= (uint8_t)((uint32_t)(q[c] & 0xF) << (word_shift % 8));
    }
}

/* ------------------------------------------------------------------------
 * Quantize + pack an fp16 NHWC tensor into packed NHWC with C' channels,
 * C' = ceil(C/32)*32 (reading 14: whole 32-channel granules, i.e. >= 16-byte
 * pixel rows for both widths); channels [C, C') are 0.
 * (section 1; reading 1, reading 7 for the zero padding value.)
 * ---------------------------------------------------------------------- */
ORACLE_API int64_t oracle_padded_channels(int64_t C, int bits)
{
    (void)bits;
    return (C + 31) / 32 * 32;
}

ORACLE_API void oracle_quantize(const uint16_t *x, int64_t N, int64_t H, int64_t W,
                                int64_t C, float inv_scale, int bits, uint8_t *xq,
                                int nthreads)
{
    int64_t Cp = oracle_padded_channels(C, bits);
    int64_t npix = N * H * W;
    int64_t row_bytes = Cp * bits / 8;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t pix = 0; pix < npix; ++pix) {
        int8_t q[4096];                          /* one pixel row; C' <= 4096 */
        for (int64_t c = 0; c < Cp; ++c)
            q[c] = (c < C) ? (int8_t)oracle_quantize_value(
                                 oracle_half_to_float(x[pix * C + c]), inv_scale, bits)
                           : 0;
        oracle_pack(q, Cp, bits, xq + pix * row_bytes);
    }
}

/* Output spatial size, floor form (reading 6): P = (H + 2 pad - R)/stride + 1 */
ORACLE_API int64_t oracle_out_dim(int64_t H, int64_t R, int64_t stride, int64_t pad)
{
    int64_t t = H + 2 * pad - R;
    if (t < 0) return 0;
    return t / stride + 1;
}

/* ------------------------------------------------------------------------
 * Direct convolution with exact integer accumulation.
 *   acc[n,p,q,k] = sum_{r<R, s<S, c<C} x[n, p*st-pad+r, q*st-pad+s, c] * w[k,r,s,c]
 * out-of-range x = 0 (zero padding, reading 7).
 * PAPER.md:56 (section 2.1): convolution over W, H, I, O, R, S, N equals the
 * GEMM (N*H*W, I*R*S) x (I*R*S, O); SPEC.md:61-64 source_coord
 * direct_conv.  x is packed NHWC with C channels, w packed KRSC (reading 8).
 * Accumulates in int64; returns -1 if any sum leaves int32 (the plan's
 * overflow guard, section 3.2.1, makes that impossible for
 * accepted shapes), else 0.
 * pix_list: NULL for all N*P*Q output pixels, else npix linear output pixel
 * indices m = (n*P + p)*Q + q, and acc has npix*K entries in that order.
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_conv_s32_fmt(const uint8_t *x, const uint8_t *w,
                                   int64_t N, int64_t H, int64_t W, int64_t C,
                                   int64_t K, int64_t R, int64_t S,
                                   int64_t stride, int64_t pad, int bits, int x_uns,
                                   const int64_t *pix_list, int64_t npix,
                                   int32_t *acc, int nthreads)
{
    int64_t P = oracle_out_dim(H, R, stride, pad);
    int64_t Q = oracle_out_dim(W, S, stride, pad);
    int64_t row_bytes = C * bits / 8;
    int64_t n_out = pix_list ? npix : N * P * Q;
    int overflow = 0;

    /* unpack both operands to one int16 per channel: x in its format (reading
     * 16), w signed */
    int16_t *xs = (int16_t *)malloc((size_t)(N * H * W * C) * sizeof(int16_t));
    int16_t *ws = (int16_t *)malloc((size_t)(K * R * S * C) * sizeof(int16_t));
    if (!xs || !ws) { free(xs); free(ws); return -2; }
    for (int64_t pix = 0; pix < N * H * W; ++pix)
        oracle_unpack_fmt(x + pix * row_bytes, C, bits, x_uns, xs + pix * C);
    for (int64_t t = 0; t < K * R * S; ++t)
        oracle_unpack_fmt(w + t * row_bytes, C, bits, 0, ws + t * C);

#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) reduction(| : overflow)
    for (int64_t i = 0; i < n_out; ++i) {
        int64_t m = pix_list ? pix_list[i] : i;
        int64_t n = m / (P * Q);
        int64_t p = (m / Q) % P;
        int64_t q = m % Q;
        for (int64_t k = 0; k < K; ++k) {
            int64_t sum = 0;
            for (int64_t r = 0; r < R; ++r) {
                int64_t h = p * stride - pad + r;
                if (h < 0 || h >= H) continue;
                for (int64_t s = 0; s < S; ++s) {
                    int64_t ww = q * stride - pad + s;
                    if (ww < 0 || ww >= W) continue;
                    const int16_t *xp = xs + ((n * H + h) * W + ww) * C;
                    const int16_t *wp = ws + ((k * R + r) * S + s) * C;
                    for (int64_t c = 0; c < C; ++c)
                        sum += (int64_t)xp[c] * (int64_t)wp[c];
                }
            }
            if (sum > INT32_MAX || sum < INT32_MIN) overflow |= 1;
            acc[i * K + k] = (int32_t)sum;
        }
    }
    free(xs);
    free(ws);
    return overflow ? -1 : 0;
}

/* Signed activations (reading 3): the format-0 case of oracle_conv_s32_fmt. */
ORACLE_API int oracle_conv_s32(const uint8_t *x, const uint8_t *w,
                               int64_t N, int64_t H, int64_t W, int64_t C,
                               int64_t K, int64_t R, int64_t S,
                               int64_t stride, int64_t pad, int bits,
                               const int64_t *pix_list, int64_t npix,
                               int32_t *acc, int nthreads)
{
    return oracle_conv_s32_fmt(x, w, N, H, W, C, K, R, S, stride, pad, bits, 0, pix_list, npix, acc, nthreads);
}

/* ------------------------------------------------------------------------
 * Requantize one accumulator (section 3.2.2: "relu, batch
 * normalization, and bias addition ... the result data are finally clipped to
 * lower bits and packed"; reading 4 order, reading 5 rounding):
 *   f = (float) acc            (int -> binary32, round to nearest even)
 *   v = fmaf(f, scale, shift)  (one rounding)
 *   r = nearbyint(v)           (ties to even)
 *   y = clamp(r, lo, hi), lo = 0 with ReLU else -2^(b-1), hi = 2^(b-1)-1
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_requant_value(int32_t acc, float scale, float shift, int relu, int bits)
{
    float f = (float)acc;
    float v = fmaf(f, scale, shift);
    float r = nearbyintf(v);
    float lo = relu ? 0.0f : lo_of(bits);
    float c = fminf(fmaxf(r, lo), hi_of(bits));
    return (int)c;
}

/* ------------------------------------------------------------------------
 * Requantize with a fused residual add (PAPER.md:200
 * section 3.2.2 names the epilogue's elementwise work -- "relu, batch
 * normalization, and bias addition" -- and the residual add of a ResNet block,
 * relu(bn(conv(x)) + identity), is the same class of work).  DESIGN reading 15:
 *   u = fmaf((float)acc, scale, shift)       the conv's BN / bias, one rounding
 *   v = fmaf((float)skip, res_scale, u)      + the skip code rescaled, one rounding
 *   y = clamp(rne(v), lo, hi), lo = 0 with ReLU (ReLU after the add)
 * skip = the skip tensor's code at the same (pixel, channel), res_scale one
 * fp32 per layer (the skip tensor's scale relative to the output's).
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_requant_res_value(int32_t acc, float scale, float shift, int skip, float res_scale,
                                        int relu, int bits)
{
    float f = (float)acc;
    float u = fmaf(f, scale, shift);
    float v = fmaf((float)skip, res_scale, u);
    float r = nearbyintf(v);
    float lo = relu ? 0.0f : lo_of(bits);
    float c = fminf(fmaxf(r, lo), hi_of(bits));
    return (int)c;
}

/* Requantize an [M, K] accumulator matrix and pack each row into K*b/8 bytes.
 * scale_shift = [scale_0..scale_{K-1}, shift_0..shift_{K-1}]. */
ORACLE_API void oracle_requant(const int32_t *acc, int64_t M, int64_t K,
                               const float *scale_shift, int relu, int bits,
                               uint8_t *y, int nthreads)
{
    int64_t row_bytes = K * bits / 8;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        int8_t q[8192];
        for (int64_t k = 0; k < K; ++k)
            q[k] = (int8_t)oracle_requant_value(acc[m * K + k], scale_shift[k],
                                                scale_shift[K + k], relu, bits);
        oracle_pack(q, K, bits, y + m * row_bytes);
    }
}

/* As oracle_requant, with the residual add of reading 15: skip is a packed
 * [M, K*b/8] tensor (the same layout as y). */
ORACLE_API void oracle_requant_res(const int32_t *acc, int64_t M, int64_t K,
                                   const float *scale_shift, const uint8_t *skip, float res_scale,
                                   int relu, int bits, uint8_t *y, int nthreads)
{
    int64_t row_bytes = K * bits / 8;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        int8_t q[8192], sk[8192];
        oracle_unpack(skip + m * row_bytes, K, bits, sk);
        for (int64_t k = 0; k < K; ++k)
            q[k] = (int8_t)oracle_requant_res_value(acc[m * K + k], scale_shift[k], scale_shift[K + k],
                                                    sk[k], res_scale, relu, bits);
        oracle_pack(q, K, bits, y + m * row_bytes);
    }
}

/* ------------------------------------------------------------------------
 * Requantize into a code format (reading 16): as oracle_requant_value /
 * oracle_requant_res_value with the clamp bounds of the output format --
 * unsigned output codes: y = clamp(rne(v), 0, 2^b - 1) (the lower bound 0 is
 * the ReLU); signed: reading 4's bounds.
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_requant_value_fmt(int32_t acc, float scale, float shift, int relu, int bits, int y_uns)
{
    float f = (float)acc;
    float v = fmaf(f, scale, shift);
    float r = nearbyintf(v);
    float lo = (relu || y_uns) ? 0.0f : (float)code_lo(bits, 0);
    float c = fminf(fmaxf(r, lo), (float)code_hi(bits, y_uns));
    return (int)c;
}

ORACLE_API int oracle_requant_res_value_fmt(int32_t acc, float scale, float shift, int skip, float res_scale,
                                            int relu, int bits, int y_uns)
{
    float f = (float)acc;
    float u = fmaf(f, scale, shift);
    float v = fmaf((float)skip, res_scale, u);
    float r = nearbyintf(v);
    float lo = (relu || y_uns) ? 0.0f : (float)code_lo(bits, 0);
    float c = fminf(fmaxf(r, lo), (float)code_hi(bits, y_uns));
    return (int)c;
}

/* [M, K] accumulators -> packed rows of format y_uns; with skip != NULL the
 * residual add of reading 15, the skip codes read in format skip_uns. */
ORACLE_API void oracle_requant_fmt(const int32_t *acc, int64_t M, int64_t K, const float *scale_shift,
                                   const uint8_t *skip, int skip_uns, float res_scale,
                                   int relu, int bits, int y_uns, uint8_t *y, int nthreads)
{
    int64_t row_bytes = K * bits / 8;
#pragma omp parallel for num_threads(nthreads) schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        int16_t q[8192], sk[8192];
        if (skip) oracle_unpack_fmt(skip + m * row_bytes, K, bits, skip_uns, sk);
        for (int64_t k = 0; k < K; ++k)
            q[k] = (int16_t)(skip ? oracle_requant_res_value_fmt(acc[m * K + k], scale_shift[k], scale_shift[K + k],
                                                                 sk[k], res_scale, relu, bits, y_uns)
                                  : oracle_requant_value_fmt(acc[m * K + k], scale_shift[k], scale_shift[K + k],
                                                             relu, bits, y_uns));
        oracle_pack_fmt(q, K, bits, y + m * row_bytes);
    }
}

/* The whole per-layer path: conv_s32 then requant+pack. */
ORACLE_API int oracle_conv_q(const uint8_t *x, const uint8_t *w,
                             int64_t N, int64_t H, int64_t W, int64_t C,
                             int64_t K, int64_t R, int64_t S,
                             int64_t stride, int64_t pad, int bits,
                             const float *scale_shift, int relu,
                             const int64_t *pix_list, int64_t npix,
                             uint8_t *y, int nthreads)
{
    int64_t P = oracle_out_dim(H, R, stride, pad);
    int64_t Q = oracle_out_dim(W, S, stride, pad);
    int64_t M = pix_list ? npix : N * P * Q;
    int32_t *acc = (int32_t *)malloc((size_t)(M * K) * sizeof(int32_t));
    if (!acc) return -2;
    int rc = oracle_conv_s32(x, w, N, H, W, C, K, R, S, stride, pad, bits,
                             pix_list, npix, acc, nthreads);
    oracle_requant(acc, M, K, scale_shift, relu, bits, y, nthreads);
    free(acc);
    return rc;
}

/* ------------------------------------------------------------------------
 * Max pooling over packed codes (the pooling glue between the stem conv and
 * layer1 of ResNet; section 1 evaluates
 * "ResNet-18 and ResNet-50", whose stem is conv1 -> 3x3/2 max pool).
 *   y[n,p,q,c] = max over the in-range taps (r,s) of x[n, p*st-pad+r, q*st-pad+s, c]
 * Out-of-range taps are skipped (the padding never wins; torch semantics).
 * Quantization is monotone, so the max of the codes is the code of the max.
 * Output spatial size: floor form (reading 6).  Returns -1 if some window has
 * no in-range tap (not possible for pad < R), else 0.
 * ---------------------------------------------------------------------- */
ORACLE_API int oracle_maxpool_fmt(const uint8_t *x, int64_t N, int64_t H, int64_t W, int64_t C,
                                  int64_t R, int64_t stride, int64_t pad, int bits, int uns,
                                  uint8_t *y, int nthreads)
{
    int64_t P = oracle_out_dim(H, R, stride, pad);
    int64_t Q = oracle_out_dim(W, R, stride, pad);
    int64_t row_bytes = C * bits / 8;
    int empty = 0;
#pragma omp parallel for num_threads(nthreads) schedule(static) reduction(| : empty)
    for (int64_t m = 0; m < N * P * Q; ++m) {
        int64_t n = m / (P * Q), p = (m / Q) % P, q = m % Q;
        int16_t best[4096], v[4096];   /* codes compared in their format (reading 16) */
        int any = 0;
        for (int64_t r = 0; r < R; ++r) {
            int64_t h = p * stride - pad + r;
            if (h < 0 || h >= H) continue;
            for (int64_t s = 0; s < R; ++s) {
                int64_t w = q * stride - pad + s;
                if (w < 0 || w >= W) continue;
                oracle_unpack_fmt(x + ((n * H + h) * W + w) * row_bytes, C, bits, uns, v);
                for (int64_t c = 0; c < C; ++c)
                    if (!any || v[c] > best[c]) best[c] = v[c];
                any = 1;
            }
        }
        if (!any) { empty |= 1; memset(best, 0, (size_t)C * sizeof(int16_t)); }
        oracle_pack_fmt(best, C, bits, y + m * row_bytes);
    }
    return empty ? -1 : 0;
}

ORACLE_API int oracle_maxpool(const uint8_t *x, int64_t N, int64_t H, int64_t W, int64_t C,
                              int64_t R, int64_t stride, int64_t pad, int bits,
                              uint8_t *y, int nthreads)
{
    return oracle_maxpool_fmt(x, N, H, W, C, R, stride, pad, bits, 0, y, nthreads);
}
