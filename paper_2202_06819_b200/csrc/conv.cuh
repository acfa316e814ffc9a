// conv.cuh -- the implicit-GEMM quantized convolution kernel for sm_100a.
//
// GEMM view (section 2.1): rows m = (n,p,q) output pixels
// (M = N*P*Q), columns = K output channels, depth = R*S*C.  The im2col matrix
// (Fig. 1) is never materialized: each k-block's A tile (BM
// consecutive output pixels x KCH channels of one filter tap (r,s)) is fetched
// by one TMA im2col-mode load from the packed NHWC input; out-of-bounds taps
// (zero padding) are zero-filled by the TMA unit and never read from HBM.
// The T4 design's block/warp/WMMA-atom tiling (Fig. 1) becomes
// one CTA tile = one tcgen05.mma M=128 x N=BN instruction stream, accumulating
// s32 in TMEM; the register-level packing of section 3.2
// becomes a per-thread epilogue: tcgen05.ld gives a thread one output pixel's
// BN channels, so requantize + pack happen in registers with no shuffles, and
// the packed tile (BITS/32 of the s32 size, Fig. 7) is staged in
// shared memory and written by one TMA store straight into the next layer's
// packed NHWC layout (section 3.3's layout consistency).
//
// INT4: sm_100a has no 4-bit integer MMA kind (tcgen05 kinds: f16, tf32,
// f8f6f4, i8).  Packed s4 tiles are TMA-loaded at half the bytes, then a
// transform warpgroup expands every nibble v to the byte 16*v (exact s8) in the
// UMMA swizzled layout; both operands are scaled by 16, so the accumulator
// holds 256*acc and the epilogue shifts it back (exact).
//
// Warp roles (persistent CTA, one per SM):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane)
//   warps 2..    epilogue: 4 warpgroups (INT8) / 2 (INT4), each warp owning the
//                32 TMEM lanes (= tile rows = output pixels) of its quadrant
//   last 4 warps INT4 only: s4 -> s8 transform
// Pipelines: smem ring full/empty(/ready) mbarriers; TMEM double-buffered
// accumulator acc_full/acc_empty; buffer b is drained by its own warpgroups,
// so the requantization of two tiles and the mainloop of a third overlap.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include "ptx.cuh"

namespace convq {

constexpr int BM = 128;
constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA

struct ConvParams {
    int N, H, W, C, K, R, S, stride, pad;
    int P, Q;
    int M;          // N*P*Q
    int row_bytes;  // packed bytes per input pixel row = C*BITS/8
    int num_cblk;   // channel chunks per tap = C / KCH
    int num_kb;     // k-blocks per tile = R*S*num_cblk
    int n_tiles;    // ceil(K / BN)
    int num_tiles;  // m_tiles * n_tiles
    int relu;
    int cvt_magic;       // |acc| <= 2^22 guaranteed: int->float via the 1.5*2^23 add (FMA pipe)
    int one;             // = 1, opaque to the compiler (keeps an integer add on the FMA pipe)
    const float *scale;  // [2K] scale then shift
    int32_t *y32;        // s32 output (OUT_S32)
};

template <int BITS, int BN, int KCH, int OUT_S32, int CG>
struct ConvCfg {
    // CG = CTAs per tile (1, or 2 = a CTA pair running tcgen05.mma.cta_group::2
    // with M = 256: each CTA stages its own 128 A rows and BN/2 B rows).
    static constexpr int BNL = BN / CG;                     // B rows staged per CTA
    static constexpr int LOAD_ROW = KCH * BITS / 8;        // packed bytes per row per k-block
    static constexpr int A_S8 = BM * KCH;                   // s8 A tile bytes
    static constexpr int B_S8 = BNL * KCH;
    static constexpr int A_PK = BITS == 4 ? BM * LOAD_ROW : 0;
    static constexpr int B_PK = BITS == 4 ? BNL * LOAD_ROW : 0;
    static constexpr int STAGE_BYTES = A_S8 + B_S8 + A_PK + B_PK;
    static constexpr int STAGE_TX = (BM + BNL) * LOAD_ROW;   // TMA bytes per stage per CTA
    static constexpr int OUT_ROW = BN * BITS / 8;            // packed output bytes per pixel row
    static constexpr int OUT_SUBW = OUT_ROW < 128 ? OUT_ROW : 128;  // TMA store box width
    static constexpr int OUT_NSUB = OUT_ROW / OUT_SUBW;
    static constexpr int OUT_BYTES = OUT_S32 ? 0 : BM * OUT_ROW;   // staging per TMEM buffer
    static constexpr int NUM_EPI = BITS == 8 ? 4 : 2;               // epilogue warpgroups
    static constexpr int EPI_PER_BUF = NUM_EPI / 2;                 // warpgroups per TMEM buffer
    static constexpr int EPI_COLS = BN / EPI_PER_BUF;               // columns one warpgroup drains
    static constexpr int CW = BITS == 8 ? 16 : 32;                  // columns per tcgen05.ld (16 B packed)
    static constexpr int SS_BYTES = OUT_S32 ? 0 : 2 * BN * 4;       // scale+shift of one n-block
    static constexpr int BAR_BYTES = 1024;
    static constexpr int STAGES_FIT = (SMEM_LIMIT - 1024 - BAR_BYTES - 2 * (OUT_BYTES + SS_BYTES)) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 12 ? 12 : STAGES_FIT;
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 2 * (OUT_BYTES + SS_BYTES) + BAR_BYTES;
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int EPI_WARP0 = 2;                             // warps 2..: epilogue warpgroups
    static constexpr int XF_WARP0 = EPI_WARP0 + 4 * NUM_EPI;        // INT4 transform warps
    static constexpr int NUM_THREADS = 32 * (XF_WARP0 + (BITS == 4 ? 4 : 0));
    static constexpr uint32_t IDESC = idesc_i8(BM * CG, BN);
    static_assert(STAGES >= 2, "tile does not fit shared memory");
    static_assert(KCH == 32 || KCH == 64 || KCH == 128, "KCH");
    static_assert(BN % (32 * CG) == 0 && BN >= 32 * CG && BN <= 256, "BN");
    static_assert(CG == 1 || CG == 2, "CG");
    static_assert(TMEM_COLS <= 512, "TMEM");
};

// Swizzle<B,4,3> on a byte offset inside a tile whose rows are `span` bytes
// (span = 128/64/32 -> SW128/SW64/SW32, 16 -> none): XOR the 16-byte chunk
// index with the 128-byte-line index bits, as TMA and UMMA both apply it.
template <int SPAN>
__device__ __forceinline__ uint32_t swz(uint32_t off) {
    constexpr uint32_t MASK = SPAN / 16 - 1;
    return off ^ (((off >> 7) & MASK) << 4);
}

// s4 nibbles -> s8 bytes holding 16*v (nibble moved to the high half).
// w: 8 nibbles, channel i at bits [4i,4i+4).  lo/hi: channels 0-3 / 4-7.
__device__ __forceinline__ void expand_s4(uint32_t w, uint32_t &lo, uint32_t &hi) {
    uint32_t even = (w << 4) & 0xF0F0F0F0u;  // byte i = nibble 2i << 4
    uint32_t odd = w & 0xF0F0F0F0u;          // byte i = nibble 2i+1 << 4
    lo = __byte_perm(even, odd, 0x5140);
    hi = __byte_perm(even, odd, 0x7362);
}

// Expand a packed s4 tile [rows][KCH/2 bytes] (TMA-swizzled for its span) into
// an s8 tile [rows][KCH bytes] in the UMMA K-major swizzled layout.
template <int KCH>
__device__ __forceinline__ void expand_tile(const uint8_t *src, uint8_t *dst, int rows, int tid, int nthr) {
    constexpr int PW = KCH / 2;      // packed row bytes
    constexpr int PPR = PW / 16;     // 16-byte pieces per packed row
    for (int i = tid; i < rows * PPR; i += nthr) {
        int row = i / PPR, j = i - row * PPR;
        uint4 v = *reinterpret_cast<const uint4 *>(src + swz<PW>(row * PW + j * 16));
        uint32_t o[8];
        expand_s4(v.x, o[0], o[1]);
        expand_s4(v.y, o[2], o[3]);
        expand_s4(v.z, o[4], o[5]);
        expand_s4(v.w, o[6], o[7]);
        *reinterpret_cast<uint4 *>(dst + swz<KCH>(row * KCH + (2 * j) * 16)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4 *>(dst + swz<KCH>(row * KCH + (2 * j + 1) * 16)) = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

// Requantize (section 3.2.2; DESIGN readings 4-5):
//   y = clamp(rne(fmaf((float)acc, scale, shift)), lo, hi)
// computed without the quarter-rate FRND/F2I conversions: clamp first (the
// bounds are integers, so clamp-then-round == round-then-clamp, and NaN -> lo
// through max.f32 either way), then add 1.5*2^23: for |u| <= 2^22 the IEEE
// add rounds u to the nearest integer (ties to even) and leaves it, two's
// complement, in the low mantissa bits.  Returns those bits; the caller
// takes the low byte / nibble as the packed code.
constexpr float RNE_MAGIC = 12582912.0f;  // 1.5 * 2^23
// (float)acc, exact, for |acc| <= 2^22: the word 0x4B400000 + acc is the
// float 1.5*2^23 + acc; subtracting 1.5*2^23 is exact.  Both steps run on the
// FMA pipe (integer multiply-add by a runtime 1 that the compiler cannot fold
// into an ALU add, then a float add) instead of one ALU-pipe I2FP: the
// epilogue is ALU-bound (FMNMX clamps, PRMT packing).
__device__ __forceinline__ float small_int_to_float(int acc, int one) {
    int w;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(w) : "r"(acc), "r"(one), "r"(0x4B400000));
    return __fsub_rn(__int_as_float(w), RNE_MAGIC);
}
template <bool MAGIC>
__device__ __forceinline__ uint32_t requant_bits(int acc, float sc, float sh, float lo, float hi, int one) {
    float f = MAGIC ? small_int_to_float(acc, one) : __int2float_rn(acc);
    float u = __fmaf_rn(f, sc, sh);
    u = fminf(fmaxf(u, lo), hi);
    return __float_as_uint(__fadd_rn(u, RNE_MAGIC));
}
// low bytes of four requant_bits results -> one packed s8 word
__device__ __forceinline__ uint32_t pack4_low_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// low nibbles of eight requant_bits results -> one packed s4 word
__device__ __forceinline__ uint32_t pack8_low_nibbles(const uint32_t *r) {
    uint32_t b01 = (r[0] & 0xFu) | ((r[1] << 4) & 0xF0u);
    uint32_t b23 = (r[2] & 0xFu) | ((r[3] << 4) & 0xF0u);
    uint32_t b45 = (r[4] & 0xFu) | ((r[5] << 4) & 0xF0u);
    uint32_t b67 = (r[6] & 0xFu) | ((r[7] << 4) & 0xF0u);
    return __byte_perm(__byte_perm(b01, b23, 0x0040), __byte_perm(b45, b67, 0x0040), 0x5410);
}

template <int BITS, int BN, int KCH, int OUT_S32, int CG>
__global__ void __launch_bounds__(ConvCfg<BITS, BN, KCH, OUT_S32, CG>::NUM_THREADS, 1)
    conv_igemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_y, const ConvParams p) {
    using Cfg = ConvCfg<BITS, BN, KCH, OUT_S32, CG>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by offset (pointer arithmetic on the shared array keeps
    // the compiler's shared-space inference: LDS/STS instead of generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

    // ---- carve shared memory (every tile 1024-byte aligned; identical offsets
    // in both CTAs of a pair, as cta_group::2 descriptors require)
    uint8_t *a_s8 = smem;                               // [STAGES][BM*KCH]
    uint8_t *b_s8 = a_s8 + STAGES * Cfg::A_S8;          // [STAGES][BNL*KCH]
    uint8_t *a_pk = b_s8 + STAGES * Cfg::B_S8;          // INT4: [STAGES][BM*KCH/2]
    uint8_t *b_pk = a_pk + STAGES * Cfg::A_PK;          // INT4: [STAGES][BNL*KCH/2]
    uint8_t *out_stage = b_pk + STAGES * Cfg::B_PK;     // [2][OUT_NSUB][BM][OUT_SUBW]
    float *ss_smem = reinterpret_cast<float *>(out_stage + 2 * Cfg::OUT_BYTES);  // [2][2*BN]
    uint64_t *bars = reinterpret_cast<uint64_t *>(out_stage + 2 * (Cfg::OUT_BYTES + Cfg::SS_BYTES));
    uint64_t *full = bars;                  // TMA -> (transform | MMA)
    uint64_t *empty = bars + STAGES;        // MMA -> TMA
    uint64_t *ready = bars + 2 * STAGES;    // transform -> MMA (INT4)
    uint64_t *acc_full = bars + 3 * STAGES; // MMA -> epilogue [2]
    uint64_t *acc_empty = acc_full + 2;     // epilogue -> MMA [2]
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(acc_empty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;     // position in the CTA pair
    const int tile0 = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
    const int tstep = CG == 2 ? (int)num_clusters_x() : (int)gridDim.x;
    // INT8 pairs count both CTAs' TMA bytes on the leader's full barrier; INT4
    // pairs expand locally, then both CTAs' transform warps arrive on the
    // leader's ready barrier.
    constexpr bool PAIR_TX = CG == 2 && BITS == 8;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tm_a);
        tma_prefetch_desc(&tm_b);
        if (!OUT_S32) tma_prefetch_desc(&tm_y);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&ready[s], 4 * CG);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4 * Cfg::EPI_PER_BUF * CG);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (CG == 2) tmem_alloc_cg2<Cfg::TMEM_COLS>(tmem_holder);
        else tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();   // barriers of both CTAs initialised before any remote use
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    const int PQ = p.P * p.Q;

    if (warp == 0) {
        // =========================== TMA producer ===========================
        if (lane == 0) {
            const uint64_t pol_a = policy_evict_normal();  // activations: re-read by R*S taps and n-tiles
            const uint64_t pol_b = policy_evict_last();    // weights: re-read by every m-tile
            uint8_t *a_dst = BITS == 4 ? a_pk : a_s8;
            uint8_t *b_dst = BITS == 4 ? b_pk : b_s8;
            constexpr int A_LD = BITS == 4 ? Cfg::A_PK : Cfg::A_S8;
            constexpr int B_LD = BITS == 4 ? Cfg::B_PK : Cfg::B_S8;
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                const int m_blk = tile / p.n_tiles, n_blk = tile - m_blk * p.n_tiles;
                const int m0 = m_blk * (BM * CG) + (int)rank * BM;   // this CTA's first output pixel
                const int n0 = m0 / PQ, rem = m0 - n0 * PQ;
                const int p0 = rem / p.Q, q0 = rem - p0 * p.Q;
                const int h0 = p0 * p.stride - p.pad, w0 = q0 * p.stride - p.pad;
                const int brow = n_blk * BN + (int)rank * Cfg::BNL;  // this CTA's B rows
                int r = 0, s = 0, cblk = 0, kcol = 0;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if constexpr (PAIR_TX) {
                        const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], CG * Cfg::STAGE_TX);
                        tma_load_im2col_4d_cg2(a_dst + stage * A_LD, &tm_a, fb, cblk * Cfg::LOAD_ROW, w0, h0, n0,
                                               (uint16_t)s, (uint16_t)r, pol_a);
                        tma_load_2d_cg2(b_dst + stage * B_LD, &tm_b, fb, kcol + cblk * Cfg::LOAD_ROW, brow, pol_b);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_TX);
                        tma_load_im2col_4d(a_dst + stage * A_LD, &tm_a, &full[stage], cblk * Cfg::LOAD_ROW, w0, h0, n0,
                                           (uint16_t)s, (uint16_t)r, pol_a);
                        tma_load_2d(b_dst + stage * B_LD, &tm_b, &full[stage], kcol + cblk * Cfg::LOAD_ROW, brow,
                                    pol_b);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    if (++cblk == p.num_cblk) {            // next filter tap (r, s)
                        cblk = 0;
                        kcol += p.row_bytes;
                        if (++s == p.S) { s = 0; ++r; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // =========================== MMA issuer =============================
        if (lane == 0 && rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep, ++local) {
                const int buf = local & 1;
                const uint32_t aphase = (local >> 1) & 1;
                mbar_wait(&acc_empty[buf], aphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + buf * BN;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(BITS == 4 ? &ready[stage] : &full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(a_s8 + stage * Cfg::A_S8);
                    const uint32_t b_addr = smem_u32(b_s8 + stage * Cfg::B_S8);
#pragma unroll
                    for (int k = 0; k < KCH / 32; ++k) {
                        const uint64_t ad = umma_desc_kmajor(a_addr + 32 * k, KCH);
                        const uint64_t bd = umma_desc_kmajor(b_addr + 32 * k, KCH);
                        if constexpr (CG == 2) mma_i8_cg2(d_tmem, ad, bd, Cfg::IDESC, (kb | k) != 0);
                        else mma_i8(d_tmem, ad, bd, Cfg::IDESC, (kb | k) != 0);
                    }
                    // frees the smem stage (in both CTAs) when these MMAs complete
                    if constexpr (CG == 2) mma_commit_cg2_mc(&empty[stage], 0x3);
                    else mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                // accumulator ready for the epilogue (of both CTAs)
                if constexpr (CG == 2) mma_commit_cg2_mc(&acc_full[buf], 0x3);
                else mma_commit(&acc_full[buf]);
            }
        }
    } else if (warp < Cfg::XF_WARP0) {
        // =========================== epilogue ===============================
        // TMEM buffer b (every other tile) is drained by EPI_PER_BUF warpgroups,
        // each owning EPI_COLS of its BN columns; each buffer has its own
        // staging tile and scale/shift copy, so one buffer's TMA store and the
        // other buffer's requantization overlap.  In a CTA pair each CTA drains
        // its own 128 rows (its TMEM half) and releases the leader's buffer.
        constexpr int EPB = Cfg::EPI_PER_BUF;
        const int e = (warp - Cfg::EPI_WARP0) >> 2;
        const int b = e / EPB;                     // TMEM buffer
        const int half = e % EPB;                  // column part
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;          // tile row = output pixel
        const int ptid = (e % EPB) * 128 + (threadIdx.x & 127);  // thread index within the buffer's group
        const bool leader = ptid == 0;
        const uint32_t bar_id = 1 + b, bar_n = 128 * EPB;
        uint8_t *stage_b = out_stage + b * Cfg::OUT_BYTES;
        float *ss_b = ss_smem + b * 2 * BN;
        const uint32_t acc_empty_leader = CG == 2 ? mapa_shared(smem_u32(&acc_empty[b]), 0) : 0;
        const float lo = p.relu ? 0.f : -(float)(1 << (BITS - 1));
        const float hi = (float)((1 << (BITS - 1)) - 1);
        const int one = p.one;
        int j = 0;
        for (int tile = tile0 + b * tstep; tile < p.num_tiles; tile += 2 * tstep, ++j) {
            const int m_blk = tile / p.n_tiles, n_blk = tile - m_blk * p.n_tiles;
            const int mrow0 = m_blk * (BM * CG) + (int)rank * BM;
            const int m = mrow0 + row;
            if (!OUT_S32) {
                if (leader) tma_store_wait_read0();   // staging of this buffer's previous tile read out
                for (int i = ptid; i < 2 * BN; i += bar_n) {   // this n-block's scale and shift
                    const int col = n_blk * BN + (i % BN);
                    ss_b[i] = col < p.K ? __ldg(p.scale + (i < BN ? 0 : p.K) + col) : 0.f;
                }
                named_bar_sync(bar_id, bar_n);
            }
            mbar_wait(&acc_full[b], j & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + b * BN + half * Cfg::EPI_COLS;
#pragma unroll 1
            for (int c = 0; c < Cfg::EPI_COLS / Cfg::CW; ++c) {
                uint32_t v[Cfg::CW];
                if constexpr (Cfg::CW == 16) tmem_ld_32x32b_x16(taddr + c * Cfg::CW, v);
                else tmem_ld_32x32b_x32(taddr + c * Cfg::CW, v);
                if (c == Cfg::EPI_COLS / Cfg::CW - 1) {  // this group's columns are in registers
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(acc_empty_leader);
                        else mbar_arrive(&acc_empty[b]);
                    }
                }
                const int ccol = half * Cfg::EPI_COLS + c * Cfg::CW;   // column within the tile
                const int col0 = n_blk * BN + ccol;
                if (OUT_S32) {
                    if (m < p.M) {
                        int32_t *dst = p.y32 + (int64_t)m * p.K + col0;
                        if (col0 + Cfg::CW <= p.K) {
#pragma unroll
                            for (int q = 0; q < Cfg::CW; q += 4) {
                                int4 t;
                                t.x = BITS == 4 ? ((int)v[q] >> 8) : (int)v[q];
                                t.y = BITS == 4 ? ((int)v[q + 1] >> 8) : (int)v[q + 1];
                                t.z = BITS == 4 ? ((int)v[q + 2] >> 8) : (int)v[q + 2];
                                t.w = BITS == 4 ? ((int)v[q + 3] >> 8) : (int)v[q + 3];
                                *reinterpret_cast<int4 *>(dst + q) = t;
                            }
                        } else {
                            for (int q = 0; q < Cfg::CW && col0 + q < p.K; ++q)
                                dst[q] = BITS == 4 ? ((int)v[q] >> 8) : (int)v[q];
                        }
                    }
                } else {
                    uint32_t r[Cfg::CW];
                    const float4 *s4 = reinterpret_cast<const float4 *>(ss_b + ccol);
                    const float4 *h4 = reinterpret_cast<const float4 *>(ss_b + BN + ccol);
                    auto requant_chunk = [&](auto magic) {
#pragma unroll
                        for (int q = 0; q < Cfg::CW / 4; ++q) {
                            const float4 sa = s4[q], sb = h4[q];
                            const int x0 = BITS == 4 ? ((int)v[4 * q] >> 8) : (int)v[4 * q];
                            const int x1 = BITS == 4 ? ((int)v[4 * q + 1] >> 8) : (int)v[4 * q + 1];
                            const int x2 = BITS == 4 ? ((int)v[4 * q + 2] >> 8) : (int)v[4 * q + 2];
                            const int x3 = BITS == 4 ? ((int)v[4 * q + 3] >> 8) : (int)v[4 * q + 3];
                            r[4 * q] = requant_bits<decltype(magic)::value>(x0, sa.x, sb.x, lo, hi, one);
                            r[4 * q + 1] = requant_bits<decltype(magic)::value>(x1, sa.y, sb.y, lo, hi, one);
                            r[4 * q + 2] = requant_bits<decltype(magic)::value>(x2, sa.z, sb.z, lo, hi, one);
                            r[4 * q + 3] = requant_bits<decltype(magic)::value>(x3, sa.w, sb.w, lo, hi, one);
                        }
                    };
                    if (p.cvt_magic) requant_chunk(std::true_type{});
                    else requant_chunk(std::false_type{});
                    // 16 packed bytes = this chunk (16 s8 or 32 s4 columns)
                    const int byte0 = ccol * BITS / 8;
                    uint8_t *sub = stage_b + (byte0 / Cfg::OUT_SUBW) * (BM * Cfg::OUT_SUBW);
                    const int inrow = byte0 % Cfg::OUT_SUBW;
                    uint4 pk;
                    if constexpr (BITS == 8) {
                        pk = make_uint4(pack4_low_bytes(r[0], r[1], r[2], r[3]), pack4_low_bytes(r[4], r[5], r[6], r[7]),
                                        pack4_low_bytes(r[8], r[9], r[10], r[11]),
                                        pack4_low_bytes(r[12], r[13], r[14], r[15]));
                    } else {
                        pk = make_uint4(pack8_low_nibbles(r), pack8_low_nibbles(r + 8), pack8_low_nibbles(r + 16),
                                        pack8_low_nibbles(r + 24));
                    }
                    *reinterpret_cast<uint4 *>(sub + swz<Cfg::OUT_SUBW>(row * Cfg::OUT_SUBW + inrow)) = pk;
                }
            }
            if (!OUT_S32) {
                fence_proxy_async_smem();  // st.shared -> visible to the TMA (async proxy)
                named_bar_sync(bar_id, bar_n);
                if (leader) {
#pragma unroll
                    for (int s = 0; s < Cfg::OUT_NSUB; ++s)
                        tma_store_2d(&tm_y, stage_b + s * (BM * Cfg::OUT_SUBW), n_blk * Cfg::OUT_ROW + s * Cfg::OUT_SUBW,
                                     mrow0);
                    tma_store_commit();
                }
            }
        }
        if (!OUT_S32 && leader) tma_store_wait0();
    } else {
        // =========================== INT4 transform =========================
        if constexpr (BITS == 4) {
            const int tid = threadIdx.x - 32 * Cfg::XF_WARP0;  // 0..127
            const uint32_t ready0 = CG == 2 ? mapa_shared(smem_u32(&ready[0]), 0) : 0;
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    expand_tile<KCH>(a_pk + stage * Cfg::A_PK, a_s8 + stage * Cfg::A_S8, BM, tid, 128);
                    expand_tile<KCH>(b_pk + stage * Cfg::B_PK, b_s8 + stage * Cfg::B_S8, Cfg::BNL, tid, 128);
                    fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05.mma
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(ready0 + 8u * stage);
                        else mbar_arrive(&ready[stage]);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();   // the pair's MMAs and remote arrivals are complete
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_cg2<Cfg::TMEM_COLS>(tmem_base);
        else tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace convq
