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
// Stages: one pipeline stage holds NSUB k-blocks (each a (tap, channel-block)
// pair: KCH channels of one filter tap), filled by NSUB im2col + NSUB weight
// loads, consumed by NSUB*KCH/32 MMAs and released by ONE tcgen05.commit: the
// issuing thread's per-stage handshake (barrier wait + commit, several hundred
// cycles) is amortised over >= ~1000 cycles of tensor work.
//
// Warp roles (persistent CTA, one per SM; CG = 2: a CTA pair per tile):
//   warps 0..    epilogue: 4 warpgroups (INT8) / 2 (INT4), each warp owning the
//                32 TMEM lanes (= tile rows = output pixels) of its quadrant
//   next 4 warps INT4 only: s4 -> s8 transform
//   next warp    TMA producer (converged warp, one elected lane issues)
//   last warp    TMEM allocator + MMA issuer (converged warp, one elected lane)
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
#ifndef CONVQ_MMA_1T
#define CONVQ_MMA_1T 0
#endif
constexpr bool kMma1T = CONVQ_MMA_1T != 0;
// Two MMA-issuing warps taking alternate tiles (CONVQ_DUAL_MMA=1; OFF by default:
// parity-green, but the ResNet-50 step measured no faster -- 1.40 vs 1.34-1.38 ms): a
// warp's per-tile control path (barrier waits, fences, commits: ~650-700 cycles,
// profiles/r01_timeline_cta0.txt) then overlaps the other warp's MMA execution
// instead of adding to it.  Tile t: warp t % 2, TMEM buffer t % NBUF, smem
// stages from t * (stages per tile) -- fixed when every unit has the same K range.
#ifndef CONVQ_DUAL_MMA
#define CONVQ_DUAL_MMA 0
#endif
constexpr int kNumMma = CONVQ_DUAL_MMA ? 2 : 1;
#ifdef CONVQ_INSTRUMENT
constexpr bool kInstrument = true;
#else
constexpr bool kInstrument = false;
#endif
// per-CTA trace counters (cycles): where the control loops wait
enum { TR_PROD_EMPTY = 0, TR_MMA_FULL, TR_MMA_ACC, TR_EPI_ACC, TR_MMA_ISSUE, TR_TOTAL, TR_TILES, TR_T0, TR_T1,
       TR_TPDL, TR_TFULL, TR_TACC, TR_EPI_SLAB, TR_EPI_BODY, TR_EPI_STORE, TR_SLOTS = 15 };
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA


struct ConvParams {
    int N, H, W, C, K, R, S, stride, pad;
    int pad_w;      // left padding of the im2col W walk (= pad, or 0 for the space-to-depth stem's window view)
    int P, Q;
    int M;          // N*P*Q
    int row_bytes;  // packed bytes per input pixel row = C*BITS/8
    int num_cblk;   // channel chunks per tap = ceil(C / KCH)
    int num_kb;     // k-blocks per tile = R*S*num_cblk
    int n_tiles;    // ceil(K / BN)
    int num_tiles;  // m_tiles * n_tiles
    int relu;
    int rotate;          // rotate each CTA's k-block start (see the producer)
    int a_gemm;          // 1x1 / stride 1 / pad 0: A is the input as a [M][C] matrix (tiled TMA, no im2col)
    int probe;           // measurement only (bits): 1 = no MMAs, 2 = no loads, 4 = no epilogue work
    int epi_wait;        // epilogue acc_full wait: 0 spin, 1 suspend-time hint, 2 nanosleep back-off
    int out_policy;      // L2 policy of the packed output stores: 0 none, 1 evict_last, 2 evict_first
    unsigned epi_wait_ns;
    unsigned long long *trace;  // measurement only: per-CTA wait-cycle counters (TRACE_SLOTS each), or null
    unsigned long long *tl;     // measurement only: CTA 0's event timeline (clock64), [64 regions][256], or null
    // duplicate-aware (halo) mode, stride 1 only:
    int Wp;              // padded input width W + 2 pad = MMA-row pitch of an output row
    int rpt;             // output rows per 128-row tile
    int tiles_per_img;   // ceil(P / rpt)
    int m_tiles;         // N * tiles_per_img
    int halo_tx;         // bytes of one halo TMA box
    const float *scale;  // [2K] scale then shift
    const uint8_t *skip; // OUT_RES: packed skip tensor [M][K*BITS/8] (the output's layout), read by the epilogue
    float res_scale;     // OUT_RES: the skip code's scale relative to the output's (DESIGN reading 15)
    // code formats (DESIGN reading 16, unsigned post-ReLU codes)
    int x_uns;           // activations are unsigned codes: A format u8 in the instruction descriptor
    int y_uns;           // output codes are unsigned: clamp to [0, 2^b - 1]
    int code_hi;         // INT4 ReLU epilogue: the largest output code (7 signed, 15 unsigned)
    uint32_t skip_xor;   // OUT_RES: code -> biased unsigned (0x80 / 0x8 per code for signed skips, 0 unsigned)
    float skip_off;      // OUT_RES: 2^23 + that bias (the skip code as an exact float, see the epilogue)
    int32_t *y32;        // s32 output (OUT = OUT_S32)
    uint8_t *y8;         // packed output for direct stores (OUT = OUT_DIRECT)
    int out_row;         // packed output bytes per pixel row = K*BITS/8
    // split-K (stream-K style work units, "the dimension of K is
    // reduced"): a tile's k-blocks are cut into `splits` ranges processed by
    // different CTAs; partial s32 sums meet in `ws` and the last arriving
    // warp of each 32-row region requantizes.  splits = 1: plain tiles.
    int splits;
    int num_units;       // num_tiles * splits
    // shared-memory carve-up chosen on the host (plan.cuh launch_conv): the
    // weight-stationary region is sized to THIS layer's weight block (not the
    // 64 KB budget), and every byte left over goes to pipeline stages
    int stages;          // smem ring depth, 2 <= stages <= MAX_STAGES
    int wsb;             // bytes of the resident weight regions (WS; s8 block + INT4 packed block)
    int wsb_s8;          // bytes of the s8 resident block (the INT4 packed block follows it)
    // Cross-launch completion counters (conv_q_plan_set_deps; NULL dep_in = wait for
    // the whole previous grid with griddepcontrol.wait): dep_in counts the input
    // tensor's codes in memory (complete at dep_in_total = N*H*W*C), dep_skip the
    // residual skip's (dep_skip_total = N*P*Q*K); every epilogue warp adds the codes
    // it wrote to dep_out once its stores are complete.
    const unsigned *dep_in;
    const unsigned *dep_skip;
    unsigned *dep_out;
    unsigned dep_in_total, dep_skip_total;
    int halo_rows;       // input rows of one halo box (halo modes)
    int32_t *ws;         // [num_tiles*CG][4*EPB regions][EPI_COLS][32] partial sums (kept zero between runs)
    unsigned *cnt;       // per-region arrival counters (kept zero between runs)
    FastDiv fd_ntiles, fd_PQ, fd_Q, fd_cblk, fd_S, fd_tpi, fd_splits, fd_Wp;
};

// Output path of the epilogue.
constexpr int OUT_TMA = 0;     // packed codes staged in smem, written by TMA stores
constexpr int OUT_S32 = 1;     // raw int32 accumulators, direct global stores (debug / parity)
constexpr int OUT_DIRECT = 2;
constexpr int OUT_RELU = 4;    // flag: INT8 ReLU-specialised epilogue (OUT_TMA | OUT_RELU, OUT_DIRECT | OUT_RELU)
constexpr int OUT_RES = 8;     // flag: fused residual add (OUT_TMA | OUT_RES, OUT_DIRECT | OUT_RES; runtime ReLU)
// flag with OUT_RELU, INT8: unsigned output codes (reading 16) -- F2IP.U8 saturates to
// [0, 255], which IS the ReLU + upper clamp (no sign masking)
constexpr int OUT_U = 16;

// Epilogue warpgroups (INT8: CONVQ_EPI_WG8, default 4; INT4: 2) and TMEM
// accumulator buffers (512 columns / BN, at most 4, at most one per warpgroup);
// shared with the host's TMA-store box computation (convq.cu).
#ifndef CONVQ_EPI_WG8
#define CONVQ_EPI_WG8 4
#endif
#ifndef CONVQ_EPI_WG4
#define CONVQ_EPI_WG4 2
#endif
// INT8 epilogue: double-buffered 32-column TMEM loads (A/B build option)
#ifndef CONVQ_TMEM_PIPE
#define CONVQ_TMEM_PIPE 0
#endif
// MMA warp, im2col / tiled path: commit a unit's accumulator only after the next
// unit's first stage of MMAs is issued (A/B build option)
#ifndef CONVQ_LATE_ACC
#define CONVQ_LATE_ACC 0
#endif
constexpr int epi_warpgroups(int bits) { return bits == 8 ? CONVQ_EPI_WG8 : CONVQ_EPI_WG4; }
constexpr int tmem_buffers(int bits, int bn) {
    return (512 / bn) < epi_warpgroups(bits) ? ((512 / bn) < 4 ? 512 / bn : 4)
                                              : (epi_warpgroups(bits) < 4 ? epi_warpgroups(bits) : 4);
}
// All-warps epilogue (CONVQ_EPI_ALLW, default on): with only two TMEM buffers
// (256-column accumulators) every INT8 epilogue warpgroup drains EVERY tile
// (BN/4 columns each) instead of half of them draining every other tile.  The
// buffer is then drained ~2x sooner and released to the MMA warp earlier --
// measured (profiles/r01_timeline_cta0.txt) the two-buffer 1x1 layers were
// paced by the epilogue's per-buffer drain time, not by its instruction rate.
#ifndef CONVQ_EPI_ALLW
#define CONVQ_EPI_ALLW 1
#endif
constexpr bool epi_all_warps(int bits, int nbuf) { return CONVQ_EPI_ALLW && bits == 8 && nbuf == 2; }
constexpr int epi_per_buf(int bits, int nbuf) {
    return epi_all_warps(bits, nbuf) ? epi_warpgroups(bits) : epi_warpgroups(bits) / nbuf;
}

template <int BITS, int BN, int KCH, int OUT, int CG, int NSUB, int HALO = 0>
struct ConvCfg {
    // CG = CTAs per tile (1, or 2 = a CTA pair running tcgen05.mma.cta_group::2
    // with M = 256: each CTA stages its own 128 A rows and BN/2 B rows).
    // HALO bit 0: duplicate-aware A operand (section 3.1, Alg. 1):
    // per (tile, channel block) ONE halo box of the padded input is loaded and
    // every filter tap reads its A rows as a shifted window of it.
    // HALO bit 1 (WS): weight-stationary -- every tile of a persistent CTA has the
    // same N block (grid = a multiple of the N-tile count), so the CTA loads its
    // BN x R*S*C weight block ONCE into a resident region and the pipeline
    // stages carry only activations (with bit 0: one halo box per stage).
    static constexpr bool HA = (HALO & 1) != 0;
    static constexpr bool WS = (HALO & 2) != 0;
    // HALO bit 2 (S2H, with WS): the s2d stem's window operand -- one tiled box of
    // consecutive 16-byte s2d pixels per tile; tap row jr and K step kk read it
    // through a SWIZZLE_NONE descriptor at pixel offset jr*Wp + 2*kk, LBO = 16 B
    static constexpr bool S2H = (HALO & 4) != 0;
    static constexpr bool HB = HA || S2H;                    // stage = one halo box
    // HALO bit 3 (MT2, weight-stationary halo modes): a work unit is TWO 128-row
    // m-groups -- one halo box covering both, MMAs into two BN-column TMEM halves,
    // one accumulator round trip (barrier waits, commits) per 256 rows: the MMA
    // warp's per-tile control path (~650 cycles) is amortised over twice the work
    static constexpr int MT = (HALO & 8) ? 2 : 1;
    static constexpr int TBW = MT * BN;                      // TMEM columns of one accumulator buffer
    static constexpr int WSB = WS ? 65536 : 0;               // resident weight region (budget; plan-time check)
    // INT4 weight-stationary: the packed block lands here once and the transform
    // warps expand it ONCE into the s8 resident region (not once per k-block stage)
    static constexpr int WSB_PK = WS && BITS == 4 ? WSB / 2 : 0;
    static constexpr int HBOX = WS && HB ? (KCH == 64 && MT == 1 ? 20480 : 32768) : 0;   // WS halo stage (budget)
    static constexpr int B_TILE = BN / CG * KCH;             // one resident k-block of this CTA's weight rows
    static constexpr int BNL = BN / CG;                     // B rows staged per CTA
    static constexpr int LOAD_ROW = KCH * BITS / 8;        // packed bytes per row per k-block
    static constexpr int A_SUB = HB ? HBOX : BM * KCH;      // s8 A sub-tile bytes (one k-block / WS halo box)
    static constexpr int B_SUB = WS ? 0 : BNL * KCH;
    static constexpr int AMT = HB ? 1 : MT;                 // A sub-tiles per k-block (generic MT2: one per m-group)
    static constexpr int A_S8 = NSUB * AMT * A_SUB;         // per stage
    static constexpr int B_S8 = NSUB * B_SUB;
    // packed INT4 A staging per k-block (halo modes: the box lives in the halo buffers --
    // or, weight-stationary, the packed box of the stage, expanded into the stage's s8 box)
    static constexpr int A_PK_SUB = BITS != 4 ? 0 : !HB ? BM * LOAD_ROW : (WS && HA ? HBOX / 2 : 0);
    static constexpr int B_PK_SUB = BITS == 4 && !WS ? BNL * LOAD_ROW : 0;
    static constexpr int A_PK = NSUB * AMT * A_PK_SUB;        // (generic MT2: one packed A tile per m-group)
    static constexpr int B_PK = NSUB * B_PK_SUB;
    static constexpr int STAGE_BYTES = A_S8 + B_S8 + A_PK + B_PK;
    static constexpr int SUB_TX = ((HB ? 0 : AMT * BM) + (WS ? 0 : BNL)) * LOAD_ROW;  // TMA bytes per k-block per CTA
    static constexpr int HALO_BYTES = HA && !WS ? 32768 : 0;  // one halo buffer (budget; checked at plan time)
    // INT4 halo: the TMA lands the packed s4 box here; the transform warps expand
    // it once per (tile, channel block) into the s8 halo buffer (not once per tap)
    static constexpr int HALO_PK = BITS == 4 ? HALO_BYTES / 2 : 0;
    static constexpr int OUT_ROW = BN * BITS / 8;            // packed output bytes per pixel row
    static constexpr int OUTP = OUT & 3;                     // output path
    static constexpr bool RELU8 = BITS == 8 && (OUT & OUT_RELU) != 0;
    static constexpr bool U8 = RELU8 && (OUT & OUT_U) != 0;          // unsigned u8 output codes
    static constexpr bool RELU4 = BITS == 4 && (OUT & OUT_RELU) != 0;  // INT4 ReLU epilogue (runtime top code)
    static constexpr bool RES = (OUT & OUT_RES) != 0;          // residual add: v = fmaf(skip, res_scale, u)
    // residual with TMA-store output and one m-group per unit: each epilogue warp
    // TMA-loads its 32-row skip slab into its output staging slab (same box, same
    // swizzle as the store), reads each 16-byte skip chunk from the address its
    // packed output chunk then overwrites, and stores the slab as usual -- the
    // skip tensor moves as coalesced bulk copies issued before the accumulator
    // wait, not as one 16-byte load per thread and row
    static constexpr bool SKIP_TMA = RES && (OUT & 3) == OUT_TMA && MT == 1;
    static constexpr int OUT_BYTES = OUTP == OUT_TMA ? BM * OUT_ROW : 0;   // staging per TMEM buffer
    static constexpr int NUM_EPI = epi_warpgroups(BITS);            // epilogue warpgroups
    // TMEM accumulator buffers: as many as the 512 columns allow (max 4), so
    // up to NBUF tiles are in the epilogue while the MMA fills the next one
    static constexpr int NBUF = tmem_buffers(BITS, TBW);
    static constexpr bool ALLW = epi_all_warps(BITS, NBUF);         // every warpgroup drains every buffer
    static constexpr int EPI_PER_BUF = epi_per_buf(BITS, NBUF);     // warpgroups per TMEM buffer
    static constexpr int EPI_COLS = BN / EPI_PER_BUF;               // columns one warp drains (of its 32 rows)
    static constexpr int EPI_ROW = EPI_COLS * BITS / 8;             // packed bytes of one row of a warp's slab
    static constexpr int EPI_SUBW = EPI_ROW < 128 ? EPI_ROW : 128;  // TMA store box width (= swizzle span)
    static constexpr int EPI_NSUB = EPI_ROW / EPI_SUBW;
    static constexpr int SLAB = 32 * EPI_ROW;                       // one warp's staging slab
    static constexpr int CW = BITS == 8 ? 16 : 32;                  // columns per tcgen05.ld (16 B packed)
    // per TMEM buffer, three slots (tile j of the buffer uses slot j % 3): the
    // tile's BN scales then BN shifts (fp32), bulk-copied from global one tile
    // ahead by the buffer's first epilogue warp; the epilogue reads them with
    // LDS (per-chunk global loads were the epilogue's top stall).  Three slots
    // let every warp release its TMEM buffer before requantizing its last chunk:
    // the copy for tile j+1 starts once the buffer's warps have released tile
    // j-1, i.e. have finished tile j-2, the previous user of slot (j+1) % 3.
    static constexpr int SS_BYTES = OUTP == OUT_S32 ? 0 : 3 * 8 * BN;
    static constexpr int BAR_BYTES = 1024;
    static constexpr int stages_with(int nhalo) {
        return (SMEM_LIMIT - 1024 - BAR_BYTES - WSB - WSB_PK - NBUF * (OUT_BYTES + SS_BYTES) - nhalo * (HALO_BYTES + HALO_PK)) /
               STAGE_BYTES;
    }
    // halo buffers in flight: the halo load of tile t+NHALO-1 overlaps tiles
    // t..t+NHALO-2, so more buffers hide more TMA latency; keep >= 2 tiles of
    // weight stages ((9/NSUB) stages per tile, 3x3 filters)
    static constexpr int HST = NSUB >= 9 ? 1 : (9 + NSUB - 1) / NSUB;
    static constexpr int NHALO = !HA || WS ? 0 : stages_with(4) >= 2 * HST ? 4 : stages_with(3) >= 2 * HST ? 3 : 2;
    static constexpr int STAGES_FIT = stages_with(NHALO);
    static constexpr int MAX_STAGES = 12;
    // stages with the full weight-stationary budget (the minimum the config
    // guarantees; the launch uses stages_for(wsb) >= STAGES for the real block)
    static constexpr int STAGES = STAGES_FIT > MAX_STAGES ? MAX_STAGES : STAGES_FIT;
    // (1024: base alignment of the dynamic smem; + 1024: the ring end rounded up to 1 KB)
    static constexpr int FIXED_BYTES = 2048 + NBUF * (OUT_BYTES + SS_BYTES) + NHALO * (HALO_BYTES + HALO_PK) + BAR_BYTES;
    static constexpr int SMEM = FIXED_BYTES + WSB + WSB_PK + STAGES * STAGE_BYTES;
    static int stages_for(int wsb) {
        const int st = (SMEM_LIMIT - FIXED_BYTES - wsb) / STAGE_BYTES;
        return st > MAX_STAGES ? MAX_STAGES : st;
    }
    static int smem_for(int wsb, int stages) { return FIXED_BYTES + wsb + stages * STAGE_BYTES; }
    static constexpr int TMEM_COLS = NBUF * TBW < 32 ? 32 : NBUF * TBW;
    // Warp layout: epilogue warpgroups first, then (INT4) the transform
    // warpgroup, then the TMA producer and the MMA issuer as the two highest
    // warp ids -- the SMSP arbiter favours higher warp ids, so the two
    // single-thread control loops are never starved by epilogue math.
    static constexpr int EPI_WARP0 = 0;
    static constexpr int XF_WARP0 = 4 * NUM_EPI;                    // INT4 transform warps
    static constexpr int PROD_WARP = XF_WARP0 + (BITS == 4 ? 4 : 0);
    static constexpr int MMA_WARP = PROD_WARP + 1;
    static constexpr int NUM_THREADS = 32 * (MMA_WARP + kNumMma);
    static constexpr uint32_t IDESC = idesc_i8(BM * CG, BN);
    static constexpr bool FITS = STAGES >= 2 && (!HB || (OUTP != OUT_TMA && (BITS == 8 || HA))) &&
                                 (!(OUT & OUT_U) || (BITS == 8 && (OUT & OUT_RELU))) &&
                                 (!RES || (OUTP != OUT_S32 && !(OUT & OUT_RELU))) &&
                                 (!WS || ((BITS == 8 || !S2H) && (!HB || NSUB == 1))) &&   // INT4 WS: generic / halo
                                 (!S2H || (WS && !HA && KCH == 64)) &&
                                 (MT == 1 || (WS && HB) || (WS && CG == 1 && !HB));  // else never instantiated
    static_assert(KCH == 32 || KCH == 64 || KCH == 128, "KCH");
    static_assert(NSUB >= 1 && NSUB <= 4, "NSUB");
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
// The float part is I2FP, FFMA and max(., lo) (NaN -> lo, and the lower clamp:
// lo is an integer, so rne(max(u, lo)) == max(rne(u), lo)); rounding and the
// upper clamp are done by the conversion to the packed code.
__device__ __forceinline__ float requant_f(int acc, float sc, float sh, float lo) {
    return fmaxf(__fmaf_rn(__int2float_rn(acc), sc, sh), lo);
}
// INT4: one F2I (round-to-nearest-even, saturating to s32) per code; the upper
// clamp is the saturation of the s4 packing instruction (I2IP.S4.SAT).
__device__ __forceinline__ int requant_int(int acc, float sc, float sh, float lo) {
    int r;
    asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(requant_f(acc, sc, sh, lo)));
    return r;
}
// INT8: two codes -> two packed s8 bytes in ONE instruction.  The PTX pair
// "cvt.rni.s32.f32 x2 ; cvt.pack.sat.s8.s32.b32" (kept adjacent in one asm
// block) is fused by ptxas into F2IP.S8.F32 (round-to-nearest-even, saturate to
// [-128, 127], pack with the upper bytes of c): d = c << 16 | q(a) << 8 | q(b).
// Measured on B200 (scripts/micro/pipe_rates.cu, epi_rates.cu): the separate
// F2I runs at 16 lanes/clk/SM -- the epilogue's old ceiling -- while F2IP and
// I2FP run at 64, so a code now costs I2FP + FFMA + FMNMX + half an F2IP.
__device__ __forceinline__ uint32_t pack2_f32_s8(float a, float b, uint32_t c) {
    uint32_t d;
    asm("{\n .reg .s32 ia, ib;\n cvt.rni.s32.f32 ia, %1;\n cvt.rni.s32.f32 ib, %2;\n"
        " cvt.pack.sat.s8.s32.b32 %0, ia, ib, %3;\n}" : "=r"(d) : "f"(a), "f"(b), "r"(c));
    return d;
}
// (a0, a1) * (b0, b1) + (c0, c1) with ONE packed fp32 FMA (sm_100 FFMA2): two
// independent IEEE round-to-nearest fmas, bit-identical to two __fmaf_rn.
__device__ __forceinline__ void fma2_rn(float a0, float a1, float b0, float b1, float c0, float c1, float &d0,
                                        float &d1) {
    asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n mov.b64 c, {%6, %7};\n"
        " fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
        : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// two-wide RN add of one scalar (add.rn.f32x2)
__device__ __forceinline__ void add2_rn(float a0, float a1, float b, float &d0, float &d1) {
    asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %4};\n"
        " add.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}" : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b));
}
// two-wide RN multiply (mul.rn.f32x2)
__device__ __forceinline__ void mul2_rn(float a0, float a1, float b, float &d0, float &d1) {
    asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %4};\n"
        " mul.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}" : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b));
}
// four float values -> one packed s8 word (value 0 in byte 0)
__device__ __forceinline__ uint32_t pack4_f32_s8(float u0, float u1, float u2, float u3) {
    return pack2_f32_s8(u1, u0, pack2_f32_s8(u3, u2, 0u));
}
// Unsigned codes (reading 16): "cvt.rni.s32.f32 x2 ; cvt.pack.sat.u8.s32.b32" -> one
// F2IP.U8 per two codes: round to nearest even, saturate to [0, 255] (the
// ReLU and the upper clamp at once), pack.
__device__ __forceinline__ uint32_t pack2_f32_u8(float a, float b, uint32_t c) {
    uint32_t d;
    asm("{\n .reg .s32 ia, ib;\n cvt.rni.s32.f32 ia, %1;\n cvt.rni.s32.f32 ib, %2;\n"
        " cvt.pack.sat.u8.s32.b32 %0, ia, ib, %3;\n}" : "=r"(d) : "f"(a), "f"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t pack4_f32_u8(float u0, float u1, float u2, float u3) {
    return pack2_f32_u8(u1, u0, pack2_f32_u8(u3, u2, 0u));
}
// clamp(rne(u), 0, 255) in one F2I.U8 (64 lanes/clk/SM; the s32 F2I runs at 16)
__device__ __forceinline__ int f2u8_rn(float u) {
    int r;
    asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(u));
    return r;
}
// cvt.pack.sat.u4.s32.b32 d, a, b, c:  d = c << 8 | sat_u4(a) << 4 | sat_u4(b)
__device__ __forceinline__ uint32_t pack2_u4(int a, int b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t pack8_sat_u4(const int *r) {
    return pack2_u4(r[1], r[0], pack2_u4(r[3], r[2], pack2_u4(r[5], r[4], pack2_u4(r[7], r[6], 0u))));
}
// ReLU on four packed s8 codes: PRMT with sign-replicating selectors gives
// 0xFF for every negative byte; clear those bytes.  Two instructions per word.
__device__ __forceinline__ uint32_t relu_s8x4(uint32_t w) {
    uint32_t m;   // prmt.b32: selector nibble bit 3 = replicate the sign of the selected byte
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(m) : "r"(w));
    return w & ~m;
}
// cvt.pack.sat.s4.s32.b32 d, a, b, c:  d = c << 8 | sat4(a) << 4 | sat4(b)
__device__ __forceinline__ uint32_t pack2_s4(int a, int b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.s4.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// eight codes -> one packed s4 word (code 0 in the low nibble), saturating to [-8, 7]
__device__ __forceinline__ uint32_t pack8_sat_s4(const int *r) {
    return pack2_s4(r[1], r[0], pack2_s4(r[3], r[2], pack2_s4(r[5], r[4], pack2_s4(r[7], r[6], 0u))));
}

// ---------------------------------------------------------------- unfused epilogue
// Standalone requantize + repack of an s32 accumulator matrix [M][K] (the
// conv kernel's CONV_Q_OUT_S32 output) into packed [M][K*BITS/8] -- the SAME
// arithmetic as the fused epilogue (readings 4-5), as a separate HBM pass.  It
// exists for the NEXT-3 ablation (fused vs unfused epilogue, PAPER.md:375-377
// section 4.4) and as the boundary's explicit re-layout step.  One thread per
// 16-byte output vector (16 s8 / 32 s4 codes of one row): 4 / 8 x 16-byte
// accumulator loads, scale/shift through the read-only cache.
template <int BITS>
__global__ void __launch_bounds__(256) requant_kernel(const int4 *__restrict__ acc, const float *__restrict__ scale,
                                                     uint4 *__restrict__ y, int total, int K, int vpr, int relu,
                                                     FastDiv fd_vpr) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int CW = BITS == 8 ? 16 : 32;     // codes per 16-byte output vector
    const float lo = relu ? 0.f : -(float)(1 << (BITS - 1));
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int m = fd_vpr.div(o);
        const int c0 = (o - m * vpr) * CW;
        int a[CW];
        const int4 *src = acc + ((int64_t)m * K + c0) / 4;
#pragma unroll
        for (int i = 0; i < CW / 4; ++i) {
            const int4 t = __ldcs(src + i);
            a[4 * i] = t.x; a[4 * i + 1] = t.y; a[4 * i + 2] = t.z; a[4 * i + 3] = t.w;
        }
        const float4 *s4 = reinterpret_cast<const float4 *>(scale + c0);
        const float4 *h4 = reinterpret_cast<const float4 *>(scale + K + c0);
        uint32_t w[4];
        if constexpr (BITS == 8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 sa = __ldg(s4 + q), sb = __ldg(h4 + q);
                float u0, u1, u2, u3;
                fma2_rn(__int2float_rn(a[4 * q]), __int2float_rn(a[4 * q + 1]), sa.x, sa.y, sb.x, sb.y, u0, u1);
                fma2_rn(__int2float_rn(a[4 * q + 2]), __int2float_rn(a[4 * q + 3]), sa.z, sa.w, sb.z, sb.w, u2, u3);
                w[q] = pack4_f32_s8(u0, u1, u2, u3);
                if (relu) w[q] = relu_s8x4(w[q]);
            }
        } else {
            int r[CW];
#pragma unroll
            for (int q = 0; q < CW / 4; ++q) {
                const float4 sa = __ldg(s4 + q), sb = __ldg(h4 + q);
                r[4 * q] = requant_int(a[4 * q], sa.x, sb.x, lo);
                r[4 * q + 1] = requant_int(a[4 * q + 1], sa.y, sb.y, lo);
                r[4 * q + 2] = requant_int(a[4 * q + 2], sa.z, sb.z, lo);
                r[4 * q + 3] = requant_int(a[4 * q + 3], sa.w, sb.w, lo);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = pack8_sat_s4(r + 8 * q);
        }
        __stcs(y + o, make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// Work unit -> (tile, k-block range).  splits == 1 (every non-split config)
// takes the division-free branch: these run once per tile in the single-thread
// control loops, where a few dozen extra instructions per tile show up on
// layers with one k-block per tile.  split*num_kb < 2^31 is checked at plan time.
__device__ __forceinline__ void unit_range(const ConvParams &p, int unit, int &tile, int &kb_lo, int &kb_hi) {
    if (p.splits == 1) {
        tile = unit;
        kb_lo = 0;
        kb_hi = p.num_kb;
    } else {
        tile = p.fd_splits.div(unit);
        const int split = unit - tile * p.splits;
        kb_lo = p.fd_splits.div(split * p.num_kb);
        kb_hi = p.fd_splits.div((split + 1) * p.num_kb);
    }
}

// Expand one k-block (A rows then B rows) with all loads of a thread issued
// before its first store: ITEMS 16-byte pieces per thread in flight (ILP)
// instead of one shared-memory round trip per piece.
template <int KCH, int ROWS_A, int ROWS_B, int NTHR>
__device__ __forceinline__ void expand_kblock(const uint8_t *a_src, uint8_t *a_dst, const uint8_t *b_src,
                                              uint8_t *b_dst, int tid) {
    constexpr int PW = KCH / 2, PPR = PW / 16;
    constexpr int TA = ROWS_A * PPR, T = (ROWS_A + ROWS_B) * PPR;
    constexpr int ITEMS = (T + NTHR - 1) / NTHR;
    uint4 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int i = tid + k * NTHR;
        if (T % NTHR == 0 || i < T) {
            const bool a = i < TA;
            const int ii = a ? i : i - TA;
            const int row = ii / PPR, j = ii - row * PPR;
            v[k] = *reinterpret_cast<const uint4 *>((a ? a_src : b_src) + swz<PW>(row * PW + j * 16));
        }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int i = tid + k * NTHR;
        if (T % NTHR == 0 || i < T) {
            const bool a = i < TA;
            const int ii = a ? i : i - TA;
            const int row = ii / PPR, j = ii - row * PPR;
            uint32_t o[8];
            expand_s4(v[k].x, o[0], o[1]);
            expand_s4(v[k].y, o[2], o[3]);
            expand_s4(v[k].z, o[4], o[5]);
            expand_s4(v[k].w, o[6], o[7]);
            uint8_t *dst = a ? a_dst : b_dst;
            *reinterpret_cast<uint4 *>(dst + swz<KCH>(row * KCH + (2 * j) * 16)) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4 *>(dst + swz<KCH>(row * KCH + (2 * j + 1) * 16)) = make_uint4(o[4], o[5], o[6], o[7]);
        }
    }
}

// Spin (lane 0, the warp waits at the shuffle) until a completion counter reaches
// `target`.  Bounded: a counter that never completes (not zeroed, a mismatched
// producer) traps after ~10 s instead of hanging the device.  No acquire / fence
// after it: an acquire load or a full / proxy fence would also wait for this
// warp's TMA loads in flight; the producer's codes reached L2 (store completion +
// fence) before its add, and the TMA loads issued after this loop read L2.
__device__ __forceinline__ void wait_counter(const unsigned *c, unsigned target) {
    if ((threadIdx.x & 31) == 0) {
        long long spins = 0;
        while (ld_relaxed_gpu(c) < target) {
            if (++spins > (1ll << 24)) __trap();
            __nanosleep(64);
        }
    }
    __syncwarp();
}

template <int BITS, int BN, int KCH, int OUT, int CG, int NSUB, int HALO>
__global__ void __launch_bounds__(ConvCfg<BITS, BN, KCH, OUT, CG, NSUB, HALO>::NUM_THREADS, 1)
    conv_igemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_y, const __grid_constant__ CUtensorMap tm_s,
                      const ConvParams p) {
    using Cfg = ConvCfg<BITS, BN, KCH, OUT, CG, NSUB, HALO>;
    // measurement hooks (wait-cycle trace, probe modes) exist only in the
    // CONVQ_INSTRUMENT build (libconvq_instr.so); compiled out otherwise
    unsigned long long *const trace = kInstrument ? p.trace : nullptr;
    // timeline (instrumented build, CTA 0): region 0 producer after each empty
    // wait, 1/2/3 MMA warp per tile after acc_empty / first full wait / acc_full
    // commit, 4+w / 24+w epilogue warp w per tile after acc_full / after its store
    unsigned long long *const tl = kInstrument && blockIdx.x == 0 ? p.tl : nullptr;
#define CONVQ_TL(region, idx) \
    do { if (tl && lane == 0) tl[(region) * 256 + ((idx) & 255)] = (unsigned long long)clock64(); } while (0)
    const int probe = kInstrument ? p.probe : 0;
    static_assert(Cfg::FITS, "tile does not fit shared memory");
    const int STAGES = p.stages;      // runtime ring depth (host: all smem left after the fixed regions)
    constexpr int MAXST = Cfg::MAX_STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment by offset (pointer arithmetic on the shared array keeps
    // the compiler's shared-space inference: LDS/STS instead of generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);

    // ---- carve shared memory (every tile 1024-byte aligned; identical offsets
    // in both CTAs of a pair, as cta_group::2 descriptors require)
    constexpr bool HA = Cfg::HA, WS = Cfg::WS, S2H = Cfg::S2H;
    uint8_t *b_res = smem;                              // WS: [num_kb][BN rows][KCH] resident weights
    uint8_t *b_res_pk = smem + (WS ? p.wsb_s8 : 0);     // INT4 WS: [num_kb][BN rows][KCH/2] packed, expanded once
    uint8_t *a_s8 = smem + (WS ? p.wsb : 0);            // [STAGES][NSUB][BM*KCH] (WS halo: [STAGES][HBOX])
    uint8_t *b_s8 = a_s8 + STAGES * Cfg::A_S8;          // [STAGES][NSUB][BNL*KCH]
    uint8_t *a_pk = b_s8 + STAGES * Cfg::B_S8;          // INT4: [STAGES][NSUB][BM*KCH/2]
    uint8_t *b_pk = a_pk + STAGES * Cfg::A_PK;          // INT4: [STAGES][NSUB][BNL*KCH/2]
    // [NBUF][EPB][4 quads] slabs [EPI_NSUB][32][EPI_SUBW]: 1024-byte aligned (swizzled TMA boxes)
    // whatever the runtime ring depth (INT4 stage sizes need not be multiples of 1 KB)
    uint8_t *out_stage = smem + ((b_pk + STAGES * Cfg::B_PK - smem + 1023) & ~1023);
    float *ss_stage = reinterpret_cast<float *>(out_stage + Cfg::NBUF * Cfg::OUT_BYTES);  // [NBUF][3 slots][2][BN]
    uint8_t *halo_buf = out_stage + Cfg::NBUF * (Cfg::OUT_BYTES + Cfg::SS_BYTES);   // HALO: [NHALO][HALO_BYTES]
    uint8_t *halo_pk = halo_buf + Cfg::NHALO * Cfg::HALO_BYTES;  // INT4 halo: [NHALO][HALO_PK] packed boxes
    uint64_t *bars = reinterpret_cast<uint64_t *>(halo_pk + Cfg::NHALO * Cfg::HALO_PK);
    uint64_t *full = bars;                  // TMA -> (transform | MMA)
    uint64_t *empty = bars + MAXST;         // MMA -> TMA
    uint64_t *ready = bars + 2 * MAXST;     // transform -> MMA (INT4)
    uint64_t *acc_full = bars + 3 * MAXST;  // MMA -> epilogue [NBUF]
    uint64_t *acc_empty = acc_full + 4;     // epilogue -> MMA [NBUF]
    uint64_t *hempty = acc_empty + 4;       // HALO: MMA -> TMA, halo buffer free [NHALO <= 4]
    uint64_t *bfull = hempty;               // WS (no separate halo buffers): resident weights loaded
    uint64_t *ss_full = hempty + 4;         // scale/shift bulk copy -> epilogue [NBUF][3 slots]
    uint64_t *skbar = ss_full + 12;         // SKIP_TMA: per epilogue warp, its skip slab landed [16]
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(skbar + 16);
    // dual MMA warps: per smem stage, the last global stage index whose fill an
    // MMA warp has waited for.  A parity wait on a stage is only valid once the
    // stage's PREVIOUS fill has completed -- and TMA fills of different stages
    // can complete out of order, so this is tracked per stage.
    volatile int *stage_done = reinterpret_cast<volatile int *>(tmem_holder + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const long long t_start = trace ? clock64() : 0;
    if (trace && threadIdx.x == 0) trace[blockIdx.x * TR_SLOTS + TR_T0] = globaltimer_ns();
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;     // position in the CTA pair
    const int tile0 = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
    const int tstep = CG == 2 ? (int)num_clusters_x() : (int)gridDim.x;
    // CTA pairs: every CTA's TMA loads complete on its OWN full barrier (a load
    // that signals the peer CTA's barrier is serialised by the TMA unit -- one in
    // flight, ~1000 cycles each, measured in scripts/micro/tma_bw.cu).  The
    // follower relays each filled stage to the leader's `ready` barrier: INT4 by
    // its transform warps (after expanding), INT8 by its otherwise idle MMA warp.
    constexpr bool PAIR8 = CG == 2 && BITS == 8;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tm_a);
        tma_prefetch_desc(&tm_b);
        if (Cfg::OUTP == OUT_TMA) tma_prefetch_desc(&tm_y);
        if (Cfg::SKIP_TMA) tma_prefetch_desc(&tm_s);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&ready[s], BITS == 4 ? 4 * CG : 1);
        }
        for (int h = 0; h < Cfg::NHALO; ++h) mbar_init(&hempty[h], 1);
        if (WS) mbar_init(bfull, 1);
        if (WS && BITS == 4) mbar_init(&hempty[2], 4 * CG);   // bready: the expanded s8 weight blocks (both CTAs)
        if (WS && CG == 2) mbar_init(&hempty[1], 1);   // leader: the follower's weight block is loaded
        for (int b = 0; b < Cfg::NBUF; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4 * Cfg::EPI_PER_BUF * CG);
            for (int k = 0; k < 3; ++k) mbar_init(&ss_full[3 * b + k], 1);
        }
        for (int i = 0; i < STAGES; ++i) stage_done[i] = -1;
        if (Cfg::SKIP_TMA)
            for (int w = 0; w < 4 * Cfg::NUM_EPI; ++w) mbar_init(&skbar[w], 1);
        fence_mbar_init();
    }
    if (warp == Cfg::MMA_WARP) {
        if constexpr (CG == 2) tmem_alloc_cg2<Cfg::TMEM_COLS>(tmem_holder);
        else tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync();   // barriers of both CTAs initialised before any remote use
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // PDL: everything above (barrier init, TMEM alloc, descriptor prefetch)
    // overlapped the previous kernel's tail; global memory is touched only
    // after pdl_wait() in the producer and epilogue roles.
    if (threadIdx.x == 0) pdl_launch_dependents();

    const int PQ = p.P * p.Q;

    if (warp == Cfg::PROD_WARP) {
        // =========================== TMA producer ===========================
        // The whole warp runs the loop (converged, uniform operands); one
        // elected lane issues the expect-tx and the TMA loads.
        const uint64_t pol_a = policy_evict_normal();  // activations: re-read by R*S taps and n-tiles
        const uint64_t pol_b = policy_evict_last();    // weights: re-read by every m-tile
        uint8_t *a_dst = BITS == 4 ? a_pk : a_s8;
        uint8_t *b_dst = BITS == 4 ? b_pk : b_s8;
        constexpr int A_LD = BITS == 4 ? Cfg::A_PK : Cfg::A_S8;
        constexpr int B_LD = BITS == 4 ? Cfg::B_PK : Cfg::B_S8;
        constexpr int A_LD_SUB = BITS == 4 ? Cfg::A_PK_SUB : Cfg::A_SUB;
        constexpr int B_LD_SUB = BITS == 4 ? Cfg::B_PK_SUB : Cfg::B_SUB;
        int stage = 0;
        uint32_t phase = 0;
        int tl_n = 0;
        if constexpr (WS) {
            // weight-stationary: this CTA's BN x (R*S*C) weight block, once, as
            // num_kb k-block tiles [BN rows][KCH] (tap-major k order).  Weights
            // are constant across layers' launches, so this load is issued
            // BEFORE the PDL wait and overlaps the previous kernel's tail.
            if (tile0 < p.num_tiles && elect_one()) {
                const int brow = (tile0 - p.fd_ntiles.div(tile0) * p.n_tiles) * BN + (int)rank * Cfg::BNL;
                mbar_arrive_expect_tx(bfull, (uint32_t)(p.num_kb * Cfg::BNL * Cfg::LOAD_ROW));
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    const int tap = p.fd_cblk.div(kb), cb = kb - tap * p.num_cblk;
                    uint8_t *dst = BITS == 4 ? b_res_pk + kb * (Cfg::BNL * Cfg::LOAD_ROW) : b_res + kb * Cfg::B_TILE;
                    tma_load_2d(dst, &tm_b, bfull, tap * p.row_bytes + cb * Cfg::LOAD_ROW, brow, pol_b);
                }
            }
            __syncwarp();
        }
        // activations (the previous layer's output) only after the previous grid
        // completed -- or, with completion counters, after its last codes are in memory
        if (p.dep_in) wait_counter(p.dep_in, p.dep_in_total);
        else pdl_wait();
        if (trace && lane == 0) trace[blockIdx.x * TR_SLOTS + TR_TPDL] = globaltimer_ns();
        if constexpr (WS && (HA || S2H)) {
            // one stage = one halo box per (tile, channel block); no weights
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                const int m_blk = p.fd_ntiles.div(tile);
                const int rt = m_blk * CG + (int)rank;            // this CTA's row tile
                const int n = p.fd_tpi.div(rt);                   // (>= N: all-OOB box, rows masked)
                const int p0 = (rt - n * p.tiles_per_img) * p.rpt;
                for (int cblk = 0; cblk < p.num_cblk; ++cblk) {
                    {
                        const long long t0 = trace ? clock64() : 0;
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_PROD_EMPTY, clock64() - t0);
                    }
                    CONVQ_TL(0, tl_n++);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&full[stage], p.halo_tx);
                        // (INT4: the packed box; the transform warps expand it into the stage's s8 box)
                        tma_load_4d(BITS == 4 ? a_pk + stage * Cfg::A_PK : a_s8 + stage * Cfg::A_S8, &tm_a, &full[stage],
                                    cblk * Cfg::LOAD_ROW, -p.pad_w, p0 - p.pad, n, pol_a);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        } else if constexpr (HA) {
            // one halo box per (tile, channel block) + the filter taps' weight
            // k-blocks in groups of NSUB; the halo rides on the first group's barrier
            int hcount = 0;
            const int RS = p.R * p.S;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                const int m_blk = p.fd_ntiles.div(tile), n_blk = tile - m_blk * p.n_tiles;
                const int rt = m_blk * CG + (int)rank;            // this CTA's row tile
                const int n = p.fd_tpi.div(rt);                   // (>= N: all-OOB box, rows masked)
                const int p0 = (rt - n * p.tiles_per_img) * p.rpt;
                const int brow = n_blk * BN + (int)rank * Cfg::BNL;
                for (int cblk = 0; cblk < p.num_cblk; ++cblk, ++hcount) {
                    const int hb = hcount % Cfg::NHALO;
                    const uint32_t hph = (hcount / Cfg::NHALO) & 1;
                    for (int tap = 0; tap < RS;) {
                        const int nsub = min(NSUB, RS - tap);
                        {
                            const long long t0 = trace ? clock64() : 0;
                            mbar_wait(&empty[stage], phase ^ 1);
                            if (tap == 0) mbar_wait(&hempty[hb], hph ^ 1);
                            if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_PROD_EMPTY, clock64() - t0);
                        }
                        if (elect_one()) {
                            const int tx = nsub * Cfg::SUB_TX + (tap == 0 ? p.halo_tx : 0);
                            if (probe & 2) {
                                mbar_arrive(&full[stage]);
                            } else {
                                {
                                    mbar_arrive_expect_tx(&full[stage], tx);
                                    if (tap == 0)
                                        tma_load_4d(BITS == 4 ? halo_pk + hb * Cfg::HALO_PK : halo_buf + hb * Cfg::HALO_BYTES,
                                                    &tm_a, &full[stage], cblk * Cfg::LOAD_ROW, -p.pad, p0 - p.pad, n, pol_a);
                                    for (int j = 0; j < nsub; ++j)
                                        tma_load_2d(b_dst + stage * B_LD + j * B_LD_SUB, &tm_b, &full[stage],
                                                    (tap + j) * p.row_bytes + cblk * Cfg::LOAD_ROW, brow, pol_b);
                                }
                            }
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        tap += nsub;
                    }
                }
            }
        } else
        for (int unit = tile0; unit < p.num_units; unit += tstep) {
            int tile, kb_lo, kb_hi;
            unit_range(p, unit, tile, kb_lo, kb_hi);
            const int m_blk = p.fd_ntiles.div(tile), n_blk = tile - m_blk * p.n_tiles;
            const int m0 = m_blk * (BM * CG * Cfg::AMT) + (int)rank * BM;   // this CTA's first output pixel
            // MT2: m-group g starts at row m0 + 128 g (its own im2col origin)
            int n0g[Cfg::AMT], h0g[Cfg::AMT], w0g[Cfg::AMT];
#pragma unroll
            for (int g = 0; g < Cfg::AMT; ++g) {
                const int mg = m0 + g * BM;
                const int n0 = p.fd_PQ.div(mg), rem = mg - n0 * PQ;
                const int p0 = p.fd_Q.div(rem), q0 = rem - p0 * p.Q;
                n0g[g] = n0;
                h0g[g] = p0 * p.stride - p.pad;
                w0g[g] = q0 * p.stride - p.pad_w;
            }
            const int brow = n_blk * BN + (int)rank * Cfg::BNL;  // this CTA's B rows
            const int nk = kb_hi - kb_lo;
            // optional rotated k-block order (CTA c starts at k-block 7c mod nk; any
            // order is bit-exact for integer accumulation)
            const int rot = (p.rotate && !WS) ? (int)(((unsigned)(blockIdx.x / CG) * 7u) % (unsigned)nk) : 0;
            for (int kb = 0; kb < nk; kb += NSUB) {
                const int nsub = min(NSUB, nk - kb);   // ragged last stage of a tile
                {
                    const long long t0 = trace ? clock64() : 0;
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_PROD_EMPTY, clock64() - t0);
                }
                CONVQ_TL(0, tl_n++);
                if (elect_one()) {
                    if (probe & 2) mbar_arrive(&full[stage]);   // measurement: no loads
                    else mbar_arrive_expect_tx(&full[stage], nsub * Cfg::SUB_TX);
                }
                __syncwarp();
                // lane j issues the loads of the stage's j-th k-block: the (tap,
                // channel block) decomposition and the TMA issue run lane-parallel
                // instead of NSUB times through one thread
                if (lane < nsub && !(probe & 2)) {
                    int k = kb + lane + rot;
                    if (k >= nk) k -= nk;
                    k += kb_lo;
                    const int tap = p.fd_cblk.div(k), cblk = k - tap * p.num_cblk;
                    const int r = p.fd_S.div(tap), s = tap - r * p.S;
                    uint8_t *bd = b_dst + stage * B_LD + lane * B_LD_SUB;
#pragma unroll
                    for (int g = 0; g < Cfg::AMT; ++g) {
                        uint8_t *ad = a_dst + stage * A_LD + (lane * Cfg::AMT + g) * A_LD_SUB;
                        if (p.a_gemm)
                            tma_load_2d(ad, &tm_a, &full[stage], cblk * Cfg::LOAD_ROW, m0 + g * BM, pol_a);
                        else
                            tma_load_im2col_4d(ad, &tm_a, &full[stage], cblk * Cfg::LOAD_ROW, w0g[g], h0g[g], n0g[g],
                                               (uint16_t)s, (uint16_t)r, pol_a);
                    }
                    if (!WS) tma_load_2d(bd, &tm_b, &full[stage], tap * p.row_bytes + cblk * Cfg::LOAD_ROW, brow, pol_b);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp >= Cfg::MMA_WARP) {
        // =========================== MMA issuer =============================
        const int mw = warp - Cfg::MMA_WARP;                 // which MMA warp
        // (split-K units have ragged K ranges; an odd buffer count would share
        // TMEM buffers between the two warps)
        const int nmma = p.splits == 1 && Cfg::NBUF % 2 == 0 ? kNumMma : 1;
        // smem stages per unit (uniform when splits == 1)
        const int s_unit = (WS && (HA || S2H)) ? p.num_cblk
                         : HA ? p.num_cblk * ((p.R * p.S + NSUB - 1) / NSUB) : (p.num_kb + NSUB - 1) / NSUB;
        // Whole warp (converged) waits; one elected lane issues the MMAs and
        // commits.  Descriptors: base + byte offset >> 4 in the start-address
        // field (addresses < 2^18, so the 14-bit field never carries).
        // CONVQ_MMA_1T=1 (measured slower: the compiler cannot keep the descriptors
        // in uniform registers and emits an R2UR waterfall per MMA): the MMA loop on lane 0 alone -- no
        // elect / warp-sync / divergence checks per stage on this single-thread
        // critical path (the per-tile control loop is serialised with the MMA
        // execution; see profiles/r01_timeline_cta0.txt)
        auto mma_elect = [&]() { return kMma1T ? true : elect_one(); };
        auto mma_sync = [&]() { if (!kMma1T) __syncwarp(); };
        if (rank == 0 && (!kMma1T || lane == 0) && mw < nmma) {
            // A format: s8 (bit 7 set) or, for unsigned activation codes (reading 16), u8
            const uint32_t idesc = p.x_uns ? (Cfg::IDESC & ~(1u << 7)) : Cfg::IDESC;
            const uint64_t a_desc0 = umma_desc_kmajor(smem_u32(a_s8), KCH);
            const uint64_t b_desc0 = umma_desc_kmajor(smem_u32(b_s8), KCH);
            // HALO: descriptor start-address delta of tap t's window, (r*Wp + s)*KCH bytes (3x3 table)
            const uint64_t a_desc_h = umma_desc_kmajor(smem_u32(halo_buf), KCH);
            uint32_t toff[9];
#pragma unroll
            for (int t = 0; t < 9; ++t) toff[t] = (uint32_t)(((t / 3) * p.Wp + (t % 3)) * KCH) >> 4;
            const uint64_t b_desc_res = umma_desc_kmajor(smem_u32(b_res), KCH);   // WS: resident k-block 0
            if (WS && BITS == 8) mbar_wait(bfull, 0);
            if (WS && BITS == 8 && CG == 2) mbar_wait(&hempty[1], 0);   // the follower's weight rows
            if (WS && BITS == 4) mbar_wait(&hempty[2], 0);   // INT4: both CTAs' blocks expanded to s8
            int stage = 0;
            uint32_t phase = 0;
            int hcount = 0;
            int gsi = 0;   // global index of the current smem stage
            // before a parity wait on stage gsi: the stage's previous fill (gsi - STAGES)
            // must be complete, i.e. its consumer has already waited past it
            auto mma_gate = [&]() {
                if (nmma > 1)
                    while (stage_done[stage] < gsi - STAGES) {
                    }
            };
            auto mma_mark = [&]() {
                if (nmma > 1 && lane == 0) stage_done[stage] = gsi;
            };
            // CONVQ_LATE_ACC (generic path): the previous unit's accumulator buffer whose
            // acc_full commit waits until this unit's first MMAs are issued (-1: none)
            int pend_buf = -1;
            constexpr bool LATE = CONVQ_LATE_ACC && !HA && !S2H;
            for (int unit = tile0 + mw * tstep, local = mw; unit < p.num_units; unit += nmma * tstep, local += nmma) {
                int tile, kb_lo, kb_hi;
                unit_range(p, unit, tile, kb_lo, kb_hi);
                if (nmma > 1) {   // this unit's first stage in the producer's global sequence
                    const int gs = local * s_unit;
                    gsi = gs;
                    stage = gs % STAGES;
                    phase = (uint32_t)(gs / STAGES) & 1u;
                    hcount = local * p.num_cblk;
                }
                const int buf = local % Cfg::NBUF;
                const uint32_t aphase = (local / Cfg::NBUF) & 1;
                {
                    const long long t0 = trace ? clock64() : 0;
                    mbar_wait(&acc_empty[buf], aphase ^ 1);
                    CONVQ_TL(1, local);
                    if (trace && lane == 0) {
                        atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_ACC, clock64() - t0);
                        atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_TILES, 1ull);
                    }
                }
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + buf * Cfg::TBW;
                if constexpr (WS && (HA || S2H)) {
                    // one stage = this tile's halo box of channel block cblk; tap t
                    // reads it at row offset r*Wp + s, its weights from the resident
                    // k-block t*num_cblk + cblk
                    for (int cblk = 0; cblk < p.num_cblk; ++cblk) {
                        long long t0 = trace ? clock64() : 0;
                        mma_gate();
                        mbar_wait(BITS == 4 ? &ready[stage] : &full[stage], phase);   // INT4: expanded box(es)
                        if (PAIR8) mbar_wait(&ready[stage], phase);   // the follower's halo box
                        mma_mark();
                        if (cblk == 0) CONVQ_TL(2, local);
                        if (trace && lane == 0) {
                            const long long t1 = clock64();
                            atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_FULL, t1 - t0);
                            t0 = t1;
                        }
                        tc_fence_after();
                        if (probe & 1) {
                            if (mma_elect()) {
                                mbar_arrive(&empty[stage]);
                                if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[stage]), 1));
                            }
                        } else if (S2H && mma_elect()) {
                            // s2d window: tap row jr, K step kk = s2d pixels 2kk, 2kk+1 of
                            // every row's window -> box pixel offset jr*Wp + 2kk
                            const uint64_t ad_s = umma_desc_kmajor_none(smem_u32(a_s8) + stage * Cfg::A_S8, 16, 128);
#pragma unroll
                            for (int g = 0; g < Cfg::MT; ++g)   // MT2: m-group g = box pixels from 128 g
                            for (int jr = 0; jr < p.R; ++jr) {
                                const uint64_t bd = b_desc_res + (uint64_t)((jr * Cfg::B_TILE) >> 4);
#pragma unroll
                                for (int kk = 0; kk < 2; ++kk) {
                                    const uint64_t ad = ad_s + (uint64_t)(g * BM + jr * p.Wp + 2 * kk);
                                    if constexpr (CG == 2) mma_i8_cg2(d_tmem + g * BN, ad, bd + 2 * kk, idesc, (jr | kk) != 0);
                                    else mma_i8(d_tmem + g * BN, ad, bd + 2 * kk, idesc, (jr | kk) != 0);
                                }
                            }
                            if constexpr (CG == 2) mma_commit_cg2_mc(&empty[stage], 0x3);
                            else mma_commit(&empty[stage]);
                        } else if (!S2H && mma_elect()) {
                            const uint64_t ad_s = a_desc0 + (uint64_t)((stage * Cfg::A_S8) >> 4);
                            if (p.R == 3 && p.S == 3) {   // 3x3: fully unrolled, tap offsets in registers
#pragma unroll
                                for (int g = 0; g < Cfg::MT; ++g)   // MT2: m-group g = halo rows from 128 g
#pragma unroll
                                for (int t = 0; t < 9; ++t) {
                                    const uint64_t ad = ad_s + toff[t] + (uint64_t)((g * BM * KCH) >> 4);
                                    const uint64_t bd = b_desc_res + (uint64_t)(((t * p.num_cblk + cblk) * Cfg::B_TILE) >> 4);
#pragma unroll
                                    for (int k = 0; k < KCH / 32; ++k) {
                                        if constexpr (CG == 2) mma_i8_cg2(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, (cblk | t | k) != 0);
                                        else mma_i8(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, (cblk | t | k) != 0);
                                    }
                                }
                            } else {                       // any R x S: tap (r, s) at row offset r*Wp + s
#pragma unroll
                                for (int g = 0; g < Cfg::MT; ++g) {
                                    int t = 0;
                                    for (int r = 0; r < p.R; ++r)
                                        for (int s_ = 0; s_ < p.S; ++s_, ++t) {
                                            const uint64_t ad = ad_s + (uint64_t)((uint32_t)((r * p.Wp + s_) * KCH) >> 4) +
                                                                (uint64_t)((g * BM * KCH) >> 4);
                                            const uint64_t bd = b_desc_res + (uint64_t)(((t * p.num_cblk + cblk) * Cfg::B_TILE) >> 4);
#pragma unroll
                                            for (int k = 0; k < KCH / 32; ++k) {
                                                if constexpr (CG == 2) mma_i8_cg2(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, (cblk | t | k) != 0);
                                                else mma_i8(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, (cblk | t | k) != 0);
                                            }
                                        }
                                }
                            }
                            if constexpr (CG == 2) mma_commit_cg2_mc(&empty[stage], 0x3);
                            else mma_commit(&empty[stage]);
                        }
                        mma_sync();
                        if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_ISSUE, clock64() - t0);
                        ++gsi;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                } else if constexpr (HA) {
                    // filter tap (r, s) reads the halo rows starting at r*Wp + s:
                    // the duplicate-aware load of PAPER.md Alg. 1, with the
                    // "genuine index" remap done by the UMMA descriptor start
                    // address (any R x S; the 3x3 tap offsets are precomputed in toff[])
                    const int RS = p.R * p.S;
                    const int hst = (RS + NSUB - 1) / NSUB;   // stages (weight groups of NSUB taps) per halo box
                    const bool k3x3 = p.R == 3 && p.S == 3;
                    auto tap_off = [&](int t) -> uint64_t {
                        if (k3x3) {
                            uint32_t o = toff[0];
#pragma unroll
                            for (int i = 1; i < 9; ++i) o = t == i ? toff[i] : o;   // register select, no local memory
                            return o;
                        }
                        const int r = p.fd_S.div(t);
                        return (uint64_t)((uint32_t)((r * p.Wp + (t - r * p.S)) * KCH) >> 4);
                    };
                    for (int cblk = 0; cblk < p.num_cblk; ++cblk, ++hcount) {
                        const int hb = hcount % Cfg::NHALO;
                        const uint64_t ad_h = a_desc_h + (uint64_t)((hb * Cfg::HALO_BYTES) >> 4);
                        auto halo_stage = [&](const int g, const int hst_) {
                            long long t0 = trace ? clock64() : 0;
                            mma_gate();
                            mbar_wait(BITS == 4 ? &ready[stage] : &full[stage], phase);   // INT4: expanded
                            if (PAIR8) mbar_wait(&ready[stage], phase);   // the follower's half of the stage
                            mma_mark();
                            if (trace && lane == 0) {
                                const long long t1 = clock64();
                                atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_FULL, t1 - t0);
                                t0 = t1;
                            }
                            tc_fence_after();
                            if (mma_elect()) {
                                if (probe & 1) {
                                    mbar_arrive(&empty[stage]);
                                    if (g == hst_ - 1) mbar_arrive(&hempty[hb]);
                                    if constexpr (CG == 2) {
                                        mbar_arrive_cluster(mapa_shared(smem_u32(&empty[stage]), 1));
                                        if (g == hst_ - 1) mbar_arrive_cluster(mapa_shared(smem_u32(&hempty[hb]), 1));
                                    }
                                } else {
                                    const uint64_t bd0 = b_desc0 + (uint64_t)((stage * Cfg::B_S8) >> 4);
#pragma unroll
                                    for (int j = 0; j < NSUB; ++j) {
                                        const int t = g * NSUB + j;
                                        if (t < RS) {
                                            const uint64_t ad = ad_h + tap_off(t);
                                            const uint64_t bd = bd0 + (uint64_t)((j * Cfg::B_SUB) >> 4);
#pragma unroll
                                            for (int k = 0; k < KCH / 32; ++k) {
                                                const uint32_t acc = (cblk | t | k) != 0;
                                                if constexpr (CG == 2) mma_i8_cg2(d_tmem, ad + 2 * k, bd + 2 * k, idesc, acc);
                                                else mma_i8(d_tmem, ad + 2 * k, bd + 2 * k, idesc, acc);
                                            }
                                        }
                                    }
                                    if constexpr (CG == 2) mma_commit_cg2_mc(&empty[stage], 0x3);
                                    else mma_commit(&empty[stage]);
                                    if (g == hst_ - 1) {             // last use of this halo buffer
                                        if constexpr (CG == 2) mma_commit_cg2_mc(&hempty[hb], 0x3);
                                        else mma_commit(&hempty[hb]);
                                    }
                                }
                            }
                            mma_sync();
                            if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_ISSUE, clock64() - t0);
                            ++gsi;
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        };
                        if (k3x3) {   // 3x3: unrolled, tap offsets resolved at compile time
#pragma unroll
                            for (int g = 0; g < Cfg::HST; ++g) halo_stage(g, Cfg::HST);
                        } else {
#pragma unroll 1
                            for (int g = 0; g < hst; ++g) halo_stage(g, hst);
                        }
                    }
                } else
                for (int kb = kb_lo; kb < kb_hi; kb += NSUB) {
                    const int nsub = min(NSUB, kb_hi - kb);
                    long long t0 = trace ? clock64() : 0;
                    mma_gate();
                    mbar_wait(BITS == 4 ? &ready[stage] : &full[stage], phase);
                    if (PAIR8) mbar_wait(&ready[stage], phase);   // the follower's half of the stage
                    mma_mark();
                    if (kb == kb_lo) CONVQ_TL(2, local);
                    if (trace && lane == 0) {
                        const long long t1 = clock64();
                        atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_FULL, t1 - t0);
                        if (local == 0 && kb == kb_lo) trace[blockIdx.x * TR_SLOTS + TR_TFULL] = globaltimer_ns();
                        t0 = t1;
                    }
                    tc_fence_after();
                    if (mma_elect()) {
                        if (probe & 1) {                // measurement: no MMAs
                            if constexpr (CG == 2) {
                                mbar_arrive(&empty[stage]);
                                mbar_arrive_cluster(mapa_shared(smem_u32(&empty[stage]), 1));
                            } else {
                                mbar_arrive(&empty[stage]);
                            }
                        } else {
                            const uint64_t ad0 = a_desc0 + (uint64_t)((stage * Cfg::A_S8) >> 4);
                            const uint64_t bd0 = b_desc0 + (uint64_t)((stage * Cfg::B_S8) >> 4);
#pragma unroll
                            for (int j = 0; j < NSUB; ++j) {
                                if (j < nsub) {
                                    const uint64_t bd = WS ? b_desc_res + (uint64_t)(((kb + j) * Cfg::B_TILE) >> 4)
                                                           : bd0 + (uint64_t)((j * Cfg::B_SUB) >> 4);
#pragma unroll
                                    for (int g = 0; g < Cfg::AMT; ++g) {   // MT2: m-group g -> TMEM columns g*BN
                                        const uint64_t ad = ad0 + (uint64_t)(((j * Cfg::AMT + g) * Cfg::A_SUB) >> 4);
#pragma unroll
                                        for (int k = 0; k < KCH / 32; ++k) {
                                            const uint32_t acc = (kb - kb_lo + j + k) != 0;
                                            if constexpr (CG == 2) mma_i8_cg2(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, acc);
                                            else mma_i8(d_tmem + g * BN, ad + 2 * k, bd + 2 * k, idesc, acc);
                                        }
                                    }
                                }
                            }
                            // frees the smem stage (in both CTAs) when these MMAs complete
                            if constexpr (CG == 2) mma_commit_cg2_mc(&empty[stage], 0x3);
                            else mma_commit(&empty[stage]);
                        }
                    }
                    mma_sync();
                    if (trace && lane == 0) atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_MMA_ISSUE, clock64() - t0);
                    ++gsi;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    if (LATE && pend_buf >= 0) {   // the previous unit's accumulator, behind these MMAs
                        if (mma_elect()) {
                            if constexpr (CG == 2) mma_commit_cg2_mc(&acc_full[pend_buf], 0x3);
                            else mma_commit(&acc_full[pend_buf]);
                        }
                        mma_sync();
                        pend_buf = -1;
                    }
                }
                // accumulator ready for the epilogue (of both CTAs)
                if (LATE) {
                    pend_buf = buf;
                } else {
                    if (mma_elect()) {
                        if constexpr (CG == 2) mma_commit_cg2_mc(&acc_full[buf], 0x3);
                        else mma_commit(&acc_full[buf]);
                    }
                    mma_sync();
                }
                CONVQ_TL(3, local);
            }
            if (LATE && pend_buf >= 0) {   // the last unit's accumulator
                if (mma_elect()) {
                    if constexpr (CG == 2) mma_commit_cg2_mc(&acc_full[pend_buf], 0x3);
                    else mma_commit(&acc_full[pend_buf]);
                }
                mma_sync();
            }
        } else if (PAIR8 && rank != 0 && mw == 0) {
            // follower CTA: relay every stage its own TMA loads filled to the
            // leader's ready barrier (same stage sequence as the producer)
            const uint32_t ready0 = mapa_shared(smem_u32(&ready[0]), 0);
            if (WS) {   // this CTA's weight rows are resident -> tell the leader
                mbar_wait(bfull, 0);
                if (elect_one()) mbar_arrive_cluster(mapa_shared(smem_u32(&hempty[1]), 0));
                __syncwarp();
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = tile0; unit < p.num_units; unit += tstep) {
                int nst;
                if constexpr (WS && (HA || S2H)) {
                    nst = p.num_cblk;
                } else if constexpr (HA) {
                    nst = p.num_cblk * ((p.R * p.S + NSUB - 1) / NSUB);
                } else {
                    int tile, kb_lo, kb_hi;
                    unit_range(p, unit, tile, kb_lo, kb_hi);
                    nst = (kb_hi - kb_lo + NSUB - 1) / NSUB;
                }
                for (int i = 0; i < nst; ++i) {
                    mbar_wait(&full[stage], phase);
                    if (elect_one()) mbar_arrive_cluster(ready0 + 8u * stage);
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
        __syncwarp();   // reconverge the MMA warp (lane 0 ran the loop alone) before the aligned barriers
    } else if (warp < Cfg::XF_WARP0) {
        // =========================== epilogue ===============================
        // Every warp works on its own: TMEM buffer b (every other tile) is
        // drained by EPI_PER_BUF warpgroups; a warp owns the 32 rows of its
        // TMEM lane quadrant and EPI_COLS columns.  Scale/shift come straight
        // from L1 (warp-uniform loads), and with TMA output each warp stages
        // its 32-row slab and issues its own bulk store: no CTA-level barrier
        // anywhere in the epilogue.  In a CTA pair each CTA drains its own 128
        // rows (its TMEM half) and releases the leader's buffer.
        constexpr int EPB = Cfg::EPI_PER_BUF;
        constexpr bool ALLW = Cfg::ALLW;
        const int e = (warp - Cfg::EPI_WARP0) >> 2;
        const int b0 = ALLW ? 0 : e / EPB;         // first TMEM buffer (ALLW: every buffer in turn)
        const int half = ALLW ? e : e % EPB;       // column part
        const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;          // tile row = output pixel
        int b = b0;                                // this unit's TMEM buffer
        uint8_t *slab = out_stage + b * Cfg::OUT_BYTES + (half * 4 + quad) * Cfg::SLAB;
        uint32_t acc_empty_leader = CG == 2 ? mapa_shared(smem_u32(&acc_empty[b]), 0) : 0;
        const float lo = (p.relu || p.y_uns) ? 0.f : -(float)(1 << (BITS - 1));
        const uint64_t out_pol = p.out_policy == 1 ? policy_evict_last() : p.out_policy == 2 ? policy_evict_first() : 0;
        constexpr bool relu8 = Cfg::RELU8;   // ReLU specialisation (p.relu == 1 guaranteed by the dispatch)
        // scale/shift of the j-th tile of this buffer -> slot j % 3, issued by the
        // buffer's first warp one tile ahead (see SS_BYTES)
        const bool ss_smem = Cfg::OUTP != OUT_S32 && p.splits == 1;
        const bool ss_issuer = ss_smem && half == 0 && quad == 0;
        auto ss_issue = [&](int u, int bb, int jj) {
            if (u < p.num_units && elect_one()) {
                const int n0 = (u - p.fd_ntiles.div(u) * p.n_tiles) * BN;
                const uint32_t bytes = 4u * (uint32_t)min(BN, p.K - n0);
                uint64_t *barp = &ss_full[3 * bb + jj % 3];
                const uint32_t bar = smem_u32(barp);
                const uint32_t dst = smem_u32(ss_stage + (3 * bb + jj % 3) * 2 * BN);
                mbar_arrive_expect_tx(barp, 2 * bytes);
                bulk_load_g2s(dst, p.scale + n0, bytes, bar);
                bulk_load_g2s(dst + 4 * BN, p.scale + p.K + n0, bytes, bar);
            }
            __syncwarp();
        };
        if (ss_issuer && !(probe & 4))   // constants: before the PDL wait
            for (int bb = ALLW ? 0 : b0; bb < (ALLW ? Cfg::NBUF : b0 + 1); ++bb) ss_issue(tile0 + bb * tstep, bb, 0);
        // outputs are written only after the previous kernel completed (with row
        // flags, every tensor a launch touches has its own buffer: no WAR hazard)
        if (!p.dep_in) pdl_wait();
        // count, per output image row n*P + p = m / Q, the pixels x columns this warp
        // wrote (lanes grouped by row with ballots; <= a few rows per 32 pixels)
        unsigned warp_total = 0;   // codes this warp wrote (counted per unit, added at exit)
        if constexpr (Cfg::RES) {   // the residual skip (an earlier layer's output) is in memory
            if (p.dep_skip) wait_counter(p.dep_skip, p.dep_skip_total);
        }
        int j = 0;    // this unit's index among the units of its buffer
        for (int unit = tile0 + b0 * tstep, lu = 0; unit < p.num_units;
             unit += (ALLW ? 1 : Cfg::NBUF) * tstep, ++lu) {
            if constexpr (ALLW) {
                b = lu % Cfg::NBUF;
                j = lu / Cfg::NBUF;
                slab = out_stage + b * Cfg::OUT_BYTES + (half * 4 + quad) * Cfg::SLAB;
                if constexpr (CG == 2) acc_empty_leader = mapa_shared(smem_u32(&acc_empty[b]), 0);
            } else {
                j = lu;
            }
            const int tile = p.splits == 1 ? unit : p.fd_splits.div(unit);
            const int m_blk = p.fd_ntiles.div(tile), n_blk = tile - m_blk * p.n_tiles;
            const int mrow0 = m_blk * (BM * CG * Cfg::AMT) + (int)rank * BM;
            int m = mrow0 + row;
            // halo modes: MMA row r of the unit -> (output row within the tile,
            // padded column); the S-1 right-most padded columns and rows past the
            // tile are discarded (m = M)
            auto halo_m = [&](int r) {
                const int rt = m_blk * CG + (int)rank;
                const int n = p.fd_tpi.div(rt);
                const int pl = p.fd_Wp.div(r), qq = r - pl * p.Wp;
                const int pp = (rt - n * p.tiles_per_img) * p.rpt + pl;
                const bool ok = rt < p.m_tiles && pl < p.rpt && pp < p.P && qq < p.Q;
                return ok ? (n * p.P + pp) * p.Q + qq : p.M;
            };
            if constexpr (HA || S2H) m = halo_m(row);
            // residual (OUT_RES): the skip tensor's 16-byte chunk at (row mm, this chunk's bytes)
            auto load_skip = [&](int mm, int c) -> uint4 {
                const int gbyte = n_blk * Cfg::OUT_ROW + half * Cfg::EPI_ROW + c * 16;
                if (mm < p.M && gbyte < p.out_row)
                    return __ldcs(reinterpret_cast<const uint4 *>(p.skip + (int64_t)mm * p.out_row + gbyte));
                return make_uint4(0u, 0u, 0u, 0u);
            };
            // OUT_RES: this thread's skip chunks of every m-group, loaded before the
            // accumulator wait (the skip tensor is an earlier layer's output), so
            // their latency overlaps the tile's mainloop
            constexpr int NCH = Cfg::EPI_COLS / Cfg::CW;
            constexpr bool SKT = Cfg::SKIP_TMA;
            uint4 skp[Cfg::RES && !SKT ? Cfg::MT : 1][Cfg::RES && !SKT ? NCH : 1];
            if constexpr (SKT) {
                // the warp's skip slab -> its (free) output staging slab, one bulk copy per
                // 128-byte column block, completing on the warp's own barrier
                if (p.splits == 1) {
                    if (lane == 0) {
                        tma_store_wait_read0();   // the slab's previous store has read it out
                        mbar_arrive_expect_tx(&skbar[warp], (uint32_t)Cfg::SLAB);
#pragma unroll
                        for (int s = 0; s < Cfg::EPI_NSUB; ++s)
                            tma_load_2d(slab + s * (32 * Cfg::EPI_SUBW), &tm_s, &skbar[warp],
                                        n_blk * Cfg::OUT_ROW + half * Cfg::EPI_ROW + s * Cfg::EPI_SUBW, mrow0 + quad * 32,
                                        policy_evict_first());
                    }
                    __syncwarp();
                }
            } else if constexpr (Cfg::RES) {
                if (p.splits == 1) {
#pragma unroll
                    for (int g = 0; g < Cfg::MT; ++g) {
                        const int mg = Cfg::MT == 1 ? m : (HA || S2H) ? halo_m(g * BM + row) : mrow0 + g * BM + row;
#pragma unroll
                        for (int c = 0; c < NCH; ++c) skp[g][c] = load_skip(mg, c);
                    }
                }
            }
            {
                const long long t0 = trace ? clock64() : 0;
                mbar_wait_relaxed(&acc_full[b], j & 1, p.epi_wait, p.epi_wait_ns);
                CONVQ_TL(4 + warp, j);
                if (trace && lane == 0 && warp == Cfg::EPI_WARP0) {
                    atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_EPI_ACC, clock64() - t0);
                    if (j == 0) trace[blockIdx.x * TR_SLOTS + TR_TACC] = globaltimer_ns();
                }
            }
            tc_fence_after();
            if (probe & 4) {   // measurement: release the accumulator untouched
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(acc_empty_leader);
                    else mbar_arrive(&acc_empty[b]);
                }
                continue;
            }
            if (ss_issuer) ss_issue(unit + Cfg::NBUF * tstep, b, j + 1);
            const uint32_t taddr0 = tmem_base + ((uint32_t)(quad * 32) << 16) + b * Cfg::TBW + half * Cfg::EPI_COLS;
            // TMEM -> registers, software-pipelined: the load of chunk c+1 is in
            // flight while chunk c is requantized (tcgen05.wait::ld waits for all
            // of this thread's loads, so each wait covers exactly one chunk).
            auto release_acc = [&]() {   // every column of this warp is in registers
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(acc_empty_leader);
                    else mbar_arrive(&acc_empty[b]);
                }
            };
            // scale/shift of this tile's columns: the buffer's smem slot (filled by
            // the MMA warp's bulk copy) or, for split-K units, global memory
            const float *ss_b = ss_stage + (3 * b + j % 3) * 2 * BN;
            // process(): requantize + pack one chunk (CW columns) -> its 16 packed bytes
            // (S32 mode: stores the raw accumulators itself); put(): store a packed chunk.
            // Split so a caller can compute the next chunk -- whose scale/shift LDS would
            // otherwise be ordered behind this chunk's staging STS (possible smem alias)
            // -- before storing this one.
            auto process = [&](const uint32_t (&v)[Cfg::CW], const int c, auto smem_tag, const uint4 sk_in) -> uint4 {
                    constexpr bool SMEM_SS = decltype(smem_tag)::value;
                    const int ccol = half * Cfg::EPI_COLS + c * Cfg::CW;   // column within the tile
                    const int col0 = n_blk * BN + ccol;
                    if (Cfg::OUTP == OUT_S32) {
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
                        // SKIP_TMA: this chunk's skip codes sit in the staging slab at the very
                        // address the packed output chunk is written to below
                        uint4 sk = sk_in;
                        if constexpr (Cfg::SKIP_TMA) {
                            if (SMEM_SS) {
                                const int sb = c * 16;
                                sk = *reinterpret_cast<const uint4 *>(
                                    slab + (sb / Cfg::EPI_SUBW) * (32 * Cfg::EPI_SUBW) +
                                    swz<Cfg::EPI_SUBW>(lane * Cfg::EPI_SUBW + sb % Cfg::EPI_SUBW));
                            }
                        }
                        // (smem slot: columns past K hold stale values; their codes are never stored)
                        const bool full = SMEM_SS || col0 + Cfg::CW <= p.K;
                        const float4 *s4 = reinterpret_cast<const float4 *>(SMEM_SS ? ss_b + ccol : p.scale + col0);
                        const float4 *h4 = reinterpret_cast<const float4 *>(SMEM_SS ? ss_b + BN + ccol : p.scale + p.K + col0);
                        // scale / shift of columns 4q..4q+3 of this chunk
                        auto ss4 = [&](int q, float4 &sa, float4 &sb) {
                            if (full) {
                                sa = SMEM_SS ? s4[q] : __ldg(s4 + q);
                                sb = SMEM_SS ? h4[q] : __ldg(h4 + q);
                            } else {
                                float t[8];
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const bool ok = col0 + 4 * q + e < p.K;  // columns past K are never stored
                                    t[e] = ok ? __ldg(p.scale + col0 + 4 * q + e) : 0.f;
                                    t[4 + e] = ok ? __ldg(p.scale + p.K + col0 + 4 * q + e) : 0.f;
                                }
                                sa = make_float4(t[0], t[1], t[2], t[3]);
                                sb = make_float4(t[4], t[5], t[6], t[7]);
                            }
                        };
                        uint4 pk;   // 16 packed bytes = this chunk (16 s8 or 32 s4 columns)
                        if constexpr (BITS == 8) {
                            // u = fma((float)acc, scale, shift); the F2IP pair conversion
                            // rounds (RNE) and saturates to [-128, 127]; ReLU (lo = 0)
                            // then clears the negative bytes of each packed word.  (Equal
                            // to clamp(rne(u), lo, hi) for every finite u; u is never NaN
                            // for finite scale/shift, the documented precondition.)
                            // Four columns at a time: 8 scale/shift registers live, not 32.
                            uint32_t w4[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                float4 sa, sb;
                                ss4(q, sa, sb);
                                float u0, u1, u2, u3;
                                fma2_rn(__int2float_rn((int)v[4 * q]), __int2float_rn((int)v[4 * q + 1]), sa.x, sa.y,
                                        sb.x, sb.y, u0, u1);
                                fma2_rn(__int2float_rn((int)v[4 * q + 2]), __int2float_rn((int)v[4 * q + 3]), sa.z,
                                        sa.w, sb.z, sb.w, u2, u3);
                                if constexpr (Cfg::RES) {
                                    // v = fmaf(skip, res_scale, u) (reading 15); skip byte -> exact float as
                                    // (2^23 + (byte ^ bias)) - (2^23 + bias), bias 0x80 for a signed skip,
                                    // 0 for an unsigned one (reading 16): one PRMT per code + one FADD2 per
                                    // two codes (the subtraction is exact: integers below 2^24)
                                    const uint32_t wv = (&sk.x)[q] ^ p.skip_xor;
                                    float k0, k1, k2, k3;
                                    add2_rn(__uint_as_float(__byte_perm(wv, 0x4B000000u, 0x7650)),
                                            __uint_as_float(__byte_perm(wv, 0x4B000000u, 0x7651)), -p.skip_off, k0, k1);
                                    add2_rn(__uint_as_float(__byte_perm(wv, 0x4B000000u, 0x7652)),
                                            __uint_as_float(__byte_perm(wv, 0x4B000000u, 0x7653)), -p.skip_off, k2, k3);
                                    fma2_rn(k0, k1, p.res_scale, p.res_scale, u0, u1, u0, u1);
                                    fma2_rn(k2, k3, p.res_scale, p.res_scale, u2, u3, u2, u3);
                                }
                                if constexpr (Cfg::U8) {
                                    w4[q] = pack4_f32_u8(u0, u1, u2, u3);       // unsigned codes: clamp [0, 255]
                                } else if (Cfg::RES && p.y_uns) {
                                    w4[q] = pack4_f32_u8(u0, u1, u2, u3);
                                } else {
                                    w4[q] = pack4_f32_s8(u0, u1, u2, u3);
                                    if (relu8 || p.relu) w4[q] = relu_s8x4(w4[q]);
                                }
                            }
                            pk = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                        } else {
                            int r[Cfg::CW];
#pragma unroll
                            for (int q = 0; q < Cfg::CW / 4; ++q) {
                                float4 sa, sb;
                                ss4(q, sa, sb);
                                if constexpr (Cfg::RELU4) {
                                    // ReLU epilogue: the MMA holds 256*acc (a4), and (float)(256 acc) * 2^-8
                                    // == (float)acc exactly (power-of-two scaling commutes with RN, no
                                    // underflow for integers), so one I2FP + half an FMUL2 replace the
                                    // shift; clamp(rne(u), 0, 255) in one F2I.U8 (4x the s32 F2I rate),
                                    // and the nibble pack below saturates at the top code (7 signed /
                                    // 15 unsigned, reading 16) -- no separate min
                                    float f0, f1, f2, f3, u0, u1, u2, u3;
                                    mul2_rn(__int2float_rn((int)v[4 * q]), __int2float_rn((int)v[4 * q + 1]), 0.00390625f,
                                            f0, f1);
                                    mul2_rn(__int2float_rn((int)v[4 * q + 2]), __int2float_rn((int)v[4 * q + 3]),
                                            0.00390625f, f2, f3);
                                    fma2_rn(f0, f1, sa.x, sa.y, sb.x, sb.y, u0, u1);
                                    fma2_rn(f2, f3, sa.z, sa.w, sb.z, sb.w, u2, u3);
                                    r[4 * q] = f2u8_rn(u0);
                                    r[4 * q + 1] = f2u8_rn(u1);
                                    r[4 * q + 2] = f2u8_rn(u2);
                                    r[4 * q + 3] = f2u8_rn(u3);
                                } else if constexpr (Cfg::RES) {
                                    // codes 4q..4q+3 = nibbles 4(q%2).. of skip word q/2; nibble -> exact
                                    // float as (2^23 + (nib ^ bias)) - (2^23 + bias), bias 8 for a signed
                                    // skip, 0 unsigned (reading 16); ReLU / clamp after the add
                                    const uint32_t wv = (&sk.x)[q >> 1] ^ p.skip_xor;
                                    const float sav[4] = {sa.x, sa.y, sa.z, sa.w}, sbv[4] = {sb.x, sb.y, sb.z, sb.w};
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const uint32_t nib = (wv >> (4 * (4 * (q & 1) + e))) & 0xFu;
                                        const float kf = __fsub_rn(__uint_as_float(0x4B000000u | nib), p.skip_off);
                                        const float u = __fmaf_rn(__int2float_rn((int)v[4 * q + e] >> 8), sav[e], sbv[e]);
                                        const float vv = fmaxf(__fmaf_rn(kf, p.res_scale, u), lo);
                                        asm("cvt.rni.s32.f32 %0, %1;" : "=r"(r[4 * q + e]) : "f"(vv));
                                    }
                                } else {
                                    r[4 * q] = requant_int((int)v[4 * q] >> 8, sa.x, sb.x, lo);
                                    r[4 * q + 1] = requant_int((int)v[4 * q + 1] >> 8, sa.y, sb.y, lo);
                                    r[4 * q + 2] = requant_int((int)v[4 * q + 2] >> 8, sa.z, sb.z, lo);
                                    r[4 * q + 3] = requant_int((int)v[4 * q + 3] >> 8, sa.w, sb.w, lo);
                                }
                            }
                            if (Cfg::RELU4 && !p.y_uns)   // ReLU codes in [0, 255] -> saturated at 7 by the s4 pack
                                pk = make_uint4(pack8_sat_s4(r), pack8_sat_s4(r + 8), pack8_sat_s4(r + 16),
                                                pack8_sat_s4(r + 24));
                            else if (Cfg::RELU4 || (Cfg::RES && p.y_uns))   // codes >= 0: unsigned packing (top 15)
                                pk = make_uint4(pack8_sat_u4(r), pack8_sat_u4(r + 8), pack8_sat_u4(r + 16),
                                                pack8_sat_u4(r + 24));
                            else
                                pk = make_uint4(pack8_sat_s4(r), pack8_sat_s4(r + 8), pack8_sat_s4(r + 16),
                                                pack8_sat_s4(r + 24));
                        }
                        return pk;
                    }
                    return make_uint4(0u, 0u, 0u, 0u);
            };
            auto put = [&](const int c, const uint4 pk) {
                    if constexpr (Cfg::OUTP != OUT_S32) {
                        const int sbyte = c * 16;                 // byte within this warp's slab row
                        if constexpr (Cfg::OUTP == OUT_TMA) {
                            if (c == 0) {   // the slab must have been read out by this warp's previous store
                                if (lane == 0) tma_store_wait_read0();   // (waited as late as possible)
                                __syncwarp();
                            }
                            uint8_t *sub = slab + (sbyte / Cfg::EPI_SUBW) * (32 * Cfg::EPI_SUBW);
                            *reinterpret_cast<uint4 *>(sub + swz<Cfg::EPI_SUBW>(lane * Cfg::EPI_SUBW + sbyte % Cfg::EPI_SUBW)) = pk;
                        } else {
                            const int gbyte = n_blk * Cfg::OUT_ROW + half * Cfg::EPI_ROW + sbyte;
                            if (m < p.M && gbyte < p.out_row) {
                                uint8_t *dst = p.y8 + (int64_t)m * p.out_row + gbyte;
                                if (p.out_policy) st_global_v4_hint(dst, pk, out_pol);
                                else *reinterpret_cast<uint4 *>(dst) = pk;
                            }
                        }
                    }
            };
            uint32_t va[Cfg::CW], vb[Cfg::CW];
            uint32_t taddr = taddr0;
            bool emit = true;   // this warp writes the region's outputs
            // TMA store of this warp's staged slab (m-group g's 32 rows)
            auto store_slab = [&](int g) {
                if (Cfg::OUTP == OUT_TMA && emit) {
                    fence_proxy_async_smem();  // st.shared -> visible to the TMA (async proxy)
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int s = 0; s < Cfg::EPI_NSUB; ++s) {
                            const int c0 = n_blk * Cfg::OUT_ROW + half * Cfg::EPI_ROW + s * Cfg::EPI_SUBW;
                            const int c1 = mrow0 + g * BM + quad * 32;
                            if (p.out_policy) tma_store_2d_hint(&tm_y, slab + s * (32 * Cfg::EPI_SUBW), c0, c1, out_pol);
                            else tma_store_2d(&tm_y, slab + s * (32 * Cfg::EPI_SUBW), c0, c1);
                        }
                        tma_store_commit();
                    }
                }
            };
            if (p.splits > 1) {
                // split-K: add this partial into the region's workspace (column-major
                // [col][32 rows], so each red instruction covers 128 contiguous bytes);
                // the warp whose arrival completes the region requantizes the sum and
                // leaves the workspace and counter zero for the next run.  s32
                // addition is associative: bit-exact in any arrival order.
                const int region = (tile * CG + (int)rank) * (4 * EPB) + half * 4 + quad;
                int32_t *wsr = p.ws + (int64_t)region * (32 * Cfg::EPI_COLS) + lane;
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    tmem_ld_issue<Cfg::CW>(taddr + c * Cfg::CW, va);
                    tmem_ld_wait_regs(va);
#pragma unroll
                    for (int q = 0; q < Cfg::CW; ++q) red_add_s32(wsr + (c * Cfg::CW + q) * 32, (int)va[q]);
                }
                release_acc();
                __threadfence();
                __syncwarp();
                unsigned old = 0;
                if (lane == 0) old = atomicAdd(p.cnt + region, 1u);
                old = __shfl_sync(0xffffffffu, old, 0);
                emit = old == (unsigned)(p.splits - 1);
                if (emit) {
                    __threadfence();
#pragma unroll 1
                    for (int c = 0; c < NCH; ++c) {
#pragma unroll
                        for (int q = 0; q < Cfg::CW; ++q) {
                            va[q] = (uint32_t)__ldcg(wsr + (c * Cfg::CW + q) * 32);
                            __stcg(wsr + (c * Cfg::CW + q) * 32, 0);
                        }
                        put(c, process(va, c, std::false_type{}, Cfg::RES ? load_skip(m, c) : make_uint4(0u, 0u, 0u, 0u)));
                    }
                    if (lane == 0) p.cnt[region] = 0u;
                }
            } else {
                // the MMA warp's copy of this tile's scale/shift (long done by now)
                if (Cfg::OUTP != OUT_S32) mbar_wait(&ss_full[3 * b + j % 3], (j / 3) & 1);
                if constexpr (SKT) {   // this warp's skip slab (issued before the accumulator wait)
                    mbar_wait(&skbar[warp], (uint32_t)(lu & 1));
                }
                // MT2: the unit's two m-groups sit in TMEM columns [g*BN, (g+1)*BN)
                for (int g = 0; g < Cfg::MT; ++g) {
                    taddr = taddr0 + g * BN;
                    if constexpr (Cfg::MT > 1) m = (HA || S2H) ? halo_m(g * BM + row) : mrow0 + g * BM + row;
                    const bool last = g == Cfg::MT - 1;
                    auto skr = [&](int c) -> uint4 { return skp[Cfg::RES && !SKT ? g : 0][Cfg::RES && !SKT ? c : 0]; };
                    if constexpr (BITS == 8 && NCH % 2 == 0 && CONVQ_TMEM_PIPE && NCH > 2) {
                        // 32 columns per tcgen05.ld, double-buffered: the next 32 columns'
                        // load is in flight while these are requantized (tcgen05.wait::ld
                        // waits for every outstanding load, so the wait follows the work)
                        uint32_t v32[2][32];
                        tmem_ld_issue<32>(taddr, v32[0]);
                        tmem_ld_wait_regs(v32[0]);
#pragma unroll
                        for (int c = 0; c < NCH; c += 2) {
                            const int cur = (c / 2) & 1;
                            const bool more = c + 2 < NCH;
                            if (more) tmem_ld_issue<32>(taddr + (c + 2) * Cfg::CW, v32[cur ^ 1]);
                            const uint4 pk0 = process(reinterpret_cast<const uint32_t(&)[Cfg::CW]>(v32[cur][0]), c,
                                                      std::true_type{}, skr(c));
                            const uint4 pk1 = process(reinterpret_cast<const uint32_t(&)[Cfg::CW]>(v32[cur][16]), c + 1,
                                                      std::true_type{}, skr(c + 1));
                            put(c, pk0);
                            put(c + 1, pk1);
                            if (more) {
                                tmem_ld_wait_regs(v32[cur ^ 1]);
                                if (last && c + 4 >= NCH) release_acc();   // every column of this warp is in registers
                            }
                        }
                    } else if constexpr (BITS == 8 && NCH % 2 == 0) {
                        // 32 columns per tcgen05.ld (two 16-byte output pieces): half
                        // the exposed TMEM-load round trips of a 16-column loop
                        uint32_t v32[32];
#pragma unroll
                        for (int c = 0; c < NCH; c += 2) {
                            tmem_ld_issue<32>(taddr + c * Cfg::CW, v32);
                            tmem_ld_wait_regs(v32);
                            if (last && c + 2 >= NCH) release_acc();
                            // both chunks' requant (and scale/shift loads) before either staging store
                            const uint4 pk0 = process(reinterpret_cast<const uint32_t(&)[Cfg::CW]>(v32[0]), c,
                                                      std::true_type{}, skr(c));
                            const uint4 pk1 = process(reinterpret_cast<const uint32_t(&)[Cfg::CW]>(v32[16]), c + 1,
                                                      std::true_type{}, skr(c + 1));
                            put(c, pk0);
                            put(c + 1, pk1);
                        }
                    } else {
                        tmem_ld_issue<Cfg::CW>(taddr, va);
                        tmem_ld_wait_regs(va);
#pragma unroll
                        for (int c = 0; c < NCH; c += 2) {
                            const bool more1 = c + 1 < NCH;
                            if (more1) tmem_ld_issue<Cfg::CW>(taddr + (c + 1) * Cfg::CW, vb);
                            else if (last) release_acc();   // every column of this warp is in registers
                            put(c, process(va, c, std::true_type{}, skr(c)));
                            if (more1) {
                                tmem_ld_wait_regs(vb);
                                const bool more2 = c + 2 < NCH;
                                if (more2) tmem_ld_issue<Cfg::CW>(taddr + (c + 2) * Cfg::CW, va);
                                else if (last) release_acc();
                                put(c + 1, process(vb, c + 1, std::true_type{}, skr(c + 1)));
                                if (more2) tmem_ld_wait_regs(va);
                            }
                        }
                    }
                    if constexpr (Cfg::MT > 1) store_slab(g);   // the slab is reused by the next group
                }
            }
            if constexpr (Cfg::MT == 1) store_slab(0);
            if (p.dep_out && emit) {   // this unit's codes written by this warp (valid pixels x columns)
                const int cols = min(Cfg::EPI_COLS, p.K - (n_blk * BN + half * Cfg::EPI_COLS));
#pragma unroll
                for (int g = 0; g < Cfg::MT; ++g) {
                    const int mg = Cfg::MT == 1 ? m : (HA || S2H) ? halo_m(g * BM + row) : mrow0 + g * BM + row;
                    const unsigned valid = __ballot_sync(0xffffffffu, mg < p.M);
                    if (cols > 0) warp_total += (unsigned)(__popc(valid) * cols);
                }
            }
            CONVQ_TL(24 + warp, j);
        }
        // before exit the staging smem must have been read out by the TMA (.read); the
        // writes themselves need not be complete (grid completion flushes them) unless a
        // completion counter is raised below -- waiting only for the reads lets the CTA
        // leave (and the next layer's CTA take the SM) a global-write latency earlier
        if (Cfg::OUTP == OUT_TMA && lane == 0) {
            if (p.dep_out) tma_store_wait0();
            else tma_store_wait_read0();
        }
        if (p.dep_out) {
            // once per warp at its exit: every store of this warp is complete (TMA:
            // lane 0's wait_group 0 above + a proxy fence; direct stores: every lane's
            // membar), then one relaxed add of the codes it wrote
            if constexpr (Cfg::OUTP == OUT_TMA) {
                if (lane == 0) fence_proxy_async_global();
            } else {
                __threadfence();
            }
            __syncwarp();
            if (lane == 0 && warp_total) atomicAdd(p.dep_out, warp_total);
        }
#undef CONVQ_TL
    } else if (warp < Cfg::PROD_WARP) {
        // =========================== INT4 transform =========================
        if constexpr (BITS == 4 && WS && HA) {
            // weight-stationary halo: the packed weight block is expanded once; every stage
            // is one packed halo box (tile, channel block), expanded into the stage's s8 box
            const int tid = threadIdx.x - 32 * Cfg::XF_WARP0;  // 0..127
            const uint32_t ready0 = CG == 2 ? mapa_shared(smem_u32(&ready[0]), 0) : 0;
            if (tile0 < p.num_tiles) {
                mbar_wait(bfull, 0);
                for (int kb = 0; kb < p.num_kb; ++kb)
                    expand_tile<KCH>(b_res_pk + kb * (Cfg::BNL * Cfg::LOAD_ROW), b_res + kb * Cfg::B_TILE, Cfg::BNL,
                                     tid, 128);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&hempty[2]), 0));
                    else mbar_arrive(&hempty[2]);
                }
            }
            const int halo_pix = p.halo_tx / Cfg::LOAD_ROW;  // box rows x Wp pixels
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                for (int cblk = 0; cblk < p.num_cblk; ++cblk) {
                    mbar_wait(&full[stage], phase);
                    expand_tile<KCH>(a_pk + stage * Cfg::A_PK, a_s8 + stage * Cfg::A_S8, halo_pix, tid, 128);
                    fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05.mma
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(ready0 + 8u * stage);
                        else mbar_arrive(&ready[stage]);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        } else if constexpr (BITS == 4 && HA) {
            // halo mode: per (tile, channel block) the first stage carries the packed
            // halo box -> expanded ONCE into the s8 halo buffer the filter taps'
            // shifted descriptors read; every stage carries NSUB taps' weights
            const int tid = threadIdx.x - 32 * Cfg::XF_WARP0;  // 0..127
            const uint32_t ready0 = CG == 2 ? mapa_shared(smem_u32(&ready[0]), 0) : 0;
            const int RS = p.R * p.S;
            const int halo_pix = p.halo_tx / Cfg::LOAD_ROW;  // box rows x Wp pixels
            int stage = 0, hcount = 0;
            uint32_t phase = 0;
            for (int tile = tile0; tile < p.num_tiles; tile += tstep) {
                for (int cblk = 0; cblk < p.num_cblk; ++cblk, ++hcount) {
                    const int hb = hcount % Cfg::NHALO;
                    for (int tap = 0; tap < RS; tap += NSUB) {
                        const int nsub = min(NSUB, RS - tap);
                        mbar_wait(&full[stage], phase);
                        if (tap == 0)
                            expand_tile<KCH>(halo_pk + hb * Cfg::HALO_PK, halo_buf + hb * Cfg::HALO_BYTES, halo_pix,
                                             tid, 128);
                        for (int j = 0; j < nsub; ++j)
                            expand_kblock<KCH, 0, Cfg::BNL, 128>(nullptr, nullptr, b_pk + stage * Cfg::B_PK + j * Cfg::B_PK_SUB,
                                                                b_s8 + stage * Cfg::B_S8 + j * Cfg::B_SUB, tid);
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
        } else if constexpr (BITS == 4) {
            const int tid = threadIdx.x - 32 * Cfg::XF_WARP0;  // 0..127
            const uint32_t ready0 = CG == 2 ? mapa_shared(smem_u32(&ready[0]), 0) : 0;
            if constexpr (WS) {
                // the CTA's packed weight block -> s8 resident block, once; then tell the
                // (leader's) MMA warp
                if (tile0 < p.num_tiles) {
                    mbar_wait(bfull, 0);
                    for (int kb = 0; kb < p.num_kb; ++kb)
                        expand_tile<KCH>(b_res_pk + kb * (Cfg::BNL * Cfg::LOAD_ROW), b_res + kb * Cfg::B_TILE, Cfg::BNL,
                                         tid, 128);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&hempty[2]), 0));
                        else mbar_arrive(&hempty[2]);
                    }
                }
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = tile0; unit < p.num_units; unit += tstep) {
                int tile, kb_lo, kb_hi;
                unit_range(p, unit, tile, kb_lo, kb_hi);
                for (int kb = kb_lo; kb < kb_hi; kb += NSUB) {
                    const int nsub = min(NSUB, kb_hi - kb);
                    mbar_wait(&full[stage], phase);
                    // (WS: stages carry A only; MT2: the k-block's AMT A tiles are contiguous)
                    for (int j = 0; j < nsub; ++j)
                        expand_kblock<KCH, Cfg::AMT * BM, WS ? 0 : Cfg::BNL, 128>(
                            a_pk + stage * Cfg::A_PK + j * Cfg::AMT * Cfg::A_PK_SUB,
                            a_s8 + stage * Cfg::A_S8 + j * Cfg::AMT * Cfg::A_SUB,
                            b_pk + stage * Cfg::B_PK + j * Cfg::B_PK_SUB, b_s8 + stage * Cfg::B_S8 + j * Cfg::B_SUB, tid);
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
    if (trace && threadIdx.x == 0) {
        atomicAdd(trace + blockIdx.x * TR_SLOTS + TR_TOTAL, clock64() - t_start);
        trace[blockIdx.x * TR_SLOTS + TR_T1] = globaltimer_ns();
    }
    if (warp == Cfg::MMA_WARP) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_cg2<Cfg::TMEM_COLS>(tmem_base);
        else tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace convq
