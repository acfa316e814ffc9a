// plan.cuh -- internal (not part of the C ABI): the plan structure, the
// TileConfig description and the templated launcher shared by the kernel
// translation units (kern_*.cu) and the host library (convq.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/convq.h"
#include "conv.cuh"

namespace convq {

int set_err(int code, const char *fmt, ...);   // thread-local last error (convq.cu)
extern int g_num_sms;

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess) return set_err(CONV_Q_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// FastDiv constants: s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1; then
// n / d == (umulhi(n, m) + n) >> s for 0 <= n < 2^31 (checked exhaustively at
// the boundaries by tests/test_abi_cpu.py's emulation).
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d < 1 ? 1 : d;
    uint32_t s = 0;
    while ((1ull << s) < f.d) ++s;
    f.s = s;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << s) - f.d)) / f.d) + 1);
    return f;
}

struct Cand {
    int bn, kch, cg, nsub;  // N tile, channels per k-block, CTAs per tile, k-blocks per stage
    int direct;             // packed output by direct stores (1) or smem staging + TMA store (0)
    int halo = 0;           // duplicate-aware halo A operand (stride 1 only)
    int ws = 0;             // weight-stationary: resident weight block per CTA (INT8, CG = 1)
    int split = 1;          // split-K work units per tile (1 = none)
};

// weight-stationary instantiations (BN, KCH, NSUB, halo, CG)
#define CONVQ_WS_LIST(X)                                                                        \
    X(64, 64, 1, 1, 1) X(64, 128, 1, 1, 1) X(128, 64, 1, 1, 1) X(128, 128, 1, 1, 1)            \
    X(64, 64, 1, 1, 2) X(64, 128, 1, 1, 2) X(128, 64, 1, 1, 2) X(128, 128, 1, 1, 2)            \
    X(64, 64, 1, 0, 1) X(128, 64, 1, 0, 1) X(256, 64, 1, 0, 1)                                \
    X(64, 128, 1, 0, 1) X(128, 128, 1, 0, 1) X(256, 128, 1, 0, 1)                             \
    X(64, 64, 2, 0, 1) X(128, 64, 2, 0, 1) X(256, 64, 2, 0, 1)                                \
    X(64, 128, 2, 0, 1) X(128, 128, 2, 0, 1) X(256, 128, 2, 0, 1)                             \
    X(64, 64, 1, 0, 2) X(128, 64, 1, 0, 2) X(256, 64, 1, 0, 2)                                \
    X(64, 128, 1, 0, 2) X(128, 128, 1, 0, 2) X(256, 128, 1, 0, 2)                             \
    X(64, 64, 1, 4, 1) X(64, 64, 1, 4, 2)                                                      \
    X(64, 64, 1, 9, 1) X(64, 64, 1, 12, 1) X(64, 64, 1, 9, 2) X(64, 64, 1, 12, 2)                 \
    X(64, 64, 1, 8, 1) X(64, 128, 1, 8, 1) X(128, 64, 1, 8, 1) X(128, 128, 1, 8, 1)

}  // namespace convq

struct conv_q_plan_s {
    using Cand = convq::Cand;
    int N, H, W, C, K, R, S, stride, pad, bits;
    int P, Q;
    int64_t M, Kg;
    // space-to-depth stem (conv_q_plan_s2d): the fields above describe the
    // stride-1 window convolution the kernel runs; o_* the caller's conv
    int s2d = 0;
    int pad_hi = 0;    // bottom padding of the H walk (= pad unless s2d)
    int xs_W = 0;      // s2d: stored columns of the s2d tensor (zero borders included)
    int o_H = 0, o_W = 0, o_C = 0, o_R = 0, o_S = 0, o_stride = 0, o_pad = 0;
    int row_bytes;     // C*bits/8
    int out_row;       // K*bits/8
    int relu = 0, out_mode = CONV_Q_OUT_PACKED;
    const void *skip = nullptr;   // conv_q_plan_set_residual: fused residual add (NULL = none)
    float res_scale = 0.f;
    int x_uns = 0, y_uns = 0, skip_uns = 0;   // conv_q_plan_set_formats: unsigned codes (DESIGN reading 16)
    // conv_q_plan_set_deps: cross-launch completion counters (NULL in = griddepcontrol.wait)
    const unsigned *dep_in = nullptr, *dep_skip = nullptr;
    unsigned *dep_out = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<Cand> cands;
    int sel = 0;
    int user_sel = 0;  // sel chosen explicitly (conv_q_plan_set_config / conv_q_plan_tune): the cache never overrides it
    float tuned_us = -1.f;
    int rotate = 0;    // CONV_Q_ROTATE=1: rotate each CTA's k-block start (A/B measurement)
    int probe = 0;     // CONV_Q_PROBE (measurement only; results are garbage when != 0)
    int epi_wait = 0;  // CONV_Q_EPI_WAIT / _NS: how epilogue warps wait for accumulators (A/B)
    unsigned epi_wait_ns = 0;
    int out_policy = 1; // CONV_Q_OUT_POLICY: L2 hint on output stores (0 none, 1 evict_last = default: the next layer reads them, 2 evict_first)
    int grid_pct = 100; // persistent grid as a percentage of the SMs (conv_q_plan_search's grid knob)
    unsigned long long *trace = nullptr;  // conv_q_plan_set_trace (measurement only)
    unsigned long long *tl = nullptr;     // conv_q_plan_set_timeline (measurement only)
    // tensor-map cache (re-encoded when a pointer or the config changes)
    CUtensorMap tm_a, tm_b, tm_y, tm_s;   // tm_s: the residual skip tensor (y's box / swizzle)
    const void *c_x = nullptr, *c_w = nullptr, *c_y = nullptr, *c_skip = nullptr;
    int c_sel = -1, c_mode = -1;
    // split-K workspace (zero between runs; owned by the plan)
    int32_t *ws = nullptr;
    unsigned *cnt = nullptr;
    size_t ws_bytes = 0, cnt_bytes = 0;
    ~conv_q_plan_s() {
        if (ws) cudaFree(ws);
        if (cnt) cudaFree(cnt);
    }
};


namespace convq {

// Whether a TileConfig fits shared memory (>= 2 stages) for both output modes.
template <int BITS>
inline bool cand_fits(const Cand &c) {
    if (c.ws) {
#define CONVQ_WFIT(BN_, KC_, NS_, H_, CG_)                                                             \
        if (c.bn == BN_ && c.kch == KC_ && c.nsub == NS_ && c.halo == H_ && c.cg == CG_)               \
            return (c.direct ? ConvCfg<BITS, BN_, KC_, OUT_DIRECT, CG_, NS_, 2 + H_>::FITS              \
                             : ConvCfg<BITS, BN_, KC_, OUT_TMA, CG_, NS_, 2 + H_>::FITS) &&             \
                   ConvCfg<BITS, BN_, KC_, OUT_S32, CG_, NS_, 2 + H_>::FITS;
        CONVQ_WS_LIST(CONVQ_WFIT)
#undef CONVQ_WFIT
        return false;
    }
    if (c.halo) {
#define CONVQ_HFIT(BN_, KC_, CG_, NS_)                                                              \
        if (c.bn == BN_ && c.kch == KC_ && c.cg == CG_ && c.nsub == NS_)                            \
            return ConvCfg<BITS, BN_, KC_, OUT_DIRECT, CG_, NS_, 1>::FITS && ConvCfg<BITS, BN_, KC_, OUT_S32, CG_, NS_, 1>::FITS;
#define CONVQ_HFIT_NS(BN_, KC_, CG_) CONVQ_HFIT(BN_, KC_, CG_, 3) CONVQ_HFIT(BN_, KC_, CG_, 1)
        CONVQ_HFIT_NS(64, 128, 1) CONVQ_HFIT_NS(128, 128, 1) CONVQ_HFIT_NS(256, 128, 1)
        CONVQ_HFIT_NS(64, 64, 1) CONVQ_HFIT_NS(128, 64, 1) CONVQ_HFIT_NS(256, 64, 1)
        CONVQ_HFIT_NS(64, 128, 2) CONVQ_HFIT_NS(128, 128, 2) CONVQ_HFIT_NS(256, 128, 2)
        CONVQ_HFIT_NS(64, 64, 2) CONVQ_HFIT_NS(128, 64, 2) CONVQ_HFIT_NS(256, 64, 2)
#undef CONVQ_HFIT_NS
#undef CONVQ_HFIT
        return false;
    }
#define CONVQ_FIT(BN_, KC_, NS_, CG_)                                                        \
    if (c.bn == BN_ && c.kch == KC_ && c.nsub == NS_ && c.cg == CG_)                         \
        return (c.direct ? ConvCfg<BITS, BN_, KC_, OUT_DIRECT, CG_, NS_>::FITS                \
                         : ConvCfg<BITS, BN_, KC_, OUT_TMA, CG_, NS_>::FITS) &&               \
               ConvCfg<BITS, BN_, KC_, OUT_S32, CG_, NS_>::FITS;
#define CONVQ_FITS_BN(KC_, NS_, CG_) CONVQ_FIT(64, KC_, NS_, CG_) CONVQ_FIT(128, KC_, NS_, CG_) CONVQ_FIT(256, KC_, NS_, CG_)
    CONVQ_FITS_BN(128, 2, 1) CONVQ_FITS_BN(128, 1, 1) CONVQ_FITS_BN(64, 4, 1) CONVQ_FITS_BN(64, 1, 1)
    CONVQ_FITS_BN(32, 4, 1) CONVQ_FITS_BN(32, 1, 1)
    CONVQ_FITS_BN(128, 2, 2) CONVQ_FITS_BN(128, 1, 2) CONVQ_FITS_BN(64, 4, 2) CONVQ_FITS_BN(64, 1, 2)
    CONVQ_FITS_BN(32, 4, 2) CONVQ_FITS_BN(32, 1, 2)
#undef CONVQ_FITS_BN
#undef CONVQ_FIT
    return false;
}


// ============================================================== launch
template <int BITS, int BN, int KCH, int OUT, int CG, int NSUB, int HALO = 0>
inline int launch_conv(conv_q_plan_s *p, const float *scale, void *y) {
    using Cfg = ConvCfg<BITS, BN, KCH, OUT, CG, NSUB, HALO>;
    auto kern = conv_igemm_kernel<BITS, BN, KCH, OUT, CG, NSUB, HALO>;
    // One CTA per SM: every CTA allocates up to all 512 TMEM columns, so a second
    // resident CTA would block in tcgen05.alloc until the first exits.  Configs
    // whose shared memory would let two CTAs share an SM (228 KB per SM, 1 KB
    // reserved per CTA) launch with their request padded past half of it.
    // Shared memory: the weight-stationary region holds exactly this layer's
    // BN/CG x R*S*C block (rounded to 1 KB; the 64 KB budget is the plan-time
    // bound), and the ring gets as many stages as the rest of the 227 KB allows.
    const int wsb_s8 = (HALO & 2) ? (int)ceil_div((int64_t)p->R * p->S * (p->C / KCH) * Cfg::B_TILE, 1024) * 1024 : 0;
    if (wsb_s8 > Cfg::WSB) return set_err(CONV_Q_EUNSUPPORTED, "weight block %d B exceeds the resident region", wsb_s8);
    const int wsb = wsb_s8 + (BITS == 4 ? (int)ceil_div(wsb_s8 / 2, 1024) * 1024 : 0);   // + INT4 packed block
    const int stages = Cfg::stages_for(wsb);
    const int smem = Cfg::smem_for(wsb, stages);
    const int SMEM_LAUNCH = smem > 116 * 1024 ? smem : 116 * 1024;
    static bool attr_set = false;
    if (!attr_set) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
        attr_set = true;
    }
    ConvParams prm;
    prm.stages = stages;
    prm.wsb = wsb;
    prm.wsb_s8 = wsb_s8;
    prm.N = p->N; prm.H = p->H; prm.W = p->W; prm.C = p->C; prm.K = p->K; prm.R = p->R; prm.S = p->S;
    prm.stride = p->stride; prm.pad = p->pad; prm.pad_w = p->s2d ? 0 : p->pad; prm.P = p->P; prm.Q = p->Q; prm.M = (int)p->M;
    prm.row_bytes = p->row_bytes;
    prm.num_cblk = (int)ceil_div(p->C, KCH);   // (s8 C = 16 mod 32: the last block is partly zero-filled)
    prm.num_kb = p->R * p->S * prm.num_cblk;
    prm.n_tiles = (int)ceil_div(p->K, BN);
    prm.num_tiles = (int)(ceil_div(p->M, BM * CG * ((HALO & 5) ? 1 : ((HALO & 8) ? 2 : 1))) * prm.n_tiles);   // generic MT2: 256-row units
    prm.Wp = p->s2d ? p->xs_W : p->W + 2 * p->pad;   // MMA-row pitch of an output row (halo modes)
    constexpr int MTV = (HALO & 8) ? 2 : 1;   // MT2: a unit = two 128-row m-groups
    prm.rpt = std::max(1, std::min(p->P, MTV * BM / prm.Wp));
    prm.tiles_per_img = (int)ceil_div(p->P, prm.rpt);
    prm.m_tiles = p->N * prm.tiles_per_img;
    const int halo_rows = (int)ceil_div(MTV * BM + (p->R - 1) * prm.Wp + ((HALO & 4) ? 3 : p->S - 1), prm.Wp);
    prm.halo_tx = halo_rows * prm.Wp * ((HALO & 4) ? 16 : Cfg::LOAD_ROW);   // S2H box: whole 16-byte s2d pixels
    if (HALO & 5) prm.num_tiles = (int)(ceil_div(prm.m_tiles, CG) * prm.n_tiles);
    prm.splits = HALO ? 1 : p->cands[p->sel].split;
    prm.num_units = prm.num_tiles * prm.splits;
    prm.ws = p->ws;
    prm.cnt = p->cnt;
    if (prm.splits > 1) {
        const size_t need = (size_t)prm.num_tiles * CG * 128 * BN * sizeof(int32_t);
        const size_t regions = (size_t)prm.num_tiles * CG * 4 * Cfg::EPI_PER_BUF;
        if (!p->ws || p->ws_bytes < need || p->cnt_bytes < regions * sizeof(unsigned))
            return set_err(CONV_Q_EINVAL, "split-K workspace not allocated (conv_q_plan_set_config / _tune allocate it)");
    }
    prm.fd_ntiles = make_fastdiv(prm.n_tiles);
    prm.fd_PQ = make_fastdiv(p->P * p->Q);
    prm.fd_Q = make_fastdiv(p->Q);
    prm.fd_cblk = make_fastdiv(prm.num_cblk);
    prm.fd_S = make_fastdiv(p->S);
    prm.fd_tpi = make_fastdiv(prm.tiles_per_img);
    prm.fd_splits = make_fastdiv(prm.splits);
    prm.fd_Wp = make_fastdiv(prm.Wp);
    prm.relu = p->relu;
    prm.rotate = p->rotate;
    prm.a_gemm = p->R == 1 && p->S == 1 && p->stride == 1 && p->pad == 0 && !(HALO & 1);
    prm.probe = p->probe;
    prm.epi_wait = p->epi_wait;
    prm.out_policy = p->out_policy;
    prm.epi_wait_ns = p->epi_wait_ns;
    prm.trace = p->trace;
    prm.tl = p->tl;
    prm.scale = scale;
    prm.skip = static_cast<const uint8_t *>(p->skip);
    prm.res_scale = p->res_scale;
    prm.dep_in = p->dep_in;
    prm.dep_skip = p->skip ? p->dep_skip : nullptr;
    prm.dep_out = p->dep_out;
    prm.dep_in_total = (unsigned)((int64_t)p->N * p->H * p->W * p->C);       // codes of x
    prm.dep_skip_total = (unsigned)((int64_t)p->N * p->P * p->Q * p->K);     // codes of the skip (= y's shape)
    prm.halo_rows = halo_rows;
    prm.x_uns = p->x_uns;
    prm.y_uns = p->y_uns;
    prm.code_hi = p->y_uns ? (1 << BITS) - 1 : (1 << (BITS - 1)) - 1;
    prm.skip_xor = p->skip_uns ? 0u : (BITS == 8 ? 0x80808080u : 0x88888888u);
    prm.skip_off = 8388608.f + (p->skip_uns ? 0.f : (BITS == 8 ? 128.f : 8.f));
    prm.y32 = static_cast<int32_t *>(y);
    prm.y8 = static_cast<uint8_t *>(y);
    prm.out_row = p->out_row;
    const int full = std::min(prm.num_units, g_num_sms / CG);  // persistent: one CTA (pair) per SM (pair)
    int clusters = p->grid_pct < 100 ? std::max(1, full * p->grid_pct / 100) : full;   // searched grid knob
    if (HALO & 2) {   // weight-stationary: every CTA keeps one N block -> a multiple of the N-tile count
        clusters = clusters / prm.n_tiles * prm.n_tiles;
        if (clusters < prm.n_tiles && full >= prm.n_tiles) clusters = prm.n_tiles;   // (a reduced grid: >= one per N block)
        if (clusters < 1) return set_err(CONV_Q_EUNSUPPORTED, "weight-stationary config needs n_tiles <= SMs");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * CG);
    cfg.blockDim = dim3(Cfg::NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM_LAUNCH;
    cfg.stream = p->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (griddepcontrol in the kernel)
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p->tm_a, p->tm_b, p->tm_y, p->tm_s, prm));
    return CONV_Q_OK;
}

template <int BITS, int OUT>
inline int dispatch_bn_kch(conv_q_plan_s *p, const float *scale, void *y) {
    const Cand c = p->cands[p->sel];
    if (c.ws) {
        {
#define CONVQ_WCASE(BN_, KC_, NS_, H_, CG_)                                                        \
            if (c.bn == BN_ && c.kch == KC_ && c.nsub == NS_ && c.halo == H_ && c.cg == CG_) {     \
                if constexpr (ConvCfg<BITS, BN_, KC_, OUT, CG_, NS_, 2 + H_>::FITS)                \
                    return launch_conv<BITS, BN_, KC_, OUT, CG_, NS_, 2 + H_>(p, scale, y);        \
                else                                                                               \
                    return set_err(CONV_Q_EUNSUPPORTED, "weight-stationary config unavailable for this output mode"); \
            }
            CONVQ_WS_LIST(CONVQ_WCASE)
#undef CONVQ_WCASE
        }
        return set_err(CONV_Q_EUNSUPPORTED, "no weight-stationary kernel for bn=%d kch=%d nsub=%d", c.bn, c.kch, c.nsub);
    }
    if (c.halo) {
#define CONVQ_HCASE(BN_, KC_, CG_, NS_)                                                            \
        if (c.bn == BN_ && c.kch == KC_ && c.cg == CG_ && c.nsub == NS_) {                         \
            if constexpr (ConvCfg<BITS, BN_, KC_, OUT, CG_, NS_, 1>::FITS)                         \
                return launch_conv<BITS, BN_, KC_, OUT, CG_, NS_, 1>(p, scale, y);                 \
            else                                                                                   \
                return set_err(CONV_Q_EUNSUPPORTED, "halo config unavailable for this output mode");  \
        }
#define CONVQ_HCASE_NS(BN_, KC_, CG_) CONVQ_HCASE(BN_, KC_, CG_, 3) CONVQ_HCASE(BN_, KC_, CG_, 1)
        CONVQ_HCASE_NS(64, 128, 1) CONVQ_HCASE_NS(128, 128, 1) CONVQ_HCASE_NS(256, 128, 1)
        CONVQ_HCASE_NS(64, 64, 1) CONVQ_HCASE_NS(128, 64, 1) CONVQ_HCASE_NS(256, 64, 1)
        CONVQ_HCASE_NS(64, 128, 2) CONVQ_HCASE_NS(128, 128, 2) CONVQ_HCASE_NS(256, 128, 2)
        CONVQ_HCASE_NS(64, 64, 2) CONVQ_HCASE_NS(128, 64, 2) CONVQ_HCASE_NS(256, 64, 2)
#undef CONVQ_HCASE_NS
#undef CONVQ_HCASE
        return set_err(CONV_Q_EUNSUPPORTED, "no halo kernel for bn=%d kch=%d cg=%d", c.bn, c.kch, c.cg);
    }
#define CONVQ_CASE(BN_, KC_, NS_, CG_)                                            \
    if (c.bn == BN_ && c.kch == KC_ && c.nsub == NS_ && c.cg == CG_) {          \
        if constexpr (ConvCfg<BITS, BN_, KC_, OUT, CG_, NS_>::FITS)             \
            return launch_conv<BITS, BN_, KC_, OUT, CG_, NS_>(p, scale, y);     \
        else                                                                    \
            return set_err(CONV_Q_EUNSUPPORTED, "tile config exceeds shared memory"); \
    }
#define CONVQ_CASES_BN(KC_, NS_, CG_) \
    CONVQ_CASE(64, KC_, NS_, CG_) CONVQ_CASE(128, KC_, NS_, CG_) CONVQ_CASE(256, KC_, NS_, CG_)
    CONVQ_CASES_BN(128, 2, 1) CONVQ_CASES_BN(128, 1, 1) CONVQ_CASES_BN(64, 4, 1) CONVQ_CASES_BN(64, 1, 1)
    CONVQ_CASES_BN(32, 4, 1) CONVQ_CASES_BN(32, 1, 1)
    CONVQ_CASES_BN(128, 2, 2) CONVQ_CASES_BN(128, 1, 2) CONVQ_CASES_BN(64, 4, 2) CONVQ_CASES_BN(64, 1, 2)
    CONVQ_CASES_BN(32, 4, 2) CONVQ_CASES_BN(32, 1, 2)
#undef CONVQ_CASES_BN
#undef CONVQ_CASE
    return set_err(CONV_Q_EUNSUPPORTED, "no kernel instantiation for bn=%d kch=%d nsub=%d cg=%d", c.bn, c.kch,
                   c.nsub, c.cg);
}


// one explicit instantiation per translation unit (kern_b<BITS>_o<OUT>.cu)
int dispatch_conv_8_0(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_8_1(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_8_2(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_8_4(conv_q_plan_s *p, const float *scale, void *y);   // OUT_TMA | OUT_RELU
int dispatch_conv_8_6(conv_q_plan_s *p, const float *scale, void *y);   // OUT_DIRECT | OUT_RELU
int dispatch_conv_4_0(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_4_1(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_4_2(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_8_8(conv_q_plan_s *p, const float *scale, void *y);    // OUT_TMA | OUT_RES
int dispatch_conv_8_10(conv_q_plan_s *p, const float *scale, void *y);   // OUT_DIRECT | OUT_RES
int dispatch_conv_8_20(conv_q_plan_s *p, const float *scale, void *y);   // OUT_TMA | OUT_RELU | OUT_U
int dispatch_conv_8_22(conv_q_plan_s *p, const float *scale, void *y);   // OUT_DIRECT | OUT_RELU | OUT_U
int dispatch_conv_4_4(conv_q_plan_s *p, const float *scale, void *y);    // OUT_TMA | OUT_RELU
int dispatch_conv_4_6(conv_q_plan_s *p, const float *scale, void *y);    // OUT_DIRECT | OUT_RELU
int dispatch_conv_4_8(conv_q_plan_s *p, const float *scale, void *y);
int dispatch_conv_4_10(conv_q_plan_s *p, const float *scale, void *y);

}  // namespace convq
