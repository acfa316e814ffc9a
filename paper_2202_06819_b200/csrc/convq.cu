// convq.cu -- libconvq.so: host side of the C ABI declared in include/convq.h.
//
// Responsibilities: validate shapes (incl. the
// accumulator overflow guard of PAPER.md:166 s3.2.1), derive the GEMM view
// (PAPER.md:56 s2.1), enumerate TileConfig candidates, pick one by timing on
// the device ("the best scheduling of MMA instructions varies for
// different convolution sizes"), encode the TMA tensor maps (im2col for the
// activations, tiled for weights and output) and launch the kernels.
// No CPU fallback: without a CUDA device every compute call returns
// CONV_Q_ECUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/convq.h"
#include "pack.cuh"
#include "peak.cuh"
#include "plan.cuh"

using namespace convq;

// ============================================================== errors
static thread_local std::string g_err;
static thread_local int g_status = CONV_Q_OK;

namespace convq {
int g_num_sms = 0;
int set_err(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    g_status = code;
    return code;
}
}  // namespace convq

extern "C" const char *conv_q_last_error(void) { return g_err.c_str(); }
extern "C" int conv_q_last_status(void) { return g_status; }
extern "C" int conv_q_version(void) { return 106; }

// ============================================================== driver entry points
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                      const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                       const cuuint64_t *, const int *, const int *, cuuint32_t, cuuint32_t,
                                       const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled_t g_encode_tiled = nullptr;
static PFN_encodeIm2col_t g_encode_im2col = nullptr;
static std::once_flag g_init_once;
static int g_init_status = CONV_Q_OK;
static std::string g_init_msg;

static void init_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) {
        g_init_status = CONV_Q_ECUDA;
        g_init_msg = std::string("no usable CUDA device: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) {
        g_init_status = CONV_Q_ECUDA;
        g_init_msg = "libconvq.so is built for sm_100a (B200); device is sm_" + std::to_string(major * 10 + minor);
        return;
    }
    cudaDriverEntryPointQueryResult q1, q2;
    void *f1 = nullptr, *f2 = nullptr;
    e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1);
    if (e == cudaSuccess) e = cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q2);
    if (e != cudaSuccess || !f1 || !f2) {
        g_init_status = CONV_Q_ECUDA;
        g_init_msg = "cuTensorMapEncode* driver entry points unavailable";
        return;
    }
    g_encode_tiled = reinterpret_cast<PFN_encodeTiled_t>(f1);
    g_encode_im2col = reinterpret_cast<PFN_encodeIm2col_t>(f2);
}
static int ensure_ws(conv_q_plan_s *p);
static bool aligned16(const void *ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }
static int ensure_device() {
    std::call_once(g_init_once, init_device);
    if (g_init_status != CONV_Q_OK) return set_err(g_init_status, "%s", g_init_msg.c_str());
    return CONV_Q_OK;
}

static CUtensorMapSwizzle swizzle_for(int span) {
    return span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : span == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
         : span == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                       : CU_TENSOR_MAP_SWIZZLE_NONE;
}

// ============================================================== plan
static std::string cand_name(const conv_q_plan_s *p, int i) {
    char b[64];
    char k[16] = "";
    if (p->cands[i].split > 1) snprintf(k, sizeof k, "_k%d", p->cands[i].split);
    snprintf(b, sizeof b, "bm%d_bn%d_kc%dx%d_c%d%s%s%s", 128 * p->cands[i].cg, p->cands[i].bn, p->cands[i].kch,
             p->cands[i].nsub, p->cands[i].cg, p->cands[i].direct ? "_st" : "", (p->cands[i].halo & 5) ? "_h" : "", k);
    if (p->cands[i].ws) return std::string(b) + "_w" + ((p->cands[i].halo & 8) ? "_m2" : "");
    return b;
}

// runtime-knob suffix of a searched selection ("" = the defaults)
static std::string runtime_suffix(const conv_q_plan_s *p) {
    if (p->epi_wait == 0 && p->out_policy == 1 && p->rotate == 0 && p->grid_pct == 100) return "";
    char b[48];
    snprintf(b, sizeof b, "+e%dp%dr%dg%d", p->epi_wait, p->out_policy, p->rotate, p->grid_pct);
    return b;
}

static std::string shape_key(const conv_q_plan_s *p) {
    char b[160];
    snprintf(b, sizeof b, "N%d_H%d_W%d_C%d_K%d_R%d_S%d_st%d_p%d_b%d_sm%d_m%d_r%d%s%s", p->N, p->H, p->W, p->C, p->K,
             p->R, p->S, p->stride, p->pad, p->bits, g_num_sms, p->out_mode, p->relu, p->skip ? "_res" : "",
             (p->x_uns || p->y_uns || (p->skip && p->skip_uns))
                 ? (std::string("_u") + char('0' + p->x_uns) + char('0' + p->y_uns) + char('0' + p->skip_uns)).c_str()
                 : "");
    return p->s2d ? std::string(b) + "_s2d" : std::string(b);
}

// in-process tuning cache, optionally mirrored to $CONV_Q_CACHE (one JSON object)
static std::mutex g_cache_mu;
static std::map<std::string, std::pair<std::string, float>> g_cache;
static bool g_cache_loaded = false;

static void cache_load_locked() {
    if (g_cache_loaded) return;
    g_cache_loaded = true;
    const char *path = getenv("CONV_Q_CACHE");
    if (!path) return;
    FILE *f = fopen(path, "r");
    if (!f) return;
    char line[512];
    while (fgets(line, sizeof line, f)) {
        char key[200], cfg[64];
        float us;
        if (sscanf(line, " \"%199[^\"]\": {\"config\": \"%63[^\"]\", \"us\": %f", key, cfg, &us) == 3)
            g_cache[key] = {cfg, us};
    }
    fclose(f);
}
static void cache_store_locked() {
    const char *path = getenv("CONV_Q_CACHE");
    if (!path) return;
    std::string tmp = std::string(path) + ".tmp";
    FILE *f = fopen(tmp.c_str(), "w");
    if (!f) return;
    fprintf(f, "{\n");
    size_t i = 0;
    for (auto &kv : g_cache)
        fprintf(f, "  \"%s\": {\"config\": \"%s\", \"us\": %.3f}%s\n", kv.first.c_str(), kv.second.first.c_str(),
                kv.second.second, ++i < g_cache.size() ? "," : "");
    fprintf(f, "}\n");
    fclose(f);
    rename(tmp.c_str(), path);
}


static void enumerate_candidates(conv_q_plan_s *p) {
    p->cands.clear();
    // (channels per k-block, k-blocks per stage): >= 256 channel-bytes of K per
    // stage where possible (8 MMAs per commit), plus the single-block variant
    static const int kn[][2] = {{128, 2}, {128, 1}, {64, 4}, {64, 1}, {32, 4}, {32, 1}};
    for (int direct : {0, 1})
        for (int cg : {1, 2})
            for (auto &q : kn) {
                const int kch = q[0], nsub = q[1];
                // (C = 16 mod 32, s8: a ragged last k-block per tap, kch < C so the box never
                // exceeds the channel dimension; im2col / tiled only -- no halo / WS candidates)
                const bool ragged = p->C % 32 != 0;
                if (ragged ? kch >= p->C : p->C % kch) continue;
                if (!ragged && kch < 128 && p->C % (2 * kch) == 0) continue;   // a wider k-block exists
                for (int bn : {64, 128, 256}) {
                    if (bn > 64 && bn / 2 >= p->K) continue;  // a narrower tile already covers K
                    const Cand cand{bn, kch, cg, nsub, direct};
                    if (!(p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand))) continue;
                    p->cands.push_back(cand);
                    // split-K variants (K among the tiled loops), each unit >= 2
                    // stages of K: when the tiles fill fewer than two waves, ~1 and ~2 work
                    // units per SM; up to six waves, the (at most two) splits that cut the
                    // wave-quantisation loss of the last partial wave the most
                    const int64_t tiles = ceil_div(p->M, 128 * cg) * ceil_div(p->K, bn);
                    const int64_t num_kb = (int64_t)p->R * p->S * ceil_div(p->C, kch);
                    const int sms = g_num_sms > 0 ? g_num_sms : 148;
                    const int64_t slots = sms / cg;
                    const int64_t ws = tiles * cg * 128 * bn * 4;
                    if (tiles >= 6 * slots || ws > ((int64_t)64 << 20) || 16 * num_kb >= ((int64_t)1 << 31)) continue;
                    const int max_sp = (int)std::min<int64_t>(16, num_kb / (2 * nsub));
                    if (tiles < 2 * slots) {
                        int last = 1;
                        for (int waves : {1, 2}) {
                            int sp = (int)std::min<int64_t>(ceil_div((int64_t)waves * slots, tiles), max_sp);
                            if (sp <= last) continue;
                            Cand sc = cand;
                            sc.split = sp;
                            p->cands.push_back(sc);
                            last = sp;
                        }
                    } else {
                        auto eff = [&](int64_t units) {   // busy fraction of the last (partial) wave's slots
                            const double w = (double)units / (double)slots;
                            return w / std::ceil(w);
                        };
                        const double e1 = eff(tiles);
                        std::vector<std::pair<double, int>> opts;
                        for (int sp : {2, 3, 4, 6, 8})
                            if (sp <= max_sp && tiles * sp <= 12 * slots && eff(tiles * sp) > e1 + 0.12)
                                opts.push_back({-eff(tiles * sp) + 0.01 * sp, sp});
                        std::sort(opts.begin(), opts.end());
                        for (size_t i = 0; i < opts.size() && i < 2; ++i) {
                            Cand sc = cand;
                            sc.split = opts[i].second;
                            p->cands.push_back(sc);
                        }
                    }
                }
            }
    // duplicate-aware (halo) candidates: stride-1 INT8 R x S convolutions whose
    // halo box (rows covering 128 MMA rows + the largest tap shift) fits 32 KB
    const int Wp = p->W + 2 * p->pad;
    // (any R x S up to 7 x 7: tap (r, s) reads the box at row offset r*Wp + s)
    // (not for the s2d stem plans: their stored tensor has its own window geometry, handled by
    // enumerate_s2d_halo; a regular halo box over it would not match the kernel's byte count)
    const bool halo_ok = !p->s2d && p->stride == 1 && p->R * p->S > 1 && p->R <= 7 && p->S <= 7 && Wp <= BM;
    // (INT4: the packed box is expanded once per (tile, channel block) by the transform warps)
    if (halo_ok && p->C % 64 == 0) {
        const int kch = p->C % 128 == 0 ? 128 : 64;
        const int halo_rows = (int)ceil_div(BM + (p->R - 1) * Wp + p->S - 1, Wp);
        if ((int64_t)halo_rows * Wp * kch <= 32768 && halo_rows <= 256)
            for (int nsub : {3, 1})
                for (int cg : {1, 2})
                    for (int bn : {64, 128, 256}) {
                        if (bn > 64 && bn / 2 >= p->K) continue;
                        Cand cand{bn, kch, cg, nsub, 1};
                        cand.halo = 1;
                        if (p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand)) p->cands.push_back(cand);
                    }
    }
    // weight-stationary candidates: the CTA's whole (BN/CG) x R*S*C weight block
    // stays resident in 64 KB of shared memory (as s8; INT4: loaded packed and
    // expanded once by the transform warps), stages carry only activations
    // (halo boxes for stride-1 3x3 -- INT8 only --, im2col / tiled rows otherwise)
    {
        const int kch = p->C % 128 == 0 ? 128 : p->C % 64 == 0 ? 64 : 0;
        const int sms = g_num_sms > 0 ? g_num_sms : 148;
        if (kch)
            for (int cg : {1, 2})
                for (int direct : {0, 1})
                    for (int bn : {64, 128, 256}) {
                        if (bn > 64 && bn / 2 >= p->K) continue;
                        if ((int64_t)(bn / cg) * p->R * p->S * p->C > 65536 || ceil_div(p->K, bn) > sms / cg) continue;
                        for (int nsub : {1, 2}) {
                            Cand cand{bn, kch, cg, nsub, direct};
                            cand.ws = 1;
                            if (p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand)) p->cands.push_back(cand);
                        }
                        if (cg == 1 && bn <= 128) {   // MT2: two 128-row m-groups per unit
                            Cand cand{bn, kch, 1, 1, direct};
                            cand.ws = 1;
                            cand.halo = 8;
                            if (p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand)) p->cands.push_back(cand);
                        }
                        if (halo_ok && direct) {   // (INT4: packed box per stage, expanded once per stage)
                            const int halo_rows = (int)ceil_div(BM + (p->R - 1) * Wp + p->S - 1, Wp);
                            if ((int64_t)halo_rows * Wp * kch <= (kch == 64 ? 20480 : 32768) && halo_rows <= 256) {
                                Cand cand{bn, kch, cg, 1, direct};
                                cand.ws = 1;
                                cand.halo = 1;
                                if (p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand)) p->cands.push_back(cand);
                            }
                            // MT2 (one CTA, two m-groups per accumulator round trip)
                            const int rows2 = (int)ceil_div(2 * BM + (p->R - 1) * Wp + p->S - 1, Wp);
                            if ((int64_t)rows2 * Wp * kch <= 32768 && rows2 <= 256) {
                                Cand cand{bn, kch, cg, 1, direct};
                                cand.ws = 1;
                                cand.halo = 1 | 8;
                                if (p->bits == 8 ? cand_fits<8>(cand) : cand_fits<4>(cand)) p->cands.push_back(cand);
                            }
                        }
                    }
    }
}

// s2d stem window-halo candidates (cand.halo = 4, weight-stationary, BN = 64):
// one tiled box of (rows covering 128 MMA rows + 3 tap rows) x Wp stored s2d
// pixels per tile; needs the 64-byte window (S2P = 4) and a box <= 20 KB
static void enumerate_s2d_halo(conv_q_plan_s *p) {
    if (!p->s2d || p->bits != 8 || p->row_bytes != 64 || p->xs_W > BM || p->K % 64) return;
    const int Wp = p->xs_W;
    const int halo_rows = (int)ceil_div(BM + (p->R - 1) * Wp + 3, Wp);
    if ((int64_t)halo_rows * Wp * 16 > 20480 || halo_rows > 256) return;
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    for (int cg : {1, 2}) {
        if (ceil_div(p->K, 64) > sms / cg) continue;
        Cand c{64, 64, cg, 1, 1};
        c.ws = 1;
        c.halo = 4;
        if (cand_fits<8>(c)) p->cands.push_back(c);
    }
    // MT2: two 128-row m-groups per accumulator round trip (box <= 32 KB)
    const int rows2 = (int)ceil_div(2 * BM + (p->R - 1) * Wp + 3, Wp);
    if ((int64_t)rows2 * Wp * 16 <= 32768)
        for (int cg : {1, 2}) {
            if (ceil_div(p->K, 64) > sms / cg) continue;
            Cand c{64, 64, cg, 1, 1};
            c.ws = 1;
            c.halo = 4 | 8;
            if (cand_fits<8>(c)) p->cands.push_back(c);
        }
}

static int default_candidate(const conv_q_plan_s *p) {
    const int64_t m_tiles = ceil_div(p->M, BM);
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    int pick = -1, narrow = -1;
    for (size_t i = 0; i < p->cands.size(); ++i) {
        const Cand &c = p->cands[i];
        if (c.kch != p->cands[0].kch || c.nsub != p->cands[0].nsub || c.cg != 1 || c.direct) continue;
        if (narrow < 0 || c.bn < p->cands[narrow].bn) narrow = (int)i;
        if (m_tiles * ceil_div(p->K, c.bn) >= sms && (pick < 0 || c.bn > p->cands[pick].bn)) pick = (int)i;
    }
    return pick >= 0 ? pick : std::max(narrow, 0);
}

// Select the cached tuning result for the plan's shape + epilogue, if any
// (the key includes relu / out_mode, so this runs again on set_epilogue).
static void apply_cache(conv_q_plan_s *p) {
    if (p->user_sel) return;   // an explicit conv_q_plan_set_config / _tune pick is sticky
    std::lock_guard<std::mutex> lk(g_cache_mu);
    cache_load_locked();
    auto it = g_cache.find(shape_key(p));
    if (it == g_cache.end()) return;
    // a searched entry (conv_q_plan_search) carries its runtime knobs after '+'
    std::string name = it->second.first;
    int ew = 0, pol = 1, rot = 0, grid = 100;
    const size_t plus = name.find('+');
    if (plus != std::string::npos) {
        if (sscanf(name.c_str() + plus, "+e%dp%dr%dg%d", &ew, &pol, &rot, &grid) != 4) return;
        name.resize(plus);
    }
    int found = -1;
    for (size_t i = 0; i < p->cands.size() && found < 0; ++i)
        if (cand_name(p, (int)i) == name) found = (int)i;
    // a split-K variant outside the enumerated list (the search's split knob)
    for (size_t i = 0, n = p->cands.size(); i < n && found < 0; ++i) {
        if (p->cands[i].split != 1 || p->cands[i].ws || p->cands[i].halo) continue;
        for (int sp = 2; sp <= 16 && found < 0; ++sp) {
            p->cands.push_back(p->cands[i]);
            p->cands.back().split = sp;
            if (cand_name(p, (int)p->cands.size() - 1) == name) found = (int)p->cands.size() - 1;
            else p->cands.pop_back();
        }
    }
    if (found < 0) return;
    p->sel = found;
    p->tuned_us = it->second.second;
    p->epi_wait = ew;
    p->epi_wait_ns = ew == 1 ? 20000u : ew == 2 ? 64u : 0u;
    p->out_policy = pol;
    p->rotate = rot;
    p->grid_pct = grid;
}

static conv_q_plan_t *finish_plan(conv_q_plan_s *p);

extern "C" conv_q_plan_t *conv_q_plan(int N, int H, int W, int C, int K, int R, int S, int stride, int pad,
                                      int bits) {
    g_err.clear();
    g_status = CONV_Q_OK;
    if (N < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || S < 1) {
        set_err(CONV_Q_EINVAL, "every dimension must be >= 1 (N=%d H=%d W=%d C=%d K=%d R=%d S=%d)", N, H, W, C, K, R,
                S);
        return nullptr;
    }
    if (stride < 1 || stride > 8) {
        set_err(CONV_Q_EINVAL, "stride %d outside [1,8] (TMA traversal stride limit)", stride);
        return nullptr;
    }
    if (pad < 0 || pad > 127) {
        set_err(CONV_Q_EINVAL, "pad %d outside [0,127] (im2col bounding-box corner range)", pad);
        return nullptr;
    }
    if (R - 1 > 255 || S - 1 > 255) {
        set_err(CONV_Q_EINVAL, "filter %dx%d too large (im2col offsets are 8-bit)", R, S);
        return nullptr;
    }
    if (bits != 4 && bits != 8) {
        set_err(CONV_Q_EINVAL, "bits must be 4 or 8, got %d", bits);
        return nullptr;
    }
    if (pad - (R - 1) < -128 || pad - (S - 1) < -128) {
        set_err(CONV_Q_EINVAL, "pad - (R-1) below -128 (im2col bounding-box corner range)");
        return nullptr;
    }
    int64_t P = (int64_t)H + 2 * pad - R, Q = (int64_t)W + 2 * pad - S;
    if (P < 0 || Q < 0) {
        set_err(CONV_Q_EINVAL, "output is empty: H+2pad-R=%lld, W+2pad-S=%lld", (long long)P, (long long)Q);
        return nullptr;
    }
    P = P / stride + 1;
    Q = Q / stride + 1;
    if (((int64_t)C * bits) % 128 || ((int64_t)K * bits) % 128) {
        set_err(CONV_Q_EUNSUPPORTED,
                "C*bits (%lld) and K*bits (%lld) must be multiples of 128 (16-byte pixel rows); pad C with "
                "conv_q_quantize",
                (long long)C * bits, (long long)K * bits);
        return nullptr;
    }
    // s8 with C = 16 (mod 32): the last k-block of a tap is half a 32-byte MMA K
    // step; its TMA box reads past the pixel's channels, which the tensor map
    // zero-fills (activations), so whatever weight bytes sit there add zero
    if (bits == 8 ? (C % 16 || C < 32) : C % 32) {
        set_err(CONV_Q_EUNSUPPORTED, "C=%d: the implicit-GEMM kernel needs C %% 32 == 0 (s4) / C %% 16 == 0 and "
                "C >= 32 (s8)", C);
        return nullptr;
    }
    if ((int64_t)C * bits / 8 > 65535) {
        set_err(CONV_Q_EUNSUPPORTED, "C*bits/8 = %lld bytes per pixel exceeds 65535", (long long)C * bits / 8);
        return nullptr;
    }
    // Accumulator guard (PAPER.md:166 s3.2.1): |acc| <= R*S*C*2^(b-1)*2^(b-1)
    // must fit int32.  INT4 runs on the MMA as 16x-scaled s8 operands, so its
    // MMA accumulator holds 256*acc: bound R*S*C*2^14 there (same as s8).
    const int64_t Kg = (int64_t)R * S * C;
    const int64_t bound = Kg * (int64_t)(1 << 14);
    if (bound > 2147483647LL) {
        set_err(CONV_Q_EOVERFLOW, "R*S*C = %lld: accumulator bound %lld exceeds int32", (long long)Kg,
                (long long)bound);
        return nullptr;
    }
    auto *p = new (std::nothrow) conv_q_plan_s();
    if (!p) {
        set_err(CONV_Q_ENOMEM, "plan allocation failed");
        return nullptr;
    }
    p->N = N; p->H = H; p->W = W; p->C = C; p->K = K; p->R = R; p->S = S;
    p->stride = stride; p->pad = p->pad_hi = pad; p->bits = bits;
    p->P = (int)P; p->Q = (int)Q;
    p->o_H = H; p->o_W = W; p->o_C = C; p->o_R = R; p->o_S = S; p->o_stride = stride; p->o_pad = pad;
    p->xs_W = W;
    return finish_plan(p);
}

// Common tail of plan creation: GEMM sizes, candidates, default / cached pick.
static conv_q_plan_t *finish_plan(conv_q_plan_s *p) {
    p->M = (int64_t)p->N * p->P * p->Q;
    p->Kg = (int64_t)p->R * p->S * p->C;
    if (p->M > 2147483647LL - 256) {
        set_err(CONV_Q_EUNSUPPORTED, "N*P*Q = %lld exceeds the 32-bit GEMM row index", (long long)p->M);
        delete p;
        return nullptr;
    }
    p->row_bytes = p->C * p->bits / 8;
    p->out_row = p->K * p->bits / 8;
    std::call_once(g_init_once, init_device);  // SM count for the default pick; errors surface at run
    enumerate_candidates(p);
    enumerate_s2d_halo(p);
    p->sel = default_candidate(p);
    if (const char *pr = getenv("CONV_Q_PROBE")) p->probe = atoi(pr);
    if (const char *ew = getenv("CONV_Q_EPI_WAIT")) p->epi_wait = atoi(ew);
    if (const char *en = getenv("CONV_Q_EPI_WAIT_NS")) p->epi_wait_ns = (unsigned)atoi(en);
    if (const char *op = getenv("CONV_Q_OUT_POLICY")) p->out_policy = atoi(op);
    if (const char *ro = getenv("CONV_Q_ROTATE")) p->rotate = atoi(ro) ? 1 : 0;
    apply_cache(p);
    if (p->cands[p->sel].split > 1 && ensure_device() == CONV_Q_OK && ensure_ws(p) != CONV_Q_OK) {
        delete p;
        return nullptr;
    }
    return p;
}

static int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Stride-2 stem conv as a stride-1 conv over a space-to-depth(2) view (pack.cuh):
// s2d tap rows jr in [0, R2) at s2d row p - PL + jr; in W the S2P consecutive
// s2d pixels q - PL .. q - PL + S2P - 1 form ONE k-block row of S2P*16 bytes,
// read through an im2col map whose W stride is one s2d pixel (16 B), i.e.
// overlapping windows of the stored tensor (no bytes duplicated in HBM).
extern "C" conv_q_plan_t *conv_q_plan_s2d(int N, int H, int W, int C, int K, int R, int S, int pad, int bits) {
    g_err.clear();
    g_status = CONV_Q_OK;
    if (N < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || S < 1) {
        set_err(CONV_Q_EINVAL, "every dimension must be >= 1");
        return nullptr;
    }
    if (bits != 4 && bits != 8) {
        set_err(CONV_Q_EINVAL, "bits must be 4 or 8, got %d", bits);
        return nullptr;
    }
    if (pad < 0 || pad > 64) {
        set_err(CONV_Q_EINVAL, "pad %d outside [0,64]", pad);
        return nullptr;
    }
    const int CP = bits == 8 ? 4 : 8;
    if (C > CP) {
        set_err(CONV_Q_EUNSUPPORTED, "s2d stem: C=%d > %d channels per 16-byte s2d pixel phase", C, CP);
        return nullptr;
    }
    if (((int64_t)K * bits) % 128) {
        set_err(CONV_Q_EUNSUPPORTED, "K*bits (%lld) must be a multiple of 128", (long long)K * bits);
        return nullptr;
    }
    const int64_t P = floor_div(H + 2 * pad - R, 2) + 1, Q = floor_div(W + 2 * pad - S, 2) + 1;
    if (P < 1 || Q < 1) {
        set_err(CONV_Q_EINVAL, "output is empty (P=%lld, Q=%lld)", (long long)P, (long long)Q);
        return nullptr;
    }
    const int PL = (pad + 1) / 2;                             // -floor(-pad/2)
    const int R2 = floor_div(R - 1 - pad, 2) + PL + 1;
    const int S2 = floor_div(S - 1 - pad, 2) + PL + 1;
    int S2P = 2;
    while (S2P < S2) S2P *= 2;
    if (S2P > 8) {
        set_err(CONV_Q_EUNSUPPORTED, "s2d stem: %d s2d taps in W exceed one 128-byte k-block", S2);
        return nullptr;
    }
    const int H2 = (H + 1) / 2;
    const int pad_hi = (int)P - 1 + R2 - H2 - PL;
    if (R2 > 64 || pad_hi - (R2 - 1) < -128 || pad_hi > 127) {
        set_err(CONV_Q_EUNSUPPORTED, "s2d stem: filter / padding outside the im2col corner range");
        return nullptr;
    }
    const int64_t Kg = (int64_t)R2 * S2P * 16 * 8 / bits;
    if (Kg * (int64_t)(1 << 14) > 2147483647LL) {
        set_err(CONV_Q_EOVERFLOW, "s2d stem: accumulator bound exceeds int32");
        return nullptr;
    }
    auto *p = new (std::nothrow) conv_q_plan_s();
    if (!p) {
        set_err(CONV_Q_ENOMEM, "plan allocation failed");
        return nullptr;
    }
    p->s2d = 1;
    p->N = N; p->H = H2; p->W = (int)Q; p->C = S2P * 16 * 8 / bits; p->K = K; p->R = R2; p->S = 1;
    p->stride = 1; p->pad = PL; p->pad_hi = pad_hi; p->bits = bits;
    p->P = (int)P; p->Q = (int)Q;
    p->xs_W = (int)Q + S2P - 1;
    p->o_H = H; p->o_W = W; p->o_C = C; p->o_R = R; p->o_S = S; p->o_stride = 2; p->o_pad = pad;
    return finish_plan(p);
}

extern "C" void conv_q_plan_destroy(conv_q_plan_t *p) { delete p; }

extern "C" int conv_q_plan_set_stream(conv_q_plan_t *p, void *stream) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    p->stream = static_cast<cudaStream_t>(stream);
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_epilogue(conv_q_plan_t *p, int relu, int out_mode) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if ((relu != 0 && relu != 1) || (out_mode != CONV_Q_OUT_PACKED && out_mode != CONV_Q_OUT_S32))
        return set_err(CONV_Q_EINVAL, "relu must be 0/1 and out_mode PACKED(0)/S32(1)");
    p->relu = relu;
    p->out_mode = out_mode;
    apply_cache(p);
    if (p->cands[p->sel].split > 1 && ensure_device() == CONV_Q_OK) return ensure_ws(p);
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_residual(conv_q_plan_t *p, const void *skip, float res_scale) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if (skip && !aligned16(skip)) return set_err(CONV_Q_EINVAL, "skip must be 16-byte aligned");
    if (skip && p->s2d) return set_err(CONV_Q_EUNSUPPORTED, "no residual add on the s2d stem plan");
    p->skip = skip;
    p->res_scale = skip ? res_scale : 0.f;
    apply_cache(p);
    if (p->cands[p->sel].split > 1 && ensure_device() == CONV_Q_OK) return ensure_ws(p);
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_deps(conv_q_plan_t *p, const unsigned *in_done, const unsigned *skip_done,
                                    unsigned *out_done) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if (p->s2d && in_done) return set_err(CONV_Q_EUNSUPPORTED, "the s2d stem plan reads the s2d quantize output");
    if ((in_done && (reinterpret_cast<uintptr_t>(in_done) & 3)) || (skip_done && (reinterpret_cast<uintptr_t>(skip_done) & 3)) ||
        (out_done && (reinterpret_cast<uintptr_t>(out_done) & 3)))
        return set_err(CONV_Q_EINVAL, "completion counters must be 4-byte aligned");
    if ((int64_t)p->N * p->H * p->W * p->C > 0xFFFFFFFFLL || (int64_t)p->M * p->K > 0xFFFFFFFFLL)
        return set_err(CONV_Q_EUNSUPPORTED, "tensor too large for a 32-bit completion counter");
    p->dep_in = in_done;
    p->dep_skip = skip_done;
    p->dep_out = out_done;
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_formats(conv_q_plan_t *p, int x_unsigned, int y_unsigned, int skip_unsigned) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if ((x_unsigned | y_unsigned | skip_unsigned) & ~1) return set_err(CONV_Q_EINVAL, "formats must be 0/1");
    // accumulator guard for unsigned activations (reading 16): |acc| <= R*S*C*(2^b - 1)*2^(b-1);
    // INT4's MMA accumulator holds 256*acc -> bound R*S*C*255*128 for both widths
    if (x_unsigned && p->Kg * (int64_t)(255 * 128) > 2147483647LL)
        return set_err(CONV_Q_EOVERFLOW, "R*S*C = %lld: unsigned-activation accumulator bound exceeds int32",
                       (long long)p->Kg);
    p->x_uns = x_unsigned;
    p->y_uns = y_unsigned;
    p->skip_uns = skip_unsigned;
    apply_cache(p);
    if (p->cands[p->sel].split > 1 && ensure_device() == CONV_Q_OK) return ensure_ws(p);
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_num_candidates(const conv_q_plan_t *p) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    return (int)p->cands.size();
}

extern "C" int conv_q_plan_candidate_name(const conv_q_plan_t *p, int i, char *buf, int len) {
    if (!p || !buf || len < 1) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (i < 0 || i >= (int)p->cands.size()) return set_err(CONV_Q_EINVAL, "candidate %d out of range", i);
    snprintf(buf, len, "%s", cand_name(p, i).c_str());
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_config(conv_q_plan_t *p, int i) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if (i < 0 || i >= (int)p->cands.size()) return set_err(CONV_Q_EINVAL, "candidate %d out of range", i);
    p->sel = i;
    p->user_sel = 1;
    p->tuned_us = -1.f;
    // allocate a split-K workspace now: conv_q_run never allocates
    if (p->cands[i].split > 1 && ensure_device() == CONV_Q_OK) return ensure_ws(p);
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_info(const conv_q_plan_t *p, conv_q_info_t *info) {
    if (!p || !info) return set_err(CONV_Q_EINVAL, "NULL argument");
    memset(info, 0, sizeof *info);
    info->N = p->N; info->H = p->o_H; info->W = p->o_W; info->C = p->o_C; info->K = p->K;
    info->R = p->o_R; info->S = p->o_S; info->stride = p->o_stride; info->pad = p->o_pad; info->bits = p->bits;
    info->P = p->P; info->Q = p->Q; info->M = p->M; info->Kg = p->Kg;
    info->s2d = p->s2d;
    info->x_dims[0] = p->N; info->x_dims[1] = p->H; info->x_dims[2] = p->xs_W;
    info->x_dims[3] = p->s2d ? 16 : p->row_bytes;
    info->w_dims[0] = p->K; info->w_dims[1] = p->R; info->w_dims[2] = p->S; info->w_dims[3] = p->row_bytes;
    info->x_bytes = (int64_t)info->x_dims[0] * info->x_dims[1] * info->x_dims[2] * info->x_dims[3];
    info->w_bytes = (int64_t)p->K * p->R * p->S * p->row_bytes;
    info->y_bytes = p->M * p->out_row;
    info->y_s32_bytes = p->M * p->K * 4;
    info->relu = p->relu;
    info->out_mode = p->out_mode;
    info->num_candidates = (int)p->cands.size();
    info->config_index = p->sel;
    snprintf(info->config, sizeof info->config, "%s", p->cands.empty() ? "" : (cand_name(p, p->sel) + runtime_suffix(p)).c_str());
    info->tuned_us = p->tuned_us;
    info->macs = p->M * p->K * p->Kg;
    return CONV_Q_OK;
}

static int encode_maps(conv_q_plan_s *p, const void *x, const void *w, void *y) {
    const Cand c = p->cands[p->sel];
    const int load_row = c.kch * p->bits / 8;
    const CUtensorMapSwizzle sw_ld = swizzle_for(load_row);
    // A (halo mode): tiled 4-D box {KCH bytes, Wp, halo rows, 1} of the
    // padded input starting at (w, h) = (-pad, p0-pad): the duplicate-free
    // "genuine" data of PAPER.md section 3.1; OOB (padding) is zero-filled.
    const int mt = (c.halo & 8) ? 2 : 1;   // MT2: the box covers two 128-row m-groups
    if (c.halo & 4) {
        // A (s2d window halo): the box is halo_rows WHOLE stored rows of the s2d
        // tensor [N][H2][Wp][16 B] at (0, 0, p0 - PL, n) -- every column is in
        // bounds by construction (zero borders are stored), rows outside [0, H2)
        // are zero-filled.  A stored row is Wp*16 contiguous bytes, so the map
        // views it as ONE inner row of 2*Wp 8-byte elements ({2 Wp, 1, H2, N}):
        // the TMA moves halo_rows long rows instead of halo_rows*Wp 16-byte rows
        // (same bytes, same smem image; 2 Wp <= 256 as Wp <= BM)
        const int Wp = p->xs_W;
        const int halo_rows = (int)ceil_div(mt * BM + (p->R - 1) * Wp + 3, Wp);
        cuuint64_t dims[4] = {(cuuint64_t)2 * Wp, 1, (cuuint64_t)p->H, (cuuint64_t)p->N};
        cuuint64_t strides[3] = {(cuuint64_t)16 * Wp, (cuuint64_t)16 * Wp, (cuuint64_t)16 * Wp * p->H};
        cuuint32_t box[4] = {(cuuint32_t)(2 * Wp), 1, (cuuint32_t)halo_rows, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = g_encode_tiled(&p->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void *>(x), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(x s2d halo) failed: %d", (int)r);
    } else if (c.halo & 1) {
        const int Wp = p->W + 2 * p->pad;
        const int halo_rows = (int)ceil_div(mt * BM + (p->R - 1) * Wp + p->S - 1, Wp);
        cuuint64_t dims[4] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->W, (cuuint64_t)p->H, (cuuint64_t)p->N};
        cuuint64_t strides[3] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->row_bytes * p->W,
                                 (cuuint64_t)p->row_bytes * p->W * p->H};
        cuuint32_t box[4] = {(cuuint32_t)load_row, (cuuint32_t)Wp, (cuuint32_t)halo_rows, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = g_encode_tiled(&p->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(x), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw_ld,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(x halo) failed: %d", (int)r);
    } else if (p->s2d) {
        // A (s2d stem): {window bytes, Q windows, H2, N}; window q starts at stored
        // column q and spans S2P s2d pixels, so the W stride is ONE s2d pixel
        // (16 B) while a "pixel" is row_bytes wide: overlapping windows.  H
        // walks the R2 tap rows with corners (-PL, pad_hi - (R2-1)); out-of-
        // image rows are zero-filled; columns are zero in the stored borders.
        cuuint64_t dims[4] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->Q, (cuuint64_t)p->H, (cuuint64_t)p->N};
        cuuint64_t strides[3] = {16, (cuuint64_t)16 * p->xs_W, (cuuint64_t)16 * p->xs_W * p->H};
        int lower[2] = {0, -p->pad};
        int upper[2] = {0, p->pad_hi - (p->R - 1)};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = g_encode_im2col(&p->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(x), dims, strides,
                                     lower, upper, (cuuint32_t)load_row, (cuuint32_t)BM, estr,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw_ld, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeIm2col(x s2d windows) failed: %d", (int)r);
    } else if (p->R == 1 && p->S == 1 && p->stride == 1 && p->pad == 0) {
        // A (1x1, stride 1, no padding): the im2col matrix IS the input viewed
        // as [N*H*W][C bytes]; a plain tiled 2-D load of BM rows
        cuuint64_t dims[2] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->M};
        cuuint64_t strides[1] = {(cuuint64_t)p->row_bytes};
        cuuint32_t box[2] = {(cuuint32_t)load_row, (cuuint32_t)BM};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = g_encode_tiled(&p->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(x), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw_ld,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(x 1x1) failed: %d", (int)r);
    } else
    // A: packed NHWC activations, im2col mode ("im2col layout"),
    // {C bytes, W, H, N}; the bounding box walks output pixels with the conv
    // stride; the corners make out-of-image taps read as zero (padding).
    {
        cuuint64_t dims[4] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->W, (cuuint64_t)p->H, (cuuint64_t)p->N};
        cuuint64_t strides[3] = {(cuuint64_t)p->row_bytes, (cuuint64_t)p->row_bytes * p->W,
                                 (cuuint64_t)p->row_bytes * p->W * p->H};
        int lower[2] = {-p->pad, -p->pad};                          // {W, H}
        int upper[2] = {p->pad - (p->S - 1), p->pad - (p->R - 1)};  // {W, H}
        cuuint32_t estr[4] = {1, (cuuint32_t)p->stride, (cuuint32_t)p->stride, 1};
        CUresult r = g_encode_im2col(&p->tm_a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(x), dims, strides,
                                     lower, upper, (cuuint32_t)load_row, (cuuint32_t)BM, estr,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw_ld, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeIm2col(x) failed: %d", (int)r);
    }
    // B: packed KRSC weights as a 2-D [K][R*S*C bytes] matrix, tiled.
    {
        cuuint64_t dims[2] = {(cuuint64_t)p->R * p->S * p->row_bytes, (cuuint64_t)p->K};
        cuuint64_t strides[1] = {(cuuint64_t)p->R * p->S * p->row_bytes};
        cuuint32_t box[2] = {(cuuint32_t)load_row, (cuuint32_t)(c.bn / c.cg)};  // this CTA's share of the N tile
        cuuint32_t estr[2] = {1, 1};
        CUresult r = g_encode_tiled(&p->tm_b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(w), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw_ld,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(w) failed: %d", (int)r);
    }
    // Y: packed NHWC output as a 2-D [M][K*bits/8 bytes] matrix (== the next
    // layer's x; PAPER.md:261 layout consistency).  Unused in S32 mode.
    if (p->out_mode == CONV_Q_OUT_PACKED && !c.direct) {
        // one box = one epilogue warp's 32-row slab (or a 128-byte column block of it)
        const int num_epi = epi_warpgroups(p->bits);
        const int nbuf = tmem_buffers(p->bits, ((c.halo & 8) ? 2 : 1) * c.bn);   // the kernel's rule (MT2: 2*BN TMEM columns per buffer)
        const int epb = epi_per_buf(p->bits, nbuf);   // the kernel's rule (all-warps epilogue for 2 buffers)
        (void)num_epi;
        const int epi_row = c.bn / epb * p->bits / 8;
        const int subw = epi_row < 128 ? epi_row : 128;
        cuuint64_t dims[2] = {(cuuint64_t)p->out_row, (cuuint64_t)p->M};
        cuuint64_t strides[1] = {(cuuint64_t)p->out_row};
        cuuint32_t box[2] = {(cuuint32_t)subw, 32u};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = g_encode_tiled(&p->tm_y, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, y, dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(subw), CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(y) failed: %d", (int)r);
        // the residual skip tensor has y's layout: the same box and swizzle, so the
        // epilogue can TMA-load a warp's skip slab into its output staging slab
        memset(&p->tm_s, 0, sizeof p->tm_s);
        if (p->skip) {
            r = g_encode_tiled(&p->tm_s, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(p->skip), dims, strides,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_for(subw),
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return set_err(CONV_Q_ECUDA, "cuTensorMapEncodeTiled(skip) failed: %d", (int)r);
        }
    } else {
        memset(&p->tm_y, 0, sizeof p->tm_y);
        memset(&p->tm_s, 0, sizeof p->tm_s);
    }
    p->c_x = x; p->c_w = w; p->c_y = y; p->c_sel = p->sel; p->c_mode = p->out_mode; p->c_skip = p->skip;
    return CONV_Q_OK;
}


// Split-K workspace for the selected config: partial sums + region counters,
// zeroed once here and left zero by every run (the kernel's last arriving warp
// clears what it consumed).  Grows only; never allocated during graph capture.
static int ensure_ws(conv_q_plan_s *p) {
    const Cand &c = p->cands[p->sel];
    if (c.split <= 1) return CONV_Q_OK;
    const int64_t tiles = ceil_div(p->M, 128 * c.cg) * ceil_div(p->K, c.bn);
    const size_t need = (size_t)tiles * c.cg * 128 * c.bn * sizeof(int32_t);
    const size_t cnt_need = (size_t)tiles * c.cg * 16 * sizeof(unsigned);   // <= 4 warps x 4 column parts
    if (p->ws && p->ws_bytes >= need && p->cnt_bytes >= cnt_need) return CONV_Q_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(p->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
        return set_err(CONV_Q_EINVAL, "split-K workspace must be allocated before graph capture (run or select the config once first)");
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    if (p->ws) cudaFree(p->ws);
    if (p->cnt) cudaFree(p->cnt);
    p->ws = nullptr;
    p->cnt = nullptr;
    p->ws_bytes = p->cnt_bytes = 0;
    CUDA_TRY(cudaMalloc(&p->ws, need));
    CUDA_TRY(cudaMalloc(&p->cnt, cnt_need));
    CUDA_TRY(cudaMemset(p->ws, 0, need));
    CUDA_TRY(cudaMemset(p->cnt, 0, cnt_need));
    CUDA_TRY(cudaDeviceSynchronize());
    p->ws_bytes = need;
    p->cnt_bytes = cnt_need;
    return CONV_Q_OK;
}

extern "C" int conv_q_run(conv_q_plan_t *p, const void *x, const void *w, const float *scale, void *y) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if (!x || !w || !scale || !y) return set_err(CONV_Q_EINVAL, "NULL tensor pointer");
    if (!aligned16(x) || !aligned16(w) || !aligned16(scale) || !aligned16(y))
        return set_err(CONV_Q_EINVAL, "tensor pointers must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    if (p->cands[p->sel].split > 1 && !p->ws)   // allocated by plan creation / set_config / set_epilogue / tune
        return set_err(CONV_Q_EINVAL, "split-K workspace missing (select the config with conv_q_plan_set_config)");
    if (p->c_x != x || p->c_w != w || p->c_y != y || p->c_sel != p->sel || p->c_mode != p->out_mode ||
        p->c_skip != p->skip) {
        rc = encode_maps(p, x, w, y);
        if (rc) return rc;
    }
    const bool s32 = p->out_mode == CONV_Q_OUT_S32;
    const bool direct = p->cands[p->sel].direct != 0;
    if (p->skip) {   // fused residual add (reading 15): packed output only, runtime ReLU
        if (s32) return set_err(CONV_Q_EINVAL, "the residual add needs the packed output mode");
        if (p->bits == 8) return direct ? dispatch_conv_8_10(p, scale, y) : dispatch_conv_8_8(p, scale, y);
        return direct ? dispatch_conv_4_10(p, scale, y) : dispatch_conv_4_8(p, scale, y);
    }
    // ReLU epilogues (unsigned output codes clamp at 0: the ReLU, reading 16)
    const bool relu = p->relu || p->y_uns;
    if (p->bits == 8) {
        if (s32) return dispatch_conv_8_1(p, scale, y);
        if (relu && p->y_uns) return direct ? dispatch_conv_8_22(p, scale, y) : dispatch_conv_8_20(p, scale, y);
        if (relu) return direct ? dispatch_conv_8_6(p, scale, y) : dispatch_conv_8_4(p, scale, y);
        return direct ? dispatch_conv_8_2(p, scale, y) : dispatch_conv_8_0(p, scale, y);
    }
    if (s32) return dispatch_conv_4_1(p, scale, y);
    if (relu) return direct ? dispatch_conv_4_6(p, scale, y) : dispatch_conv_4_4(p, scale, y);
    return direct ? dispatch_conv_4_2(p, scale, y) : dispatch_conv_4_0(p, scale, y);
}

// Time every candidate (a7): `warmup` untimed runs, then 3 rounds of `reps`
// back-to-back launches (PDL overlaps each launch's prologue with the previous
// kernel, as in a layer sequence), score = the median round's mean.  us[i]
// receives candidate i's score (or -1 if it failed to run).  Restores the
// previous selection.  Returns the index of the fastest candidate.
// The `reps` back-to-back launches of a round are captured into a CUDA graph
// and the graph is replayed: the device time of the launch sequence (PDL
// between them, as in a layer chain) without the host's per-launch cost --
// measured ~4 us per conv_q_run and ~13 us through the Python binding, which
// exceeds the device time of small-batch layers and would make eager timing
// pick configs by host overhead.
// A timing session: the plan's stream (or a private non-blocking one when the
// plan uses the legacy / per-thread stream -- graph capture needs one) and two
// events; time_sel() scores the plan's current selection + runtime knobs.
struct TimingSession {
    conv_q_plan_s *p;
    cudaStream_t user_stream, ts;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc = CONV_Q_OK;
    explicit TimingSession(conv_q_plan_s *plan) : p(plan), user_stream(plan->stream), ts(plan->stream) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaError_t e = cudaStreamIsCapturing(p->stream, &cs);
        if (e != cudaSuccess) { rc = set_err(CONV_Q_ECUDA, "cudaStreamIsCapturing: %s", cudaGetErrorString(e)); return; }
        if (cs != cudaStreamCaptureStatusNone) { rc = set_err(CONV_Q_EINVAL, "tuning cannot run inside a graph capture"); return; }
        if (ts == nullptr || ts == cudaStreamLegacy || ts == cudaStreamPerThread) {
            if ((e = cudaStreamSynchronize(ts)) != cudaSuccess ||
                (e = cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking)) != cudaSuccess) {
                rc = set_err(CONV_Q_ECUDA, "timing stream: %s", cudaGetErrorString(e));
                ts = user_stream;
                return;
            }
        }
        p->stream = ts;
        if ((e = cudaEventCreate(&e0)) != cudaSuccess || (e = cudaEventCreate(&e1)) != cudaSuccess)
            rc = set_err(CONV_Q_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(e));
    }
    // `warmup` runs (+ tensor maps encoded), then 3 rounds of one CUDA-graph
    // replay of `reps` captured launches; *us = the median round's mean
    int time_sel(const void *x, const void *w, const float *scale, void *y, int warmup, int reps, float *us) {
        int r = ensure_ws(p);   // split-K workspace (grows only), before any timed run
        for (int k = 0; k < warmup + 1 && !r; ++k) r = conv_q_run(p, x, w, scale, y);
        if (r) return r;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaError_t ce = cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) return set_err(CONV_Q_ECUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(ce));
        for (int j = 0; j < reps && !r; ++j) r = conv_q_run(p, x, w, scale, y);
        ce = cudaStreamEndCapture(ts, &graph);
        if (!r && ce != cudaSuccess) r = set_err(CONV_Q_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(ce));
        if (!r) {
            ce = cudaGraphInstantiate(&exec, graph, 0);
            if (ce != cudaSuccess) r = set_err(CONV_Q_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ce));
        }
        float rt[3] = {0.f, 0.f, 0.f};
        if (!r) {
            cudaGraphLaunch(exec, ts);   // upload / first-replay costs outside the timed rounds
            for (int k = 0; k < 3; ++k) {
                cudaEventRecord(e0, ts);
                cudaGraphLaunch(exec, ts);
                cudaEventRecord(e1, ts);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                rt[k] = ms * 1000.f / reps;
            }
            ce = cudaGetLastError();
            if (ce != cudaSuccess) r = set_err(CONV_Q_ECUDA, "candidate graph replay: %s", cudaGetErrorString(ce));
        }
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (r) return r;
        std::sort(rt, rt + 3);
        *us = rt[1];
        return CONV_Q_OK;
    }
    // synchronise, restore the plan's stream; the first error wins
    int finish(int r) {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        cudaError_t e = cudaStreamSynchronize(ts);
        if (ts != user_stream) cudaStreamDestroy(ts);
        p->stream = user_stream;
        if (r) return r;
        if (e != cudaSuccess) return set_err(CONV_Q_ECUDA, "candidate run failed: %s", cudaGetErrorString(e));
        return CONV_Q_OK;
    }
};

static int time_candidates(conv_q_plan_s *p, const void *x, const void *w, const float *scale, void *y, int warmup,
                           int reps, float *us) {
    TimingSession t(p);
    if (t.rc) return t.finish(t.rc);
    int best = -1, rc = CONV_Q_OK;
    float best_us = 0.f;
    const int saved = p->sel;
    for (int i = 0; i < (int)p->cands.size() && !rc; ++i) {
        p->sel = i;
        float u = 0.f;
        if ((rc = t.time_sel(x, w, scale, y, warmup, reps, &u))) break;
        if (us) us[i] = u;
        if (best < 0 || u < best_us) {
            best = i;
            best_us = u;
        }
    }
    p->sel = saved;
    rc = t.finish(rc);
    return rc ? rc : best;
}

extern "C" int conv_q_plan_time(conv_q_plan_t *p, const void *x, const void *w, const float *scale, void *y,
                                int warmup, int reps, float *us) {
    if (!p || !us) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (warmup < 0 || reps < 1) return set_err(CONV_Q_EINVAL, "warmup >= 0 and reps >= 1 required");
    int rc = ensure_device();
    if (rc) return rc;
    TimingSession t(p);
    if (t.rc) return t.finish(t.rc);
    rc = t.time_sel(x, w, scale, y, warmup, reps, us);
    return t.finish(rc);
}

extern "C" int conv_q_plan_time_candidates(conv_q_plan_t *p, const void *x, const void *w, const float *scale,
                                           void *y, int warmup, int reps, float *us) {
    if (!p || !us) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (warmup < 0 || reps < 1) return set_err(CONV_Q_EINVAL, "warmup >= 0 and reps >= 1 required");
    int rc = ensure_device();
    if (rc) return rc;
    for (size_t i = 0; i < p->cands.size(); ++i) us[i] = -1.f;
    rc = time_candidates(p, x, w, scale, y, warmup, reps, us);
    if (rc >= 0 && p->cands[p->sel].split > 1) ensure_ws(p);
    return rc;
}

extern "C" int conv_q_plan_tune(conv_q_plan_t *p, const void *x, const void *w, const float *scale, void *y,
                                int warmup, int reps) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
    if (warmup < 0 || reps < 1) return set_err(CONV_Q_EINVAL, "warmup >= 0 and reps >= 1 required");
    int rc = ensure_device();
    if (rc) return rc;
    std::vector<float> us(p->cands.size(), -1.f);
    const int best = time_candidates(p, x, w, scale, y, warmup, reps, us.data());
    if (best < 0) return best;
    p->sel = best;
    p->user_sel = 1;
    p->tuned_us = us[best];
    if ((rc = ensure_ws(p))) return rc;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        cache_load_locked();
        g_cache[shape_key(p)] = {cand_name(p, best), us[best]};
        cache_store_locked();
    }
    return best;
}

// ============================================================== learned search (NEXT-4)
// The plan's enlarged schedule space (include/convq.h conv_q_plan_space):
// TileConfig knobs taken from the candidate list (only values that occur, so
// the space stays dense) x runtime knobs.  A point is valid when its
// TileConfig knobs name a candidate of the list and its runtime knobs apply.
namespace {
enum { KB_BN, KB_KBLK, KB_CG, KB_MODE, KB_DIRECT, KB_SPLIT, KB_EPI, KB_POL, KB_ROT, KB_GRID, KB_COUNT };
const int kSplits[] = {1, 2, 3, 4, 6, 8};
const int kGrids[] = {100, 75, 50};
const int kEpiWait[] = {0, 1, 2};
const unsigned kEpiWaitNs[] = {0, 20000, 64};

struct PlanSpace {
    conv_q_plan_s *p;
    std::vector<int> bns, cgs;
    std::vector<std::pair<int, int>> kblks, modes;   // (kch, nsub), (ws, halo)
    std::map<std::vector<int>, int> base;            // (bn, kblk, cg, mode, direct) -> candidate index (split 1)
    int sizes[KB_COUNT];
    explicit PlanSpace(conv_q_plan_s *plan) : p(plan) {
        for (const Cand &c : p->cands) {
            if (c.split != 1) continue;
            if (std::find(bns.begin(), bns.end(), c.bn) == bns.end()) bns.push_back(c.bn);
            if (std::find(cgs.begin(), cgs.end(), c.cg) == cgs.end()) cgs.push_back(c.cg);
            const std::pair<int, int> kb{c.kch, c.nsub}, md{c.ws, c.halo};
            if (std::find(kblks.begin(), kblks.end(), kb) == kblks.end()) kblks.push_back(kb);
            if (std::find(modes.begin(), modes.end(), md) == modes.end()) modes.push_back(md);
        }
        std::sort(bns.begin(), bns.end());
        std::sort(cgs.begin(), cgs.end());
        std::sort(kblks.begin(), kblks.end());
        std::sort(modes.begin(), modes.end());
        for (size_t i = 0; i < p->cands.size(); ++i) {
            const Cand &c = p->cands[i];
            if (c.split != 1) continue;
            std::vector<int> k = {idx(bns, c.bn), idx(kblks, std::make_pair(c.kch, c.nsub)), idx(cgs, c.cg),
                                  idx(modes, std::make_pair(c.ws, c.halo)), c.direct};
            if (!base.count(k)) base[k] = (int)i;
        }
        sizes[KB_BN] = (int)bns.size();
        sizes[KB_KBLK] = (int)kblks.size();
        sizes[KB_CG] = (int)cgs.size();
        sizes[KB_MODE] = (int)modes.size();
        sizes[KB_DIRECT] = 2;
        sizes[KB_SPLIT] = 6;
        sizes[KB_EPI] = 3;
        sizes[KB_POL] = 3;
        sizes[KB_ROT] = 2;
        sizes[KB_GRID] = 3;
    }
    template <class T>
    static int idx(const std::vector<T> &v, const T &x) {
        return (int)(std::find(v.begin(), v.end(), x) - v.begin());
    }
    // candidate index of the point's TileConfig (split 1), or -1
    int base_of(const int *k) const {
        auto it = base.find(std::vector<int>{k[KB_BN], k[KB_KBLK], k[KB_CG], k[KB_MODE], k[KB_DIRECT]});
        return it == base.end() ? -1 : it->second;
    }
    bool valid(const int *k) const {
        const int b = base_of(k);
        if (b < 0) return false;
        const Cand &c = p->cands[b];
        const int split = kSplits[k[KB_SPLIT]];
        if (split > 1) {   // split-K: im2col / tiled configs, the enumeration's limits
            if (c.ws || c.halo) return false;
            const int64_t tiles = ceil_div(p->M, 128 * c.cg) * ceil_div(p->K, c.bn);
            const int64_t num_kb = (int64_t)p->R * p->S * (p->C / c.kch);
            if (split > std::min<int64_t>(16, num_kb / (2 * c.nsub))) return false;
            if (tiles * c.cg * 128 * c.bn * 4 > ((int64_t)64 << 20) || 16 * num_kb >= ((int64_t)1 << 31)) return false;
        }
        // (a reduced weight-stationary grid keeps >= one CTA per N block: plan.cuh)
        return !(k[KB_ROT] && c.ws);   // the kernel ignores rotation for resident weights
    }
    // select the point on the plan: TileConfig (+ a split-K variant appended to
    // the candidate list when missing) and the runtime knobs
    void apply(const int *k) {
        Cand c = p->cands[base_of(k)];
        c.split = kSplits[k[KB_SPLIT]];
        int sel = -1;
        for (size_t i = 0; i < p->cands.size(); ++i) {
            const Cand &d = p->cands[i];
            if (d.bn == c.bn && d.kch == c.kch && d.cg == c.cg && d.nsub == c.nsub && d.direct == c.direct &&
                d.halo == c.halo && d.ws == c.ws && d.split == c.split) { sel = (int)i; break; }
        }
        if (sel < 0) {
            p->cands.push_back(c);
            sel = (int)p->cands.size() - 1;
        }
        p->sel = sel;
        p->epi_wait = kEpiWait[k[KB_EPI]];
        p->epi_wait_ns = kEpiWaitNs[k[KB_EPI]];
        p->out_policy = k[KB_POL];
        p->rotate = k[KB_ROT];
        p->grid_pct = kGrids[k[KB_GRID]];
    }
};

struct SearchCtx {
    PlanSpace *sp;
    TimingSession *ts;
    const void *x, *w;
    const float *scale;
    void *y;
    int warmup, reps;
    int fatal = CONV_Q_OK;
};

int search_valid(void *ctx, const int *k) { return static_cast<SearchCtx *>(ctx)->sp->valid(k) ? 1 : 0; }

double search_cost(void *ctx, const int *k) {
    SearchCtx *s = static_cast<SearchCtx *>(ctx);
    if (s->fatal) return -1.0;
    s->sp->apply(k);
    float us = 0.f;
    const int rc = s->ts->time_sel(s->x, s->w, s->scale, s->y, s->warmup, s->reps, &us);
    if (rc) {
        // a launch error leaves the context usable (EUNSUPPORTED / EINVAL are host-side);
        // a device fault is sticky: stop measuring
        if (cudaPeekAtLastError() != cudaSuccess || rc == CONV_Q_ECUDA) s->fatal = rc;
        return -1.0;
    }
    return us;
}
}  // namespace

extern "C" int conv_q_plan_space(const conv_q_plan_t *p, int *n_knobs, int *knob_sizes, long long *n_valid) {
    if (!p || !n_knobs || !knob_sizes) return set_err(CONV_Q_EINVAL, "NULL argument");
    PlanSpace sp(const_cast<conv_q_plan_t *>(p));
    *n_knobs = KB_COUNT;
    long long total = 1;
    for (int i = 0; i < KB_COUNT; ++i) {
        knob_sizes[i] = sp.sizes[i];
        total *= sp.sizes[i];
    }
    if (n_valid) {
        long long nv = 0;
        int k[KB_COUNT];
        for (long long v = 0; v < total; ++v) {
            long long r = v;
            for (int i = KB_COUNT - 1; i >= 0; --i) { k[i] = (int)(r % sp.sizes[i]); r /= sp.sizes[i]; }
            nv += sp.valid(k);
        }
        *n_valid = nv;
    }
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_set_point(conv_q_plan_t *p, const int *knobs) {
    if (!p || !knobs) return set_err(CONV_Q_EINVAL, "NULL argument");
    PlanSpace sp(p);
    for (int i = 0; i < KB_COUNT; ++i)
        if (knobs[i] < 0 || knobs[i] >= sp.sizes[i]) return set_err(CONV_Q_EINVAL, "knob %d out of range", i);
    if (!sp.valid(knobs)) return set_err(CONV_Q_EUNSUPPORTED, "not a valid point of the plan's space");
    sp.apply(knobs);
    p->user_sel = 1;
    p->tuned_us = -1.f;
    if (p->cands[p->sel].split > 1) {
        const int rc = ensure_device();
        if (rc) return rc;
        return ensure_ws(p);
    }
    return CONV_Q_OK;
}

extern "C" int conv_q_plan_get_point(const conv_q_plan_t *p, int *knobs) {
    if (!p || !knobs) return set_err(CONV_Q_EINVAL, "NULL argument");
    PlanSpace sp(const_cast<conv_q_plan_t *>(p));
    const Cand &c = p->cands[p->sel];
    knobs[KB_BN] = PlanSpace::idx(sp.bns, c.bn);
    knobs[KB_KBLK] = PlanSpace::idx(sp.kblks, std::make_pair(c.kch, c.nsub));
    knobs[KB_CG] = PlanSpace::idx(sp.cgs, c.cg);
    knobs[KB_MODE] = PlanSpace::idx(sp.modes, std::make_pair(c.ws, c.halo));
    knobs[KB_DIRECT] = c.direct;
    knobs[KB_SPLIT] = (int)(std::find(std::begin(kSplits), std::end(kSplits), c.split) - std::begin(kSplits));
    knobs[KB_EPI] = p->epi_wait;
    knobs[KB_POL] = p->out_policy;
    knobs[KB_ROT] = p->rotate;
    knobs[KB_GRID] = (int)(std::find(std::begin(kGrids), std::end(kGrids), p->grid_pct) - std::begin(kGrids));
    for (int i = 0; i < KB_COUNT; ++i)
        if (knobs[i] < 0 || knobs[i] >= sp.sizes[i] || (i == KB_EPI && p->epi_wait_ns != kEpiWaitNs[p->epi_wait]))
            return set_err(CONV_Q_EUNSUPPORTED, "the current selection is not a point of the plan's space (knob %d)", i);
    return sp.valid(knobs) ? CONV_Q_OK : set_err(CONV_Q_EUNSUPPORTED, "the current selection is not a valid point");
}

extern "C" int conv_q_plan_search(conv_q_plan_t *p, const void *x, const void *w, const float *scale, void *y,
                                  const conv_q_search_opts_t *opts, int warmup, int reps, float *best_us,
                                  double *history_us) {
    if (!p || !x || !w || !scale || !y) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (warmup < 0 || reps < 1) return set_err(CONV_Q_EINVAL, "warmup >= 0 and reps >= 1 required");
    int rc = ensure_device();
    if (rc) return rc;
    PlanSpace sp(p);
    TimingSession ts(p);
    if (ts.rc) return ts.finish(ts.rc);
    // saved selection + runtime knobs (restored if the search fails)
    const int s_sel = p->sel, s_ew = p->epi_wait, s_pol = p->out_policy, s_rot = p->rotate, s_grid = p->grid_pct;
    const unsigned s_ns = p->epi_wait_ns;
    SearchCtx ctx{&sp, &ts, x, w, scale, y, warmup, reps};
    int best[KB_COUNT];
    std::vector<double> hist(opts ? std::max(opts->trials, 1) : 128);
    const int n = conv_q_search(KB_COUNT, sp.sizes, search_valid, search_cost, &ctx, opts, best, hist.data(), nullptr);
    rc = ts.finish(ctx.fatal ? ctx.fatal : (n < 0 ? n : CONV_Q_OK));
    if (rc) {
        p->sel = s_sel; p->epi_wait = s_ew; p->epi_wait_ns = s_ns; p->out_policy = s_pol; p->rotate = s_rot;
        p->grid_pct = s_grid;
        return rc;
    }
    if (history_us)
        for (int i = 0; i < n; ++i) history_us[i] = hist[i] > 0 ? hist[i] : -1.0;
    double bu = -1;
    for (int i = 0; i < n; ++i)
        if (hist[i] > 0 && (bu < 0 || hist[i] < bu)) bu = hist[i];
    sp.apply(best);
    p->user_sel = 1;
    p->tuned_us = (float)bu;
    if (best_us) *best_us = (float)bu;
    if ((rc = ensure_ws(p))) return rc;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        cache_load_locked();
        g_cache[shape_key(p)] = {cand_name(p, p->sel) + runtime_suffix(p), (float)bu};
        cache_store_locked();
    }
    return n;
}

// ============================================================== quantize / pack
extern "C" int conv_q_padded_channels(int C, int bits) {
    if (C < 1 || (bits != 4 && bits != 8)) return set_err(CONV_Q_EINVAL, "C >= 1 and bits in {4,8} required");
    return (C + 31) / 32 * 32;  // 32-channel granule (reading 14): >= 16-byte rows for s4 and s8
}

static int grid_for(int64_t items, int threads) {
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    int64_t blocks = ceil_div(items, threads);
    int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread blocks per SM
    return (int)std::max<int64_t>(1, std::min(blocks, cap));
}

extern "C" int conv_q_quantize(const void *x_fp16, int N, int H, int W, int C, float inv_scale, int bits, void *xq,
                               void *stream) {
    if (!x_fp16 || !xq) return set_err(CONV_Q_EINVAL, "NULL tensor pointer");
    if (N < 1 || H < 1 || W < 1 || C < 1) return set_err(CONV_Q_EINVAL, "dimensions must be >= 1");
    if (bits != 4 && bits != 8) return set_err(CONV_Q_EINVAL, "bits must be 4 or 8");
    if (!aligned16(xq)) return set_err(CONV_Q_EINVAL, "xq must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    const int Cp = conv_q_padded_channels(C, bits);
    const int64_t npix = (int64_t)N * H * W;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (Cp == C && aligned16(x_fp16)) {
        const int64_t n_out_vec = npix * C * bits / 128;
        const int grid = grid_for(ceil_div(n_out_vec, 4), 256);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const uint4 *xs = static_cast<const uint4 *>(x_fp16);
        uint4 *ys = static_cast<uint4 *>(xq);
        if (bits == 8)
            CUDA_TRY(cudaLaunchKernelEx(&cfg, quantize_flat_kernel<8, 4>, xs, ys, n_out_vec, inv_scale));
        else
            CUDA_TRY(cudaLaunchKernelEx(&cfg, quantize_flat_kernel<4, 4>, xs, ys, n_out_vec, inv_scale));
    } else {
        const int vec_per_pix = Cp * bits / 128;
        const int grid = grid_for(npix * vec_per_pix, 256);
        if (bits == 8)
            quantize_padded_kernel<8><<<grid, 256, 0, st>>>(static_cast<const __half *>(x_fp16),
                                                           static_cast<uint4 *>(xq), npix, C, vec_per_pix, inv_scale);
        else
            quantize_padded_kernel<4><<<grid, 256, 0, st>>>(static_cast<const __half *>(x_fp16),
                                                           static_cast<uint4 *>(xq), npix, C, vec_per_pix, inv_scale);
    }
    CUDA_TRY(cudaGetLastError());
    return CONV_Q_OK;
}

extern "C" int conv_q_pack_weights(const int8_t *w, int K, int R, int S, int C, int bits, void *wp, void *stream) {
    if (!w || !wp) return set_err(CONV_Q_EINVAL, "NULL tensor pointer");
    if (K < 1 || R < 1 || S < 1 || C < 1) return set_err(CONV_Q_EINVAL, "dimensions must be >= 1");
    if (bits != 4 && bits != 8) return set_err(CONV_Q_EINVAL, "bits must be 4 or 8");
    if (((int64_t)C * bits) % 128) return set_err(CONV_Q_EUNSUPPORTED, "C*bits must be a multiple of 128");
    if (!aligned16(w) || !aligned16(wp)) return set_err(CONV_Q_EINVAL, "pointers must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    const int64_t n_out_vec = (int64_t)K * R * S * C * bits / 128;
    const int grid = grid_for(n_out_vec, 256);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (bits == 8)
        pack_weights_kernel<8><<<grid, 256, 0, st>>>(w, static_cast<uint4 *>(wp), n_out_vec);
    else
        pack_weights_kernel<4><<<grid, 256, 0, st>>>(w, static_cast<uint4 *>(wp), n_out_vec);
    CUDA_TRY(cudaGetLastError());
    return CONV_Q_OK;
}

// Unfused epilogue: s32 [M][K] -> packed [M][K*bits/8] (conv.cuh requant_kernel)
extern "C" int conv_q_requant(const int32_t *acc, int64_t M, int K, const float *scale, int relu, int bits, void *y,
                              void *stream) {
    if (!acc || !scale || !y) return set_err(CONV_Q_EINVAL, "NULL tensor pointer");
    if (M < 1 || K < 1) return set_err(CONV_Q_EINVAL, "M and K must be >= 1");
    if (bits != 4 && bits != 8) return set_err(CONV_Q_EINVAL, "bits must be 4 or 8");
    if (relu != 0 && relu != 1) return set_err(CONV_Q_EINVAL, "relu must be 0 or 1");
    if (((int64_t)K * bits) % 128) return set_err(CONV_Q_EUNSUPPORTED, "K*bits must be a multiple of 128");
    if (!aligned16(acc) || !aligned16(scale) || !aligned16(y)) return set_err(CONV_Q_EINVAL, "pointers must be 16-byte aligned");
    const int vpr = (int)((int64_t)K * bits / 128);
    if (M * vpr >= ((int64_t)1 << 31)) return set_err(CONV_Q_EUNSUPPORTED, "more than 2^31 output vectors");
    int rc = ensure_device();
    if (rc) return rc;
    const int total = (int)(M * vpr);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ceil_div(total, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int4 *a = reinterpret_cast<const int4 *>(acc);
    uint4 *ys = static_cast<uint4 *>(y);
    if (bits == 8)
        CUDA_TRY(cudaLaunchKernelEx(&cfg, requant_kernel<8>, a, scale, ys, total, K, vpr, relu, make_fastdiv(vpr)));
    else
        CUDA_TRY(cudaLaunchKernelEx(&cfg, requant_kernel<4>, a, scale, ys, total, K, vpr, relu, make_fastdiv(vpr)));
    return CONV_Q_OK;
}

// R x R max pooling of packed codes (pack.cuh maxpool_kernel)
extern "C" int conv_q_maxpool(const void *x, int N, int H, int W, int C, int R, int stride, int pad, int bits,
                              void *y, void *stream) {
    return conv_q_maxpool_fmt(x, N, H, W, C, R, stride, pad, bits, 0, y, stream);
}

extern "C" int conv_q_maxpool_fmt(const void *x, int N, int H, int W, int C, int R, int stride, int pad, int bits,
                                  int uns, void *y, void *stream) {
    if (uns != 0 && uns != 1) return set_err(CONV_Q_EINVAL, "uns must be 0 or 1");
    if (!x || !y) return set_err(CONV_Q_EINVAL, "NULL tensor pointer");
    if (N < 1 || H < 1 || W < 1 || C < 1 || R < 1 || stride < 1) return set_err(CONV_Q_EINVAL, "dimensions must be >= 1");
    if (bits != 4 && bits != 8) return set_err(CONV_Q_EINVAL, "bits must be 4 or 8");
    if (pad < 0 || pad >= R) return set_err(CONV_Q_EINVAL, "pad must be in [0, R)");
    if (H + 2 * pad < R || W + 2 * pad < R) return set_err(CONV_Q_EINVAL, "output is empty");
    if (((int64_t)C * bits) % 128) return set_err(CONV_Q_EUNSUPPORTED, "C*bits must be a multiple of 128");
    if (!aligned16(x) || !aligned16(y)) return set_err(CONV_Q_EINVAL, "pointers must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - R) / stride + 1;
    const int vpp = (int)((int64_t)C * bits / 128);
    const int64_t total = (int64_t)N * P * Q * vpp;
    if (total >= ((int64_t)1 << 31) || (int64_t)N * H * W * vpp >= ((int64_t)1 << 40))
        return set_err(CONV_Q_EUNSUPPORTED, "max pool output exceeds 2^31 16-byte vectors");
    if (R != 2 && R != 3) return set_err(CONV_Q_EUNSUPPORTED, "max pool window R=%d (2 or 3 supported)", R);
    const int grid = (int)ceil_div(total, 256);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint4 *xs = static_cast<const uint4 *>(x);
    uint4 *ys = static_cast<uint4 *>(y);
    const FastDiv fv = make_fastdiv(vpp), fq = make_fastdiv(Q), fp = make_fastdiv(P);
    if (R == 3 && stride == 2) {
        // the ResNet stem pool: 4 output rows per thread, shared horizontal maxima
        constexpr int T = 4;
        const int groups = (int)ceil_div(P, T);
        const int64_t total4 = (int64_t)N * groups * Q * vpp;
        cfg.gridDim = dim3((unsigned)ceil_div(total4, 256));
        auto k4 = uns ? (bits == 8 ? maxpool3s2_rows_kernel<8, true, T> : maxpool3s2_rows_kernel<4, true, T>)
                      : (bits == 8 ? maxpool3s2_rows_kernel<8, false, T> : maxpool3s2_rows_kernel<4, false, T>);
        CUDA_TRY(cudaLaunchKernelEx(&cfg, k4, xs, ys, N, H, W, P, Q, vpp, pad, groups, fv, fq, make_fastdiv(groups)));
        return CONV_Q_OK;
    }
    auto kern = uns ? (bits == 8 ? (R == 3 ? maxpool_kernel<8, 3, true> : maxpool_kernel<8, 2, true>)
                                 : (R == 3 ? maxpool_kernel<4, 3, true> : maxpool_kernel<4, 2, true>))
                    : (bits == 8 ? (R == 3 ? maxpool_kernel<8, 3> : maxpool_kernel<8, 2>)
                                 : (R == 3 ? maxpool_kernel<4, 3> : maxpool_kernel<4, 2>));
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, xs, ys, N, H, W, P, Q, vpp, stride, pad, fv, fq, fp));
    return CONV_Q_OK;
}

// s2d stem input / weights (pack.cuh s2d_quantize_kernel / s2d_weights_kernel)
extern "C" int conv_q_s2d_quantize(const conv_q_plan_t *p, const void *x_fp16, float inv_scale, void *xs,
                                   void *stream) {
    if (!p || !x_fp16 || !xs) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (!p->s2d) return set_err(CONV_Q_EINVAL, "plan was not created by conv_q_plan_s2d");
    if (!aligned16(xs)) return set_err(CONV_Q_EINVAL, "xs must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    const int64_t total = (int64_t)p->N * p->H * p->xs_W;
    if (total >= ((int64_t)1 << 31)) return set_err(CONV_Q_EUNSUPPORTED, "s2d tensor exceeds 2^31 pixels");
    // one thread per stored s2d pixel (no grid-stride loop: every thread's loads
    // are in flight at once; the kernel is a single HBM pass)
    const int grid = (int)ceil_div(total, 256);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int PL = p->pad;
    // RGB with W % 8 == 0 and a 16-byte aligned image: 4 s2d columns per thread,
    // 16-byte loads (rows are 6*W bytes, a multiple of 48; the stored row has
    // PL + W/2 + right-border columns, every border column written as zeros)
    if (p->o_C == 3 && p->o_W % 8 == 0 && (reinterpret_cast<uintptr_t>(x_fp16) & 15) == 0 &&
        p->xs_W >= PL + p->o_W / 2) {
        const int G = p->o_W / 8, TR = G + (p->xs_W - p->o_W / 2);
        const int64_t tv = (int64_t)p->N * p->H * TR;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)ceil_div(tv, 256));
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        auto kv = p->bits == 8 ? s2d_quantize_c3v_kernel<8> : s2d_quantize_c3v_kernel<4>;
        CUDA_TRY(cudaLaunchKernelEx(&cfg, kv, static_cast<const __half *>(x_fp16), static_cast<uint4 *>(xs), p->N,
                                    p->o_H, p->o_W, p->H, p->xs_W, PL, G, TR, inv_scale, make_fastdiv(TR),
                                    make_fastdiv(p->H)));
        return CONV_Q_OK;
    }
    // (even W keeps every row's 6*W-byte offset 4-byte aligned)
    const bool c3 = p->o_C == 3 && p->o_W % 2 == 0 && (reinterpret_cast<uintptr_t>(x_fp16) & 3) == 0;
    auto kern = p->bits == 8 ? (c3 ? s2d_quantize_kernel<8, true> : s2d_quantize_kernel<8, false>)
                             : (c3 ? s2d_quantize_kernel<4, true> : s2d_quantize_kernel<4, false>);
    kern<<<grid, 256, 0, st>>>(static_cast<const __half *>(x_fp16), static_cast<uint4 *>(xs), p->N, p->o_H, p->o_W,
                               p->o_C, p->H, p->xs_W, PL, inv_scale, make_fastdiv(p->xs_W), make_fastdiv(p->H));
    CUDA_TRY(cudaGetLastError());
    return CONV_Q_OK;
}

extern "C" int conv_q_s2d_pack_weights(const conv_q_plan_t *p, const int8_t *w_krsc, void *w_packed, void *stream) {
    if (!p || !w_krsc || !w_packed) return set_err(CONV_Q_EINVAL, "NULL argument");
    if (!p->s2d) return set_err(CONV_Q_EINVAL, "plan was not created by conv_q_plan_s2d");
    if (!aligned16(w_packed)) return set_err(CONV_Q_EINVAL, "w_packed must be 16-byte aligned");
    int rc = ensure_device();
    if (rc) return rc;
    const int S2P = p->row_bytes / 16;
    const int64_t total = (int64_t)p->K * p->R * S2P;
    const int grid = grid_for(total, 256);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (p->bits == 8)
        s2d_weights_kernel<8><<<grid, 256, 0, st>>>(w_krsc, static_cast<uint4 *>(w_packed), p->K, p->o_R, p->o_S,
                                                    p->o_C, p->R, S2P, p->pad, p->o_pad);
    else
        s2d_weights_kernel<4><<<grid, 256, 0, st>>>(w_krsc, static_cast<uint4 *>(w_packed), p->K, p->o_R, p->o_S,
                                                    p->o_C, p->R, S2P, p->pad, p->o_pad);
    CUDA_TRY(cudaGetLastError());
    return CONV_Q_OK;
}

// ============================================================== peak
extern "C" int conv_q_int8_peak(int iters, double *ops_per_s) {
    if (iters < 1 || !ops_per_s) return set_err(CONV_Q_EINVAL, "iters >= 1 and non-NULL output required");
    int rc = ensure_device();
    if (rc) return rc;
    const int smem = 1024 + (128 + 256) * 128 + 64;
    CUDA_TRY(cudaFuncSetAttribute(int8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int *sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(int)));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    int8_peak_kernel<<<g_num_sms, 128, smem>>>(std::min(iters, 1024), sink);  // warm-up
    cudaEventRecord(e0);
    int8_peak_kernel<<<g_num_sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return set_err(CONV_Q_ECUDA, "peak kernel failed: %s", cudaGetErrorString(e));
    *ops_per_s = 2.0 * 128 * 256 * 32 * (double)iters * g_num_sms / (ms * 1e-3);
    return CONV_Q_OK;
}

// Measurement only: MMA pipeline handshake probe (see peak.cuh).  Returns the
// achieved INT8 ops/s for `groups` groups of G MMAs (M=128, N=n) with at most
// S-1 groups in flight (S=1: no waits).
extern "C" CONVQ_API int conv_q_mma_pipe_probe(int groups, int G, int S, int n, double *ops_per_s) {
    if (groups < 1 || G < 1 || S < 1 || S > 16 || n < 16 || n > 256 || (n % 16) || !ops_per_s)
        return set_err(CONV_Q_EINVAL, "bad probe arguments");
    int rc = ensure_device();
    if (rc) return rc;
    const int smem = 1024 + (128 + 256) * 128 + 256;
    CUDA_TRY(cudaFuncSetAttribute(mma_pipe_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int *sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(int)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma_pipe_probe_kernel<<<g_num_sms, 128, smem>>>(std::min(groups, 64), G, S, n, sink);
    cudaEventRecord(e0);
    mma_pipe_probe_kernel<<<g_num_sms, 128, smem>>>(groups, G, S, n, sink);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return set_err(CONV_Q_ECUDA, "probe kernel failed: %s", cudaGetErrorString(e));
    *ops_per_s = 2.0 * 128 * n * 32 * (double)groups * G * g_num_sms / (ms * 1e-3);
    return CONV_Q_OK;
}

// Measurement only: per-primitive single-thread cycles of the MMA warp (see micro_probe_kernel).
extern "C" CONVQ_API int conv_q_micro_probe(int mode, int iters, int n, double *cycles_per_iter) {
    if (mode < 0 || mode > 9 || iters < 1 || n < 16 || n > 256 || (n % 16) || !cycles_per_iter)
        return set_err(CONV_Q_EINVAL, "bad probe arguments");
    int rc = ensure_device();
    if (rc) return rc;
    const int smem = 1024 + (128 + 256) * 128 + 256;
    void (*kerns[10])(int, int, long long *) = {micro_probe_kernel<0>, micro_probe_kernel<1>, micro_probe_kernel<2>,
                                                micro_probe_kernel<3>, micro_probe_kernel<4>, micro_probe_kernel<5>,
                                                micro_probe_kernel<6>, micro_probe_kernel<7>, micro_probe_kernel<8>,
                                                micro_probe_kernel<9>};
    CUDA_TRY(cudaFuncSetAttribute(kerns[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    long long *out = nullptr;
    CUDA_TRY(cudaMalloc(&out, sizeof(long long)));
    kerns[mode]<<<1, 128, smem>>>(iters, n, out);
    long long h = 0;
    cudaError_t e = cudaMemcpy(&h, out, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(out);
    if (e != cudaSuccess) return set_err(CONV_Q_ECUDA, "probe kernel failed: %s", cudaGetErrorString(e));
    *cycles_per_iter = (double)h / iters;
    return CONV_Q_OK;
}

// Measurement only: CTA-pair (cta_group::2, M=256) variant of the probe above.
extern "C" CONVQ_API int conv_q_mma_pipe_probe2(int groups, int G, int S, int n, double *ops_per_s) {
    if (groups < 1 || G < 1 || S < 1 || S > 16 || n < 32 || n > 256 || (n % 32) || !ops_per_s)
        return set_err(CONV_Q_EINVAL, "bad probe arguments");
    int rc = ensure_device();
    if (rc) return rc;
    const int smem = 1024 + (128 + 256) * 128 + 256;
    CUDA_TRY(cudaFuncSetAttribute(mma_pipe_probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int *sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(int)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g_num_sms / 2 * 2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int gw = std::min(groups, 64);
    CUDA_TRY(cudaLaunchKernelEx(&cfg, mma_pipe_probe2_kernel, gw, G, S, n, sink));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    CUDA_TRY(cudaLaunchKernelEx(&cfg, mma_pipe_probe2_kernel, groups, G, S, n, sink));
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return set_err(CONV_Q_ECUDA, "probe2 kernel failed: %s", cudaGetErrorString(e));
    *ops_per_s = 2.0 * 256 * n * 32 * (double)groups * G * (g_num_sms / 2) / (ms * 1e-3);
    return CONV_Q_OK;
}

// Measurement only: per-CTA wait-cycle counters (see conv.cuh TR_*): the
// caller passes a device buffer of >= 8 * grid u64 (zeroed), or NULL to stop.
extern "C" CONVQ_API int conv_q_plan_set_trace(conv_q_plan_t *p, void *counters) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
#ifndef CONVQ_INSTRUMENT
    if (counters) return set_err(CONV_Q_EUNSUPPORTED, "tracing needs the CONVQ_INSTRUMENT build (libconvq_instr.so)");
#endif
    p->trace = static_cast<unsigned long long *>(counters);
    return CONV_Q_OK;
}

// Measurement only: CTA 0's event timeline (clock64 per event, [64][256] u64,
// zeroed by the caller; see conv.cuh CONVQ_TL), or NULL to stop.
extern "C" CONVQ_API int conv_q_plan_set_timeline(conv_q_plan_t *p, void *buf) {
    if (!p) return set_err(CONV_Q_EINVAL, "NULL plan");
#ifndef CONVQ_INSTRUMENT
    if (buf) return set_err(CONV_Q_EUNSUPPORTED, "timelines need the CONVQ_INSTRUMENT build (libconvq_instr.so)");
#endif
    p->tl = static_cast<unsigned long long *>(buf);
    return CONV_Q_OK;
}
