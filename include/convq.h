/*
 * convq.h -- C ABI of libconvq.so: B200 (sm_100a) quantized INT8/INT4
 * implicit-GEMM 2-D convolution with s32 accumulation, input quantize/pack,
 * and a fused requantize + repack epilogue that writes the next layer's
 * packed NHWC layout.
 *
 * The operation (section 2.1): a convolution over feature map
 * width W, height H, input channels I (= C here), output channels O (= K),
 * kernel R x S, batch N "can be translated into matrix multiplication of
 * (N*H*W, I*R*S) x (I*R*S, O)".  Output spatial size uses floor:
 *   P = (H + 2*pad - R)/stride + 1,   Q = (W + 2*pad - S)/stride + 1.
 * For every output pixel (n,p,q) and output channel k:
 *   acc[n,p,q,k] = sum_{r,s,c} x[n, p*stride-pad+r, q*stride-pad+s, c] * w[k,r,s,c]
 * (out-of-range x reads as 0), then (section 3.2.2: "relu, batch
 * normalization, and bias addition ... finally clipped to lower bits and
 * packed"):
 *   y[n,p,q,k] = clamp(rne(fmaf((float)acc, scale[k], shift[k])), lo, hi)
 *   lo = relu ? 0 : -2^(bits-1),  hi = 2^(bits-1) - 1
 * packed into `bits`-bit two's-complement codes (section 1:
 * "8 consecutive values (in 32-bit) into a packed vector of 4-bit elements").
 *
 * Conventions for every entry point:
 *   - Tensor pointers are DEVICE pointers unless stated, 16-byte aligned.
 *     The caller owns every tensor; the library never frees them.
 *   - Calls are asynchronous on the plan's (or the given) CUDA stream; kernel
 *     faults surface at the next synchronisation, as usual in CUDA.
 *   - Functions returning int return CONV_Q_OK (0) or a negative CONV_Q_E*
 *     code; conv_q_plan returns NULL on error.  conv_q_last_error() then holds
 *     a thread-local message.
 *   - Packed layouts (bits = 8 or 4), channel-innermost:
 *       s8: byte c of a pixel row = (uint8) q[c]
 *       s4: 32-bit word c/8 holds q[c] & 0xF at bits 4*(c mod 8)
 *           (little-nibble-first), i.e. byte c/2, low nibble = even c.
 *     One pixel row is C*bits/8 bytes and must be a multiple of 16 bytes.
 *   - x : packed NHWC  [N][H][W][C*bits/8]
 *     w : packed KRSC  [K][R][S][C*bits/8]   (C innermost)
 *     scale: 2*K floats [scale_0..scale_{K-1}, shift_0..shift_{K-1}]
 *     y : packed NHWC  [N][P][Q][K*bits/8]   (== next layer's x), or
 *         int32 NHWC   [N][P][Q][K] in CONV_Q_OUT_S32 mode (raw accumulators).
 */
#ifndef CONVQ_H
#define CONVQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CONVQ_API __attribute__((visibility("default")))
#else
#define CONVQ_API
#endif

/* status codes */
#define CONV_Q_OK            0
#define CONV_Q_EINVAL       (-1)  /* bad argument: dims < 1, stride/pad/bits out of range, NULL or misaligned pointer */
#define CONV_Q_EUNSUPPORTED (-2)  /* valid conv the kernels do not cover, e.g. C*bits or K*bits not a multiple of 128 */
#define CONV_Q_EOVERFLOW    (-3)  /* R*S*C*2^(2*bits-2) may exceed int32 (accumulator guard, PAPER.md:166 s3.2.1) */
#define CONV_Q_ECUDA        (-4)  /* a CUDA runtime/driver call failed (no device, launch failure, ...) */
#define CONV_Q_ENOMEM       (-5)  /* host or device allocation failed */

/* output modes (conv_q_plan_set_epilogue) */
#define CONV_Q_OUT_PACKED    0    /* requantize + repack to bits-bit NHWC (default) */
#define CONV_Q_OUT_S32       1    /* raw int32 accumulators (debug / parity) */

typedef struct conv_q_plan_s conv_q_plan_t;   /* opaque; owned by the library */

typedef struct conv_q_info_s {
    int N, H, W, C, K, R, S, stride, pad, bits;
    int P, Q;                 /* output spatial size (floor) */
    int64_t M;                /* GEMM rows  = N*P*Q */
    int64_t Kg;               /* GEMM depth = R*S*C */
    int64_t x_bytes, w_bytes, y_bytes, y_s32_bytes;
    int relu, out_mode;
    int num_candidates;       /* TileConfig candidates valid for this shape */
    int config_index;         /* currently selected candidate */
    char config[64];          /* its name, e.g. "bm128_bn256_kc128x1_c1_st" (see conv_q_plan_candidate_name) */
    float tuned_us;           /* per-launch time of the selected config if tuned, else -1 */
    int64_t macs;             /* M * K * Kg: multiply-accumulates of one run */
    /* (ABI 1.01) tensor shapes conv_q_run expects, in bytes of the innermost dim:
     *   x [x_dims[0]][x_dims[1]][x_dims[2]][x_dims[3] bytes]
     *   w [w_dims[0]][w_dims[1]][w_dims[2]][w_dims[3] bytes]
     * (== [N][H][W][C*bits/8] and [K][R][S][C*bits/8] for conv_q_plan; the
     * s2d tensors for conv_q_plan_s2d, whose other fields describe the
     * caller's stride-2 conv). */
    int s2d;
    int x_dims[4];
    int w_dims[4];
} conv_q_info_t;

/*
 * Create a plan for one convolution shape (the paper's problem statement,
 * N, H, W, I(=C), O(=K), R, S, plus stride and pad).
 * bits in {4, 8} applies to x, w and y.  Host-only: validates the shape,
 * derives P, Q, M, Kg, enumerates the valid TileConfig candidates and picks a
 * default (conv_q_plan_tune re-picks by timing).  Needs a CUDA device only to
 * read its SM count; on a machine without one the plan is still created and
 * conv_q_run returns CONV_Q_ECUDA.
 * Errors (NULL + last_error):
 *   EINVAL       any dim < 1, stride not in [1,8], pad not in [0,127],
 *                R-1 or S-1 > 255, P or Q < 1, bits not in {4,8}
 *   EUNSUPPORTED C*bits or K*bits not a multiple of 128; s4: C not a multiple of
 *                32; s8: C < 32 (C = 16 mod 32 is accepted: the last channel block
 *                of each tap is zero-filled by the TMA)
 *                (pad C with conv_q_quantize), or C*bits/8 > 65535
 *   EOVERFLOW    R*S*C * 2^(2*bits-2) > 2^31-1
 */
CONVQ_API conv_q_plan_t *conv_q_plan(int N, int H, int W, int C, int K, int R, int S,
                           int stride, int pad, int bits);

/*
 * Stem convolution (ABI 1.01): a stride-2 R x S convolution with pad `pad`
 * over an image with few channels (C <= 4 for bits = 8, C <= 8 for bits = 4),
 * e.g. ResNet's conv1 7x7/2 over RGB -- the same operation and output
 * (P = (H+2pad-R)/2 + 1, y packed NHWC [N][P][Q][K*bits/8]) as
 * conv_q_plan(N,H,W,C,K,R,S,2,pad,bits) on the channel-padded input, computed
 * as a stride-1 convolution over a space-to-depth(2) view (DESIGN.md s6
 * "stem"): no 32-channel padding of C=3 (10.7x wasted MMA work and operand
 * bytes at 7x7/2) and 128/64-byte operand rows instead of 32-byte ones.
 *   x : conv_q_s2d_quantize output, [N][ceil(H/2)][Q + S2P - 1][16 B]
 *       (info.x_dims; 16-byte s2d pixels = 2x2 input pixels x 4 (s8) / 8 (s4)
 *       channel codes, index (2*dh+dw)*CP + c, zero borders)
 *   w : conv_q_s2d_pack_weights output, [K][R2][1][S2P*16 B] (info.w_dims)
 * conv_q_run / _tune / _set_epilogue / _set_config / _info work as for any
 * plan.  Errors: as conv_q_plan, plus EUNSUPPORTED when C exceeds the phase
 * width or the filter needs more than 8 s2d taps in W.
 */
CONVQ_API conv_q_plan_t *conv_q_plan_s2d(int N, int H, int W, int C, int K, int R, int S, int pad, int bits);

/* fp16 NHWC image [N][H][W][C] (device) -> the plan's s2d tensor xs (device,
 * info.x_dims bytes, 16-byte aligned), quantized exactly as conv_q_quantize:
 * q = clamp(rne(fp32(x) * inv_scale), lo, hi), NaN -> lo.  Errors: EINVAL. */
CONVQ_API int conv_q_s2d_quantize(const conv_q_plan_t *plan, const void *x_fp16, float inv_scale, void *xs,
                                  void *stream);

/* int8 KRSC codes [K][R][S][C] (device, the caller's unpadded C) -> the plan's
 * window weights (device, info.w_dims bytes).  Once per model. */
CONVQ_API int conv_q_s2d_pack_weights(const conv_q_plan_t *plan, const int8_t *w_krsc, void *w_packed,
                                      void *stream);

/*
 * Run the plan: y = requant(conv(x, w), scale) (or raw s32 accumulators).
 * x, w, scale, y: device pointers in the layouts above, 16-byte aligned.
 * One launch of the implicit-GEMM kernel on the plan's stream.  Never
 * allocates: a split-K config (name suffix "_k<s>": s CTAs share one output
 * tile's K loop, and meet in a plan-owned s32 workspace of
 * ceil(M/BM)*BM*K*4 bytes + counters, zeroed once and left zero by every run)
 * gets its workspace when it is selected (conv_q_plan / _set_config /
 * _set_epilogue / _set_residual / _tune), so a run may be graph-captured.
 * Errors: EINVAL (NULL / misaligned pointer), ECUDA (no device, launch failure).
 * One run in flight per plan is allowed (the plan caches tensor maps and owns
 * the split-K workspace).
 */
CONVQ_API int conv_q_run(conv_q_plan_t *plan, const void *x, const void *w, const float *scale, void *y);

/*
 * Fused residual add (ABI 1.03; SURVEY 8(f) NEXT-2 -- a ResNet block's
 * relu(bn(conv(x)) + identity); section 3.2.2 puts the elementwise
 * "relu, batch normalization, and bias addition" in the epilogue).  With a
 * non-NULL skip every later conv_q_run / conv_q_plan_tune computes, per
 * output (pixel m, channel k), DESIGN reading 15:
 *   u = fmaf((float)acc, scale[k], shift[k]);  v = fmaf((float)skip[m,k], res_scale, u)
 *   y = clamp(rne(v), lo, hi)       (ReLU, if enabled, after the add)
 * skip: device packed tensor in y's layout [N][P][Q][K*bits/8] (16-byte
 * aligned, caller-owned, read only; e.g. the block input or the downsample
 * conv's output); res_scale: one fp32 per layer.  NULL disables.  The pointer
 * is stored in the plan (a captured CUDA graph keeps the one it was captured
 * with).  Errors: EINVAL (misaligned skip; S32 output mode at run time),
 * EUNSUPPORTED (s2d stem plans).
 */
CONVQ_API int conv_q_plan_set_residual(conv_q_plan_t *plan, const void *skip, float res_scale);

/* Stream for subsequent runs (a cudaStream_t; NULL = legacy default stream). */
CONVQ_API int conv_q_plan_set_stream(conv_q_plan_t *plan, void *stream);

/* relu in {0,1}; out_mode CONV_Q_OUT_PACKED or CONV_Q_OUT_S32.  Re-selects the
 * tuning cache's config for (shape, relu, out_mode) when it holds one. */
CONVQ_API int conv_q_plan_set_epilogue(conv_q_plan_t *plan, int relu, int out_mode);

/* TileConfig candidates: count, names, manual selection.
 * Name = bm<MMA rows>_bn<N tile>_kc<channels per k-block>x<k-blocks per stage>
 *        _c<CTAs per tile (2 = cta_group::2 pair)>[_st: direct 16-byte stores,
 *        else smem staging + TMA store][_h: duplicate-aware halo A operand]
 *        [_k<s>: split-K over s work units][_w: weight-stationary (the CTA's
 *        weight block resident in shared memory)][_m2: a work unit is two
 *        128-row m-groups sharing one accumulator round trip]. */
CONVQ_API int conv_q_plan_num_candidates(const conv_q_plan_t *plan);
CONVQ_API int conv_q_plan_candidate_name(const conv_q_plan_t *plan, int index, char *buf, int buflen);
CONVQ_API int conv_q_plan_set_config(conv_q_plan_t *plan, int index);

/*
 * Per-shape tile configuration picked by timing ("the best
 * scheduling of MMA instructions varies for different convolution sizes";
 * the B200 analog of the paper's exhaustive search, Table 1).
 * Times every candidate on the given (caller-owned, valid) buffers with CUDA
 * events -- `warmup` untimed runs, then 3 rounds of `reps` back-to-back
 * launches (as in a layer sequence, where each launch's prologue overlaps the
 * previous kernel), scored by the median round's mean -- selects the
 * fastest and records it in the in-process cache (and in the JSON file named
 * by $CONV_Q_CACHE, if set).  y is overwritten.  Synchronises the stream.
 * Returns the selected index (>= 0) or an error code.
 */
CONVQ_API int conv_q_plan_tune(conv_q_plan_t *plan, const void *x, const void *w, const float *scale,
                     void *y, int warmup, int reps);

/*
 * (ABI 1.04) Time every candidate exactly as conv_q_plan_tune does and write
 * candidate i's per-launch time in microseconds to us[i] (host array of
 * conv_q_plan_num_candidates floats; -1 if it did not run), WITHOUT changing
 * the selection or the cache.  Returns the fastest index or an error code.
 * Used by the per-shape sweep and the ablation (scripts/ablation.py).
 */
CONVQ_API int conv_q_plan_time_candidates(conv_q_plan_t *plan, const void *x, const void *w, const float *scale,
                                          void *y, int warmup, int reps, float *us);

/*
 * (ABI 1.06) Learned, diversity-aware schedule search:
 * the exploration module of PAPER.md:282-298 (section 3.4, Figs. 12-13) with
 * the settings of PAPER.md:309-314 (section 4.1).  Host-only; no device work.
 *
 * A space is n_knobs categorical knobs, knob i taking values 0..knob_sizes[i]-1
 * (1 <= n_knobs <= CONV_Q_SEARCH_MAX_KNOBS; the product of the sizes < 2^60).
 *   valid(ctx, knobs): nonzero when the point exists (NULL: every point);
 *   cost(ctx, knobs):  the measured cost of the point, > 0, lower is better
 *                      (e.g. microseconds); <= 0 marks a failed point.
 * Every batch measures `batch` never-measured points: the first batch random,
 * then the (batch - 1) best points of simulated annealing over a cost model
 * (pairwise ranking loss on the measurements so far) plus one random point;
 * diversity != 0: each annealing chain makes two mutants and half of all
 * mutants are kept by configuration diversity before competing with their
 * parents (the paper's proposal); 0: one mutant per chain (AutoTVM).
 * Stops after `trials` measurements or when the space is exhausted.
 * best_knobs (host, n_knobs ints) receives the fastest measured point;
 * history_cost (host, trials doubles) / history_knobs (host, trials*n_knobs
 * ints), if not NULL, receive every measurement in order.
 * Returns the number of measurements (>= 1) or an error code (EINVAL: bad
 * arguments; ECUDA: no point measured successfully).  Deterministic for a seed.
 */
#define CONV_Q_SEARCH_MAX_KNOBS 16
typedef struct conv_q_search_opts {
    int trials;          /* hardware measurements in total (default 128) */
    int batch;           /* measurements per model round (default 32 = 31 picks + 1 random) */
    int sa_iters;        /* annealing iterations (500) */
    int sa_early_stop;   /* stop when the optimal set is unchanged this long (50) */
    int sa_points;       /* parallel annealing chains (128) */
    int diversity;       /* 1: diversity-aware selection (default), 0: plain mutation */
    float sa_temp0;      /* start temperature (1.0) */
    float sa_cool;       /* temperature decrease per iteration (0.002) */
    unsigned long long seed;
} conv_q_search_opts_t;
typedef int (*conv_q_valid_fn)(void *ctx, const int *knobs);
typedef double (*conv_q_cost_fn)(void *ctx, const int *knobs);
CONVQ_API void conv_q_search_opts_default(conv_q_search_opts_t *opts);
CONVQ_API int conv_q_search(int n_knobs, const int *knob_sizes, conv_q_valid_fn valid, conv_q_cost_fn cost,
                            void *ctx, const conv_q_search_opts_t *opts, int *best_knobs, double *history_cost,
                            int *history_knobs);

/*
 * (ABI 1.06) The plan's enlarged schedule space (NEXT-4): the TileConfig
 * knobs of the candidate list -- BN, k-block (channels x k-blocks per stage),
 * CTAs per tile, operand mode (im2col/tiled, halo, weight-stationary, WS halo,
 * WS MT2, WS halo MT2), output path (TMA store / direct) -- crossed with
 * runtime knobs: split-K {1,2,3,4,6,8} (im2col/tiled configs), epilogue
 * accumulator wait {spin, suspend hint, nanosleep}, output L2 policy {none,
 * evict_last, evict_first}, k-block start rotation {off, on}, persistent
 * grid {100, 75, 50 % of the SMs}.  *n_knobs (<= CONV_Q_SEARCH_MAX_KNOBS) and
 * knob_sizes[] describe it; *n_valid receives the number of valid points.
 */
CONVQ_API int conv_q_plan_space(const conv_q_plan_t *plan, int *n_knobs, int *knob_sizes, long long *n_valid);

/* (ABI 1.06) Select one point of conv_q_plan_space (knobs: host, n_knobs ints):
 * its TileConfig (a split-K variant is appended to the candidate list when
 * needed; its workspace is allocated here) and runtime knobs.  EINVAL: a knob
 * out of range; EUNSUPPORTED: not a valid point. */
CONVQ_API int conv_q_plan_set_point(conv_q_plan_t *plan, const int *knobs);
/* (ABI 1.06) The current selection as a point of conv_q_plan_space (knobs: host,
 * n_knobs ints) -- e.g. to copy a searched pick to another plan of the same
 * shape.  EUNSUPPORTED when the selection is not a point of the space (a
 * split-K count outside {1,2,3,4,6,8}, a runtime knob set by environment). */
CONVQ_API int conv_q_plan_get_point(const conv_q_plan_t *plan, int *knobs);

/*
 * (ABI 1.06) conv_q_search over conv_q_plan_space, each point timed on the
 * device exactly as conv_q_plan_tune times a candidate (`warmup` runs, 3
 * rounds of `reps` graph-captured launches, median round).  Selects the
 * fastest point (TileConfig -- a split-K variant is appended to the candidate
 * list when needed -- and its runtime knobs), records it in the tuning cache
 * under the plan's shape key (name = candidate name + "+e<wait>p<policy>r<rot>g<grid %>"),
 * writes its time to *best_us and every measured time (-1 = failed) to
 * history_us (host, opts->trials doubles; may be NULL).  y is overwritten.
 * Synchronises the stream.  Returns the number of measurements or an error code.
 */
CONVQ_API int conv_q_plan_search(conv_q_plan_t *plan, const void *x, const void *w, const float *scale, void *y,
                                 const conv_q_search_opts_t *opts, int warmup, int reps, float *best_us,
                                 double *history_us);

/* (ABI 1.06) Time the current selection exactly as conv_q_plan_tune times a
 * candidate (graph-captured `reps` launches, 3 rounds, median) and write its
 * per-launch microseconds to *us (host).  The per-layer table of bench.py.
 * Synchronises the stream.  y is overwritten. */
CONVQ_API int conv_q_plan_time(conv_q_plan_t *plan, const void *x, const void *w, const float *scale, void *y,
                               int warmup, int reps, float *us);

/* Fill *info (host memory). */
CONVQ_API int conv_q_plan_info(const conv_q_plan_t *plan, conv_q_info_t *info);

CONVQ_API void conv_q_plan_destroy(conv_q_plan_t *plan);

/*
 * Quantize + pack (section 1).  x_fp16: device fp16 NHWC
 * [N][H][W][C]; xq: device packed NHWC with C' = conv_q_padded_channels(C,bits)
 * channels ([N][H][W][C'*bits/8] bytes); channels [C, C') are written as 0.
 *   q = clamp(rne(fp32(x) * inv_scale), -2^(bits-1), 2^(bits-1)-1); NaN -> lo.
 * stream: cudaStream_t or NULL.  Errors: EINVAL, ECUDA.
 */
CONVQ_API int conv_q_quantize(const void *x_fp16, int N, int H, int W, int C, float inv_scale,
                    int bits, void *xq, void *stream);

/* C' = C rounded up to a multiple of 32 channels: one 32-byte tcgen05 K step
 * for s8 and a whole 16-byte pixel row for s4 (reading 14). */
CONVQ_API int conv_q_padded_channels(int C, int bits);

/*
 * Pack weights once per model (off the per-run path): w_krsc is a device int8
 * [K][R][S][C] array of codes already in [-2^(bits-1), 2^(bits-1)-1] (values
 * outside are truncated to their low `bits` bits); w_packed receives
 * [K][R][S][C*bits/8] bytes.  C*bits must be a multiple of 128.
 */
CONVQ_API int conv_q_pack_weights(const int8_t *w_krsc, int K, int R, int S, int C, int bits,
                        void *w_packed, void *stream);

/*
 * Unfused epilogue (ABI 1.04): requantize + repack an s32 accumulator matrix
 * acc [M][K] (device; e.g. conv_q_run's CONV_Q_OUT_S32 output, M = N*P*Q) into
 * packed y [M][K*bits/8] (device) with exactly the fused epilogue's arithmetic
 * (section 3.2.2; DESIGN readings 4-5):
 *   y = clamp(rne(fmaf((float)acc, scale[k], shift[k])), lo, hi), lo = relu ? 0 : -2^(bits-1).
 * A separate HBM pass (4 + bits/8 bytes per output) -- the design the fused
 * epilogue replaces; kept for the NEXT-3 ablation (section 4.4)
 * and for callers that need the s32 accumulators too.  scale: 2*K floats.
 * Errors: EINVAL (NULL / misaligned pointer, M or K < 1, relu not 0/1, bits),
 * EUNSUPPORTED (K*bits not a multiple of 128, > 2^31 output vectors), ECUDA.
 */
CONVQ_API int conv_q_requant(const int32_t *acc, int64_t M, int K, const float *scale, int relu, int bits, void *y,
                             void *stream);

/*
 * R x R max pooling of packed codes (ABI 1.02; the pooling glue of a ResNet
 * stem: conv1 -> 3x3/2 max pool -> layer1; the networks of
 * PAPER.md:40 section 1).  x: device packed NHWC [N][H][W][C*bits/8];
 * y: device packed NHWC [N][P][Q][C*bits/8], P = (H+2pad-R)/stride + 1 (floor),
 * Q likewise.  y[n,p,q,c] = max of x[n, p*stride-pad+r, q*stride-pad+s, c] over
 * the in-range taps (padding never wins); max of signed codes, exact.
 * Errors: EINVAL (NULL / misaligned pointer, dims < 1, pad not in [0,R),
 * empty output), EUNSUPPORTED (C*bits not a multiple of 128, R not in {2,3},
 * more than 2^31 output vectors), ECUDA.
 */
CONVQ_API int conv_q_maxpool(const void *x, int N, int H, int W, int C, int R, int stride, int pad, int bits,
                             void *y, void *stream);

/*
 * As conv_q_maxpool over codes of format uns (ABI 1.05; DESIGN reading 16):
 * uns = 1 compares unsigned codes [0, 2^bits - 1] (post-ReLU activations),
 * uns = 0 signed codes (== conv_q_maxpool).  Errors: as conv_q_maxpool, plus
 * EINVAL for uns not 0/1.
 */
CONVQ_API int conv_q_maxpool_fmt(const void *x, int N, int H, int W, int C, int R, int stride, int pad, int bits,
                                 int uns, void *y, void *stream);

/*
 * Code formats of a plan (ABI 1.05; SURVEY 8(f) NEXT-2 "unsigned u8/u4
 * post-ReLU activations"; DESIGN reading 16 -- the paper's codes are signed,
 * SPEC.md:274, and a ReLU epilogue (section 3.2.2) leaves the
 * sign bit unused).  Each flag 0 = signed two's-complement codes (the
 * default), 1 = unsigned codes [0, 2^bits - 1]; same packed layout either way:
 *   x_unsigned     the activations x are read as unsigned (tcgen05 A format u8;
 *                  INT4 nibbles expand to 16*v as before)
 *   y_unsigned     the packed output is written as unsigned codes:
 *                  y = clamp(rne(v), 0, 2^bits - 1) -- the lower bound is the
 *                  ReLU, so it applies whatever conv_q_plan_set_epilogue's relu
 *   skip_unsigned  the residual skip tensor (conv_q_plan_set_residual) holds
 *                  unsigned codes
 * Weights stay signed.  Ownership: none.  The plan re-applies the tuning cache
 * (its key includes the formats).  Errors: EINVAL (NULL plan, flag not 0/1),
 * EOVERFLOW (x_unsigned with R*S*C*255*128 > 2^31 - 1: the accumulator guard
 * of PAPER.md:166 section 3.2.1 for unsigned activations).
 */
CONVQ_API int conv_q_plan_set_formats(conv_q_plan_t *plan, int x_unsigned, int y_unsigned, int skip_unsigned);

/*
 * Cross-launch completion counters (ABI 1.05): dataflow between consecutive
 * conv launches of a layer chain (the packed output of one layer IS the next
 * layer's input, section 3.3).  Instead of waiting for the whole
 * previous grid to complete and flush (griddepcontrol.wait), the launch waits
 * for a counter of the codes its input holds; every producer warp adds the
 * codes it wrote once its stores are complete.  Each argument is ONE device
 * uint32 counter, caller-owned, 4-byte aligned, ZERO at the start of every run
 * of the chain (e.g. one memset per step):
 *   in_done    the input x is complete when it reaches N*H*W*C (the count its
 *              producer adds); NULL: wait for the whole preceding kernel
 *              instead (griddepcontrol.wait).
 *   skip_done  the residual skip is complete at N*P*Q*K; NULL: the skip is
 *              complete before the launch.
 *   out_done   incremented by N*P*Q*K in total as this launch's codes reach
 *              global memory; the next layer's in_done.  NULL: not counted.
 * With in_done set, every buffer the launch writes must not be read by a
 * kernel still running (true in a chain of distinct per-layer outputs).
 * Tuning (conv_q_plan_tune / _time_candidates) needs the counters cleared.
 * Errors: EINVAL (NULL plan, misaligned counters), EUNSUPPORTED (in_done on an
 * s2d stem plan, tensors with more than 2^32 - 1 codes).
 */
CONVQ_API int conv_q_plan_set_deps(conv_q_plan_t *plan, const unsigned *in_done, const unsigned *skip_done,
                                   unsigned *out_done);

/* Thread-local status code of the last failed call on this thread (0 if none). */
CONVQ_API int conv_q_last_status(void);

/* Thread-local message for the last error on this thread ("" if none). */
CONVQ_API const char *conv_q_last_error(void);

/* ABI version (major*100 + minor). */
CONVQ_API int conv_q_version(void);

/*
 * Measurement only (roofline denominator): run a tcgen05.mma
 * kind::i8 loop (M=128, N=256, K=32, operands resident in shared memory, no
 * HBM traffic) on every SM for `iters` MMAs per CTA and report the achieved
 * dense INT8 rate in ops/s (2 ops per MAC) in *ops_per_s.  Synchronises.
 */
CONVQ_API int conv_q_int8_peak(int iters, double *ops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* CONVQ_H */
