"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
closed forms, values the paper/spec print, special cases that reduce to a
library routine (numpy's IEEE fp16 decode, torch float64 conv2d), brute force
through a different route (explicit im2col lowering + GEMM), and
invariants.  CPU only."""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import workloads as wl


# ---------------------------------------------------------------- fp16 decode
def test_half_decode_all_codes_match_ieee():
    """Every binary16 code decodes to numpy's IEEE value (library routine)."""
    codes = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = codes.view(np.float16).astype(np.float32)
    got = np.array([oracle.half_to_float(int(c)) for c in codes], dtype=np.float32)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint32), ref[~nan].view(np.uint32))  # incl. -0


# ---------------------------------------------------------------- quantize
@pytest.mark.parametrize("bits", [4, 8])
def test_quantize_exact_multiples(bits):
    """x = j / inv_scale exactly representable -> q = clamp(j)."""
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    for inv in (1.0, 4.0, 0.25, 32.0):
        for j in range(-300, 301):
            f = j / inv
            assert oracle.quantize_value(f, inv, bits) == min(max(j, lo), hi)


def test_quantize_ties_to_even():
    cases = {0.5: 0, 1.5: 2, 2.5: 2, 3.5: 4, -0.5: 0, -1.5: -2, -2.5: -2, 126.5: 126, 125.5: 126}
    for f, q in cases.items():
        assert oracle.quantize_value(f, 1.0, 8) == q, f
    # s4: 6.5 -> 6, 7.5 -> 8 -> clamped 7, -7.5 -> -8
    assert oracle.quantize_value(6.5, 1.0, 4) == 6
    assert oracle.quantize_value(7.5, 1.0, 4) == 7
    assert oracle.quantize_value(-7.5, 1.0, 4) == -8


def test_quantize_specials():
    for bits in (4, 8):
        lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
        assert oracle.quantize_value(65504.0, 1.0, bits) == hi
        assert oracle.quantize_value(-65504.0, 1.0, bits) == lo
        assert oracle.quantize_value(math.inf, 1.0, bits) == hi
        assert oracle.quantize_value(-math.inf, 1.0, bits) == lo
        assert oracle.quantize_value(-0.0, 1.0, bits) == 0
        assert oracle.quantize_value(math.nan, 1.0, bits) == lo       # reading 5: NaN -> lo
        assert oracle.quantize_value(1e-8, 1.0, bits) == 0


def test_quantize_tensor_padding_and_layout():
    """C=3 pads to C'=32 (reading 14) with zero codes; real channels equal
    the scalar quantizer; pixel order is NHWC."""
    g = np.random.default_rng(1)
    x = g.standard_normal((2, 3, 5, 3)).astype(np.float16)
    for bits, cp in ((8, 32), (4, 32)):
        assert oracle.padded_channels(3, bits) == cp
        xq = oracle.quantize(x, 7.0, bits)
        assert xq.shape == (2, 3, 5, cp * bits // 8)
        codes = oracle.unpack(xq, cp, bits)
        assert np.all(codes[..., 3:] == 0)
        for idx in itertools.product(range(2), range(3), range(5), range(3)):
            assert codes[idx] == oracle.quantize_value(float(x[idx]), 7.0, bits)


# ---------------------------------------------------------------- pack
def test_pack_spec_words():
    """SPEC.md:226 [1..8] <-> 0x87654321; SPEC.md:235-237 0 and 0xFFFFFFFF."""
    w = oracle.pack(np.array([1, 2, 3, 4, 5, 6, 7, 8], dtype=np.int8), 4)
    assert int(w.view("<u4")[0]) == 0x87654321
    assert list(oracle.unpack(np.array([0x21, 0x43, 0x65, 0x87], np.uint8), 8, 4)) == [1, 2, 3, 4, 5, 6, 7, -8]
    assert list(oracle.unpack(np.zeros(4, np.uint8), 8, 4)) == [0] * 8
    assert list(oracle.unpack(np.full(4, 0xFF, np.uint8), 8, 4)) == [-1] * 8
    assert int(oracle.pack(np.full(8, -1, np.int8), 4).view("<u4")[0]) == 0xFFFFFFFF
    assert int(oracle.pack(np.full(8, -8, np.int8), 4).view("<u4")[0]) == 0x88888888
    assert list(oracle.pack(np.array([-128, -1, 0, 127], np.int8), 8)) == [0x80, 0xFF, 0x00, 0x7F]


@pytest.mark.parametrize("bits", [4, 8])
def test_pack_roundtrip_random(bits):
    g = np.random.default_rng(2)
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    q = g.integers(lo, hi + 1, size=(10000, 8), dtype=np.int8)
    p = oracle.pack(q, bits)
    assert p.shape == (10000, 8 * bits // 8)
    assert np.array_equal(oracle.unpack(p, 8, bits), q)
    # and bytes -> codes -> bytes is the identity on every byte value
    b = np.arange(256, dtype=np.uint8).reshape(-1, 8 * bits // 8) if bits == 8 else \
        np.arange(256, dtype=np.uint8).repeat(4).reshape(-1, 4)
    assert np.array_equal(oracle.pack(oracle.unpack(b, 8, bits), bits), b)


# ---------------------------------------------------------------- conv_s32
def _lowered_gemm(xc, wc, stride, pad):
    """Independent route (section 2.1, Fig. 1): materialize the im2col
    matrix L[(n,p,q), (r,s,c)] by enumerating source coordinates,
    then one int64 matrix product with the weight matrix."""
    N, H, W, C = xc.shape
    K, R, S, _ = wc.shape
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    L = np.zeros((N * P * Q, R * S * C), dtype=np.int64)
    row = 0
    for n in range(N):
        for p in range(P):
            for q in range(Q):
                col = 0
                for r in range(R):
                    for s in range(S):
                        h, w = p * stride - pad + r, q * stride - pad + s
                        if 0 <= h < H and 0 <= w < W:
                            L[row, col:col + C] = xc[n, h, w]
                        col += C
                row += 1
    Wm = wc.reshape(K, R * S * C).astype(np.int64).T
    return (L @ Wm).reshape(N, P, Q, K)


@pytest.mark.parametrize("bits", [4, 8])
def test_conv_brute_force_lowered_gemm(bits):
    g = np.random.default_rng(3)
    per16 = 128 // bits
    for trial in range(24):
        N = int(g.integers(1, 3))
        H, W = int(g.integers(1, 6)), int(g.integers(1, 6))
        C = per16 * int(g.integers(1, 3))
        K = int(g.integers(1, 5))
        R, S = int(g.choice([1, 3])), int(g.choice([1, 3, 2]))
        stride = int(g.integers(1, 3))
        pad = int(g.integers(0, 2))
        if (H + 2 * pad - R) < 0 or (W + 2 * pad - S) < 0:
            continue
        x = wl.random_bytes(g, (N, H, W, C * bits // 8))
        w = wl.random_bytes(g, (K, R, S, C * bits // 8))
        got = oracle.conv_s32(x, w, C, stride, pad, bits)
        ref = _lowered_gemm(oracle.unpack(x, C, bits), oracle.unpack(w, C, bits), stride, pad)
        assert np.array_equal(got, ref), (N, H, W, C, K, R, S, stride, pad)


@pytest.mark.parametrize("bits", [4, 8])
def test_conv_matches_torch_float64(bits):
    """Library cross-check: torch conv2d in float64 on integer-valued tensors is
    exact (every partial sum is an integer < 2^53)."""
    g = np.random.default_rng(4)
    for (N, H, W, C, K, R, S, st, pad) in [(2, 9, 7, 64, 16, 3, 3, 1, 1), (1, 11, 11, 32, 8, 5, 5, 2, 2),
                                            (1, 8, 8, 128, 12, 1, 1, 2, 0), (2, 7, 6, 32, 20, 7, 7, 3, 3),
                                            (1, 6, 6, 64, 4, 3, 1, 1, 0)]:
        if C * bits % 128:
            continue
        x = wl.random_bytes(g, (N, H, W, C * bits // 8))
        w = wl.random_bytes(g, (K, R, S, C * bits // 8))
        got = oracle.conv_s32(x, w, C, st, pad, bits)
        xt = torch.from_numpy(oracle.unpack(x, C, bits).astype(np.float64)).permute(0, 3, 1, 2)
        wt = torch.from_numpy(oracle.unpack(w, C, bits).astype(np.float64)).permute(0, 3, 1, 2)
        ref = torch.nn.functional.conv2d(xt, wt, stride=st, padding=pad).permute(0, 2, 3, 1).numpy()
        assert np.array_equal(got, ref.astype(np.int64))


def test_conv_all_ones_tap_counts():
    """SPEC.md:76 (4x4 input, 3x3, pad 1): 144 im2col cells, 100 valid taps, 44
    pad taps. With all-ones x and w, y[p,q,k] = taps(p,q) * C: 4C corners, 6C
    edges, 9C inside; sum over (p,q) = 100*C for every k."""
    C, K = 16, 3
    x = np.ones((1, 4, 4, C), np.int8).view(np.uint8)
    w = np.ones((K, 3, 3, C), np.int8).view(np.uint8)
    y = oracle.conv_s32(x, w, C, 1, 1, 8)[0]
    taps = np.array([[4, 6, 6, 4], [6, 9, 9, 6], [6, 9, 9, 6], [4, 6, 6, 4]])
    for k in range(K):
        assert np.array_equal(y[:, :, k], taps * C)
        assert y[:, :, k].sum() == 100 * C
    assert 9 * 16 == 144 and 144 - 100 == 44


def test_conv_identity_and_zero():
    """zero in -> zero out; 1x1 identity weights -> output = input."""
    g = np.random.default_rng(5)
    for bits in (4, 8):
        C = 128 // bits * 2
        x = wl.random_bytes(g, (2, 5, 6, C * bits // 8))
        ident = np.eye(C, dtype=np.int8).reshape(C, 1, 1, C)
        w = oracle.pack(ident, bits)
        y = oracle.conv_s32(x, w, C, 1, 0, bits)
        assert np.array_equal(y, oracle.unpack(x, C, bits).astype(np.int32))
        z = oracle.conv_s32(np.zeros_like(x), wl.random_bytes(g, (7, 3, 3, C * bits // 8)), C, 1, 1, bits)
        assert not z.any()


def test_conv_1x1_is_explicit_gemm():
    g = np.random.default_rng(6)
    C, K = 64, 24
    x = wl.random_bytes(g, (3, 4, 5, C))
    w = wl.random_bytes(g, (K, 1, 1, C))
    y = oracle.conv_s32(x, w, C, 1, 0, 8)
    A = x.view(np.int8).reshape(-1, C).astype(np.int64)
    B = w.view(np.int8).reshape(K, C).astype(np.int64)
    assert np.array_equal(y.reshape(-1, K), A @ B.T)


def test_conv_extremes_largest_kg():
    """All x = w = -128 at 3x3x512: interior acc = 4608 * 16384 = 75,497,472 (> 2^24)."""
    C = 512
    x = np.full((1, 3, 3, C), 0x80, np.uint8)
    w = np.full((2, 3, 3, C), 0x80, np.uint8)
    y = oracle.conv_s32(x, w, C, 1, 1, 8)
    assert y[0, 1, 1, 0] == 4608 * 16384 == 75497472
    assert y[0, 0, 0, 1] == 4 * 512 * 16384


def test_conv_pixel_sampling_equals_full():
    g = np.random.default_rng(7)
    C = 64
    x = wl.random_bytes(g, (2, 9, 8, C))
    w = wl.random_bytes(g, (16, 3, 3, C))
    full = oracle.conv_s32(x, w, C, 2, 1, 8)
    pix = np.array([0, 5, 17, full.shape[1] * full.shape[2] * 2 - 1], np.int64)
    part = oracle.conv_s32(x, w, C, 2, 1, 8, pix=pix)
    assert np.array_equal(part, full.reshape(-1, 16)[pix])


def test_table1_ops_and_gemm_shapes():
    """PAPER.md:323 Table 1 OPs = 1,849,688,064 for every stage at N=8;
    SPEC.md:58-60 GEMM shapes."""
    for L in wl.paper_table1_layers():
        P, Q = oracle.out_dim(L.H, L.R, 1, 1), oracle.out_dim(L.W, L.S, 1, 1)
        assert 2 * 8 * P * Q * L.K * L.C * L.R * L.S == 1849688064
    assert 8 * 56 * 56 == 25088 and 64 * 9 == 576
    assert 8 * oracle.out_dim(7, 3, 1, 1) ** 2 == 392 and 512 * 9 == 4608
    assert oracle.out_dim(56, 3, 2, 1) == 28      # floor reading 6: (56+2-3)/2 = 27.5
    assert oracle.out_dim(224, 7, 2, 3) == 112


# ---------------------------------------------------------------- requant
def test_requant_scale_one_is_saturating_cast():
    for acc in range(-300, 301):
        assert oracle.requant_value(acc, 1.0, 0.0, False, 8) == min(max(acc, -128), 127)
        assert oracle.requant_value(acc, 1.0, 0.0, False, 4) == min(max(acc, -8), 7)
        assert oracle.requant_value(acc, 1.0, 0.0, True, 8) == min(max(acc, 0), 127)


def test_requant_half_ties_even():
    """scale 0.5: 1->0, 3->2, 5->2, -1->0, -3->-2 (round half to even)."""
    for acc, y in {1: 0, 3: 2, 5: 2, 7: 4, -1: 0, -3: -2, -5: -2, 2: 1}.items():
        assert oracle.requant_value(acc, 0.5, 0.0, False, 8) == y


def test_requant_power_of_two_scales_exact():
    """scale 2^-k, shift 0: y = clamp(round_half_even(acc / 2^k)) computed exactly
    with rationals (Python round() on Fraction is half-to-even)."""
    g = np.random.default_rng(8)
    for k in range(0, 12):
        for acc in g.integers(-(1 << 20), 1 << 20, size=300):
            exact = round(Fraction(int(acc), 1 << k))
            assert oracle.requant_value(int(acc), 2.0 ** -k, 0.0, False, 8) == min(max(exact, -128), 127)


def test_requant_shift_and_relu():
    assert oracle.requant_value(10, 1.0, 0.5, False, 8) == 10      # 10.5 -> 10
    assert oracle.requant_value(11, 1.0, 0.5, False, 8) == 12      # 11.5 -> 12
    assert oracle.requant_value(-10, 1.0, -0.5, True, 8) == 0
    assert oracle.requant_value(-10, 1.0, 20.25, True, 4) == 7


def test_requant_int_to_float_rounding():
    """(float)acc rounds to nearest even before the FMA: -(2^24+1) -> -2^24, so
    with scale 2^-25 the product is exactly -0.5 -> 0 (an exact-rational
    evaluation without that rounding would give -1)."""
    acc = -((1 << 24) + 1)
    assert oracle.requant_value(acc, 2.0 ** -25, 0.0, False, 8) == 0
    assert round(Fraction(acc, 1 << 25)) == -1


@pytest.mark.parametrize("relu", [False, True])
def test_requant_single_rounding_fma_exact(relu):
    """Reading 5 (PAPER.md:200 s3.2.2 epilogue order): the
    multiply-add rounds ONCE.  40 000 adversarial (acc, scale, shift) triples
    whose exact value sits within half an ulp of a half-integer (a quarter of
    them exact ties) are evaluated with exact rationals and one binary32
    rounding (tests/exact_fp.py); the oracle must match every one, and the
    set must contain cases where mul-then-add (two roundings) gives another
    code -- so a two-rounding oracle fails this pin."""
    import exact_fp
    g = np.random.default_rng(2202)
    acc, scale, shift = exact_fp.near_tie_cases(g, 40000, 8)
    n = acc.size
    # one case per output channel of a 1 x 8000 accumulator row (vectorised oracle calls)
    got = np.concatenate([
        oracle.unpack(oracle.requant(acc[i:i + 8000].astype(np.int32).reshape(1, -1),
                                     np.concatenate([scale[i:i + 8000], shift[i:i + 8000]]), relu, 8), 8000, 8)[0]
        for i in range(0, n, 8000)])
    ref = np.array([exact_fp.requant_exact(int(a), float(s), float(h), relu, 8)
                    for a, s, h in zip(acc, scale, shift)])
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (bad[:5], acc[bad[:5]], scale[bad[:5]], shift[bad[:5]], got[bad[:5]], ref[bad[:5]])
    two = exact_fp.requant_two_roundings(acc, scale, shift, relu, 8)
    differ = int(np.count_nonzero(two != ref))
    assert differ >= 500, differ                  # the pin separates fmaf from mul-then-add
    # exact ties (float64 evaluation is exact for these short operands): round
    # half to even decides, and every tie lands on an even code
    f = acc.astype(np.float64) * scale.astype(np.float64) + shift.astype(np.float64)
    ties = (np.arange(n) % 4 == 0) & (f - np.floor(f) == 0.5)
    assert np.count_nonzero(ties) >= n // 5
    assert np.all(ref[ties] % 2 == 0)


def test_requant_pack_rows():
    acc = np.array([[1, -1, 200, -200, 3, 4, 5, 6]], np.int32)
    ss = np.concatenate([np.ones(8), np.zeros(8)]).astype(np.float32)
    y = oracle.requant(acc, ss, False, 4)
    assert int(y.view("<u4").reshape(-1)[0]) == 0x654387F1
    assert list(oracle.unpack(y, 8, 4)[0]) == [1, -1, 7, -8, 3, 4, 5, 6]
    y8 = oracle.requant(acc, ss, True, 8)
    assert list(y8[0]) == [1, 0, 127, 0, 3, 4, 5, 6]


# ---------------------------------------------------------------- guard arithmetic
def test_accumulator_bits_paper():
    """PAPER.md:166 section 3.2.1: 2^4 * 2^4 * 128 = 2^15 -> 16 bits."""
    def bits_required(a, b, terms):
        return math.ceil(math.log2((1 << a) * (1 << b) * terms)) + 1

    def channels_to_saturate(acc_bits, a, b, taps):
        return math.ceil((1 << (acc_bits - 1)) / ((1 << a) * (1 << b) * taps))

    assert bits_required(4, 4, 128) == 16
    assert bits_required(8, 8, 256) == 25
    assert channels_to_saturate(32, 4, 4, 9) == 932068
    assert channels_to_saturate(16, 4, 4, 1) == 128


# ---------------------------------------------------------------- max pool (NEXT-2 glue)
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("N,H,W,C,R,st,pad", [(2, 9, 8, 64, 3, 2, 1), (1, 12, 12, 32, 3, 2, 1),
                                               (1, 7, 5, 32, 2, 2, 0), (1, 6, 6, 64, 3, 1, 1)])
def test_maxpool_matches_torch(bits, N, H, W, C, R, st, pad):
    """Library cross-check: torch max_pool2d (float64, -inf padding) on the
    unpacked codes, repacked by the (pinned) pack."""
    g = np.random.default_rng(31 + H)
    x = wl.random_bytes(g, (N, H, W, C * bits // 8))
    got = oracle.maxpool(x, C, R, st, pad, bits)
    xt = torch.from_numpy(oracle.unpack(x, C, bits).astype(np.float64)).permute(0, 3, 1, 2)
    ref = torch.nn.functional.max_pool2d(xt, R, st, pad).permute(0, 2, 3, 1).numpy().astype(np.int8)
    assert got.shape[:3] == ref.shape[:3]
    assert np.array_equal(oracle.unpack(got, C, bits), ref)


def test_maxpool_closed_forms():
    """All-equal input -> the same code everywhere (padding never wins, even for
    the most negative code); a single maximum reaches exactly the windows that
    cover it."""
    x = np.full((1, 5, 5, 32), 0x80, np.uint8)                # every code -128
    assert np.all(oracle.maxpool(x, 32, 3, 2, 1, 8) == 0x80)
    x = np.zeros((1, 6, 6, 32), np.uint8)
    x[0, 3, 2, 5] = 100
    y = oracle.unpack(oracle.maxpool(x, 32, 3, 2, 1, 8), 32, 8)
    hit = {(p, q) for p in range(3) for q in range(3) if abs(2 * p - 3) <= 1 and abs(2 * q - 2) <= 1}
    for p in range(3):
        for q in range(3):
            assert y[0, p, q, 5] == (100 if (p, q) in hit else 0)
    assert np.all(np.delete(y, 5, axis=3) == 0)



# ---------------------------------------------------------------- residual epilogue (NEXT-2, reading 15)
def test_requant_res_zero_scale_is_plain_requant():
    g = np.random.default_rng(41)
    for _ in range(2000):
        acc, sc, sh = int(g.integers(-(1 << 20), 1 << 20)), float(np.float32(g.uniform(1e-4, 1e-2))), \
            float(np.float32(g.uniform(-3, 3)))
        sk = int(g.integers(-128, 128))
        for relu in (False, True):
            assert oracle.requant_res_value(acc, sc, sh, sk, 0.0, relu, 8) == oracle.requant_value(acc, sc, sh, relu, 8)


def test_requant_res_unit_scales_add_integers():
    """scale = res_scale = 1, shift = 0: y = clamp(acc + skip) (every step exact)."""
    for acc in range(-150, 151, 7):
        for sk in range(-128, 128, 5):
            assert oracle.requant_res_value(acc, 1.0, 0.0, sk, 1.0, False, 8) == min(max(acc + sk, -128), 127)
            assert oracle.requant_res_value(acc, 1.0, 0.0, sk, 1.0, True, 8) == min(max(acc + sk, 0), 127)
    for acc in range(-12, 13):
        for sk in range(-8, 8):
            assert oracle.requant_res_value(acc, 1.0, 0.0, sk, 1.0, False, 4) == min(max(acc + sk, -8), 7)


@pytest.mark.parametrize("relu", [False, True])
def test_requant_res_exact_two_roundings(relu):
    """Reading 15's two single-rounded FMAs, against exact rationals: random
    cases plus near-tie cases (the shift puts u next to a half-integer, the
    skip term moves it by a non-dyadic amount)."""
    import exact_fp
    g = np.random.default_rng(4242 + relu)
    acc, sc, sh = exact_fp.near_tie_cases(g, 6000, 8)
    sk = g.integers(-128, 128, acc.size)
    rs = np.float32(g.uniform(0.05, 1.5))
    K = acc.size
    skip = oracle.pack(sk.astype(np.int8).reshape(1, K), 8)
    got = oracle.unpack(oracle.requant_res(acc.astype(np.int32).reshape(1, K), np.concatenate([sc, sh]), skip,
                                           float(rs), relu, 8), K, 8)[0]
    ref = np.array([exact_fp.requant_res_exact(int(a), float(s), float(h), int(k), float(rs), relu, 8)
                    for a, s, h, k in zip(acc, sc, sh, sk)])
    assert np.array_equal(got, ref), np.nonzero(got != ref)[0][:5]
    # scalar entry point == packed entry point
    for i in range(0, K, 97):
        assert oracle.requant_res_value(int(acc[i]), float(sc[i]), float(sh[i]), int(sk[i]), float(rs), relu, 8) \
            == ref[i]
