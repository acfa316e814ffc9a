"""Pins for the oracle's unsigned code formats (DESIGN reading 16; SURVEY 8(f)
NEXT-2 "unsigned u8/u4 post-ReLU activations"; section 3.2.2 --
the ReLU of the epilogue makes every post-ReLU code non-negative, so the sign
bit of a signed code is wasted).  Pinned against values fixed by the format
definitions, a library routine (torch float64 conv2d / max_pool2d), an
algebraic identity through the already-pinned signed path, and exact
rationals.  CPU only."""
import numpy as np
import pytest
import torch

import exact_fp
import oracle
import workloads as wl


# ---------------------------------------------------------------- unpack / pack
def test_unpack_fmt_every_byte():
    """u8: a byte IS its value; s8: two's complement (== the pinned oracle.unpack)."""
    b = np.arange(256, dtype=np.uint8)
    assert list(oracle.unpack_fmt(b, 256, 8, True)) == list(range(256))
    assert list(oracle.unpack_fmt(b, 256, 8, False)) == [v - 256 if v >= 128 else v for v in range(256)]
    assert np.array_equal(oracle.unpack_fmt(b, 256, 8, False), oracle.unpack(b, 256, 8).astype(np.int16))
    # u4: byte i holds channel 2i (low nibble) and 2i+1 (high nibble), read unsigned
    u4 = oracle.unpack_fmt(b, 512, 4, True)
    assert list(u4[0::2]) == [v & 15 for v in range(256)] and list(u4[1::2]) == [v >> 4 for v in range(256)]


def test_unpack_fmt_spec_words():
    """SPEC.md:226's word 0x87654321 read as unsigned nibbles is [1..8] (the top
    nibble 8 is -8 only in the signed format); 0xFFFFFFFF is 15 everywhere."""
    w = np.array([0x21, 0x43, 0x65, 0x87], np.uint8)
    assert list(oracle.unpack_fmt(w, 8, 4, True)) == [1, 2, 3, 4, 5, 6, 7, 8]
    assert list(oracle.unpack_fmt(w, 8, 4, False)) == [1, 2, 3, 4, 5, 6, 7, -8]
    assert list(oracle.unpack_fmt(np.full(4, 0xFF, np.uint8), 8, 4, True)) == [15] * 8


@pytest.mark.parametrize("bits", [4, 8])
def test_pack_fmt_roundtrip(bits):
    g = np.random.default_rng(16)
    q = g.integers(0, 1 << bits, size=(2000, 32)).astype(np.int16)
    p = oracle.pack_fmt(q, bits)
    assert np.array_equal(oracle.unpack_fmt(p, 32, bits, True), q)
    # signed values pack exactly as the pinned signed pack
    s = g.integers(-(1 << (bits - 1)), 1 << (bits - 1), size=(500, 32))
    assert np.array_equal(oracle.pack_fmt(s.astype(np.int16), bits), oracle.pack(s.astype(np.int8), bits))


# ---------------------------------------------------------------- conv with unsigned activations
@pytest.mark.parametrize("bits", [4, 8])
def test_conv_unsigned_matches_torch_float64(bits):
    """Library cross-check: torch float64 conv2d on the unsigned activation values
    and signed weight values (exact: |acc| < 2^53)."""
    g = np.random.default_rng(61 + bits)
    for N, H, W, C, K, R, st, pad in [(2, 7, 6, 64, 5, 3, 1, 1), (1, 9, 9, 32, 3, 3, 2, 1), (1, 5, 4, 32, 4, 1, 1, 0)]:
        x = wl.random_bytes(g, (N, H, W, C * bits // 8))
        w = wl.random_bytes(g, (K, R, R, C * bits // 8))
        acc = oracle.conv_s32(x, w, C, st, pad, bits, x_uns=True)
        xt = torch.from_numpy(oracle.unpack_fmt(x, C, bits, True).astype(np.float64)).permute(0, 3, 1, 2)
        wt = torch.from_numpy(oracle.unpack(w, C, bits).astype(np.float64)).permute(0, 3, 1, 2)
        ref = torch.nn.functional.conv2d(xt, wt, stride=st, padding=pad).permute(0, 2, 3, 1).numpy()
        assert np.array_equal(acc, ref.astype(np.int64))


@pytest.mark.parametrize("bits", [4, 8])
def test_conv_unsigned_identity_through_signed(bits):
    """u = s + 2^b [s < 0] for every code, so by linearity
    acc_u = acc_s + 2^b * conv(mask, w), mask = 1 where the signed code is negative.
    Both right-hand terms come from the (separately pinned) signed path."""
    g = np.random.default_rng(77 + bits)
    N, H, W, C, K = 2, 6, 5, 64, 6
    x = wl.random_bytes(g, (N, H, W, C * bits // 8))
    w = wl.random_bytes(g, (K, 3, 3, C * bits // 8))
    neg = (oracle.unpack(x, C, bits) < 0).astype(np.int8)
    mask = oracle.pack(neg, bits)
    acc_u = oracle.conv_s32(x, w, C, 1, 1, bits, x_uns=True).astype(np.int64)
    acc_s = oracle.conv_s32(x, w, C, 1, 1, bits).astype(np.int64)
    acc_m = oracle.conv_s32(mask, w, C, 1, 1, bits).astype(np.int64)
    assert np.array_equal(acc_u, acc_s + (1 << bits) * acc_m)
    assert np.any(acc_m != 0)


def test_conv_unsigned_extremes():
    """All activations 255 and all weights -128 at 3x3x512: acc = -255*128*4608
    at interior pixels (= -150 405 120, inside int32: the plan guard's bound for
    unsigned codes, R*S*C*255*128 < 2^31)."""
    x = np.full((1, 3, 3, 512), 0xFF, np.uint8)
    w = np.full((1, 3, 3, 512), 0x80, np.uint8)
    acc = oracle.conv_s32(x, w, 512, 1, 1, 8, x_uns=True)
    assert acc[0, 1, 1, 0] == -255 * 128 * 9 * 512
    assert acc[0, 0, 0, 0] == -255 * 128 * 4 * 512


# ---------------------------------------------------------------- requant into unsigned codes
def test_requant_fmt_closed_forms():
    """scale 1, shift 0: every step exact, y = clamp(acc, 0, 2^b - 1) for unsigned
    output codes (the ReLU is the lower clamp); the signed format equals the
    pinned requant_value."""
    for acc in range(-300, 301, 3):
        assert oracle.requant_value_fmt(acc, 1.0, 0.0, False, 8, True) == min(max(acc, 0), 255)
        assert oracle.requant_value_fmt(acc, 1.0, 0.0, True, 8, True) == min(max(acc, 0), 255)
        assert oracle.requant_value_fmt(acc, 1.0, 0.0, False, 4, True) == min(max(acc, 0), 15)
        for relu in (False, True):
            for bits in (4, 8):
                assert oracle.requant_value_fmt(acc, 1.0, 0.0, relu, bits, False) == \
                    oracle.requant_value(acc, 1.0, 0.0, relu, bits)
    # ties to even near the top of the unsigned range: 254.5 -> 254, 255.5 -> 256 -> 255
    assert oracle.requant_value_fmt(509, 0.5, 0.0, True, 8, True) == 254
    assert oracle.requant_value_fmt(511, 0.5, 0.0, True, 8, True) == 255
    assert oracle.requant_value_fmt(29, 0.5, 0.0, True, 4, True) == 14      # 14.5 -> 14


@pytest.mark.parametrize("bits", [8, 4])
def test_requant_fmt_exact_single_rounding(bits):
    """Near-tie (acc, scale, shift) around half-integers of the whole unsigned
    range [0, 2^b - 1], against exact rationals with one rounding (reading 5)."""
    g = np.random.default_rng(1600 + bits)
    hi = (1 << bits) - 1
    acc, sc, sh = exact_fp.near_tie_cases(g, 8000, bits, k_lo=-2, k_hi=hi + 1)
    K = acc.size
    y = oracle.requant_fmt(acc.astype(np.int32).reshape(1, K), np.concatenate([sc, sh]), True, bits, True)
    got = oracle.unpack_fmt(y, K, bits, True)[0]
    ref = np.array([exact_fp.requant_exact(int(a), float(s), float(h), True, bits, uns=True)
                    for a, s, h in zip(acc, sc, sh)])
    assert np.array_equal(got, ref), np.nonzero(got != ref)[0][:5]
    assert np.count_nonzero(ref > (hi >> 1)) > K // 4     # the upper half of the range is exercised


def test_requant_res_fmt_unit_scales():
    """scale = res_scale = 1, shift 0: y = clamp(acc + skip) with the skip read in
    its own format and y clamped to the output format."""
    for acc in range(-300, 301, 11):
        for sk in range(0, 256, 7):
            skb = np.array([[sk]], np.uint8)
            y = oracle.requant_fmt(np.array([[acc]], np.int32), np.array([1.0, 0.0], np.float32), True, 8, True,
                                   skip=skb, skip_uns=True, res_scale=1.0)
            assert int(y[0, 0]) == min(max(acc + sk, 0), 255)
            s_signed = sk - 256 if sk >= 128 else sk
            y = oracle.requant_fmt(np.array([[acc]], np.int32), np.array([1.0, 0.0], np.float32), True, 8, True,
                                   skip=skb, skip_uns=False, res_scale=1.0)
            assert int(y[0, 0]) == min(max(acc + s_signed, 0), 255)
            assert oracle.requant_res_value_fmt(acc, 1.0, 0.0, sk, 1.0, True, 8, True) == min(max(acc + sk, 0), 255)


def test_requant_res_fmt_exact():
    g = np.random.default_rng(1615)
    acc, sc, sh = exact_fp.near_tie_cases(g, 4000, 8, k_lo=0, k_hi=255)
    sk = g.integers(0, 256, acc.size)
    rs = float(np.float32(0.37))
    K = acc.size
    y = oracle.requant_fmt(acc.astype(np.int32).reshape(1, K), np.concatenate([sc, sh]), True, 8, True,
                           skip=sk.astype(np.uint8).reshape(1, K), skip_uns=True, res_scale=rs)
    got = oracle.unpack_fmt(y, K, 8, True)[0]
    ref = np.array([exact_fp.requant_res_exact(int(a), float(s), float(h), int(k), rs, True, 8, uns=True)
                    for a, s, h, k in zip(acc, sc, sh, sk)])
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- max pool over unsigned codes
@pytest.mark.parametrize("bits", [8, 4])
def test_maxpool_unsigned_matches_torch(bits):
    g = np.random.default_rng(91 + bits)
    N, H, W, C = 2, 9, 8, 64
    x = wl.random_bytes(g, (N, H, W, C * bits // 8))
    got = oracle.maxpool(x, C, 3, 2, 1, bits, uns=True)
    xt = torch.from_numpy(oracle.unpack_fmt(x, C, bits, True).astype(np.float64)).permute(0, 3, 1, 2)
    ref = torch.nn.functional.max_pool2d(xt, 3, 2, 1).permute(0, 2, 3, 1).numpy().astype(np.int64)
    assert np.array_equal(oracle.unpack_fmt(got, C, bits, True), ref)
    # a plausible mistake -- comparing the bytes as signed -- gives another result here
    assert not np.array_equal(got, oracle.maxpool(x, C, 3, 2, 1, bits))
