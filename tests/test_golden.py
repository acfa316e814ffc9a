"""The oracle against values printed in the paper / its spec (tests/golden/,
each entry with its citation).  CPU only."""
import json
import math
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_values.json")
G = json.load(open(GOLDEN))


def test_table1_ops_every_stage():
    """PAPER.md:323 Table 1: 2 * N * P * Q * K * C * R * S = 1,849,688,064 at N = 8 for stages 2-5,
    with P, Q from the oracle's output-size rule (reading 6)."""
    t = G["table1"]
    for s in t["stages"]:
        P, Q = oracle.out_dim(s["H"], 3, 1, 1), oracle.out_dim(s["W"], 3, 1, 1)
        assert (P, Q) == (s["H"], s["W"])
        assert 2 * t["N"] * P * Q * s["K"] * s["C"] * 9 == t["ops"]
    # the paper's speed-up row is baseline / searched (context only: T4 numbers)
    for s in t["stages"]:
        assert f"{s['baseline_us'] / s['searched_us']:.2f}x" == s["speedup"]


def test_accumulator_bits():
    """16 bits for INT4 x INT4 x 128 terms; ~1e6 channels saturate s32 (3x3)."""
    a = G["accumulator_bits"]
    assert math.ceil(math.log2(16 * 16 * 128)) + 1 == a["int4_128ch_bits"]
    c = a["int4_3x3_channels_to_saturate_32bit"]
    assert 16 * 16 * 9 * c >= 2 ** 31 > 16 * 16 * 9 * (c - 1)
    # the oracle's conv reaches the bound exactly: all -8 codes, C = 128 -> 2^4*2^4*... = 8*8*9*128
    C = 128
    x = oracle.pack(np.full((1, 3, 3, C), -8, np.int8), 4).reshape(1, 3, 3, C // 2)
    w = oracle.pack(np.full((1, 3, 3, C), -8, np.int8), 4).reshape(1, 3, 3, C // 2)
    y = oracle.conv_s32(x, w, C, 1, 0, 4)
    assert int(y[0, 0, 0, 0]) == 64 * 9 * C


def test_pack_int4_words():
    """SPEC.md:226,235-237 (section 3.2.3 Fig. 9)."""
    p = G["pack_int4"]
    w = oracle.pack(np.array(p["codes"], np.int8), 4)
    # code 8 does not fit a signed nibble: the spec's example packs raw nibbles; 8 == -8 mod 16
    assert int(w.view("<u4")[0]) == p["word"]
    assert list(oracle.unpack(np.frombuffer(np.uint32(p["all_ones_word"]).tobytes(), np.uint8), 8, 4)) == \
        [p["all_ones_signed"]] * 8


def test_duplicate_structure_4x4_3x3():
    """SPEC.md:76 (Alg. 1): 144 cells, 100 valid, 16 genuine, 84 duplicates, 44 pad --
    measured through the oracle's conv: one-hot inputs count the taps that reference each pixel."""
    d = G["duplicates_4x4_3x3"]
    H, W, R, S = d["H"], d["W"], d["R"], d["S"]
    C = 16
    P, Q = oracle.out_dim(H, R, d["stride"], d["pad"]), oracle.out_dim(W, S, d["stride"], d["pad"])
    assert P * Q * R * S == d["cells"]
    w = np.zeros((1, R, S, C), np.int8)
    w[..., 0] = 1
    refs = 0
    genuine = 0
    for h in range(H):
        for ww in range(W):
            x = np.zeros((1, H, W, C), np.int8)
            x[0, h, ww, 0] = 1
            y = oracle.conv_s32(x.view(np.uint8), w.view(np.uint8), C, d["stride"], d["pad"], 8)
            n = int(y.sum())          # taps (output pixel, filter tap) that read input pixel (h, ww)
            refs += n
            genuine += n > 0
    assert refs == d["valid"]
    assert genuine == d["genuine"]
    assert refs - genuine == d["duplicates"]
    assert d["cells"] - refs == d["pad_cells"]


def test_requant_ties():
    """SURVEY 8(c) closed form: RNE ties at scale 0.5."""
    r = G["requant_ties"]
    K = len(r["acc"])
    ss = np.concatenate([np.full(K, r["scale"], np.float32), np.full(K, r["shift"], np.float32)])
    y = oracle.requant(np.array([r["acc"]], np.int32), ss, False, 8)
    assert list(oracle.unpack(y, K, 8)[0]) == r["y"]
