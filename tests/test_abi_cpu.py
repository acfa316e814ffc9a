"""Host-side tests of the C ABI (no GPU needed): the library loads, exports
every symbol include/convq.h declares, validates shapes with the documented
error codes, and refuses to compute without a CUDA device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

import paper_2202_06819_b200 as cq
from paper_2202_06819_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return cq.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "convq.h")).read()
    return sorted(set(re.findall(r"CONVQ_API[^;(]*?\b(conv_q_\w+)\s*\(", src)))


def test_header_declares_the_paper_entry_points():
    syms = header_symbols()
    for s in ("conv_q_plan", "conv_q_run", "conv_q_quantize", "conv_q_pack_weights", "conv_q_plan_tune",
              "conv_q_plan_info", "conv_q_plan_destroy", "conv_q_last_error"):
        assert s in syms
    assert len(syms) >= 16


def test_library_exports_every_header_symbol(lib):
    for s in header_symbols():
        assert hasattr(lib, s), s
    out = os.popen(f"nm -D --defined-only {cq.LIB_PATH}").read()
    exported = set(re.findall(r" T (conv_q_\w+)", out))
    assert set(header_symbols()) <= exported
    assert lib.conv_q_version() == 106


@pytest.mark.parametrize("args,code", [
    ((0, 56, 56, 64, 64, 3, 3, 1, 1, 8), cq.EINVAL),      # N < 1
    ((1, 56, 56, 64, 64, 3, 3, 0, 1, 8), cq.EINVAL),      # stride 0
    ((1, 56, 56, 64, 64, 3, 3, 9, 1, 8), cq.EINVAL),      # stride > 8 (TMA traversal stride)
    ((1, 56, 56, 64, 64, 3, 3, 1, 128, 8), cq.EINVAL),    # pad > 127
    ((1, 56, 56, 64, 64, 3, 3, 1, 1, 5), cq.EINVAL),      # bits
    ((1, 2, 2, 64, 64, 5, 5, 1, 0, 8), cq.EINVAL),        # empty output
    ((1, 56, 56, 24, 64, 3, 3, 1, 1, 8), cq.EUNSUPPORTED),  # C*bits not multiple of 128
    ((1, 56, 56, 64, 40, 3, 3, 1, 1, 4), cq.EUNSUPPORTED),  # K*bits not multiple of 128
    ((1, 56, 56, 16, 64, 3, 3, 1, 1, 8), cq.EUNSUPPORTED),  # s8 C < 32 (pad with quantize)
    ((1, 8, 8, 16384, 64, 3, 3, 1, 1, 8), cq.EOVERFLOW),  # R*S*C*2^14 > 2^31-1
])
def test_plan_validation_codes(lib, args, code):
    with pytest.raises(cq.ConvQError) as ei:
        cq.ConvPlan(*args)
    assert ei.value.code == code
    assert lib.conv_q_last_status() == code
    assert lib.conv_q_last_error()


def test_overflow_guard_boundary(lib):
    """Kg*2^14 <= 2^31-1  <=>  Kg <= 131071 (PAPER.md:166 s3.2.1 bound, exact form)."""
    cq.ConvPlan(1, 4, 4, 14560, 16, 3, 3, 1, 1, 8)          # Kg = 131040: accepted
    with pytest.raises(cq.ConvQError) as ei:
        cq.ConvPlan(1, 4, 4, 14592, 16, 3, 3, 1, 1, 8)      # Kg = 131328: rejected
    assert ei.value.code == cq.EOVERFLOW


def test_plan_info_gemm_view(lib):
    """PAPER.md:56 (N*H*W, I*R*S) x (I*R*S, O); floor output size for stride 2."""
    p = cq.ConvPlan(8, 56, 56, 64, 64, 3, 3, 1, 1, 8)
    i = p.info()
    assert (i.P, i.Q, i.M, i.Kg) == (56, 56, 25088, 576)
    assert 2 * i.macs == 1849688064                                  # PAPER.md:323 Table 1 OPs
    assert i.x_bytes == 8 * 56 * 56 * 64 and i.y_bytes == 25088 * 64
    q = cq.ConvPlan(1, 56, 56, 64, 128, 3, 3, 2, 1, 4)
    assert (q.info().P, q.info().Q) == (28, 28)
    assert q.info().y_bytes == 28 * 28 * 64
    assert i.num_candidates >= 1 and i.config.startswith("bm128_")
    assert p.candidates()[i.config_index] == i.config


def test_stem_s2d_plan_geometry(lib):
    """ResNet conv1 7x7/2 p3 over 224x224x3 as a stride-1 conv over the s2d view:
    same P, Q and output bytes as the direct conv; 4 s2d tap rows x one 64-byte
    window (4 s2d pixels x 16 B) per row -> Kg = 4*64 (vs 49*32 = 1568 with
    C padded to 32); the s2d tensor holds Q+3 stored columns."""
    p = cq.StemPlan(256, 224, 224, 3, 64, 7, 7, 3, 8)
    i = p.info()
    assert (i.H, i.W, i.C, i.R, i.S, i.stride, i.pad) == (224, 224, 3, 7, 7, 2, 3) and i.s2d == 1
    assert (i.P, i.Q, i.M) == (112, 112, 256 * 112 * 112)
    assert i.Kg == 4 * 64 and i.y_bytes == 256 * 112 * 112 * 64
    assert i.x_dims == (256, 112, 115, 16) and i.w_dims == (64, 4, 1, 64)
    assert i.x_bytes == 256 * 112 * 115 * 16
    assert p.macs == 256 * 112 * 112 * 64 * 7 * 7 * 3                     # useful MACs
    q = cq.StemPlan(16, 224, 224, 3, 64, 7, 7, 3, 4)                       # INT4: 8 nibbles per phase
    assert q.info().w_dims == (64, 4, 1, 64) and q.info().Kg == 4 * 128
    r = cq.StemPlan(1, 33, 29, 3, 32, 3, 3, 1, 8)                          # odd sizes, 3x3/2 p1
    assert (r.info().P, r.info().Q) == (17, 15)
    assert r.info().w_dims == (32, 2, 1, 32) and r.info().x_dims == (1, 17, 16, 16)
    for args, code in (((1, 224, 224, 5, 64, 7, 7, 3, 8), cq.EUNSUPPORTED),   # C > 4 channels per phase (s8)
                       ((1, 224, 224, 3, 40, 7, 7, 3, 8), cq.EUNSUPPORTED),   # K*bits % 128
                       ((1, 224, 224, 3, 64, 19, 19, 9, 8), cq.EUNSUPPORTED),  # > 8 s2d taps in W
                       ((0, 224, 224, 3, 64, 7, 7, 3, 8), cq.EINVAL)):
        with pytest.raises(cq.ConvQError) as ei:
            cq.StemPlan(*args)
        assert ei.value.code == code, args
    i0 = cq.ConvPlan(1, 8, 8, 64, 64, 3, 3, 1, 1, 8).info()
    assert i0.s2d == 0 and i0.x_dims == (1, 8, 8, 64) and i0.w_dims == (64, 3, 3, 64)
    # the only duplicate-aware candidates of an s2d plan are its window-halo ones
    # (a regular halo box over the stored s2d tensor would not match the kernel's
    # TMA byte count -- a round-2 regression that hung a GPU test)
    for plan in (p, q, r):
        assert all("_h_w" in n for n in plan.candidates() if "_h" in n), plan.candidates()


def test_candidates_and_selection(lib):
    p = cq.ConvPlan(32, 14, 14, 256, 256, 3, 3, 1, 1, 8)
    names = p.candidates()
    assert len(names) == len(set(names)) >= 3
    p.set_config(len(names) - 1)
    assert p.info().config == names[-1]
    with pytest.raises(cq.ConvQError):
        p.set_config(len(names))


def test_padded_channels(lib):
    assert cq.padded_channels(3, 8) == 32 and cq.padded_channels(3, 4) == 32
    assert cq.padded_channels(64, 8) == 64 and cq.padded_channels(65, 4) == 96


def test_epilogue_args(lib):
    p = cq.ConvPlan(1, 8, 8, 64, 64, 1, 1, 1, 0, 8)
    p.set_epilogue(True, cq.OUT_S32)
    assert p.info().relu == 1 and p.info().out_mode == cq.OUT_S32
    with pytest.raises(cq.ConvQError):
        p.set_epilogue(True, 7)


def test_no_cpu_fallback(lib):
    """Without a device every compute entry point fails loudly (ECUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    p = cq.ConvPlan(1, 8, 8, 64, 64, 1, 1, 1, 0, 8)
    buf = ctypes.create_string_buffer(1 << 16)
    addr = (ctypes.addressof(buf) + 15) // 16 * 16
    rc = lib.conv_q_run(p._h, ctypes.c_void_p(addr), ctypes.c_void_p(addr), ctypes.c_void_p(addr),
                        ctypes.c_void_p(addr), )
    assert rc == cq.ECUDA
    assert lib.conv_q_quantize(ctypes.c_void_p(addr), 1, 1, 1, 64, ctypes.c_float(1.0), 8,
                               ctypes.c_void_p(addr), None) == cq.ECUDA
    assert lib.conv_q_run(p._h, None, ctypes.c_void_p(addr), ctypes.c_void_p(addr),
                          ctypes.c_void_p(addr)) == cq.EINVAL
    assert lib.conv_q_run(p._h, ctypes.c_void_p(addr + 4), ctypes.c_void_p(addr), ctypes.c_void_p(addr),
                          ctypes.c_void_p(addr)) == cq.EINVAL


def test_fastdiv_constants_exact():
    """The kernels' control loops divide by per-launch constants with
    q = (umulhi(n, m) + n) >> s, s = ceil(log2 d), m = floor(2^32 (2^s - d)/d) + 1
    (plan.cuh make_fastdiv).  Exact for every 0 <= n < 2^31 at the boundaries
    that can fail (multiples of d and their neighbours, the top of the range)."""
    import random
    rnd = random.Random(6819)
    ds = list(range(1, 2100)) + [rnd.randrange(1, 2 ** 31) for _ in range(2000)] + \
        [2 ** k + e for k in range(31) for e in (-1, 0, 1) if 2 ** k + e >= 1]
    for d in ds:
        s = (d - 1).bit_length()
        m = ((1 << 32) * ((1 << s) - d)) // d + 1
        assert m < 1 << 32
        top = (2 ** 31 - 1) // d * d
        for n in {0, 1, d - 1, d, d + 1, 2 ** 31 - 1, top, top - 1, rnd.randrange(0, 2 ** 31)}:
            if 0 <= n < 2 ** 31:
                assert (((n * m) >> 32) + n) >> s == n // d, (d, n)


def test_plan_ragged_channel_block_s8(lib):
    """s8 needs only C*8 % 128 == 0 -- C = 16 (mod 32) is accepted (C >= 32):
    im2col / tiled candidates whose k-block is narrower than C; the last block of each tap
    reads zero-filled channels (no halo / weight-stationary candidates)."""
    for C in (48, 80, 112):
        p = cq.ConvPlan(2, 9, 11, C, 64, 3, 3, 1, 1, 8)
        names = p.candidates()
        assert names and all("_h" not in n and "_w" not in n for n in names)
        assert all(int(n.split("_kc")[1].split("x")[0]) < C for n in names)
    with pytest.raises(cq.ConvQError) as ei:      # s4: C*4 = 192 is not a multiple of 128
        cq.ConvPlan(1, 8, 8, 48, 64, 3, 3, 1, 1, 4)
    assert ei.value.code == cq.EUNSUPPORTED
