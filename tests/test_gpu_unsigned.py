"""Unsigned post-ReLU code formats on the GPU (-m gpu; DESIGN reading 16,
SURVEY 8(f) NEXT-2): conv_q_plan_set_formats / conv_q_maxpool_fmt against the
oracle's *_fmt functions (pinned in tests/test_oracle_unsigned.py), bit-exact.

* every candidate of representative shapes (3x3 halo / weight-stationary / MT2,
  1x1, strided, split-K, CTA pairs) with unsigned activations in and unsigned
  (u8 / u4) codes out, batch large enough for several work units per CTA;
* the mixed cases: unsigned input with signed output (no ReLU), signed input
  with unsigned output, raw s32 accumulators of unsigned activations;
* the residual epilogue with an unsigned or a signed skip into unsigned codes;
* unsigned max pooling;
* the bench chains with unsigned activations end to end.
"""
import numpy as np
import pytest

import oracle
import workloads as wl
from oracle import check

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cq():
    import paper_2202_06819_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


R50 = dict((l.name, l) for l, _ in wl.resnet50_layers())
SHAPES = [(R50["l1.b0.c2"], 16, 8), (R50["l3.b1.c3"], 16, 8), (R50["l2.b0.c2"], 8, 8), (R50["l4.b1.c1"], 16, 8),
          (wl.CFG1, 1, 8), (R50["l1.b0.c2"], 8, 4), (R50["l3.b1.c2"], 8, 4), (wl.CFG1, 1, 4)]


@pytest.mark.parametrize("L,N,bits", SHAPES)
def test_unsigned_every_candidate(cq, L, N, bits):
    """x unsigned -> y unsigned (the post-ReLU chain format): every candidate,
    packed codes and raw s32 accumulators."""
    g = wl.rng(16, L.K + N + bits)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    pix = check.sample_pixels(N, L.P, L.Q, g, 256)
    ref32 = oracle.conv_s32(x, w, L.C, L.stride, L.pad, bits, pix=pix, x_uns=True)
    refq = oracle.requant_fmt(ref32, ss, True, bits, True)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True, x_uns=True, y_uns=True)
    M = N * L.P * L.Q
    xd, wd, sd = dev(x), dev(w), dev(ss)
    y = torch.empty((M, L.K * bits // 8), dtype=torch.uint8, device="cuda")
    y32 = torch.empty((M, L.K), dtype=torch.int32, device="cuda")
    for ci, name in enumerate(plan.candidates()):
        plan.set_config(ci)
        plan.set_epilogue(True, cq.OUT_PACKED)
        y.fill_(0xA5)
        plan.run(xd, wd, sd, y)
        plan.set_epilogue(True, cq.OUT_S32)
        y32.fill_(-7777777)
        plan.run(xd, wd, sd, y32)
        torch.cuda.synchronize()
        got = y.cpu().numpy()[pix]
        assert np.array_equal(got, refq), (name, check.first_diff(got, refq))
        assert np.array_equal(y32.cpu().numpy()[pix], ref32), name


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("x_uns,y_uns,relu", [(True, False, False), (True, False, True), (False, True, False),
                                              (False, True, True)])
def test_mixed_formats(cq, bits, x_uns, y_uns, relu):
    L, N = R50["l2.b1.c2"], 4
    g = wl.rng(17, int(x_uns) + 2 * int(y_uns) + 4 * int(relu) + bits)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    pix = check.sample_pixels(N, L.P, L.Q, g, 256)
    ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, relu, pix=pix, x_uns=x_uns, y_uns=y_uns)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=relu, x_uns=x_uns, y_uns=y_uns)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
    for ci, name in enumerate(plan.candidates()):
        plan.set_config(ci)
        y.fill_(0x3C)
        plan.run(xd, wd, sd, y)
        torch.cuda.synchronize()
        got = y.cpu().numpy()[pix]
        assert np.array_equal(got, ref), (name, check.first_diff(got, ref))


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("skip_uns", [True, False])
def test_residual_unsigned(cq, bits, skip_uns):
    """Residual epilogue into unsigned codes, the skip read in its own format,
    every candidate."""
    for L, N in ((R50["l1.b0.c3"], 4), (wl.Layer("k3", 14, 14, 256, 256, 3, 3, 1, 1), 4)):
        g = wl.rng(18, L.K + bits + int(skip_uns))
        x, w, ss = wl.layer_inputs(g, L, N, bits)
        skip = wl.random_bytes(g, (N, L.P, L.Q, L.K * bits // 8))
        rs = wl.res_scale(g)
        pix = check.sample_pixels(N, L.P, L.Q, g, 256)
        ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, True, pix=pix, skip=skip, res_scale=rs,
                            x_uns=True, y_uns=True, skip_uns=skip_uns)
        plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
        plan.set_formats(True, True, skip_uns)
        xd, wd, sd, kd = dev(x), dev(w), dev(ss), dev(skip)
        plan.set_residual(kd, rs)
        y = torch.empty((N * L.P * L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
        for ci, name in enumerate(plan.candidates()):
            plan.set_config(ci)
            y.fill_(0x5A)
            plan.run(xd, wd, sd, y)
            torch.cuda.synchronize()
            got = y.cpu().numpy()[pix]
            assert np.array_equal(got, ref), (L.name, name, check.first_diff(got, ref))


@pytest.mark.parametrize("bits", [8, 4])
def test_maxpool_unsigned(cq, bits):
    g = np.random.default_rng(900 + bits)
    for N, H, W, C in ((2, 112, 112, 64), (3, 9, 7, 32)):
        x = wl.random_bytes(g, (N, H, W, C * bits // 8))
        got = cq.maxpool(dev(x), C, 3, 2, 1, bits, uns=True).cpu().numpy()
        ref = oracle.maxpool(x, C, 3, 2, 1, bits, uns=True)
        assert np.array_equal(got, ref), check.first_diff(got, ref)


def test_unsigned_overflow_guard(cq):
    """R*S*C*255*128 > 2^31 - 1 -> EOVERFLOW for unsigned activations; the same
    shape is accepted with signed ones (R*S*C*2^14 fits)."""
    plan = cq.ConvPlan(1, 3, 3, 8192, 128, 3, 3, 1, 1, 8)
    Kg = 9 * 8192
    assert Kg * 128 * 128 <= 2**31 - 1 < Kg * 255 * 128
    with pytest.raises(cq.ConvQError):
        plan.set_formats(True, False)


@pytest.mark.parametrize("workload", ["resnet50_int8_b256_uns", "resnet18_int4_b16_uns", "resnet18_int8_b1_uns",
                                      "resnet50_int8_b256_res_uns", "resnet18_int4_b16_res_uns"])
def test_bench_chain_unsigned(cq, workload):
    """The bench chains with unsigned post-ReLU codes (stem output, pool, every
    conv in and out, residual skips), tuned as the bench tunes, sampled parity
    of every launch against the oracle."""
    from test_gpu_network import test_bench_chain_parity
    test_bench_chain_parity(cq, workload)
