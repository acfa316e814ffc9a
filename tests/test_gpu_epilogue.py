"""The INT8 epilogue's two s32 -> f32 conversions (-m gpu): I2FP, and IADD +
FADD2 (conv.cuh i2f2_small) for layers whose accumulators provably stay within
2^22 (R*S*C*max|x|*max|w| <= 2^22, plan.cuh).  Both must give the oracle's bytes
(reading 5: s32 -> f32 RN, one FMA, RNE) -- at the boundary accumulators
+-2^22, at every candidate, signed and unsigned activations, and next to a
layer just past the guard (I2FP)."""
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


def _extreme_inputs(g, N, H, W, C, K, x_uns):
    """Codes at the extremes (plus a random share) so accumulators reach +-2^22."""
    lo = 0 if x_uns else -128
    hi = 255 if x_uns else 127
    x = g.choice(np.array([lo, hi, lo, lo], np.int64), size=(N, H, W, C))
    x[0, 0, 0, :] = lo if not x_uns else hi                    # one pixel all extreme
    x[..., : C // 8] = g.integers(lo, hi + 1, size=x[..., : C // 8].shape)
    w = g.choice(np.array([-128, 127, -128], np.int64), size=(K, 1, 1, C))
    w[0] = -128                                                  # channel 0 all -128: acc = C*lo*-128
    w[1] = 127
    w[2:8] = g.integers(-128, 128, size=w[2:8].shape)
    xb = (x.astype(np.int64) & 0xFF).astype(np.uint8)
    wb = (w.astype(np.int64) & 0xFF).astype(np.uint8)
    acc = np.einsum("nhwc,kc->nhwk", x, w[:, 0, 0, :])
    return xb, wb, acc


@pytest.mark.parametrize("C,x_uns,magic", [(256, False, True), (128, True, True), (288, False, False),
                                           (160, True, False), (64, False, True)])
def test_conversion_boundary_every_candidate(cq, C, x_uns, magic):
    N, H, W, K = 2, 9, 7, 128
    g = np.random.default_rng(2200 + C)
    x, w, acc = _extreme_inputs(g, N, H, W, C, K, x_uns)
    bound = C * (255 if x_uns else 128) * 128
    assert (bound <= 1 << 22) == magic
    if magic:
        assert np.abs(acc).max() <= 1 << 22
    if C == 256 and not x_uns:
        assert np.abs(acc).max() == 1 << 22                      # the boundary itself is exercised
    # scales that keep the codes mostly unsaturated, fractional products (ties exercised)
    sc = (2.0 ** -15 * (1 + g.integers(0, 64, K) / 64.0)).astype(np.float32)
    sh = g.uniform(-2, 2, K).astype(np.float32)
    sh[::7] = 0.5
    ss = np.concatenate([sc, sh]).astype(np.float32)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    for relu in (False, True):
        plan = cq.ConvPlan(N, H, W, C, K, 1, 1, 1, 0, 8, relu=relu)
        plan.set_formats(x_uns=x_uns)
        ref = oracle.requant(acc.astype(np.int32), ss, relu, 8)
        for ci, name in enumerate(plan.candidates()):
            plan.set_config(ci)
            y = torch.full((N, H, W, K), 0xA5, dtype=torch.uint8, device="cuda")
            plan.run(xd, wd, sd, y)
            torch.cuda.synchronize()
            got = y.cpu().numpy()
            assert np.array_equal(got, ref), (C, x_uns, relu, name, check.first_diff(got, ref))
