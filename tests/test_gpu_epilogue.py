"""The INT8 epilogue's s32 -> f32 -> requant at extreme accumulators (-m gpu):
1x1 layers whose codes sit at the range ends so the accumulators reach
+-2^22 (C = 256 signed: every |acc| <= 2^22 with equality), beyond 2^22, and
with unsigned activations -- every candidate, ReLU on and off, against the
oracle's bytes (reading 5: s32 -> f32 RN, one FMA, RNE).

(An IADD + FADD2 conversion, exact for |acc| <= 2^22, was measured as a
replacement for I2FP on such layers: slower -- DESIGN.md negative results.)"""
import numpy as np
import pytest

import oracle
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
    """Codes at the extremes (plus random pixels) so accumulators reach the bound."""
    lo, hi = (0, 255) if x_uns else (-128, 127)
    x = g.choice(np.array([lo, hi, lo, lo], np.int64), size=(N, H, W, C))
    x[:, 1:3] = g.integers(lo, hi + 1, size=x[:, 1:3].shape)       # two random rows
    x[0, 0, 0, :] = hi if x_uns else lo                           # one pixel all extreme
    w = g.choice(np.array([-128, 127, -128], np.int64), size=(K, C))
    w[0] = -128                                                   # channel 0: acc = C * x * -128
    w[1] = 127
    w[2:8] = g.integers(-128, 128, size=w[2:8].shape)
    xb = (x & 0xFF).astype(np.uint8)
    wb = (w & 0xFF).astype(np.uint8).reshape(K, 1, 1, C)
    acc = np.einsum("nhwc,kc->nhwk", x, w)                        # 1x1 conv == explicit GEMM
    return xb, wb, acc


@pytest.mark.parametrize("C,x_uns", [(256, False), (128, True), (288, False), (160, True), (64, False)])
def test_extreme_accumulators_every_candidate(cq, C, x_uns):
    N, H, W, K = 2, 9, 7, 128
    g = np.random.default_rng(2200 + C)
    x, w, acc = _extreme_inputs(g, N, H, W, C, K, x_uns)
    amax = int(np.abs(acc).max())
    assert amax == C * (255 if x_uns else 128) * 128              # the layer's bound itself is reached
    if C == 256 and not x_uns:
        assert amax == 1 << 22
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
