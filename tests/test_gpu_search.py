"""NEXT-4 on the device: every point of the plan's enlarged schedule space
(conv_q_plan_space: TileConfig x split-K x epilogue wait x L2 policy x
rotation x grid) computes the same bytes as the oracle, and the learned search
(conv_q_plan_search, PAPER.md:282-298 / 309-314) leaves the plan on a
correct, faster-or-equal point.  -m gpu."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cq():
    import paper_2202_06819_b200 as m
    m.load()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _setup(L, N, bits, seed, relu=True):
    g = np.random.default_rng(seed)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, relu)
    return x, w, ss, ref


def _valid_points(cq, plan, sizes, k, seed):
    """k random valid points (set_point accepts them), covering the new split values."""
    g = np.random.default_rng(seed)
    pts = []
    tries = 0
    while len(pts) < k and tries < 20000:
        tries += 1
        pt = [int(g.integers(s)) for s in sizes]
        if len(pts) < k // 3:
            pt[5] = int(g.choice([2, 4]))   # split 3 / 6 -- not in the enumerated list
        try:
            plan.set_point(pt)
        except cq.ConvQError:
            continue
        pts.append(pt)
    return pts


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("L,N", [
    (wl.Layer("t1.stage3", 28, 28, 128, 128, 3, 3, 1, 1), 2),   # Table 1 stage-3 shape, halo / WS / pairs
    (wl.Layer("l4.c1", 7, 7, 2048, 512, 1, 1, 1, 0), 2),         # K-deep 1x1: split-K 3 / 6 / 8
    (wl.Layer("l2.ds", 20, 20, 256, 512, 1, 1, 2, 0), 1),       # strided 1x1, ragged M
])
def test_random_space_points_parity(cq, bits, L, N):
    x, w, ss, ref = _setup(L, N, bits, 4242 + bits)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    sizes, nvalid = plan.space()
    assert nvalid > 0
    xd, wd, sd = dev(x), dev(w), dev(ss)
    for pt in _valid_points(cq, plan, sizes, 24, 99 + bits):
        plan.set_point(pt)
        for rep in range(2):   # split-K workspaces must be left zero by each run
            y = torch.full((N, L.P, L.Q, L.K * bits // 8), 0xA5, dtype=torch.uint8, device="cuda")
            plan.run(xd, wd, sd, y)
            torch.cuda.synchronize()
            got = y.cpu().numpy()
            assert np.array_equal(got, ref), (L.name, bits, pt, plan.info().config, rep)


@pytest.mark.parametrize("bits", [8, 4])
def test_search_selects_correct_point(cq, bits):
    """conv_q_plan_search over cfg1-at-N=8 (Table 1 stage 2): the selected point
    is bit-exact, its time is the minimum of the history, and the search
    measured only distinct points."""
    L = wl.paper_table1_layers()[0]
    N = 8
    x, w, ss, ref = _setup(L, N, bits, 31 + bits)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    y = torch.empty((N, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device="cuda")
    r = plan.search(xd, wd, sd, y, warmup=1, reps=5, trials=48, batch=16, seed=3)
    h = [t for t in r["history_us"] if t > 0]
    assert len(r["history_us"]) == 48 and h
    assert abs(r["best_us"] - min(h)) < 1e-3
    info = plan.info()
    assert info.config == r["config"] and info.tuned_us > 0
    y.fill_(0xA5)
    plan.run(xd, wd, sd, y)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), ref), r["config"]
    # the pick copies to another plan of the shape (what the network does for repeated layers)
    other = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    other.set_point(plan.get_point())
    assert other.info().config == r["config"]
    y.fill_(0xA5)
    other.run(xd, wd, sd, y)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), ref), r["config"]


@pytest.mark.parametrize("bits", [8, 4])
def test_stem_space_points_parity(cq, bits):
    """Random points of the s2d stem plan's space (window-halo / im2col TileConfigs x
    runtime knobs) against the oracle's direct stride-2 conv on the channel-padded image."""
    N, H, W, C, K, R, S, pad = 2, 30, 40, 3, 64, 7, 7, 3
    g = np.random.default_rng(606 + bits)
    x = (g.standard_normal((N, H, W, C)) * 2).astype(np.float16)
    inv = 127 / 4 if bits == 8 else 7 / 3
    wv = wl.weight_values(g, K, R, S, C, bits)
    Cp = oracle.padded_channels(C, bits)
    w_pad = np.zeros((K, R, S, Cp), dtype=np.int8)
    w_pad[..., :C] = wv
    ss = wl.scale_shift(g, K, R * S * C, 40.0 if bits == 8 else 3.0, wl.uniform_code_std(bits), bits)
    ref = oracle.requant(oracle.conv_s32(oracle.quantize(x, inv, bits), oracle.pack(w_pad, bits), Cp, 2, pad, bits),
                         ss, True, bits)
    plan = cq.StemPlan(N, H, W, C, K, R, S, pad, bits, relu=True)
    xs = plan.quantize(dev(x), inv)
    wp = plan.pack_weights(dev(wv))
    sd = dev(ss)
    sizes, nvalid = plan.space()
    assert nvalid > 0
    for pt in _valid_points(cq, plan, sizes, 16, 808 + bits):
        plan.set_point(pt)
        y = torch.full((N, plan.P, plan.Q, K * bits // 8), 0xA5, dtype=torch.uint8, device="cuda")
        plan.run(xs, wp, sd, y)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), ref), (bits, pt, plan.info().config)
