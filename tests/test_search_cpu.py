"""NEXT-4: the learned, diversity-aware schedule search engine
(csrc/search.cpp, section 3.4 with the settings of
PAPER.md:309-314) driven through the C ABI with synthetic cost functions --
host only, no GPU.  The device leg (conv_q_plan_search) is in
tests/test_gpu_search.py.

Search-quality bar after SPEC.md:607 (the spec's desk-scale substitute for
Table 1): on a noise-free synthetic cost the search reaches within 5 % of the
exhaustive optimum in >= 18 of 20 seeds."""
import itertools
import math

import numpy as np
import pytest

import paper_2202_06819_b200 as cq

# the shape of conv_q_plan_space: BN, k-block, CTAs, mode, output path, split,
# epilogue wait, L2 policy, rotation, grid
SIZES = [3, 4, 2, 4, 2, 6, 3, 3, 2, 3]


def _synthetic(seed):
    """A noise-free cost over SIZES: log-cost additive in per-knob and a few
    pairwise terms (like tile shape x split interactions), an invalid region,
    and one narrow good corner."""
    g = np.random.default_rng(seed)
    unary = [g.uniform(0.0, 0.35, s) for s in SIZES]
    pairs = {(0, 5): g.uniform(0.0, 0.4, (3, 6)), (1, 3): g.uniform(0.0, 0.3, (4, 4)),
             (2, 9): g.uniform(0.0, 0.3, (2, 3)), (3, 4): g.uniform(0.0, 0.25, (4, 2))}

    def valid(k):
        return not (k[3] >= 2 and k[5] > 0) and not (k[3] >= 2 and k[8] == 1)   # "split / rotation only plain"

    def cost(k):
        v = sum(unary[i][k[i]] for i in range(len(SIZES)))
        v += sum(t[k[a], k[b]] for (a, b), t in pairs.items())
        return 10.0 * math.exp(v)

    pts = [k for k in itertools.product(*[range(s) for s in SIZES]) if valid(k)]
    best = min(cost(k) for k in pts)
    return cost, valid, best, len(pts)


def test_space_is_large_enough_to_need_search():
    _, _, _, n = _synthetic(0)
    assert n > 20000   # exhaustive device timing of every point is out of reach (>~200)


@pytest.mark.parametrize("diversity", [1, 0])
def test_reaches_exhaustive_optimum(diversity):
    """>= 18/20 seeds within 5 % of the exhaustive optimum in 128 measurements
    (0.2 % of the 50k-point space)."""
    hits = 0
    for seed in range(20):
        cost, valid, best, _ = _synthetic(100 + seed)
        r = cq.search(SIZES, cost, valid, trials=128, seed=seed, diversity=diversity)
        assert r["n"] == 128
        hits += min(r["history_cost"]) <= 1.05 * best
    assert hits >= 18, hits


def test_learned_beats_random_sampling():
    """The model-guided batches beat the same number of uniformly random valid points."""
    wins = 0
    for seed in range(10):
        cost, valid, best, _ = _synthetic(200 + seed)
        r = cq.search(SIZES, cost, valid, trials=96, seed=seed)
        g = np.random.default_rng(seed)
        rnd = []
        while len(rnd) < 96:
            k = [int(g.integers(s)) for s in SIZES]
            if valid(k):
                rnd.append(cost(k))
        wins += min(r["history_cost"]) < min(rnd)
    assert wins >= 9, wins


def test_only_valid_unmeasured_points_and_first_batch_random():
    cost, valid, _, _ = _synthetic(3)
    r = cq.search(SIZES, cost, valid, trials=100, batch=32, seed=7)
    keys = [tuple(k) for k in r["history_knobs"]]
    assert len(set(keys)) == len(keys) == 100               # never re-measures a point
    assert all(valid(k) for k in keys)
    assert all(math.isclose(c, cost(k)) for c, k in zip(r["history_cost"], keys))
    assert r["best"] == list(keys[int(np.argmin(r["history_cost"]))])


def test_deterministic_for_a_seed():
    cost, valid, _, _ = _synthetic(4)
    a = cq.search(SIZES, cost, valid, trials=64, seed=11)
    b = cq.search(SIZES, cost, valid, trials=64, seed=11)
    c = cq.search(SIZES, cost, valid, trials=64, seed=12)
    assert a == b
    assert a["history_knobs"] != c["history_knobs"]


def test_failed_points_rank_last():
    """cost <= 0 marks a failed point: never the best, and the search steers off them."""
    cost, valid, best, _ = _synthetic(5)

    def flaky(k):
        return -1.0 if k[0] == 0 else cost(k)

    r = cq.search(SIZES, flaky, valid, trials=128, seed=3)
    assert r["best"][0] != 0
    fails = [c for c in r["history_cost"] if c <= 0]
    first = sum(c <= 0 for c in r["history_cost"][:32])
    later = sum(c <= 0 for c in r["history_cost"][32:]) / 3.0
    assert fails and later < first   # model batches pick fewer failing points than the random first batch


def test_small_space_exhausted():
    seen = []

    def cost(k):
        seen.append(tuple(k))
        return 1.0 + k[0] + 2 * k[1]

    r = cq.search([2, 3], cost, trials=50, batch=4, seed=1)
    assert r["n"] == 6 and sorted(set(seen)) == sorted(itertools.product(range(2), range(3)))
    assert r["best"] == [0, 0]


def test_model_learns_separable_ranking():
    """On a separable 4x4x4 space the ranking model steers the second and third
    batches onto the optimum: found within 36 measurements for every seed, at a
    median position <= 16 (uniform random sampling without replacement: ~32)."""
    def cost(k):
        return 1.0 + 3 * k[0] + 2 * k[1] + k[2]

    pos = []
    for seed in range(20):
        r = cq.search([4, 4, 4], cost, trials=36, batch=12, seed=seed)
        keys = [tuple(k) for k in r["history_knobs"]]
        assert (0, 0, 0) in keys and r["best"] == [0, 0, 0]
        pos.append(keys.index((0, 0, 0)))
    assert sorted(pos)[10] <= 16, pos


def test_bad_arguments():
    with pytest.raises(cq.ConvQError):
        cq.search([], lambda k: 1.0)
    with pytest.raises(cq.ConvQError):
        cq.search([2, 0], lambda k: 1.0)
    with pytest.raises(cq.ConvQError):
        cq.search([2, 2], lambda k: 1.0, trials=0)
    with pytest.raises(cq.ConvQError):   # nothing measured successfully
        cq.search([2, 2], lambda k: -1.0, trials=4)


def test_opts_defaults_are_the_papers():
    o = cq.SearchOpts.make()
    assert (o.batch, o.sa_iters, o.sa_early_stop, o.sa_points, o.diversity) == (32, 500, 50, 128, 1)
    assert math.isclose(o.sa_temp0, 1.0) and math.isclose(o.sa_cool, 0.002, rel_tol=1e-6)


@pytest.mark.parametrize("shape", [(8, 56, 56, 64, 64, 3, 3, 1, 1), (8, 7, 7, 512, 512, 3, 3, 1, 1),
                                   (32, 14, 14, 256, 1024, 1, 1, 1, 0)])
def test_plan_space_host_only(shape):
    """conv_q_plan_space needs no GPU: the enlarged space of a ResNet shape is
    far beyond the ~80 TileConfig candidates exhaustive tuning times."""
    N, H, W, C, K, R, S, st, pad = shape
    p = cq.ConvPlan(N, H, W, C, K, R, S, st, pad, 8)
    sizes, nvalid = p.space()
    assert len(sizes) == 10 and sizes[5:] == [6, 3, 3, 2, 3]
    assert nvalid >= 10 * len(p.candidates()) and nvalid > 200


def test_plan_point_roundtrip_host_only():
    """get_point / set_point (no GPU for split-1 points): every valid split-1
    point of a shape's space round-trips, and the info() name carries the
    runtime-knob suffix when a knob is off its default."""
    p = cq.ConvPlan(8, 28, 28, 128, 128, 3, 3, 1, 1, 8)
    sizes, _ = p.space()
    pt0 = p.get_point()
    assert pt0[5:] == [0, 0, 1, 0, 0]          # split 1, spin wait, evict_last, no rotation, full grid
    n = 0
    for pt in itertools.product(*[range(s) for s in sizes[:5]]):
        for rt in ([0, 0, 1, 0, 0], [0, 1, 2, 0, 1], [0, 2, 0, 1, 2]):
            k = list(pt) + rt
            try:
                p.set_point(k)
            except cq.ConvQError as e:
                assert e.code == cq.EUNSUPPORTED
                continue
            assert p.get_point() == k
            name = p.info().config
            assert ("+" in name) == (rt != [0, 0, 1, 0, 0]), name
            n += 1
    assert n >= len([c for c in p.candidates() if "_k" not in c])
    with pytest.raises(cq.ConvQError):
        p.set_point([99] * len(sizes))
