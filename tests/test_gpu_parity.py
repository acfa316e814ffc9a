"""GPU-vs-oracle parity (bit-exact) through the C ABI.  Needs a B200: -m gpu.

Every comparison is element by element on the same seeded inputs (workloads/),
the CUDA side through paper_2202_06819_b200 (libconvq.so), the CPU side through
oracle/ (liboracle.so).  Integer and byte results must be identical."""
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


def run_conv(cq, L, N, bits, x, w, ss, relu=False, s32=False, config=None, plan=None):
    p = plan or cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits)
    p.set_epilogue(relu, cq.OUT_S32 if s32 else cq.OUT_PACKED)
    if config is not None:
        p.set_config(config)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    if s32:
        y = torch.full((N, L.P, L.Q, L.K), -7777777, dtype=torch.int32, device="cuda")
    else:
        y = torch.full((N, L.P, L.Q, L.K * bits // 8), 0xA5, dtype=torch.uint8, device="cuda")
    p.run(xd, wd, sd, y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def first_diff(a, b):
    idx = np.argwhere(a != b)
    return None if idx.size == 0 else (tuple(idx[0]), a[tuple(idx[0])], b[tuple(idx[0])], len(idx))


def check_layer(cq, L, N, bits, seed, relu=False, all_configs=True):
    g = np.random.default_rng(seed)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    ref32 = oracle.conv_s32(x, w, L.C, L.stride, L.pad, bits)
    refq = oracle.requant(ref32, ss, relu, bits)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits)
    cfgs = range(len(plan.candidates())) if all_configs else [plan.info().config_index]
    for ci in cfgs:
        name = plan.candidates()[ci]
        got32 = run_conv(cq, L, N, bits, x, w, ss, relu, True, ci, plan)
        assert np.array_equal(got32, ref32), (L, bits, name, first_diff(got32, ref32))
        gotq = run_conv(cq, L, N, bits, x, w, ss, relu, False, ci, plan)
        assert np.array_equal(gotq, refq), (L, bits, name, first_diff(gotq, refq))


# ----------------------------------------------------------------- quantize / pack
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("shape", [(2, 7, 9, 64), (1, 5, 6, 3), (3, 4, 4, 96), (1, 1, 1, 32), (2, 3, 3, 33)])
def test_quantize_parity(cq, bits, shape):
    g = np.random.default_rng(11)
    x = (g.standard_normal(shape) * 3).astype(np.float16)
    flat = x.reshape(-1)
    specials = np.array([65504, -65504, np.inf, -np.inf, np.nan, -0.0, 0.125, 0.375, -0.625, 31.875],
                        dtype=np.float16)
    flat[:min(flat.size, specials.size)] = specials[:min(flat.size, specials.size)]
    inv = 4.0 if bits == 8 else 2.0          # 0.125*(2j+1)*4 = j + 0.5: exact ties
    got = cq.quantize(dev(x), inv, bits)
    torch.cuda.synchronize()
    ref = oracle.quantize(x, inv, bits)
    assert np.array_equal(got.cpu().numpy(), ref), first_diff(got.cpu().numpy(), ref)


@pytest.mark.parametrize("bits", [8, 4])
def test_quantize_large_flat(cq, bits):
    g = np.random.default_rng(12)
    x = g.standard_normal((4, 56, 56, 64)).astype(np.float16)
    got = cq.quantize(dev(x), 127 / 4 if bits == 8 else 7 / 3, bits).cpu().numpy()
    ref = oracle.quantize(x, 127 / 4 if bits == 8 else 7 / 3, bits)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("bits", [8, 4])
def test_pack_weights_parity(cq, bits):
    g = np.random.default_rng(13)
    wv = wl.weight_values(g, 48, 3, 3, 64, bits)
    got = cq.pack_weights(dev(wv), bits).cpu().numpy()
    assert np.array_equal(got, oracle.pack(wv, bits))


# ----------------------------------------------------------------- conv
@pytest.mark.parametrize("bits", [8, 4])
def test_cfg1_parity_all_configs(cq, bits):
    """cfg1: N=1 56x56x64->64 3x3 s1 p1 (ResNet-18 stage-1 layer)."""
    check_layer(cq, wl.CFG1, 1, bits, wl.seed(1), relu=False)


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("L,N", [
    (wl.Layer("tail", 9, 11, 64, 64, 3, 3, 1, 1), 3),            # M=297: ragged tail, crosses images
    (wl.Layer("s2", 13, 13, 96, 128, 3, 3, 2, 1), 2),            # stride 2, odd size
    (wl.Layer("1x1s2", 14, 14, 128, 256, 1, 1, 2, 0), 2),        # downsample shape
    (wl.Layer("k80", 6, 6, 64, 96, 3, 3, 1, 1), 1),              # K not a multiple of the N tile
    (wl.Layer("rect", 10, 7, 64, 64, 3, 1, 1, 1), 2),            # R != S, rectangular image
    (wl.Layer("7x7", 23, 23, 32, 64, 7, 7, 2, 3), 1),            # conv1-like 7x7 s2 p3
    (wl.Layer("5x5p2", 8, 8, 64, 32, 5, 5, 1, 2), 2),
    (wl.Layer("1px", 1, 1, 128, 64, 1, 1, 1, 0), 5),             # 1x1 images
    (wl.Layer("pad3", 4, 4, 32, 64, 3, 3, 1, 3), 1),             # padding larger than the filter reach
    (wl.Layer("7x7s1", 12, 10, 64, 64, 7, 7, 1, 3), 2),          # general R x S halo (49 taps)
    (wl.Layer("1x3", 9, 20, 128, 64, 1, 3, 1, 1), 2),            # R=1 x S=3 halo, pad rows
    (wl.Layer("5x5c128", 11, 13, 128, 128, 5, 5, 1, 2), 3),      # 25 taps, 2 channel blocks
])
def test_shape_edge_parity(cq, bits, L, N):
    if (L.K * bits) % 128:
        pytest.skip("K*bits not a multiple of 128")
    check_layer(cq, L, N, bits, 1234, relu=(L.name in ("s2", "7x7")))


@pytest.mark.parametrize("L,N", [
    (wl.Layer("c48", 9, 11, 48, 64, 3, 3, 1, 1), 2),             # s8 C = 16 (mod 32): ragged last k-block
    (wl.Layer("c80s2", 13, 12, 80, 96, 3, 3, 2, 1), 1),          # stride 2, K not a tile multiple
    (wl.Layer("c112x1", 7, 9, 112, 64, 1, 1, 1, 0), 3),          # 1x1 tiled (a_gemm) path
])
def test_ragged_channel_block_s8(cq, L, N):
    """SURVEY 8(b) boundary: s8 with C = 16 (mod 32), every candidate, s32 + packed."""
    check_layer(cq, L, N, 8, 4321, relu=True)


@pytest.mark.parametrize("bits", [8, 4])
def test_fuzz_parity(cq, bits):
    g = np.random.default_rng(99 + bits)
    n_done = 0
    while n_done < 12:
        R = int(g.choice([1, 3, 5, 7]))
        S = int(g.choice([1, 3, 5, 7]))
        stride = int(g.integers(1, 3))
        pad = int(g.integers(0, 4))
        H, W = int(g.integers(1, 21)), int(g.integers(1, 21))
        if H + 2 * pad < R or W + 2 * pad < S:
            continue
        C = 32 * int(g.integers(1, 9))
        K = (16 if bits == 8 else 32) * int(g.integers(1, 17 if bits == 8 else 9))
        N = int(g.integers(1, 4))
        L = wl.Layer("fuzz", H, W, C, K, R, S, stride, pad)
        check_layer(cq, L, N, bits, int(g.integers(1 << 30)), relu=bool(g.integers(2)), all_configs=False)
        n_done += 1


@pytest.mark.parametrize("bits", [8, 4])
def test_extreme_operands(cq, bits):
    """All codes at -2^(b-1): the largest accumulators (3x3x512: 4608*2^(2b-2))."""
    L = wl.Layer("ext", 5, 5, 512, 64, 3, 3, 1, 1)
    x = np.full((1, 5, 5, 512 * bits // 8), 0x80 if bits == 8 else 0x88, np.uint8)
    w = np.full((64, 3, 3, 512 * bits // 8), 0x80 if bits == 8 else 0x88, np.uint8)
    ss = np.concatenate([np.full(64, 2.0 ** -20, np.float32), np.zeros(64, np.float32)])
    ref32 = oracle.conv_s32(x, w, 512, 1, 1, bits)
    got32 = run_conv(cq, L, 1, bits, x, w, ss, s32=True)
    assert np.array_equal(got32, ref32)
    assert np.array_equal(run_conv(cq, L, 1, bits, x, w, ss), oracle.requant(ref32, ss, False, bits))


def test_requant_ties_and_saturation(cq):
    """scale 0.5 / shift 0 on small integer accumulators: exact .5 ties -> even;
    large scale saturates to both ends."""
    L = wl.Layer("ties", 4, 4, 32, 64, 1, 1, 1, 0)
    g = np.random.default_rng(5)
    x = g.integers(-3, 4, size=(2, 4, 4, 32), dtype=np.int8).view(np.uint8)
    w = np.zeros((64, 1, 1, 32), np.int8)
    w[:, 0, 0, 0] = 1
    w = w.view(np.uint8)
    ss = np.concatenate([np.where(np.arange(64) < 32, 0.5, 100.0).astype(np.float32),
                         np.where(np.arange(64) % 3 == 0, 0.25, 0.0).astype(np.float32)])
    for relu in (False, True):
        got = run_conv(cq, L, 2, 8, x, w, ss, relu=relu)
        assert np.array_equal(got, oracle.conv_q(x, w, 32, 1, 0, 8, ss, relu))


def test_determinism(cq):
    L = wl.Layer("det", 14, 14, 256, 256, 3, 3, 1, 1)
    g = np.random.default_rng(3)
    x, w, ss = wl.layer_inputs(g, L, 4, 8)
    p = cq.ConvPlan(4, 14, 14, 256, 256, 3, 3, 1, 1, 8)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    y0 = torch.empty((4, 14, 14, 256), dtype=torch.uint8, device="cuda")
    p.run(xd, wd, sd, y0)
    ref = y0.clone()
    for _ in range(50):
        p.run(xd, wd, sd, y0)
        assert torch.equal(y0, ref)


# ----------------------------------------------------------------- full-size sampled parity
@pytest.mark.parametrize("bits,name,N", [(8, "l3.b1.c2", 256), (8, "l1.b0.c2", 256), (8, "l4.b0.ds", 256),
                                         (4, "l2.b0.c2", 256)])
def test_resnet50_fullsize_sampled(cq, bits, name, N):
    """BASELINE cfg4 sizes (batch 256) in the bench launch configuration: the
    oracle computes sampled output pixels (first/last image + random)."""
    L = dict((l.name, l) for l, _ in wl.resnet50_layers())[name]
    g = wl.rng(4, 0)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    got = run_conv(cq, L, N, bits, x, w, ss, relu=True).reshape(-1, L.K * bits // 8)
    M = N * L.P * L.Q
    pix = np.unique(np.concatenate([np.arange(0, 40), np.arange(M - 40, M),
                                    g.integers(0, M, 64)])).astype(np.int64)
    ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, True, pix=pix)
    assert np.array_equal(got[pix], ref)


def test_resnet18_chain_int8_b1(cq):
    """cfg2: ResNet-18 convs INT8 batch 1, each y is the next x byte-for-byte."""
    layers = wl.resnet18_layers()
    g = wl.rng(2, 0)
    x0 = wl.random_bytes(g, (1, 56, 56, 64))
    outs_gpu, outs_ref = [], []
    for i, (L, src) in enumerate(layers):
        gi = wl.rng(2, i + 1)
        wv = wl.random_bytes(gi, (L.K, L.R, L.S, L.C))
        sd = wl.uniform_code_std(8)
        ss = wl.scale_shift(gi, L.K, L.R * L.S * L.C, sd * 0.5, sd, 8)
        xin_g = x0 if src < 0 else outs_gpu[src]
        xin_r = x0 if src < 0 else outs_ref[src]
        outs_gpu.append(run_conv(cq, L, 1, 8, xin_g, wv, ss, relu=True))
        outs_ref.append(oracle.conv_q(xin_r, wv, L.C, L.stride, L.pad, 8, ss, True))
        assert np.array_equal(outs_gpu[-1], outs_ref[-1]), (i, L)


def test_resnet18_chain_int4_b16(cq):
    """cfg3: ResNet-18 convs INT4 (packed s4, s4 -> s8 on chip) batch 16, each y is
    the next x byte-for-byte, every output byte compared."""
    layers = wl.resnet18_layers()
    g = wl.rng(3, 0)
    x0 = wl.random_bytes(g, (16, 56, 56, 64 * 4 // 8))
    outs_gpu, outs_ref = [], []
    for i, (L, src) in enumerate(layers):
        gi = wl.rng(3, i + 1)
        wv = wl.random_bytes(gi, (L.K, L.R, L.S, L.C * 4 // 8))
        sd = wl.uniform_code_std(4)
        ss = wl.scale_shift(gi, L.K, L.R * L.S * L.C, sd * 0.5, sd, 4)
        xin_g = x0 if src < 0 else outs_gpu[src]
        xin_r = x0 if src < 0 else outs_ref[src]
        outs_gpu.append(run_conv(cq, L, 16, 4, xin_g, wv, ss, relu=True))
        outs_ref.append(oracle.conv_q(xin_r, wv, L.C, L.stride, L.pad, 4, ss, True))
        assert np.array_equal(outs_gpu[-1], outs_ref[-1]), (i, L, first_diff(outs_gpu[-1], outs_ref[-1]))


@pytest.mark.parametrize("bits,name", [(8, "l1.b0.c3"), (8, "l3.b1.c3"), (8, "l2.b1.c2"), (8, "l4.b0.c2")])
def test_resnet50_fullsize_tuned_sampled(cq, bits, name):
    """The bench's launch configuration: batch 256 with the tile config conv_q_plan_tune
    picks (a7), sampled output pixels vs the oracle."""
    L = dict((l.name, l) for l, _ in wl.resnet50_layers())[name]
    N = 256
    g = wl.rng(4, 7)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True)
    xd, wd, sd = dev(x), dev(w), dev(ss)
    y = torch.full((N, L.P, L.Q, L.K * bits // 8), 0xA5, dtype=torch.uint8, device="cuda")
    plan.tune(xd, wd, sd, y, warmup=1, reps=2)
    y.fill_(0xA5)
    plan.run(xd, wd, sd, y)
    torch.cuda.synchronize()
    got = y.cpu().numpy().reshape(-1, L.K * bits // 8)
    M = N * L.P * L.Q
    pix = np.unique(np.concatenate([np.arange(0, 40), np.arange(M - 40, M),
                                    g.integers(0, M, 96)])).astype(np.int64)
    ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, True, pix=pix)
    assert np.array_equal(got[pix], ref), (plan.info().config, first_diff(got[pix], ref))


def test_int8_peak_runs(cq):
    ops = cq.int8_peak(20000)
    assert 1e14 < ops < 6e15


# ----------------------------------------------------------------- split-K
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("L,N", [
    (wl.Layer("l4.3x3", 7, 7, 512, 512, 3, 3, 1, 1), 1),         # ResNet-18 stage 5, batch 1
    (wl.Layer("l3.s2", 28, 28, 128, 256, 3, 3, 2, 1), 1),        # stride-2 entry of stage 4
    (wl.Layer("l4.ds", 14, 14, 256, 512, 1, 1, 2, 0), 2),        # 1x1 s2 downsample
])
def test_split_k_parity(cq, bits, L, N):
    """Split-K work units (several CTAs per output tile, partial sums meeting
    in the plan's workspace): every split candidate, three runs in a row (the
    workspace must be left zero by each run), s32 and packed outputs."""
    g = np.random.default_rng(77 + bits)
    x, w, ss = wl.layer_inputs(g, L, N, bits)
    ref32 = oracle.conv_s32(x, w, L.C, L.stride, L.pad, bits)
    refq = oracle.requant(ref32, ss, True, bits)
    plan = cq.ConvPlan(N, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits)
    names = plan.candidates()
    split = [i for i, n in enumerate(names) if "_k" in n]
    assert split, names
    for ci in split:
        for rep in range(3):
            got32 = run_conv(cq, L, N, bits, x, w, ss, True, True, ci, plan)
            assert np.array_equal(got32, ref32), (names[ci], rep, first_diff(got32, ref32))
            gotq = run_conv(cq, L, N, bits, x, w, ss, True, False, ci, plan)
            assert np.array_equal(gotq, refq), (names[ci], rep, first_diff(gotq, refq))


# ----------------------------------------------------------------- s2d stem
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("N,H,W,C,K,R,S,pad", [
    (2, 30, 38, 3, 64, 7, 7, 3),      # ResNet conv1 geometry, small image, several tiles + ragged tail
    (1, 33, 29, 3, 64, 7, 7, 3),      # odd H/W: last s2d row/column half empty
    (1, 21, 19, 3, 128, 3, 3, 1),     # 3x3/2 p1 stem (2 s2d taps)
    (2, 16, 16, 1, 64, 5, 5, 2),      # C=1, 5x5/2 p2
    (1, 26, 32, 3, 64, 7, 7, 3),      # even W: the vectorised C=3 quantize path, odd H
])
def test_stem_s2d_parity(cq, bits, N, H, W, C, K, R, S, pad):
    """StemPlan (s2d quantize + window weights + stride-1 conv) == the oracle's
    direct stride-2 conv on the channel-padded quantized image, every config,
    s32 accumulators and requantized bytes."""
    g = np.random.default_rng(6819 + 7 * H + bits)
    x = (g.standard_normal((N, H, W, C)) * 2).astype(np.float16)
    inv = 127 / 4 if bits == 8 else 7 / 3
    wv = wl.weight_values(g, K, R, S, C, bits)
    Cp = oracle.padded_channels(C, bits)
    w_pad = np.zeros((K, R, S, Cp), dtype=np.int8)
    w_pad[..., :C] = wv
    xq = oracle.quantize(x, inv, bits)
    wq = oracle.pack(w_pad, bits)
    ss = wl.scale_shift(g, K, R * S * C, 40.0 if bits == 8 else 3.0, wl.uniform_code_std(bits), bits)
    ref32 = oracle.conv_s32(xq, wq, Cp, 2, pad, bits)
    refq = oracle.requant(ref32, ss, True, bits)
    plan = cq.StemPlan(N, H, W, C, K, R, S, pad, bits)
    xs = plan.quantize(dev(x), inv)
    wp = plan.pack_weights(dev(wv))
    sd = dev(ss)
    P, Q = plan.P, plan.Q
    assert ref32.shape == (N, P, Q, K)
    for ci, name in enumerate(plan.candidates()):
        plan.set_config(ci)
        plan.set_epilogue(True, cq.OUT_S32)
        y32 = torch.full((N, P, Q, K), -7777777, dtype=torch.int32, device="cuda")
        plan.run(xs, wp, sd, y32)
        torch.cuda.synchronize()
        got32 = y32.cpu().numpy()
        assert np.array_equal(got32, ref32), (name, first_diff(got32, ref32))
        plan.set_epilogue(True, cq.OUT_PACKED)
        yq = torch.full((N, P, Q, K * bits // 8), 0xA5, dtype=torch.uint8, device="cuda")
        plan.run(xs, wp, sd, yq)
        torch.cuda.synchronize()
        assert np.array_equal(yq.cpu().numpy(), refq), (name, first_diff(yq.cpu().numpy(), refq))


@pytest.mark.parametrize("bits", [8, 4])
def test_stem_s2d_fullsize_sampled(cq, bits):
    """ResNet-50 conv1 at 224x224, batch 32 (the bench's launch configuration
    shape per image): sampled output pixels vs the oracle, computed one by one."""
    N, K = 32, 64
    g = np.random.default_rng(99 + bits)
    x = g.standard_normal((N, 224, 224, 3)).astype(np.float16)
    inv = 127 / 4 if bits == 8 else 7 / 3
    wv = wl.weight_values(g, K, 7, 7, 3, bits)
    w_pad = np.zeros((K, 7, 7, 32), dtype=np.int8)
    w_pad[..., :3] = wv
    ss = wl.scale_shift(g, K, 147, 40.0 if bits == 8 else 3.0, wl.uniform_code_std(bits), bits)
    plan = cq.StemPlan(N, 224, 224, 3, K, 7, 7, 3, bits, relu=True)
    plan.tune(plan.quantize(dev(x), inv), plan.pack_weights(dev(wv)), dev(ss),
              torch.empty((N, 112, 112, K * bits // 8), dtype=torch.uint8, device="cuda"), warmup=1, reps=2)
    xs = plan.quantize(dev(x), inv)
    y = torch.empty((N, 112, 112, K * bits // 8), dtype=torch.uint8, device="cuda")
    plan.run(xs, plan.pack_weights(dev(wv)), dev(ss), y)
    torch.cuda.synchronize()
    M = N * 112 * 112
    pix = np.unique(np.concatenate([g.integers(0, M, 3000), [0, 111, 112 * 112 - 1, M - 1, 112 * 111]]))
    ref = oracle.conv_q(oracle.quantize(x, inv, bits), oracle.pack(w_pad, bits), 32, 2, 3, bits, ss, True, pix=pix)
    got = y.cpu().numpy().reshape(M, -1)[pix]
    assert np.array_equal(got, ref), first_diff(got, ref)
