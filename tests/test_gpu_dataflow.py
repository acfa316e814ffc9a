"""Cross-launch completion counters (conv_q_plan_set_deps) on the GPU (-m gpu):
the bench chains with dataflow between conv launches, every launch checked
against the oracle on sampled pixels (tile boundaries included), several steps
in a row (the counters are re-zeroed every step), and dataflow == whole-grid
dependencies byte for byte on every output."""
import numpy as np
import pytest

import workloads as wl

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cq():
    import paper_2202_06819_b200 as m
    m.load()
    return m


def _net(workload, dataflow, B=None):
    import bench
    spec = bench.workload_spec(workload)
    B = B or spec.batch
    net = bench.build_network(spec, B, torch.device("cuda", 0), dataflow=dataflow)
    g = wl.rng(spec.cfg_id, 1000)
    net.x_in.copy_(torch.from_numpy(wl.fp16_activations(g, B, *tuple(net.x_in.shape[1:]))))
    return spec, net, B


@pytest.mark.parametrize("workload,B", [("resnet18_int8_b1", None), ("resnet18_int4_b16", None),
                                        ("resnet50_int8_b256", 32), ("resnet50_int8_b256_res", 32),
                                        ("resnet18_int8_b1_res_uns", None), ("resnet50_int8_b256", None)])
def test_dataflow_chain_parity(cq, workload, B):
    import bench
    spec, net, B = _net(workload, True, B)
    net.tune(warmup=1, reps=2)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    net.set_stream(stream)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        net.step(stream)
    for _ in range(3):                   # replays: the counters are re-zeroed inside every step
        graph.replay()
    torch.cuda.synchronize()
    imgs = sorted({0, B // 2, B - 1})
    ok, bad = bench.parity_check(net, spec, imgs, n_rand=256, seed=5)
    torch.cuda.set_stream(torch.cuda.default_stream())
    assert ok, bad[:5]


@pytest.mark.parametrize("workload,B", [("resnet18_int8_b1", None), ("resnet50_int8_b256_res", 16)])
def test_dataflow_equals_grid_dependencies(cq, workload, B):
    """Same configs, same inputs: every conv output byte-identical with and without flags."""
    spec, a, B = _net(workload, True, B)
    _, b, _ = _net(workload, False, B)
    a.tune(warmup=1, reps=2)
    for ca, cb in zip(a.convs, b.convs):      # the same tile configs on both
        cb.plan.set_config(ca.plan.candidates().index(ca.plan.info().config))
    for _ in range(2):
        a.step()
        b.step()
    torch.cuda.synchronize()
    for ca, cb in zip(a.convs, b.convs):
        assert torch.equal(ca.y, cb.y), ca.name
