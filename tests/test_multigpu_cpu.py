"""Multi-process (gloo, world size 2, CPU) coverage of the batch-sharded path:
shard arithmetic, concatenated shard outputs == single-process output (the CPU
oracle stands in for the device kernel -- the sharding logic is what is under
test), and the max-over-ranks step-time reduction bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as wl


def test_shard_batch_partitions():
    for N in (1, 7, 256, 255):
        for g in (1, 2, 3, 4, 8):
            got = [wl.shard_batch(N, g, r) for r in range(g)]
            assert sum(c for _, c in got) == N
            assert got[0][0] == 0
            for (s0, c0), (s1, _) in zip(got, got[1:]):
                assert s1 == s0 + c0
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = wl.Layer("mg", 6, 5, 32, 16, 3, 3, 1, 1)
    g = wl.rng(4, 99)
    x, w, ss = wl.layer_inputs(g, L, N, 8)           # every rank draws the same global input
    wt = torch.from_numpy(w.copy())
    dist.broadcast(wt, 0)                              # weights replicated by one broadcast
    start, count = wl.shard_batch(N, world, rank)
    y = oracle.conv_q(x[start:start + count], wt.numpy(), L.C, L.stride, L.pad, 8, ss, True, nthreads=1)
    parts = [None] * world
    dist.all_gather_object(parts, y)                   # the optional final gather
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)           # bench.py: step time = max over ranks
    if rank == 0:
        ret["y"] = np.concatenate(parts, axis=0)
        ret["tmax"] = float(t.item())
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [5, 4])
def test_gloo_two_ranks_concat_equals_single(N):
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), N, ret), nprocs=world, join=True)
    L = wl.Layer("mg", 6, 5, 32, 16, 3, 3, 1, 1)
    x, w, ss = wl.layer_inputs(wl.rng(4, 99), L, N, 8)
    ref = oracle.conv_q(x, w, L.C, L.stride, L.pad, 8, ss, True)
    assert np.array_equal(ret["y"], ref)
    assert ret["tmax"] == 2.0


# ---------------------------------------------------------------- bench.py's own rank logic
def _bench_worker(rank, world, port, ret):
    """Drives bench.py's rank functions (shard_plan, replicate, max_over_ranks,
    gather_outputs) under gloo with a stubbed device arm: the oracle computes
    each rank's shard of a small ResNet-shaped layer on the host."""
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = bench.workload_spec("cfg1")
    L = wl.Layer("mg", 6, 5, 32, 16, 3, 3, 1, 1)
    Bg, B, start = bench.shard_plan(6, world, rank, "strong")
    x, w, ss = wl.layer_inputs(wl.rng(4, 98), L, Bg, 8)
    # rank-dependent garbage before the broadcast: replicate() must make every rank equal rank 0
    wt = torch.from_numpy(w.copy() if rank == 0 else np.zeros_like(w))
    st = torch.from_numpy(ss.copy() if rank == 0 else np.zeros_like(ss))
    bench.replicate([wt, st], world, dist)
    y = oracle.conv_q(x[start:start + B], wt.numpy(), L.C, L.stride, L.pad, 8, st.numpy(), True, nthreads=1)
    out = bench.gather_outputs(torch.from_numpy(y), world, dist)
    tmax = bench.max_over_ranks(10.0 + rank, world, dist, "cpu")
    tmin = bench.min_over_ranks(1.0 - rank, world, dist, "cpu")
    ret[rank] = (Bg, B, start, tmax, tmin)
    if rank == 0:
        ret["y"] = out.numpy()
    dist.destroy_process_group()


def test_bench_rank_logic_gloo_two_ranks():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_bench_worker, args=(world, _free_port(), ret), nprocs=world, join=True)
    L = wl.Layer("mg", 6, 5, 32, 16, 3, 3, 1, 1)
    x, w, ss = wl.layer_inputs(wl.rng(4, 98), L, 6, 8)
    assert ret[0][:3] == (6, 3, 0) and ret[1][:3] == (6, 3, 3)      # strong: global 6 split 3 + 3
    assert ret[0][3] == ret[1][3] == 11.0                            # max over ranks
    assert ret[0][4] == ret[1][4] == 0.0
    assert np.array_equal(ret["y"], oracle.conv_q(x, w, L.C, L.stride, L.pad, 8, ss, True))


def test_bench_shard_plan_rules():
    import bench
    assert bench.shard_plan(256, 8, 7, "strong") == (256, 32, 224)
    assert bench.shard_plan(256, 1, 0, "strong") == (256, 256, 0)
    assert bench.shard_plan(256, 4, 3, "weak") == (1024, 256, 768)
    with pytest.raises(SystemExit):
        bench.shard_plan(255, 2, 0, "strong")                        # uneven shards are rejected
