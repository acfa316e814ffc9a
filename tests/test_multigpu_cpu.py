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
