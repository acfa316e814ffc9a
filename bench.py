#!/usr/bin/env python
"""bench.py -- throughput of the quantized implicit-GEMM convolution path on B200.

Default workload (BASELINE.json configs[3], the one its "images/s at
1/2/4/8 GPU" metric is quoted on): ResNet-50 v1.5 convolutions, INT8, global
batch 256.  One step = one pass of the whole hot path over one batch:
  a1+stem  s2d quantize of the fp16 224x224x3 images, conv1 (7x7/2 as a stride-1
           window conv over the space-to-depth view), 3x3/2 max pool
  a3-a6    the 52 convolutions of layer1..layer4 through conv_q_run, each with
           the fused requantize + repack epilogue, each y the next x
           (downsample 1x1s read their block input)
i.e. all 53 convs of the network.  Weights are packed once (a2, off the
per-step path) and broadcast with one NCCL broadcast at setup; tile configs are
picked per shape by on-device timing (a7) at setup.

Timing: the timed window replays ONLY the plain CUDA graph of a step (every
kernel launched with programmatic dependent launch, nothing between them);
per-launch CUDA events are recorded in a separate window of event-instrumented
graph replays right after it (those numbers feed the per-layer table and the
roofline, never `value`).

Multi-GPU (a8): one process per GPU under torchrun.  With N > 1
the global batch is split across ranks (strong scaling, the default there;
--scaling weak gives every rank its own full batch); no collective on the data
path; the step time is the max over ranks.

After the timed windows a parity leg (the oracle, on the host) recomputes
sampled output pixels of every layer of the first and last image from the
device's own input bytes of that layer and reports `parity_ok`.

--impl reference times the CPU oracle (oracle/) on the host cores on a
bounded per-step sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as wl  # noqa: E402

UNIT = "images/s"
L2_BYTES = 126 * 1024 * 1024


# ---------------------------------------------------------------------------- workloads
class Spec:
    """A bench workload: network layers, per-GPU batch, precision, input stage."""

    def __init__(self, name, layers, batch, bits, conv1, desc, cfg_id, metric):
        # layers: (Layer, src) pairs, or (Layer, src, skip) triples for a network with residual adds
        layers = [tuple(t) + (None,) * (3 - len(t)) for t in layers]
        self.residual = any(t[2] is not None for t in layers)
        self.name, self.layers, self.batch, self.bits = name, layers, batch, bits
        self.conv1, self.desc, self.cfg_id, self.metric = conv1, desc, cfg_id, metric
        self.inv_scale = 127 / 4 if bits == 8 else 7 / 3
        self.pool = (3, 2, 1)
        self.unsigned = False     # unsigned post-ReLU codes (workload suffix _uns)


RES_SUFFIX = "_res"
UNS_SUFFIX = "_uns"


def workload_spec(name: str) -> Spec:
    if name.endswith(UNS_SUFFIX):
        # the same network with unsigned post-ReLU activation codes (NEXT-2, DESIGN reading 16)
        base = workload_spec(name[:-len(UNS_SUFFIX)])
        base.name, base.unsigned = name, True
        base.desc += ", unsigned post-ReLU codes (u%d activations)" % base.bits
        base.metric = base.metric.replace("fused requant-repack", "fused requant-repack, u%d activations" % base.bits)
        return base
    if name.endswith(RES_SUFFIX):
        # the same network with its residual adds fused into the c3 / c2 epilogues (NEXT-2)
        base = workload_spec(name[:-len(RES_SUFFIX)])
        blocks = wl.resnet50_blocks() if "resnet50" in name else wl.resnet18_blocks()
        return Spec(name, blocks, base.batch, base.bits, base.conv1,
                    base.desc + ", residual adds fused into the block-output epilogues",
                    base.cfg_id, base.metric.replace("fused requant-repack", "fused requant-repack + residual"))
    if name == "resnet50_int8_b256":
        return Spec(name, wl.resnet50_layers(), 256, 8, wl.resnet18_conv1(),
                    "ResNet-50 v1.5: conv1 (s2d stem) + 3x3/2 max pool + layer1-4 convs, INT8", 4,
                    "images/s (ResNet-50 all 53 conv layers, INT8, fused requant-repack)")
    if name == "resnet18_int8_b1":
        return Spec(name, wl.resnet18_layers(), 1, 8, wl.resnet18_conv1(),
                    "ResNet-18: conv1 (s2d stem) + 3x3/2 max pool + layer1-4 convs, INT8", 2,
                    "images/s (ResNet-18 all 20 conv layers, INT8, fused requant-repack)")
    if name == "resnet18_int4_b16":
        return Spec(name, wl.resnet18_layers(), 16, 4, wl.resnet18_conv1(),
                    "ResNet-18: conv1 (s2d stem) + 3x3/2 max pool + layer1-4 convs, INT4", 3,
                    "images/s (ResNet-18 all 20 conv layers, INT4, fused requant-repack)")
    if name == "cfg1":
        return Spec(name, [(wl.CFG1, -1)], 1, 8, None, "single INT8 conv N=1 56x56x64->64 3x3", 1,
                    "images/s (single INT8 conv 56x56x64->64 3x3, fused requant-repack)")
    raise SystemExit(f"unknown workload {name}")


def layer_ops(L, N):
    return 2 * N * L.P * L.Q * L.K * L.C * L.R * L.S


def layer_bytes(L, N, bits):
    """Algorithmic HBM bytes: referenced input pixels + weights + output."""
    if L.R == 1 and L.S == 1 and L.pad == 0:
        x_pix = N * L.P * L.Q           # a strided 1x1 only touches the sampled pixels
    else:
        x_pix = N * L.H * L.W
    return (x_pix * L.C + L.K * L.R * L.S * L.C + N * L.P * L.Q * L.K) * bits // 8


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def layer_weights(spec: Spec, i: int):
    """Seeded weight codes + [scale|shift] of conv i (i = -1: conv1), identical on every rank."""
    bits = spec.bits
    if i < 0:
        L = spec.conv1
        g = wl.rng(spec.cfg_id, 0)
    else:
        L = spec.layers[i][0]
        g = wl.rng(spec.cfg_id, i + 1)
    wv = wl.weight_values(g, L.K, L.R, L.S, L.C, bits)
    sd = wl.uniform_code_std(bits)
    ss = wl.scale_shift(g, L.K, L.R * L.S * L.C, sd * 0.5, sd, bits)
    return wv, ss


def layer_res_scale(spec: Spec, i: int) -> float:
    return wl.res_scale(wl.rng(spec.cfg_id, 500 + i))


def build_network(spec: Spec, B: int, device, world: int = 1, dist=None, dataflow=None):
    """The device network of a workload (packed weights broadcast from rank 0);
    dataflow None = auto (completion counters for per-GPU batch <= 4)."""
    import torch

    from paper_2202_06819_b200.network import ConvNet

    if dataflow is None:
        dataflow = B <= 4

    net = ConvNet(B, spec.bits, device, unsigned=spec.unsigned, dataflow=dataflow)

    def dev_params(i):
        wv, ss = layer_weights(spec, i)
        wt, st = torch.from_numpy(wv).to(device), torch.from_numpy(ss).to(device)
        replicate([wt, st], world, dist)          # one broadcast at setup (identical already)
        return wt, st

    if spec.conv1 is not None:
        wt, st = dev_params(-1)
        net.set_stem(spec.conv1, wt, st, spec.inv_scale, pool=spec.pool)
    else:
        L0 = spec.layers[0][0]
        net.set_quantize_input(L0.H, L0.W, L0.C, spec.inv_scale)
    for i, (L, src, skip) in enumerate(spec.layers):
        wt, st = dev_params(i)
        net.add_conv(L, src, wt, st, relu=True, name=L.name, skip=skip,
                     res_scale=layer_res_scale(spec, i) if skip is not None else 0.0)
    return net


# ---------------------------------------------------------------------------- rank logic
def shard_plan(batch: int, world: int, rank: int, scaling: str):
    """-> (global batch, this rank's batch, this rank's first image).  strong: the
    global batch `batch` is split into equal contiguous shards;
    weak: every rank runs its own `batch` images."""
    if scaling == "weak":
        return batch * world, batch, rank * batch
    if batch % world:
        raise SystemExit(f"strong scaling needs the global batch {batch} divisible by {world} ranks")
    start, count = wl.shard_batch(batch, world, rank)
    return batch, count, start


def replicate(tensors, world: int, dist):
    """Weights/scales replicated from rank 0 (one broadcast each, at setup)."""
    if world > 1:
        for t in tensors:
            dist.broadcast(t, 0)


def max_over_ranks(x: float, world: int, dist, device) -> float:
    """Step time = max over ranks (all_reduce MAX)."""
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def min_over_ranks(x: float, world: int, dist, device) -> float:
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def gather_outputs(y, world: int, dist):
    """The optional final gather: every rank's last-layer packed output,
    concatenated in rank order (== the 1-GPU output of the global batch)."""
    import torch
    if world == 1:
        return y.clone()
    out = torch.empty((world * y.shape[0],) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    try:
        dist.all_gather_into_tensor(out, y)
    except (RuntimeError, NotImplementedError, ValueError):   # backends without it (gloo: host tensors only)
        yc = y.cpu()
        parts = [torch.empty_like(yc) for _ in range(world)]
        dist.all_gather(parts, yc)
        out = torch.cat(parts, 0).to(y.device)
    return out


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.proc = None
        self.gpu_index = gpu_index
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 f"-lms={period_ms}", f"-i={gpu_index}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(n)
        res = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if not sm:
            # a timed region shorter than nvidia-smi's start-up + period: one sample right after it
            try:
                one = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                      f"-i={self.gpu_index}"], capture_output=True, text=True, timeout=10).stdout
                f = [x.strip() for x in one.strip().splitlines()[0].split(",")]
                res.update(sm_mhz=float(f[1]), sm_max_mhz=float(f[2]),
                           reasons=sorted(n for n, v in zip(names, f[5:9]) if v.lower() in ("active", "1", "yes")),
                           samples=1, note="timed region shorter than the sampling period: one sample right after it")
            except Exception:
                pass
        return res


# ---------------------------------------------------------------------------- parity leg
def parity_check(net, spec: Spec, imgs, n_rand: int = 64, seed: int = 0, nthreads=None):
    """Sampled oracle check of every launch of one step (images `imgs` of this
    rank's batch): each layer recomputed from the device's own input bytes of
    that layer.  -> (ok, list of failures)."""
    import torch

    from oracle import check

    g = np.random.default_rng(seed)
    idx = torch.as_tensor(list(imgs), dtype=torch.long, device=net.device)
    host = lambda t: t.index_select(0, idx).cpu().numpy()  # noqa: E731
    bad = []
    bits = spec.bits
    if net.stem is not None:
        st = net.stem
        L1 = st["layer"]
        wv, ss = layer_weights(spec, -1)
        y1 = host(st["y"])
        pix = check.sample_pixels(len(imgs), st["plan"].P, st["plan"].Q, g, n_rand)
        ok, d = check.check_stem(host(net.x_in), wv, ss, L1, bits, spec.inv_scale, st["relu"], y1, pix, nthreads,
                                 y_uns=net.in_uns)
        if not ok:
            bad.append(("conv1", d))
        ok, d = check.check_pool(y1, L1.K, st["pool"], bits, host(net.net_in), nthreads, uns=net.in_uns)
        if not ok:
            bad.append(("maxpool", d))
    for i, c in enumerate(net.convs):
        L = c.layer
        pix = check.sample_pixels(len(imgs), L.P, L.Q, g, n_rand)
        sk = net.skip_tensor(i)
        ok, d = check.check_conv(host(net.src_tensor(i)), c.w.cpu().numpy(), c.ss.cpu().numpy(), L, bits, c.relu,
                                 host(c.y), pix, nthreads, skip=None if sk is None else host(sk),
                                 res_scale=c.res_scale, x_uns=c.plan.x_uns, y_uns=c.plan.y_uns,
                                 skip_uns=c.plan.skip_uns)
        if not ok:
            bad.append((c.name, d))
    return not bad, bad


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2202_06819_b200 as cq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    cq.load()

    spec = workload_spec(args.workload)
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    B_arg = args.batch or spec.batch
    B_global, B, img0 = shard_plan(B_arg, world, rank, scaling)

    # ---- setup (off the timed path): weights, scales, plans, buffers, tuning
    # completion-counter dataflow between conv launches: measured faster only for
    # the latency-bound tiny batches (ResNet-18 b1 0.095 vs 0.101 ms, ResNet-50 b1
    # 0.214 vs 0.220); equal at b256, slower at b32 (DESIGN 6) -> on for B <= 4
    dataflow = (B <= 4) if args.dataflow == "auto" else args.dataflow == "on"
    net = build_network(spec, B, dev, world, dist, dataflow=dataflow)
    stream = torch.cuda.Stream(dev)          # all work (and graph capture) on one side stream
    torch.cuda.set_stream(stream)
    net.set_stream(stream)
    g = wl.rng(spec.cfg_id, 1000)
    x_all = wl.fp16_activations(g, B_global, *tuple(net.x_in.shape[1:]))   # the global batch, this rank's shard
    net.x_in.copy_(torch.from_numpy(x_all[img0:img0 + B]))
    tuned = {} if args.no_tune else net.tune(warmup=2, reps=10, search_trials=args.search)
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        net.step(stream)
    torch.cuda.synchronize()

    # ---- CUDA graphs: the timed steps replay the plain graph (one launch per
    # kernel, PDL between them); per-launch events live in separate graphs
    # replayed after the timed window
    nl = net.launches_per_step
    n_ev = max(3, min(args.steps, 20))
    evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(nl + 1)] for _ in range(n_ev)]

    def ev_step(e):
        k = [0]
        e[0].record(stream)

        def cb(tag):
            k[0] += 1
            e[k[0]].record(stream)
        net.step(stream, cb)

    # conv-chain window: events only at the step start, after the input stage and
    # at the step end, so the conv launches between them keep their PDL overlap
    # exactly as in the plain graph (the roofline's kernel time)
    n_in_st = len(net.stage_names)
    evc = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)] for _ in range(n_ev)]

    def chain_step(e):
        k = [0]
        e[0].record(stream)

        def cb(tag):
            k[0] += 1
            if k[0] == n_in_st:
                e[1].record(stream)
        net.step(stream, cb)
        e[2].record(stream)

    use_graph = not args.no_graph
    graph, graphs_ev, graphs_ch = None, None, None
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                net.step(stream)
            graphs_ev = []
            for e in evs:
                ge = torch.cuda.CUDAGraph()
                with torch.cuda.graph(ge, stream=stream):
                    ev_step(e)
                graphs_ev.append(ge)
            graphs_ch = []
            for e in evc:
                gc = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gc, stream=stream):
                    chain_step(e)
                graphs_ch.append(gc)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # fall back to eager launches
            print(f"[bench] CUDA graph capture failed ({ex}); eager launches", file=sys.stderr)
            use_graph, graph, graphs_ev, graphs_ch = False, None, None, None
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)] for _ in range(n_ev)]
            evc = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_ev)]

    # ---- timed region: exactly K plain steps, barrier + sync on both sides
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local % ndev)
    time.sleep(0.2)
    t0.record(stream)
    for _ in range(args.steps):
        if use_graph:
            graph.replay()
        else:
            net.step(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_per_step = max_over_ranks(t0.elapsed_time(t1), world, dist, dev) / args.steps

    # ---- per-launch durations: a separate window of event-instrumented replays
    for j in range(n_ev):
        if use_graph:
            graphs_ev[j].replay()
        else:
            ev_step(evs[j])
    for j in range(n_ev):
        if use_graph:
            graphs_ch[j].replay()
        else:
            chain_step(evc[j])
    torch.cuda.synchronize()
    chain_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evc)
    per_launch_ms = [statistics.mean(e[k].elapsed_time(e[k + 1]) for e in evs) for k in range(nl)]
    ev_step_ms = statistics.mean(e[0].elapsed_time(e[nl]) for e in evs)
    n_in = len(net.stage_names)
    in_ms = dict(zip(net.stage_names, per_launch_ms[:n_in]))
    per_layer_ms = per_launch_ms[n_in:]

    # ---- graph-timed per-layer times (each conv alone: `reps` back-to-back launches in
    # one CUDA graph, PDL between them as in the chain -- no event between launches)
    graph_layer_us = net.time_layers(warmup=2, reps=20)

    # ---- e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None if args.no_e2e else run_e2e(args, net, stream, graph, use_graph, x_all[img0:img0 + B], world,
                                           dist, dev, B_global)

    gather = None
    if args.gather:
        gather = time_gather(net.outputs[-1], world, dist, dev)

    # ---- roofline of the dominant kernel: the implicit-GEMM conv (all conv launches of a step)
    peaks, peak_src = measured_peaks()
    int8_peak_tops = 2.0 * peaks["bf16_tflops"]          # INT8 = 2 x bf16 (nominal 4.5 / 2.25 PF)
    hbm_peak = peaks["hbm_gbs"]
    bits = spec.bits
    conv_layers = [c.layer for c in net.convs]
    # the conv launches of a step: the layer chain timed as one PDL-overlapped
    # segment (conv-chain window) + conv1 from the per-launch window
    conv_ms = chain_ms + in_ms.get("stem", 0.0)
    ops_step = sum(layer_ops(L, B) for L in conv_layers) + (layer_ops(spec.conv1, B) if net.stem else 0)
    bytes_step = sum(layer_bytes(L, B, bits) for L in conv_layers)
    achieved_tops = ops_step / (conv_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_step")
        except Exception:
            traffic = None
    layer_rows = []
    ideal_sum = 0.0
    for i, c in enumerate(net.convs):
        L = c.layer
        ops, by = layer_ops(L, B), layer_bytes(L, B, bits)
        ideal = max(ops / (int8_peak_tops * 1e12), by / (hbm_peak * 1e9)) * 1e3
        ideal_sum += ideal
        t = per_layer_ms[i]
        tg = graph_layer_us[i] * 1e-3
        layer_rows.append({"layer": L.name, "shape": f"{L.H}x{L.W} {L.C}->{L.K} {L.R}x{L.S} s{L.stride}",
                           "config": c.plan.info().config,
                           "graph_us": round(graph_layer_us[i], 2), "graph_roofline_frac": round(ideal / tg, 3),
                           "graph_tops": round(ops / (tg * 1e-3) / 1e12, 1),
                           "us": round(t * 1e3, 2),
                           "tops": round(ops / (t * 1e-3) / 1e12, 1),
                           "frac_int8_peak": round(ops / (t * 1e-3) / 1e12 / int8_peak_tops, 3),
                           "gbs": round(by / (t * 1e-3) / 1e9, 1),
                           "bound": "tensor" if ops / by > int8_peak_tops * 1e12 / (hbm_peak * 1e9) else "hbm",
                           "roofline_frac": round(ideal / t, 3)})

    stem = None
    if net.stem is not None:
        L1, P1 = spec.conv1, net.stem["plan"]
        s2d_bytes = B * (L1.H * L1.W * L1.C * 2 + P1.x_bytes // B)
        y1_bytes = B * P1.P * P1.Q * L1.K * bits // 8
        pool_bytes = y1_bytes + net.net_in.numel()
        stem = {"layer": f"{L1.name} {L1.R}x{L1.S}/{L1.stride} {L1.C}->{L1.K} as s2d stride-1 window conv + "
                         f"maxpool {spec.pool[0]}x{spec.pool[0]}/{spec.pool[1]}",
                "s2d_quantize_us": round(in_ms["s2d"] * 1e3, 2),
                "s2d_quantize_gbs": round(s2d_bytes / (in_ms["s2d"] * 1e-3) / 1e9, 1),
                "conv_us": round(in_ms["stem"] * 1e3, 2),
                "conv_useful_tops": round(layer_ops(L1, B) / (in_ms["stem"] * 1e-3) / 1e12, 1),
                "maxpool_us": round(in_ms["pool"] * 1e3, 2),
                "maxpool_gbs": round(pool_bytes / (in_ms["pool"] * 1e-3) / 1e9, 1),
                "config": P1.info().config}

    k7 = None
    if rank == 0 and not args.no_k7:
        try:
            k7 = round(cq.int8_peak(200000) / 1e12, 1)
        except Exception as ex:  # measurement only
            k7 = f"failed: {ex}"

    # ---- parity leg (host oracle, after every timed window): first and last image of this rank's shard
    parity = None
    if not args.no_parity:
        net.step(stream)
        torch.cuda.synchronize()
        t = time.perf_counter()
        ok, bad = parity_check(net, spec, sorted({0, B - 1}), n_rand=args.parity_pixels)
        ok_all = min_over_ranks(1.0 if ok else 0.0, world, dist, dev) == 1.0
        parity = {"parity_ok": ok_all, "images_checked": f"first and last image of every rank's shard",
                  "launches_checked": net.launches_per_step - (1 if net.stem is not None else 0),
                  "failures": [f"{n}: {d}" for n, d in bad[:5]], "seconds": round(time.perf_counter() - t, 1)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(spec, B, budget_s=args.cpu_budget)

    if rank == 0:
        quant_ms = in_ms.get("quantize") or in_ms.get("s2d")
        line = {
            "metric": spec.metric, "value": round(B_global / (ms_per_step * 1e-3), 2), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": f"int{bits}",
            "data": "synthetic (seeded N(0,1) fp16 images, uniform weight codes, random-init ResNet shapes)",
            "config": {"workload": args.workload, "description": spec.desc, "per_gpu_batch": B,
                       "global_batch": B_global, "bits": bits, "conv_layers_per_step": len(net.convs) + bool(net.stem),
                       "kernels_per_step": nl, "input": net.input_desc, "parallelism": f"batch-shard dp{world}",
                       "l2": "inputs larger than L2: per-step working set %.2f GB >> 126 MB L2" % (
                           (bytes_step + net.x_in.numel() * 2) / 1e9),
                       "launch": ("CUDA graph per step (PDL between kernels" +
                                  (", per-row dataflow flags between conv launches)" if net.dataflow else ")"))
                                 if use_graph else "eager launches",
                       "timed_window": "plain graph replays only; conv-chain and per-launch events in separate windows"},
            "conv_tops": round(achieved_tops, 1),
            "conv_frac_int8_peak": round(achieved_tops / int8_peak_tops, 3),
            "int8_peak_k7_tops": k7,
            "step_roofline_frac": round(ideal_sum / sum(per_layer_ms), 3),
            "graph_layers_sum_ms": round(sum(graph_layer_us) * 1e-3, 4),
            "graph_step_roofline_frac": round(ideal_sum / (sum(graph_layer_us) * 1e-3), 3),
            "roofline": {"bound": "tensor", "achieved": round(achieved_tops, 1), "peak": round(int8_peak_tops, 1),
                         "unit": "TOPS", "frac": round(achieved_tops / int8_peak_tops, 4),
                         "traffic": traffic, "kernel": "conv_igemm_kernel (all conv launches of one step, conv1 incl.)",
                         "algorithmic_ops_per_step": ops_step, "algorithmic_bytes_per_step": bytes_step,
                         "kernel_ms_per_step": round(conv_ms, 4),
                         "kernel_ms_source": f"conv chain ({len(net.convs)} launches, PDL intact) between two CUDA events on the "
                                             "launch stream + conv1's per-launch event time",
                         "per_launch_sum_ms": round(sum(per_layer_ms) + in_ms.get("stem", 0.0), 4),
                         "event_window_ms_per_step": round(ev_step_ms, 4),
                         "peak_source": f"2 x bf16_tflops of MEASURED_PEAKS.json ({peak_src}, burst)"},
            "quantize": {"ms": round(quant_ms, 4), "kernel": net.stage_names[0]},
            "gpu_launches": args.steps * nl,
            "clocks": clocks, "e2e": e2e, "stem": stem, "gather": gather, "parity": parity,
            "parity_ok": None if parity is None else parity["parity_ok"],
            "tuned": len(tuned), "tuning": f"search({args.search})" if args.search else "exhaustive", "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
        if args.layers_out:
            with open(args.layers_out, "w") as f:
                json.dump({"workload": args.workload, "layers": layer_rows, "input_stage_ms": in_ms,
                           "clocks": clocks, "tuned": tuned}, f, indent=1)
        for r in layer_rows:
            print("  %-10s %-22s %-34s %8.1fus (graph %7.1fus) %7.1f TOPS %5.1f%% peak %7.1f GB/s %-6s rf=%.2f "
                  "graph rf=%.2f" % (
                      r["layer"], r["shape"], r["config"], r["us"], r["graph_us"], r["tops"], 100 * r["frac_int8_peak"],
                      r["gbs"], r["bound"], r["roofline_frac"], r["graph_roofline_frac"]), file=sys.stderr)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, net, stream, graph, use_graph, x_host_np, world, dist, dev, B_global):
    """End to end through the public API with host buffers: every step copies its
    fp16 images H2D from pinned memory and its last output D2H, inside the timed
    region.  The copies run on two copy streams (uploads, downloads),
    double-buffered, so step i+1's upload and step i's download overlap each
    other and the compute of step i (the compute is the same CUDA graph as the
    device-only number, one per buffer pair)."""
    import torch
    h_in = torch.from_numpy(x_host_np).pin_memory()
    y_last = net.outputs[-1]
    h_out = [torch.empty(y_last.shape, dtype=torch.uint8).pin_memory() for _ in range(2)]
    x_bufs = [net.x_in, torch.empty_like(net.x_in)]
    o_bufs = [y_last, torch.empty_like(y_last)]
    pipelined = use_graph
    graphs = None
    if pipelined:
        saved_x, saved_o = net.x_in, net.convs[-1].y
        net.x_in, net.convs[-1].y = x_bufs[1], o_bufs[1]
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=stream):
            net.step(stream)
        net.x_in, net.convs[-1].y = saved_x, saved_o
        graphs = [graph, g2]
    # uploads and downloads on two copy streams (separate copy engines: the H2D of
    # step i+1 and the D2H of step i move in opposite directions over the host link
    # at the same time, both overlapped with step i's compute)
    cs_in, cs_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]
    ev_dl = [torch.cuda.Event(), torch.cuda.Event()]

    def steps(k):
        if not pipelined:                       # serial fallback (eager launches)
            for _ in range(k):
                net.x_in.copy_(h_in, non_blocking=True)
                net.step(stream)
                h_out[0].copy_(y_last, non_blocking=True)
            return
        cs_in.wait_stream(stream)
        cs_out.wait_stream(stream)
        with torch.cuda.stream(cs_in):
            x_bufs[0].copy_(h_in, non_blocking=True)
        ev_in[0].record(cs_in)
        for i in range(k):
            b = i % 2
            if i + 1 < k:                       # upload step i+1's input now
                with torch.cuda.stream(cs_in):
                    if i >= 1:
                        cs_in.wait_event(ev_done[1 - b])   # step i-1 released input buffer 1-b
                    x_bufs[1 - b].copy_(h_in, non_blocking=True)
                ev_in[1 - b].record(cs_in)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_dl[b])     # step i-2's result left output buffer b
            graphs[b].replay()
            ev_done[b].record(stream)
            with torch.cuda.stream(cs_out):     # download step i's result
                cs_out.wait_event(ev_done[b])
                h_out[b].copy_(o_bufs[b], non_blocking=True)
            ev_dl[b].record(cs_out)
        stream.wait_stream(cs_in)
        stream.wait_stream(cs_out)

    steps(4)
    torch.cuda.synchronize()
    k = max(3, min(args.steps, 50))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    steps(k)
    e1.record(stream)
    torch.cuda.synchronize()
    te = max_over_ranks(e0.elapsed_time(e1) / k, world, dist, dev)
    return {"value": round(B_global / (te * 1e-3), 2), "unit": UNIT,
            "h2d_bytes_per_step": int(h_in.numel() * h_in.element_size()),
            "d2h_bytes_per_step": int(h_out[0].numel()), "ms_per_step": round(te, 4),
            "copies": "double-buffered; H2D and D2H on two copy streams, overlapped with each other and the compute"
                      if pipelined
                      else "serial"}


def time_gather(y_last, world, dist, dev):
    """The optional final gather: the ranks' last-layer packed
    outputs concatenated with one all_gather over NVLink, timed separately
    from the compute (no collective inside the step)."""
    import torch
    for _ in range(3):
        out = gather_outputs(y_last, world, dist)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(torch.cuda.current_stream())
    for _ in range(10):
        out = gather_outputs(y_last, world, dist)
    g1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    tg = max_over_ranks(g0.elapsed_time(g1) / 10, world, dist, dev)
    return {"ms": round(tg, 4), "bytes_total": int(out.numel()),
            "op": "all_gather_into_tensor" if world > 1 else "copy (1 rank)"}


# ---------------------------------------------------------------------------- CPU oracle
def _oracle_layers(spec: Spec):
    """The conv layers the oracle computes for one image (conv1 over its
    channel-padded input, as the oracle's direct convolution runs it)."""
    import oracle
    layers = [t[0] for t in spec.layers]
    if spec.conv1 is not None:
        L1 = spec.conv1
        layers = [wl.Layer(L1.name, L1.H, L1.W, oracle.padded_channels(L1.C, spec.bits), L1.K, L1.R, L1.S,
                           L1.stride, L1.pad)] + layers
    return layers


def _oracle_sample(layers, bits, frac, g):
    """Per-layer sample: random packed inputs for one image and a fraction
    `frac` of the layer's output pixels (all K channels)."""
    sample = []
    for i, L in enumerate(layers):
        x, w, ss = wl.layer_inputs(wl.rng(4, 5000 + i), L, 1, bits)
        npix = max(1, int(round(frac * L.P * L.Q)))
        pix = np.sort(g.choice(L.P * L.Q, size=npix, replace=False)).astype(np.int64)
        sample.append((L, x, w, ss, pix))
    return sample


def _oracle_step(sample, bits, nthreads):
    import oracle
    macs = 0
    for (L, x, w, ss, pix) in sample:
        oracle.conv_q(x, w, L.C, L.stride, L.pad, bits, ss, True, pix=pix, nthreads=nthreads)
        macs += pix.size * L.K * L.C * L.R * L.S
    return macs


def _per_image_macs(layers):
    return sum(L.P * L.Q * L.K * L.C * L.R * L.S for L in layers)


def cpu_baseline(spec: Spec, B, budget_s=15.0):
    """The oracle, as it stands, on the host cores over a bounded sample (all
    cores, and one thread on a tenth of the budget)."""
    import oracle
    oracle.build()
    layers = _oracle_layers(spec)
    nthreads = oracle.default_threads()
    g = np.random.default_rng(7)
    per_image = _per_image_macs(layers)

    def timed(nt, budget):
        # grow the sample until it takes about `budget` seconds (10-30 s of CPU work by default)
        frac = 0.01
        while True:
            reps = max(1, int(frac))
            sample = _oracle_sample(layers, spec.bits, min(frac, 1.0), g)
            t = time.perf_counter()
            macs = sum(_oracle_step(sample, spec.bits, nt) for _ in range(reps))
            dt = time.perf_counter() - t
            if dt >= 0.5 * budget or frac >= 256:
                break
            frac *= min(16.0, max(2.0, budget / max(dt, 1e-3)))
        desc = (f"{reps} image(s), every output pixel of every layer" if frac >= 1 else
                f"{frac * 100:.2f}% of the output pixels of every layer of one image")
        return macs / per_image / dt, f"{desc} ({macs / 1e9:.2f} GMAC in {dt:.1f} s)", dt

    v, desc, dt = timed(nthreads, budget_s)
    v1, desc1, dt1 = timed(1, budget_s / 10)
    return {"value": round(v, 4), "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{desc}, extrapolated to images/s (all {len(layers)} conv layers incl. conv1 on its "
                      f"channel-padded input)",
            "seconds": round(dt, 2), "value_1thread": round(v1, 4), "sample_1thread": desc1}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    spec = workload_spec(args.workload)
    layers = _oracle_layers(spec)
    nthreads = oracle.default_threads()
    per_image = _per_image_macs(layers)
    g = np.random.default_rng(8)
    probe = _oracle_sample(layers, spec.bits, 0.002, g)
    t = time.perf_counter()
    m = _oracle_step(probe, spec.bits, nthreads)
    rate = m / (time.perf_counter() - t)
    per_step_s = args.ref_budget / max(1, args.steps + args.warmup)
    frac = min(1.0, max(0.0005, per_step_s * rate / per_image))
    sample = _oracle_sample(layers, spec.bits, frac, g)
    for _ in range(args.warmup):
        _oracle_step(sample, spec.bits, nthreads)
    t = time.perf_counter()
    macs = 0
    for _ in range(args.steps):
        macs += _oracle_step(sample, spec.bits, nthreads)
    dt = time.perf_counter() - t
    value = macs / per_image / dt
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    line = {"impl": "reference", "metric": spec.metric, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": f"int{spec.bits}",
            "data": "synthetic", "config": {"workload": args.workload, "description": spec.desc,
                                            "per_gpu_batch": spec.batch, "bits": spec.bits},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": f"per step {frac * 100:.3f}% of the output pixels of every layer of one "
                                       f"image, extrapolated to whole images"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50_int8_b256",
                    choices=[w + r + u for w in ("resnet50_int8_b256", "resnet18_int8_b1", "resnet18_int4_b16")
                             for r in ("", RES_SUFFIX) for u in ("", UNS_SUFFIX)] + ["cfg1"])
    ap.add_argument("--batch", type=int, default=0, help="override the batch (global for strong scaling)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="strong (default for N > 1): the global batch is split across GPUs; "
                         "weak: every GPU runs its own batch")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: several ranks may share one GPU, for testing)")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--search", type=int, default=0,
                    help="tune the conv layers by the learned search over the enlarged space (NEXT-4) with this "
                         "many measurements per unique shape instead of timing every TileConfig")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--dataflow", default="auto", choices=["auto", "on", "off"],
                    help="completion counters between conv launches instead of whole-grid dependencies "
                         "(auto: on for per-GPU batch <= 4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-pixels", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k7", action="store_true", help="skip the tcgen05 kind::i8 peak microbenchmark")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--layers-out", default="")
    ap.add_argument("--gather", action="store_true",
                    help="also time the optional final all_gather of the last layer's output (reported separately)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
