#!/usr/bin/env python
"""bench.py -- throughput of the quantized implicit-GEMM convolution path on B200.

Default workload (BASELINE.json configs[3], the one its "images/s at
1/2/4/8 GPU" metric is quoted on): ResNet-50 v1.5 convolutions, INT8, batch
256 per GPU.  One step = one pass of the whole hot path over one batch:
  a1  quantize + pack the fp16 layer-1 input [B,56,56,64] (conv_q_quantize)
  a3-a6  all 52 convolutions of layer1..layer4 through conv_q_run, each with
         the fused requantize + repack epilogue, each y the next x (downsample
         1x1s read their block input; no residual add / pooling)
The stem conv1 (C=3) is timed separately and reported in "stem" (it is not
part of the step): the s2d StemPlan (fused quantize +
space-to-depth, then a stride-1 window conv).  Weights are packed once (a2, off the
per-step path) and broadcast with one NCCL broadcast at setup; tile configs
are picked per shape by on-device timing (a7) at setup.

Multi-GPU (a8): one process per GPU under torchrun; every rank runs its own
batch of 256 images (weak scaling, no collective on the data path); the step
time is the max over ranks.

--impl reference times the CPU oracle (oracle/) on the host cores on a
bounded per-step sample of the same workload (sampled output pixels of every
layer), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as wl  # noqa: E402

METRIC = "images/s (ResNet-50 conv layers, INT8, fused requant-repack)"


def metric_name(workload: str) -> str:
    """BASELINE.json's images/s metric, labelled with the workload's network and precision."""
    if workload == "resnet50_int8_b256":
        return METRIC
    if workload == "resnet18_int8_b1":
        return "images/s (ResNet-18 conv layers, INT8, fused requant-repack)"
    if workload == "resnet18_int4_b16":
        return "images/s (ResNet-18 conv layers, INT4, fused requant-repack)"
    return "images/s (single INT8 conv 56x56x64->64 3x3, fused requant-repack)"
UNIT = "images/s"
L2_BYTES = 126 * 1024 * 1024


# ---------------------------------------------------------------------------- workloads
def workload_spec(name: str):
    """-> (layers [(Layer, src)], batch, bits, conv1 Layer or None, description)."""
    if name == "resnet50_int8_b256":
        return wl.resnet50_layers(), 256, 8, wl.resnet18_conv1(), "ResNet-50 v1.5 layer1-4 convs, INT8, batch 256/GPU"
    if name == "resnet18_int8_b1":
        return wl.resnet18_layers(), 1, 8, wl.resnet18_conv1(), "ResNet-18 layer1-4 convs, INT8, batch 1/GPU"
    if name == "resnet18_int4_b16":
        return wl.resnet18_layers(), 16, 4, wl.resnet18_conv1(), "ResNet-18 layer1-4 convs, INT4, batch 16/GPU"
    if name == "cfg1":
        return [(wl.CFG1, -1)], 1, 8, None, "single INT8 conv N=1 56x56x64->64 3x3"
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
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.proc = None
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
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2202_06819_b200 as cq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cq.load()

    layers, B, bits, conv1, desc = workload_spec(args.workload)
    if args.batch:
        B = args.batch
    B_global = B * world
    if args.scaling == "strong":      # the global batch is split across ranks
        B_global = B
        _, B = wl.shard_batch(B_global, world, rank)
    g = wl.rng(4, 1000 + rank)

    # ---- setup (off the timed path): weights, scales, plans, buffers
    weights, scales, plans, outs = [], [], [], []
    x_in_f16 = torch.from_numpy(wl.fp16_activations(g, B, 56, 56, 64)).to(dev)
    inv_scale = 127 / 4 if bits == 8 else 7 / 3
    for i, (L, src) in enumerate(layers):
        gi = wl.rng(4, i + 1)                         # same weights on every rank ...
        wv = torch.from_numpy(wl.weight_values(gi, L.K, L.R, L.S, L.C, bits)).to(dev)
        wp = cq.pack_weights(wv, bits)                 # a2: once per model
        sd = wl.uniform_code_std(bits)
        ss = torch.from_numpy(wl.scale_shift(gi, L.K, L.R * L.S * L.C, sd * 0.5, sd, bits)).to(dev)
        if world > 1:                                  # ... and replicated by one broadcast
            dist.broadcast(wp, 0)
            dist.broadcast(ss, 0)
        weights.append(wp)
        scales.append(ss)
        plans.append(cq.ConvPlan(B, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, bits, relu=True))
        outs.append(torch.empty((B, L.P, L.Q, L.K * bits // 8), dtype=torch.uint8, device=dev))
    xq = torch.empty((B, 56, 56, 64 * bits // 8), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(dev)          # all work (and graph capture) on one side stream
    torch.cuda.set_stream(stream)
    for p in plans:
        p.set_stream(stream)

    def src_of(i):
        s = layers[i][1]
        return xq if s < 0 else outs[s]

    # a7: per-shape tile config picked by timing (once per unique shape)
    tuned = {}
    cq.quantize(x_in_f16, inv_scale, bits, out=xq)
    for i, (L, _) in enumerate(layers):
        key = (L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad)
        if args.no_tune:
            continue
        if key in tuned:
            plans[i].set_config(tuned[key])
        else:
            tuned[key] = plans[i].tune(src_of(i), weights[i], scales[i], outs[i], warmup=2, reps=5)
    torch.cuda.synchronize()

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        cq.quantize(x_in_f16, inv_scale, bits, out=xq, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        for i in range(len(layers)):
            plans[i].run(src_of(i), weights[i], scales[i], outs[i], stream=stream)
            if ev is not None:
                ev[2 + i].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- CUDA graphs: one step = one graph launch (no per-kernel host launch
    # cost); a second set of graphs carries per-launch timing events (external
    # event-record nodes) for the per-layer / roofline numbers.
    n_ev_steps = min(args.steps, 20)                   # per-launch events on the last steps
    evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(layers) + 2)]
           for _ in range(n_ev_steps)]
    use_graph = not args.no_graph
    graph, graphs_ev = None, None
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            graphs_ev = []
            for e in evs:
                ge = torch.cuda.CUDAGraph()
                with torch.cuda.graph(ge, stream=stream):
                    step(e)
                graphs_ev.append(ge)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as ex:  # fall back to eager launches
            print(f"[bench] CUDA graph capture failed ({ex}); eager launches", file=sys.stderr)
            use_graph, graph, graphs_ev = False, None, None
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(layers) + 2)] for _ in range(n_ev_steps)]

    def run_step(j):
        """Timed step number j of the window (j >= 0: with per-launch events)."""
        if use_graph:
            (graphs_ev[j] if j >= 0 else graph).replay()
        else:
            step(evs[j] if j >= 0 else None)

    # ---- timed region: exactly K steps, barrier + sync on both sides
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    time.sleep(0.2)
    t0.record(stream)
    for s in range(args.steps):
        run_step(s - (args.steps - n_ev_steps))
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = t0.elapsed_time(t1)
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms_max = float(t_local.item())
    ms_per_step = total_ms_max / args.steps

    # per-launch durations (the events bracket each launch on its stream)
    per_layer_ms = [statistics.mean(e[1 + i].elapsed_time(e[2 + i]) for e in evs) for i in range(len(layers))]
    quant_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)

    # ---- e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        # End to end through the public API with host buffers: every step copies
        # its fp16 input H2D from pinned memory and its last output D2H, inside
        # the timed region.  The copies run on a copy stream, double-buffered, so
        # step i+1's input upload and step i's download overlap the compute of
        # step i (the compute itself is the same CUDA graph as the device-only
        # number, one per buffer pair).
        h_in = torch.from_numpy(wl.fp16_activations(g, B, 56, 56, 64)).pin_memory()
        h_out = [torch.empty(outs[-1].shape, dtype=torch.uint8).pin_memory() for _ in range(2)]
        x_bufs = [x_in_f16, torch.empty_like(x_in_f16)]
        o_bufs = [outs[-1], torch.empty_like(outs[-1])]
        pipelined = use_graph
        if pipelined:
            saved_x, saved_o = x_in_f16, outs[-1]
            x_in_f16, outs[-1] = x_bufs[1], o_bufs[1]
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=stream):
                step()
            x_in_f16, outs[-1] = saved_x, saved_o
            graphs_e2e = [graph, g2]
        cs = torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_steps(k):
            if not pipelined:                       # serial fallback (eager launches)
                for _ in range(k):
                    x_in_f16.copy_(h_in, non_blocking=True)
                    run_step(-1)
                    h_out[0].copy_(outs[-1], non_blocking=True)
                return
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                x_bufs[0].copy_(h_in, non_blocking=True)
            ev_in[0].record(cs)
            for i in range(k):
                b = i % 2
                if i + 1 < k:                       # upload step i+1's input now
                    with torch.cuda.stream(cs):
                        if i >= 1:
                            cs.wait_event(ev_done[1 - b])   # step i-1 released buffer pair 1-b
                        x_bufs[1 - b].copy_(h_in, non_blocking=True)
                    ev_in[1 - b].record(cs)
                stream.wait_event(ev_in[b])
                graphs_e2e[b].replay()
                ev_done[b].record(stream)
                with torch.cuda.stream(cs):         # download step i's result
                    cs.wait_event(ev_done[b])
                    h_out[b].copy_(o_bufs[b], non_blocking=True)
            stream.wait_stream(cs)

        e2e_steps(4)
        torch.cuda.synchronize()
        k_e2e = max(3, min(args.steps, 50))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        e2e_steps(k_e2e)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / k_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(B_global / (float(te.item()) * 1e-3), 2), "unit": UNIT,
               "h2d_bytes_per_step": int(h_in.numel() * h_in.element_size()),
               "d2h_bytes_per_step": int(h_out[0].numel()), "ms_per_step": round(float(te.item()), 4),
               "copies": "double-buffered on a copy stream, overlapped with the previous step" if pipelined
                         else "serial"}

    # ---- optional final gather: the ranks' last-layer packed
    # outputs concatenated on every rank with one NCCL all_gather over NVLink,
    # timed separately from the compute (no collective inside the step)
    gather = None
    if args.gather:
        y_last = outs[-1]
        y_all = torch.empty((world * y_last.shape[0],) + tuple(y_last.shape[1:]), dtype=y_last.dtype, device=dev)
        def do_gather():
            if world > 1:
                dist.all_gather_into_tensor(y_all, y_last)
            else:
                y_all.copy_(y_last)
        for _ in range(3):
            do_gather()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(torch.cuda.current_stream())
        for _ in range(10):
            do_gather()
        g1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1) / 10], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms": round(float(tg.item()), 4), "bytes_total": int(y_all.numel()),
                  "op": "all_gather_into_tensor (NCCL)" if world > 1 else "copy (1 rank)"}

    # ---- stem conv1 (timed separately, not part of the step):
    # the s2d StemPlan = fused quantize + space-to-depth of the fp16 image, then
    # the stride-1 window conv (no 3 -> 32 channel padding)
    stem = None
    if conv1 is not None and not args.no_stem:
        L1 = conv1
        xs = torch.from_numpy(wl.fp16_activations(g, B, L1.H, L1.W, L1.C)).to(dev)
        p1 = cq.StemPlan(B, L1.H, L1.W, L1.C, L1.K, L1.R, L1.S, L1.pad, bits, relu=True)
        p1.set_stream(stream)
        w1 = torch.from_numpy(wl.weight_values(wl.rng(4, 0), L1.K, L1.R, L1.S, L1.C, bits)).to(dev)
        ws = p1.pack_weights(w1)
        sd1 = wl.uniform_code_std(bits)
        ss1 = torch.from_numpy(wl.scale_shift(wl.rng(4, 0), L1.K, L1.R * L1.S * L1.C, sd1 * 0.5, sd1, bits)).to(dev)
        xsq = p1.quantize(xs, inv_scale)
        y1 = torch.empty((B, L1.P, L1.Q, L1.K * bits // 8), dtype=torch.uint8, device=dev)
        if not args.no_tune:
            p1.tune(xsq, ws, ss1, y1, warmup=2, reps=5)
        for _ in range(3):
            p1.quantize(xs, inv_scale, out=xsq, stream=stream)
            p1.run(xsq, ws, ss1, y1, stream=stream)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        qt, ct = [], []
        for _ in range(10):
            ev[0].record(stream)
            p1.quantize(xs, inv_scale, out=xsq, stream=stream)
            ev[1].record(stream)
            p1.run(xsq, ws, ss1, y1, stream=stream)
            ev[2].record(stream)
            torch.cuda.synchronize()
            qt.append(ev[0].elapsed_time(ev[1]))
            ct.append(ev[1].elapsed_time(ev[2]))
        q_ms, c_ms = statistics.median(qt), statistics.median(ct)
        ms = q_ms + c_ms
        stem = {"layer": "conv1 7x7 s2 3->64 as s2d stride-1 4x1 window conv (conv_q_plan_s2d)",
                "ms": round(ms, 4), "quantize_s2d_ms": round(q_ms, 4), "conv_ms": round(c_ms, 4),
                "useful_tops": round(layer_ops(L1, B) / (c_ms * 1e-3) / 1e12, 2),
                "images_per_s": round(B / (ms * 1e-3), 1), "config": p1.info().config}

    # ---- roofline of the dominant kernel: the implicit-GEMM conv (all launches of a step)
    peaks, peak_src = measured_peaks()
    int8_peak_tops = 2.0 * peaks["bf16_tflops"]          # INT8 = 2 x bf16 (nominal 4.5 / 2.25 PF)
    hbm_peak = peaks["hbm_gbs"]
    conv_ms = sum(per_layer_ms)
    ops_step = sum(layer_ops(L, B) for L, _ in layers)
    bytes_step = sum(layer_bytes(L, B, bits) for L, _ in layers)
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
    for i, (L, _) in enumerate(layers):
        ops, by = layer_ops(L, B), layer_bytes(L, B, bits)
        ideal = max(ops / (int8_peak_tops * 1e12), by / (hbm_peak * 1e9)) * 1e3
        ideal_sum += ideal
        t = per_layer_ms[i]
        layer_rows.append({"layer": L.name, "shape": f"{L.H}x{L.W} {L.C}->{L.K} {L.R}x{L.S} s{L.stride}",
                           "config": plans[i].info().config, "us": round(t * 1e3, 2),
                           "tops": round(ops / (t * 1e-3) / 1e12, 1),
                           "frac_int8_peak": round(ops / (t * 1e-3) / 1e12 / int8_peak_tops, 3),
                           "gbs": round(by / (t * 1e-3) / 1e9, 1),
                           "bound": "tensor" if ops / by > int8_peak_tops * 1e12 / (hbm_peak * 1e9) else "hbm",
                           "roofline_frac": round(ideal / t, 3)})

    k7 = None
    if rank == 0 and not args.no_k7:
        try:
            k7 = round(cq.int8_peak(200000) / 1e12, 1)
        except Exception as ex:  # measurement only
            k7 = f"failed: {ex}"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(layers, B, bits, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": metric_name(args.workload), "value": round(B_global / (ms_per_step * 1e-3), 2), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int8" if bits == 8 else "int4",
            "data": "synthetic (seeded N(0,1) fp16 input, uniform weight codes, random-init ResNet shapes)",
            "config": {"workload": args.workload, "description": desc, "per_gpu_batch": B,
                       "global_batch": B_global, "bits": bits, "conv_layers_per_step": len(layers),
                       "kernels_per_step": len(layers) + 1, "parallelism": f"batch-shard dp{world}",
                       "l2": "inputs larger than L2: per-step working set %.2f GB >> 126 MB L2" % (
                           (bytes_step + B * 56 * 56 * 64 * 2) / 1e9),
                       "stem_conv1": "timed separately (see stem)",
                       "launch": "CUDA graph per step" if use_graph else "eager launches"},
            "conv_tops": round(achieved_tops, 1),
            "conv_frac_int8_peak": round(achieved_tops / int8_peak_tops, 3),
            "int8_peak_k7_tops": k7,
            "step_roofline_frac": round(ideal_sum / conv_ms, 3),
            "roofline": {"bound": "tensor", "achieved": round(achieved_tops, 1), "peak": round(int8_peak_tops, 1),
                         "unit": "TOPS", "frac": round(achieved_tops / int8_peak_tops, 4),
                         "traffic": traffic, "kernel": "conv_igemm_kernel (all launches of one step)",
                         "algorithmic_ops_per_step": ops_step, "algorithmic_bytes_per_step": bytes_step,
                         "kernel_ms_per_step": round(conv_ms, 4),
                         "peak_source": f"2 x bf16_tflops of MEASURED_PEAKS.json ({peak_src}, burst)"},
            "quantize": {"ms": round(quant_ms, 4),
                         "gbs": round(B * 56 * 56 * 64 * (2 + bits / 8) / (quant_ms * 1e-3) / 1e9, 1),
                         "hbm_peak_gbs": hbm_peak},
            "gpu_launches": args.steps * (len(layers) + 1),
            "clocks": clocks, "e2e": e2e, "stem": stem, "gather": gather, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
        if args.layers_out:
            with open(args.layers_out, "w") as f:
                json.dump({"workload": args.workload, "layers": layer_rows, "quantize_ms": quant_ms,
                           "clocks": clocks}, f, indent=1)
        for r in layer_rows:
            print("  %-10s %-22s %-22s %8.1fus %7.1f TOPS %5.1f%% peak %7.1f GB/s %-6s rf=%.2f" % (
                r["layer"], r["shape"], r["config"], r["us"], r["tops"], 100 * r["frac_int8_peak"], r["gbs"],
                r["bound"], r["roofline_frac"]), file=sys.stderr)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------- CPU oracle
def _oracle_sample(layers, bits, frac, g):
    """Build a per-layer sample: random packed inputs for one image and a
    fraction `frac` of the layer's output pixels (all K channels)."""
    sample = []
    for i, (L, _) in enumerate(layers):
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


def cpu_baseline(layers, B, bits, budget_s=15.0, frac=None):
    """The oracle, as it stands, on the host cores over a bounded sample."""
    import oracle
    oracle.build()
    nthreads = oracle.default_threads()
    g = np.random.default_rng(7)
    per_image_macs = sum(L.P * L.Q * L.K * L.C * L.R * L.S for L, _ in layers)
    if frac is None:  # calibrate: ~budget_s of work
        probe = _oracle_sample(layers, bits, 0.02, g)
        t = time.perf_counter()
        m = _oracle_step(probe, bits, nthreads)
        dt = time.perf_counter() - t
        rate = m / dt
        frac = max(0.005, budget_s * rate / per_image_macs)
    reps = max(1, int(frac))                       # whole images beyond one
    sample = _oracle_sample(layers, bits, min(frac, 1.0), g)
    t = time.perf_counter()
    macs = 0
    for _ in range(reps):
        macs += _oracle_step(sample, bits, nthreads)
    dt = time.perf_counter() - t
    imgs = macs / per_image_macs
    desc = (f"{reps} image(s), every output pixel of every layer" if frac >= 1 else
            f"{frac * 100:.2f}% of the output pixels of every layer of one image")
    return {"value": round(imgs / dt, 4), "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{desc} ({macs / 1e9:.2f} GMAC in {dt:.1f} s), extrapolated to images/s",
            "seconds": round(dt, 2)}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    layers, B, bits, _, desc = workload_spec(args.workload)
    nthreads = oracle.default_threads()
    per_image_macs = sum(L.P * L.Q * L.K * L.C * L.R * L.S for L, _ in layers)
    g = np.random.default_rng(8)
    total_budget = args.ref_budget
    # calibrate the per-step sample so (warmup + steps) steps fit the budget
    probe = _oracle_sample(layers, bits, 0.002, g)
    t = time.perf_counter()
    m = _oracle_step(probe, bits, nthreads)
    rate = m / (time.perf_counter() - t)
    per_step_s = total_budget / max(1, args.steps + args.warmup)
    frac = min(1.0, max(0.0005, per_step_s * rate / per_image_macs))
    sample = _oracle_sample(layers, bits, frac, g)
    for _ in range(args.warmup):
        _oracle_step(sample, bits, nthreads)
    t = time.perf_counter()
    macs = 0
    for _ in range(args.steps):
        macs += _oracle_step(sample, bits, nthreads)
    dt = time.perf_counter() - t
    imgs = macs / per_image_macs
    value = imgs / dt
    line = {"impl": "reference", "metric": metric_name(args.workload), "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": f"int{bits}",
            "data": "synthetic", "config": {"workload": args.workload, "description": desc, "per_gpu_batch": B,
                                            "bits": bits},
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
                    choices=["resnet50_int8_b256", "resnet18_int8_b1", "resnet18_int4_b16", "cfg1"])
    ap.add_argument("--batch", type=int, default=0, help="override per-GPU batch")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU runs its own batch; strong: the batch is split across GPUs")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stem", action="store_true")
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
