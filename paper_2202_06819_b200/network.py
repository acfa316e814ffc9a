"""Layer-sequence executor for the quantized conv path (product code).

A ``ConvNet`` is one device's copy of a ResNet-shaped convolution network in
the packed layout the paper's epilogue produces (section 3.3:
"the output of one convolution layer is ... the input of the next"):

  input stage   either the stem -- fp16 image -> s2d quantize -> conv1 (stride-2
                7x7 as a stride-1 window conv, StemPlan) -> 3x3/2 max pool -- or a
                plain quantize + pack of an fp16 activation tensor (a1)
  conv layers   one ConvPlan per layer (a3-a6), each reading the packed output of
                an earlier layer (or the input stage), fused requantize + repack
                epilogue writing the next layer's packed NHWC input

Weights are packed once (a2), tile configs are picked per unique shape by
on-device timing (a7), and one ``step`` launches every kernel on one stream,
so the whole step can be captured as one CUDA graph.  Argument marshalling
and buffer ownership only: every step of the path runs in libconvq.so's
kernels; there is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import (ConvPlan, StemPlan, maxpool, pack_weights, quantize, padded_channels)


@dataclass
class _Conv:
    name: str
    layer: object           # has H, W, C, K, R, S, stride, pad, P, Q
    src: int                # index of the producing conv, -1 = the input stage's output
    relu: bool
    skip: object            # residual: index of the conv whose output is added (-1 = input stage), or None
    res_scale: float
    plan: ConvPlan
    w: object               # packed weights (device uint8)
    ss: object              # [scale | shift] (device float32)
    y: object               # packed output (device uint8)
    key: tuple = field(default=())


class ConvNet:
    """Quantized conv network on one device.

    net = ConvNet(batch, bits, device)
    net.set_stem(conv1, w_codes, ss, inv_scale)      # or net.set_quantize_input(H, W, C, inv_scale)
    for L, src in layers: net.add_conv(L, src, w_codes, ss, relu=True)
    net.tune(); net.step(stream)                      # net.x_in is the fp16 input, net.outputs the results
    """

    def __init__(self, batch: int, bits: int, device, stream=None, unsigned: bool = False,
                 dataflow: bool = True):
        """unsigned: every ReLU output is written as unsigned codes [0, 2^b - 1] and
        read as unsigned activations by its consumers (DESIGN reading 16).
        dataflow: consecutive conv launches synchronise through completion
        counters (conv_q_plan_set_deps) instead of whole-grid completion; the
        counters are zeroed at the start of every step."""
        import torch
        self.torch = torch
        self.B, self.bits, self.device = batch, bits, device
        self.unsigned = unsigned
        self.dataflow = dataflow
        self.flags = None         # int32 completion counter of every conv output (zeroed per step)
        self.stream = stream
        self.convs: list[_Conv] = []
        self.stem = None
        self.x_in = None
        self.input_desc = None
        self.net_in = None        # packed tensor the first conv reads (quantized input or pooled stem output)
        self._stages = []         # ("quantize" | "s2d" | "stem" | "pool", callable) in launch order

    # ------------------------------------------------------------- input stage
    def set_quantize_input(self, H: int, W: int, C: int, inv_scale: float):
        """a1 only: fp16 [B,H,W,C] -> packed [B,H,W,C'] (conv_q_quantize)."""
        t = self.torch
        self.x_in = t.empty((self.B, H, W, C), dtype=t.float16, device=self.device)
        Cp = padded_channels(C, self.bits)
        self.net_in = t.empty((self.B, H, W, Cp * self.bits // 8), dtype=t.uint8, device=self.device)
        self.inv_scale = inv_scale
        self.in_uns = False                           # quantized fp16 input: signed codes
        self._stages = [("quantize", lambda s: quantize(self.x_in, inv_scale, self.bits, out=self.net_in, stream=s))]
        self.input_desc = f"quantize fp16 [{self.B},{H},{W},{C}]"

    def set_stem(self, conv1, w_codes, ss, inv_scale: float, pool=(3, 2, 1), relu: bool = True):
        """conv1 through the s2d StemPlan (fused quantize + space-to-depth, then a
        stride-1 window conv) followed by an R x R max pool of its packed output."""
        t = self.torch
        L = conv1
        self.x_in = t.empty((self.B, L.H, L.W, L.C), dtype=t.float16, device=self.device)
        sp = StemPlan(self.B, L.H, L.W, L.C, L.K, L.R, L.S, L.pad, self.bits, relu=relu,
                      y_uns=self.unsigned and relu)
        self.in_uns = self.unsigned and relu          # format of the pooled stem output
        xs = t.empty(sp.x_dims, dtype=t.uint8, device=self.device)
        wp = sp.pack_weights(w_codes)
        y1 = t.empty((self.B, sp.P, sp.Q, L.K * self.bits // 8), dtype=t.uint8, device=self.device)
        pr, pst, ppad = pool
        Pp, Qp = (sp.P + 2 * ppad - pr) // pst + 1, (sp.Q + 2 * ppad - pr) // pst + 1
        self.net_in = t.empty((self.B, Pp, Qp, L.K * self.bits // 8), dtype=t.uint8, device=self.device)
        self.stem = dict(layer=L, plan=sp, xs=xs, w=wp, ss=ss, y=y1, pool=pool, inv_scale=inv_scale, relu=relu)
        self.inv_scale = inv_scale
        self._stages = [
            ("s2d", lambda s: sp.quantize(self.x_in, inv_scale, out=xs, stream=s)),
            ("stem", lambda s: sp.run(xs, wp, ss, y1, stream=s)),
            ("pool", lambda s: maxpool(y1, L.K, pr, pst, ppad, self.bits, out=self.net_in, stream=s,
                                       uns=self.in_uns)),
        ]
        self.input_desc = f"stem {L.name} {L.R}x{L.S}/{L.stride} {L.C}->{L.K} (s2d) + maxpool {pr}x{pr}/{pst}"

    # ------------------------------------------------------------- conv layers
    def add_conv(self, L, src: int, w_codes, ss, relu: bool = True, name: str | None = None,
                 skip: int | None = None, res_scale: float = 0.0) -> int:
        """One conv layer reading the output of conv `src` (-1: the input stage);
        with `skip`, the epilogue adds res_scale * (the output of conv `skip`)
        before ReLU / rounding (a ResNet block's residual, DESIGN reading 15)."""
        t = self.torch
        assert src < len(self.convs) and (skip is None or skip < len(self.convs))
        x_uns = self.in_uns if src < 0 else self.convs[src].plan.y_uns
        y_uns = self.unsigned and relu
        plan = ConvPlan(self.B, L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, self.bits, relu=relu,
                        x_uns=x_uns, y_uns=y_uns)
        wp = pack_weights(w_codes, self.bits)
        y = t.empty((self.B, L.P, L.Q, L.K * self.bits // 8), dtype=t.uint8, device=self.device)
        skip_uns = False
        if skip is not None:
            sk = self.net_in if skip < 0 else self.convs[skip].y
            assert tuple(sk.shape) == tuple(y.shape), (sk.shape, y.shape)
            skip_uns = self.in_uns if skip < 0 else self.convs[skip].plan.y_uns
            if skip_uns:
                plan.set_formats(x_uns, y_uns, True)
            plan.set_residual(sk, res_scale)
        key = (L.H, L.W, L.C, L.K, L.R, L.S, L.stride, L.pad, relu, skip is not None, x_uns, y_uns, skip_uns)
        self.convs.append(_Conv(name or getattr(L, "name", f"conv{len(self.convs)}"), L, src, relu, skip, res_scale,
                                plan, wp, ss, y, key))
        return len(self.convs) - 1

    def skip_tensor(self, i: int):
        s = self.convs[i].skip
        return None if s is None else (self.net_in if s < 0 else self.convs[s].y)

    def src_tensor(self, i: int):
        s = self.convs[i].src
        return self.net_in if s < 0 else self.convs[s].y

    @property
    def outputs(self):
        return [c.y for c in self.convs]

    def set_stream(self, stream):
        self.stream = stream
        for c in self.convs:
            c.plan.set_stream(stream)
        if self.stem is not None:
            self.stem["plan"].set_stream(stream)

    # ------------------------------------------------------------- a7 tuning
    # ------------------------------------------------------------- dataflow counters
    def _apply_deps(self, on: bool):
        """Completion counters of every conv (conv_q_plan_set_deps): conv i adds the
        codes it wrote to self.flags[i]; it waits for its source's count (not for the
        input stage's: that one is waited for as a whole grid) and its skip's."""
        t = self.torch
        if on and self.flags is None:
            self.flags = t.zeros(len(self.convs), dtype=t.int32, device=self.device)
        for i, c in enumerate(self.convs):
            if not on:
                c.plan.set_deps(None, None, None)
                continue
            f = self.flags
            c.plan.set_deps(f[c.src:c.src + 1] if c.src >= 0 else None,
                            f[c.skip:c.skip + 1] if (c.skip is not None and c.skip >= 0) else None, f[i:i + 1])

    def tune(self, warmup: int = 2, reps: int = 5, search_trials: int = 0) -> dict:
        """Pick each unique shape's tile config by on-device timing (conv_q_plan_tune),
        on the network's real buffers (the input stage is run once first).
        search_trials > 0: the conv layers use the learned search over the enlarged
        space instead (conv_q_plan_search, NEXT-4) with that many measurements."""
        self._apply_deps(False)          # layers timed standalone: no flags
        self.run_input_stage(self.stream)
        if self.stem is not None:
            st = self.stem
            st["plan"].tune(st["xs"], st["w"], st["ss"], st["y"], warmup=warmup, reps=reps, stream=self.stream)
            self.run_input_stage(self.stream)
        picks = {}
        for i, c in enumerate(self.convs):
            if c.key in picks:
                if search_trials > 0:
                    c.plan.set_point(picks[c.key][2])   # TileConfig + runtime knobs of the searched pick
                else:
                    c.plan.set_config(picks[c.key][0])
            else:
                if search_trials > 0:
                    c.plan.search(self.src_tensor(i), c.w, c.ss, c.y, warmup=warmup, reps=reps, stream=self.stream,
                                  trials=search_trials)
                    idx = c.plan.info().config_index
                else:
                    idx = c.plan.tune(self.src_tensor(i), c.w, c.ss, c.y, warmup=warmup, reps=reps, stream=self.stream)
                picks[c.key] = (idx, c.plan.info().config, c.plan.get_point() if search_trials > 0 else None)
        self.torch.cuda.synchronize(self.device)
        if self.dataflow:
            self._apply_deps(True)
        return {str(k): v[1] for k, v in picks.items()}

    def time_layers(self, warmup: int = 2, reps: int = 20) -> list[float]:
        """Graph-timed microseconds per launch of every conv on the network's real
        buffers (conv_q_plan_time: `reps` back-to-back launches captured in a CUDA
        graph, PDL between them as in the chain; median of 3 replays).  Outputs are
        rewritten with identical bytes."""
        self._apply_deps(False)
        us = [c.plan.time(self.src_tensor(i), c.w, c.ss, c.y, warmup=warmup, reps=reps, stream=self.stream)
              for i, c in enumerate(self.convs)]
        self.torch.cuda.synchronize(self.device)
        if self.dataflow:
            self._apply_deps(True)
        return us

    # ------------------------------------------------------------- execution
    def run_input_stage(self, stream=None, ev=None):
        s = stream if stream is not None else self.stream
        for j, (_, f) in enumerate(self._stages):
            f(s)
            if ev is not None:
                ev(("input", j))

    def step(self, stream=None, ev=None):
        """One pass of the whole hot path over the batch; ev(tag) is called after
        every launch (per-launch timing events), tag = ("input", j) or ("conv", i)."""
        s = stream if stream is not None else self.stream
        if self.dataflow:
            if self.flags is None:
                self._apply_deps(True)
            if hasattr(s, "cuda_stream"):
                with self.torch.cuda.stream(s):
                    self.flags.zero_()   # counters start at zero every step
            else:
                self.flags.zero_()
        self.run_input_stage(s, ev)
        for i, c in enumerate(self.convs):
            c.plan.run(self.src_tensor(i), c.w, c.ss, c.y, stream=s)
            if ev is not None:
                ev(("conv", i))

    @property
    def launches_per_step(self) -> int:
        return len(self._stages) + len(self.convs)

    @property
    def stage_names(self) -> list[str]:
        return [n for n, _ in self._stages]
