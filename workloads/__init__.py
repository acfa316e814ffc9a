"""Seeded synthetic inputs and ResNet layer tables.

This module is shared by the tests, bench.py and smoke() to feed BOTH the CUDA
path and the CPU oracle the same bytes.  It holds none of the method's
arithmetic: no quantize, pack, convolution or requantization happens here --
only random numbers drawn with numpy ``default_rng`` and the shapes of the
paper's workloads (ResNet convolution layers, section 1 and
PAPER.md:309 section 4.1 "3x3 ... convolution of each stage of ResNet50").

Input recipe:
  * seed = 6819 + 1000*config_id + layer_idx (numpy default_rng)
  * fp16 activations ~ N(0, 1)
  * packed operands: uniform random bytes, i.e. every s8 code uniform in
    [-128,127] and every s4 nibble uniform in [-8,7] (weights w ~ U{lo..hi})
  * scale[k] = 2^round(log2(target/sigma_acc)) * (1 + 0.25 u_k),
    sigma_acc = sqrt(Kg) * sigma_x * sigma_w; shift[k] ~ U[-2, 2]
    (targets sigma_y ~ 40 for s8, ~3 for s4: a few % saturate, ties occur)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

import numpy as np


def seed(config_id: int, layer_idx: int = 0) -> int:
    return 6819 + 1000 * config_id + layer_idx


def rng(config_id: int, layer_idx: int = 0) -> np.random.Generator:
    return np.random.default_rng(seed(config_id, layer_idx))


@dataclass(frozen=True)
class Layer:
    name: str
    H: int
    W: int
    C: int
    K: int
    R: int
    S: int
    stride: int
    pad: int

    @property
    def P(self) -> int:
        return (self.H + 2 * self.pad - self.R) // self.stride + 1

    @property
    def Q(self) -> int:
        return (self.W + 2 * self.pad - self.S) // self.stride + 1

    def macs(self, N: int) -> int:
        return N * self.P * self.Q * self.K * self.C * self.R * self.S

    def as_dict(self):
        return asdict(self)


# --------------------------------------------------------------------------
# layer tables (torchvision topologies at 224x224)
# --------------------------------------------------------------------------
def resnet18_conv1() -> Layer:
    return Layer("conv1", 224, 224, 3, 64, 7, 7, 2, 3)


def resnet18_layers():
    """The 19 convolutions of ResNet-18 after conv1, in execution order.

    Each entry is (layer, src) where src is the index of the layer whose output
    it consumes (-1 = the chain input, the packed 56x56x64 layer1 input).
    Downsample 1x1s consume their block's input (no residual add, no pooling:
    SURVEY 8(d) cfg2)."""
    out = []
    prev = -1
    chans = [(64, 56), (128, 28), (256, 14), (512, 7)]
    cin = 64
    hin = 56
    for li, (c, hw) in enumerate(chans):
        for b in range(2):
            stride = 2 if (li > 0 and b == 0) else 1
            blk_in = prev
            name = f"l{li+1}.b{b}"
            out.append((Layer(name + ".c1", hin, hin, cin, c, 3, 3, stride, 1), blk_in))
            c1 = len(out) - 1
            out.append((Layer(name + ".c2", hw, hw, c, c, 3, 3, 1, 1), c1))
            c2 = len(out) - 1
            if stride == 2:
                out.append((Layer(name + ".ds", hin, hin, cin, c, 1, 1, 2, 0), blk_in))
            prev = c2
            cin, hin = c, hw
    return out


def resnet50_layers():
    """The 52 convolutions of ResNet-50 v1.5 after conv1 (stride on the 3x3),
    in execution order, as (layer, src) pairs like resnet18_layers()."""
    out = []
    prev = -1
    stages = [(64, 3, 56), (128, 4, 28), (256, 6, 14), (512, 3, 7)]
    cin, hin = 64, 56
    for si, (width, nblk, hw) in enumerate(stages):
        for b in range(nblk):
            stride = 2 if (si > 0 and b == 0) else 1
            blk_in = prev
            name = f"l{si+1}.b{b}"
            out.append((Layer(name + ".c1", hin, hin, cin, width, 1, 1, 1, 0), blk_in))
            c1 = len(out) - 1
            out.append((Layer(name + ".c2", hin, hin, width, width, 3, 3, stride, 1), c1))
            c2 = len(out) - 1
            out.append((Layer(name + ".c3", hw, hw, width, 4 * width, 1, 1, 1, 0), c2))
            c3 = len(out) - 1
            if b == 0:
                out.append((Layer(name + ".ds", hin, hin, cin, 4 * width, 1, 1, stride, 0), blk_in))
            prev = c3
            cin, hin = 4 * width, hw
    return out


def resnet18_blocks():
    """ResNet-18 with its residual adds, in execution order: (layer, src, skip)
    triples -- skip is the index whose output the layer's epilogue adds (-1 =
    the layer1 input) or None.  Basic block: c1 -> [ds] -> c2 + (ds or block input)."""
    out = []
    prev = -1
    chans = [(64, 56), (128, 28), (256, 14), (512, 7)]
    cin, hin = 64, 56
    for li, (c, hw) in enumerate(chans):
        for b in range(2):
            stride = 2 if (li > 0 and b == 0) else 1
            blk_in = prev
            name = f"l{li+1}.b{b}"
            out.append((Layer(name + ".c1", hin, hin, cin, c, 3, 3, stride, 1), blk_in, None))
            c1 = len(out) - 1
            ident = blk_in
            if stride == 2:
                out.append((Layer(name + ".ds", hin, hin, cin, c, 1, 1, 2, 0), blk_in, None))
                ident = len(out) - 1
            out.append((Layer(name + ".c2", hw, hw, c, c, 3, 3, 1, 1), c1, ident))
            prev = len(out) - 1
            cin, hin = c, hw
    return out


def resnet50_blocks():
    """ResNet-50 v1.5 with its residual adds, as (layer, src, skip) triples like
    resnet18_blocks().  Bottleneck: c1 -> c2 -> [ds] -> c3 + (ds or block input)."""
    out = []
    prev = -1
    stages = [(64, 3, 56), (128, 4, 28), (256, 6, 14), (512, 3, 7)]
    cin, hin = 64, 56
    for si, (width, nblk, hw) in enumerate(stages):
        for b in range(nblk):
            stride = 2 if (si > 0 and b == 0) else 1
            blk_in = prev
            name = f"l{si+1}.b{b}"
            out.append((Layer(name + ".c1", hin, hin, cin, width, 1, 1, 1, 0), blk_in, None))
            c1 = len(out) - 1
            out.append((Layer(name + ".c2", hin, hin, width, width, 3, 3, stride, 1), c1, None))
            c2 = len(out) - 1
            ident = blk_in
            if b == 0:
                out.append((Layer(name + ".ds", hin, hin, cin, 4 * width, 1, 1, stride, 0), blk_in, None))
                ident = len(out) - 1
            out.append((Layer(name + ".c3", hw, hw, width, 4 * width, 1, 1, 1, 0), c2, ident))
            prev = len(out) - 1
            cin, hin = 4 * width, hw
    return out


def res_scale(g: np.random.Generator) -> float:
    """The fp32 scale of a residual add's skip codes (uniform in [0.25, 0.75])."""
    return float(np.float32(g.uniform(0.25, 0.75)))


def paper_table1_layers():
    """PAPER.md:319-331 Table 1: the 3x3 s1 p1 convolutions of ResNet-50
    stages 2-5 (K = C), quoted at N = 8."""
    return [Layer("stage2", 56, 56, 64, 64, 3, 3, 1, 1),
            Layer("stage3", 28, 28, 128, 128, 3, 3, 1, 1),
            Layer("stage4", 14, 14, 256, 256, 3, 3, 1, 1),
            Layer("stage5", 7, 7, 512, 512, 3, 3, 1, 1)]


CFG1 = Layer("cfg1.l1.3x3", 56, 56, 64, 64, 3, 3, 1, 1)


# --------------------------------------------------------------------------
# generators (random numbers only)
# --------------------------------------------------------------------------
def fp16_activations(g: np.random.Generator, N: int, H: int, W: int, C: int) -> np.ndarray:
    return g.standard_normal((N, H, W, C), dtype=np.float32).astype(np.float16)


def random_bytes(g: np.random.Generator, shape) -> np.ndarray:
    """Uniform random bytes: a packed tensor whose codes are uniform over the
    whole signed range (s8 bytes, or two s4 nibbles per byte)."""
    return g.integers(0, 256, size=shape, dtype=np.uint8)


def weight_values(g: np.random.Generator, K: int, R: int, S: int, C: int, bits: int) -> np.ndarray:
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    return g.integers(lo, hi + 1, size=(K, R, S, C), dtype=np.int8)


def uniform_code_std(bits: int) -> float:
    """Standard deviation of a code uniform over [-2^(b-1), 2^(b-1)-1]."""
    n = 1 << bits
    return math.sqrt((n * n - 1) / 12.0)


def scale_shift(g: np.random.Generator, K: int, Kg: int, sigma_x: float, sigma_w: float,
                bits: int) -> np.ndarray:
    """[scale_0..scale_{K-1}, shift_0..shift_{K-1}] as float32 (recipe above)."""
    target = 40.0 if bits == 8 else 3.0
    sigma_acc = math.sqrt(Kg) * sigma_x * sigma_w
    base = 2.0 ** round(math.log2(target / sigma_acc))
    u = g.random(K)
    scale = (base * (1.0 + 0.25 * u)).astype(np.float32)
    shift = g.uniform(-2.0, 2.0, K).astype(np.float32)
    return np.concatenate([scale, shift]).astype(np.float32)


def layer_inputs(g: np.random.Generator, layer: Layer, N: int, bits: int):
    """(x packed bytes [N,H,W,C*b/8], w packed bytes [K,R,S,C*b/8], scale_shift)."""
    nb = layer.C * bits // 8
    x = random_bytes(g, (N, layer.H, layer.W, nb))
    w = random_bytes(g, (layer.K, layer.R, layer.S, nb))
    sd = uniform_code_std(bits)
    ss = scale_shift(g, layer.K, layer.R * layer.S * layer.C, sd, sd, bits)
    return x, w, ss


def shard_batch(global_batch: int, world: int, rank: int):
    """Contiguous batch shard of `rank`: n_i = floor(N/g) + [i < N mod g].
    Returns (first image, image count)."""
    base, extra = divmod(global_batch, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count
