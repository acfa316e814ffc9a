"""Sampled oracle checks of a whole network step (test infrastructure).

Used by tests/ and by bench.py's parity leg (after the timed region, never
inside it).  Every check recomputes sampled outputs of ONE layer with the CPU
oracle from that layer's actual input bytes (as produced on the device by the
previous layer), so a wrong byte anywhere in the chain is attributed to the
layer that produced it.  Inputs are numpy arrays copied from the device by the
caller; nothing here imports the product package.
"""
from __future__ import annotations

import numpy as np

from . import conv_q, maxpool, pack, padded_channels, quantize


def sample_pixels(n_img: int, P: int, Q: int, g: np.random.Generator, n_rand: int = 64) -> np.ndarray:
    """Linear output pixel indices (n*P + p)*Q + q over an n_img-image batch:
    the first and last pixel rows of the first and last image, both image
    corners, pixels around every 128-row tile boundary, and n_rand random ones."""
    M = n_img * P * Q
    idx = [np.arange(min(Q, M)), np.arange(max(0, M - Q), M), [0, Q - 1, (P - 1) * Q, P * Q - 1, M - 1]]
    for b in range(128, M, 128 * max(1, M // (128 * 16))):        # up to ~16 tile boundaries
        idx.append(np.arange(max(0, b - 2), min(M, b + 2)))
    idx.append(g.integers(0, M, n_rand))
    return np.unique(np.concatenate([np.asarray(a, np.int64) for a in idx]))


def first_diff(a: np.ndarray, b: np.ndarray):
    bad = np.argwhere(a != b)
    return None if bad.size == 0 else (tuple(int(i) for i in bad[0]), int(a[tuple(bad[0])]),
                                       int(b[tuple(bad[0])]), int(len(bad)))


def check_conv(x: np.ndarray, w: np.ndarray, ss: np.ndarray, L, bits: int, relu: bool, y: np.ndarray,
               pix: np.ndarray, nthreads: int | None = None, skip: np.ndarray | None = None,
               res_scale: float = 0.0, x_uns: bool = False, y_uns: bool = False, skip_uns: bool = False):
    """y (packed [n,P,Q,K*b/8] from the device) vs the oracle at pixels `pix`
    of the same n-image batch x (with `skip`: the residual epilogue, reading
    15, adding the device's own skip bytes; *_uns: unsigned code formats,
    reading 16).  Returns (ok, diff)."""
    ref = conv_q(x, w, L.C, L.stride, L.pad, bits, ss, relu, pix=pix, nthreads=nthreads, skip=skip,
                 res_scale=res_scale, x_uns=x_uns, y_uns=y_uns, skip_uns=skip_uns)
    got = y.reshape(-1, y.shape[-1])[pix]
    d = first_diff(got, ref)
    return d is None, d


def check_stem(x_fp16: np.ndarray, w_codes: np.ndarray, ss: np.ndarray, conv1, bits: int, inv_scale: float,
               relu: bool, y: np.ndarray, pix: np.ndarray, nthreads: int | None = None, y_uns: bool = False):
    """The stem conv (any implementation of conv1) vs the oracle's quantize +
    direct stride-2 conv over the channel-padded image, at pixels `pix`."""
    L = conv1
    Cp = padded_channels(L.C, bits)
    wpad = np.zeros((L.K, L.R, L.S, Cp), np.int8)
    wpad[..., :L.C] = w_codes
    xq = quantize(x_fp16, inv_scale, bits, nthreads=nthreads)
    ref = conv_q(xq, pack(wpad, bits), Cp, L.stride, L.pad, bits, ss, relu, pix=pix, nthreads=nthreads,
                 y_uns=y_uns)
    got = y.reshape(-1, y.shape[-1])[pix]
    d = first_diff(got, ref)
    return d is None, d


def check_pool(x: np.ndarray, C: int, pool, bits: int, y: np.ndarray, nthreads: int | None = None,
               uns: bool = False):
    R, st, pad = pool
    ref = maxpool(x, C, R, st, pad, bits, nthreads=nthreads, uns=uns)
    d = first_diff(y, ref)
    return d is None, d
