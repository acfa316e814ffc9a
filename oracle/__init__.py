"""CPU oracle for the quantized implicit-GEMM convolution of arXiv 2202.06819.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2202_06819_b200``) never imports it, and
it never imports the product: the two share no code, headers, tables or
helpers.  The arithmetic lives in ``oracle/oracle.c`` (plain C, built with
``-O2 -ffp-contract=off``, no fast-math); this module only marshals numpy
arrays into it.

Every function cites the passage it follows (PAPER.md / SPEC.md line numbers
under /root/reference, plus the section).  Pins live in ``tests/test_oracle_*``.
Parity unpinned: none of the functions; the synthetic
scale/shift values have no paper values, the arithmetic applied to them is
pinned by closed forms.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_float
        vp = ctypes.c_void_p
        lib.oracle_half_to_float.restype = f32
        lib.oracle_half_to_float.argtypes = [ctypes.c_uint16]
        lib.oracle_quantize_value.restype = i32
        lib.oracle_quantize_value.argtypes = [f32, f32, i32]
        lib.oracle_pack.restype = None
        lib.oracle_pack.argtypes = [vp, i64, i32, vp]
        lib.oracle_unpack.restype = None
        lib.oracle_unpack.argtypes = [vp, i64, i32, vp]
        lib.oracle_padded_channels.restype = i64
        lib.oracle_padded_channels.argtypes = [i64, i32]
        lib.oracle_quantize.restype = None
        lib.oracle_quantize.argtypes = [vp, i64, i64, i64, i64, f32, i32, vp, i32]
        lib.oracle_out_dim.restype = i64
        lib.oracle_out_dim.argtypes = [i64, i64, i64, i64]
        lib.oracle_conv_s32.restype = i32
        lib.oracle_conv_s32.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i32,
                                        vp, i64, vp, i32]
        lib.oracle_requant_value.restype = i32
        lib.oracle_requant_value.argtypes = [i32, f32, f32, i32, i32]
        lib.oracle_requant.restype = None
        lib.oracle_requant.argtypes = [vp, i64, i64, vp, i32, i32, vp, i32]
        lib.oracle_conv_q.restype = i32
        lib.oracle_conv_q.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i32,
                                      vp, i32, vp, i64, vp, i32]
        lib.oracle_requant_res_value.restype = i32
        lib.oracle_requant_res_value.argtypes = [i32, f32, f32, i32, f32, i32, i32]
        lib.oracle_requant_res.restype = None
        lib.oracle_requant_res.argtypes = [vp, i64, i64, vp, vp, f32, i32, i32, vp, i32]
        lib.oracle_unpack_fmt.restype = None
        lib.oracle_unpack_fmt.argtypes = [vp, i64, i32, i32, vp]
        lib.oracle_pack_fmt.restype = None
        lib.oracle_pack_fmt.argtypes = [vp, i64, i32, vp]
        lib.oracle_conv_s32_fmt.restype = i32
        lib.oracle_conv_s32_fmt.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, i64, i64, i32, i32,
                                            vp, i64, vp, i32]
        lib.oracle_requant_value_fmt.restype = i32
        lib.oracle_requant_value_fmt.argtypes = [i32, f32, f32, i32, i32, i32]
        lib.oracle_requant_res_value_fmt.restype = i32
        lib.oracle_requant_res_value_fmt.argtypes = [i32, f32, f32, i32, f32, i32, i32, i32]
        lib.oracle_requant_fmt.restype = None
        lib.oracle_requant_fmt.argtypes = [vp, i64, i64, vp, vp, i32, f32, i32, i32, i32, vp, i32]
        lib.oracle_maxpool_fmt.restype = i32
        lib.oracle_maxpool_fmt.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i32, i32, vp, i32]
        lib.oracle_maxpool.restype = i32
        lib.oracle_maxpool.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, i32, vp, i32]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


# --------------------------------------------------------------------------
# scalar steps
# --------------------------------------------------------------------------
def half_to_float(h: int) -> float:
    """IEEE binary16 -> binary32 decode written from the format definition
    (quantizer input, section 1)."""
    return float(_load().oracle_half_to_float(int(h) & 0xFFFF))


def quantize_value(f: float, inv_scale: float, bits: int) -> int:
    """q = clamp(rne(f * inv_scale)) -- reading 1 (section 1)."""
    return int(_load().oracle_quantize_value(float(np.float32(f)), float(np.float32(inv_scale)), bits))


def requant_value(acc: int, scale: float, shift: float, relu: bool, bits: int) -> int:
    """y = clamp(rne(fmaf((float)acc, scale, shift))) -- PAPER.md:200 section 3.2.2,
    readings 4 and 5."""
    return int(_load().oracle_requant_value(int(acc), float(np.float32(scale)),
                                            float(np.float32(shift)), int(bool(relu)), bits))


def requant_res_value(acc: int, scale: float, shift: float, skip: int, res_scale: float, relu: bool,
                      bits: int) -> int:
    """y = clamp(rne(fmaf(skip, res_scale, fmaf((float)acc, scale, shift)))) -- the
    residual epilogue of DESIGN reading 15."""
    return int(_load().oracle_requant_res_value(int(acc), float(np.float32(scale)), float(np.float32(shift)),
                                                int(skip), float(np.float32(res_scale)), int(bool(relu)), bits))


def requant_value_fmt(acc: int, scale: float, shift: float, relu: bool, bits: int, y_uns: bool) -> int:
    """requant_value into output format y_uns (reading 16: unsigned codes clamp to
    [0, 2^b - 1])."""
    return int(_load().oracle_requant_value_fmt(int(acc), float(np.float32(scale)), float(np.float32(shift)),
                                                int(bool(relu)), bits, int(bool(y_uns))))


def requant_res_value_fmt(acc: int, scale: float, shift: float, skip: int, res_scale: float, relu: bool,
                          bits: int, y_uns: bool) -> int:
    """requant_res_value into output format y_uns (readings 15, 16)."""
    return int(_load().oracle_requant_res_value_fmt(int(acc), float(np.float32(scale)), float(np.float32(shift)),
                                                    int(skip), float(np.float32(res_scale)), int(bool(relu)), bits,
                                                    int(bool(y_uns))))


def out_dim(H: int, R: int, stride: int, pad: int) -> int:
    """P = floor((H + 2 pad - R) / stride) + 1 (reading 6)."""
    return int(_load().oracle_out_dim(H, R, stride, pad))


def padded_channels(C: int, bits: int) -> int:
    """C' = ceil(C/32)*32: whole 32-channel granules (DESIGN reading 14)."""
    return int(_load().oracle_padded_channels(C, bits))


# --------------------------------------------------------------------------
# tensor steps
# --------------------------------------------------------------------------
def pack(q: np.ndarray, bits: int) -> np.ndarray:
    """Pack int8 codes along the last axis (SPEC.md:220-228 little-nibble-first)."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    C = q.shape[-1]
    rows = q.reshape(-1, C)
    out = np.empty((rows.shape[0], C * bits // 8), dtype=np.uint8)
    lib = _load()
    for i in range(rows.shape[0]):
        r = np.ascontiguousarray(rows[i])
        o = out[i]
        lib.oracle_pack(_ptr(r), C, bits, o.ctypes.data_as(ctypes.c_void_p))
    return out.reshape(*q.shape[:-1], C * bits // 8)


def unpack(p: np.ndarray, C: int, bits: int) -> np.ndarray:
    """Inverse of pack; nibbles sign-extended."""
    p = np.ascontiguousarray(p, dtype=np.uint8)
    nb = C * bits // 8
    rows = p.reshape(-1, nb)
    out = np.empty((rows.shape[0], C), dtype=np.int8)
    lib = _load()
    for i in range(rows.shape[0]):
        r = np.ascontiguousarray(rows[i])
        o = out[i]
        lib.oracle_unpack(_ptr(r), C, bits, o.ctypes.data_as(ctypes.c_void_p))
    return out.reshape(*p.shape[:-1], C)


def unpack_fmt(p: np.ndarray, C: int, bits: int, uns: bool) -> np.ndarray:
    """Unpack codes of format uns (reading 16) -> int16 [..., C]."""
    p = np.ascontiguousarray(p, dtype=np.uint8)
    nb = C * bits // 8
    rows = p.reshape(-1, nb)
    out = np.empty((rows.shape[0], C), dtype=np.int16)
    lib = _load()
    for i in range(rows.shape[0]):
        r = np.ascontiguousarray(rows[i])
        o = out[i]
        lib.oracle_unpack_fmt(_ptr(r), C, bits, int(bool(uns)), o.ctypes.data_as(ctypes.c_void_p))
    return out.reshape(*p.shape[:-1], C)


def pack_fmt(q: np.ndarray, bits: int) -> np.ndarray:
    """Pack int16 codes of either format (their low b bits, reading 2)."""
    q = np.ascontiguousarray(q, dtype=np.int16)
    C = q.shape[-1]
    rows = q.reshape(-1, C)
    out = np.empty((rows.shape[0], C * bits // 8), dtype=np.uint8)
    lib = _load()
    for i in range(rows.shape[0]):
        r = np.ascontiguousarray(rows[i])
        o = out[i]
        lib.oracle_pack_fmt(_ptr(r), C, bits, o.ctypes.data_as(ctypes.c_void_p))
    return out.reshape(*q.shape[:-1], C * bits // 8)


def quantize(x_fp16: np.ndarray, inv_scale: float, bits: int, nthreads: int | None = None) -> np.ndarray:
    """fp16 NHWC -> packed NHWC with C' channels (section 1)."""
    x = np.ascontiguousarray(x_fp16, dtype=np.float16)
    N, H, W, C = x.shape
    Cp = padded_channels(C, bits)
    out = np.empty((N, H, W, Cp * bits // 8), dtype=np.uint8)
    _load().oracle_quantize(_ptr(x.view(np.uint16)), N, H, W, C, float(np.float32(inv_scale)), bits,
                            _ptr(out), nthreads or default_threads())
    return out


def conv_s32(x: np.ndarray, w: np.ndarray, C: int, stride: int, pad: int, bits: int,
             pix: np.ndarray | None = None, nthreads: int | None = None, x_uns: bool = False) -> np.ndarray:
    """Exact integer direct convolution (section 2.1).

    x: packed NHWC uint8 [N,H,W,C*b/8]; w: packed KRSC uint8 [K,R,S,C*b/8].
    Returns int32 [N,P,Q,K], or [len(pix),K] for a list of linear output
    pixel indices m = (n*P+p)*Q+q.  x_uns: x holds unsigned codes (reading 16).
    """
    x = np.ascontiguousarray(x, dtype=np.uint8)
    w = np.ascontiguousarray(w, dtype=np.uint8)
    N, H, W, nb = x.shape
    K, R, S, nbw = w.shape
    assert nb == nbw == C * bits // 8, (nb, nbw, C, bits)
    P, Q = out_dim(H, R, stride, pad), out_dim(W, S, stride, pad)
    if pix is None:
        acc = np.empty((N, P, Q, K), dtype=np.int32)
        pl, npix = None, 0
    else:
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        acc = np.empty((pix.size, K), dtype=np.int32)
        pl, npix = _ptr(pix), pix.size
    rc = _load().oracle_conv_s32_fmt(_ptr(x), _ptr(w), N, H, W, C, K, R, S, stride, pad, bits, int(bool(x_uns)),
                                     pl, npix, _ptr(acc), nthreads or default_threads())
    if rc != 0:
        raise OverflowError(f"oracle_conv_s32 rc={rc} (accumulator left int32 or OOM)")
    return acc


def requant(acc: np.ndarray, scale_shift: np.ndarray, relu: bool, bits: int,
            nthreads: int | None = None) -> np.ndarray:
    """Requantize s32 [..., K] and pack rows (section 3.2.2)."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    K = acc.shape[-1]
    ss = np.ascontiguousarray(scale_shift, dtype=np.float32)
    assert ss.size == 2 * K
    assert K <= 8192, "oracle_requant packs one row in an 8192-code buffer"
    M = acc.size // K
    out = np.empty((M, K * bits // 8), dtype=np.uint8)
    _load().oracle_requant(_ptr(acc), M, K, _ptr(ss), int(bool(relu)), bits, _ptr(out),
                           nthreads or default_threads())
    return out.reshape(*acc.shape[:-1], K * bits // 8)


def requant_res(acc: np.ndarray, scale_shift: np.ndarray, skip: np.ndarray, res_scale: float, relu: bool,
                bits: int, nthreads: int | None = None) -> np.ndarray:
    """requant with the fused residual add (reading 15); skip: packed [..., K*b/8]
    with the same leading shape as acc."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    K = acc.shape[-1]
    ss = np.ascontiguousarray(scale_shift, dtype=np.float32)
    assert ss.size == 2 * K and K <= 8192
    M = acc.size // K
    sk = np.ascontiguousarray(skip, dtype=np.uint8).reshape(M, K * bits // 8)
    out = np.empty((M, K * bits // 8), dtype=np.uint8)
    _load().oracle_requant_res(_ptr(acc), M, K, _ptr(ss), _ptr(sk), float(np.float32(res_scale)),
                               int(bool(relu)), bits, _ptr(out), nthreads or default_threads())
    return out.reshape(*acc.shape[:-1], K * bits // 8)


def requant_fmt(acc: np.ndarray, scale_shift: np.ndarray, relu: bool, bits: int, y_uns: bool,
                skip: np.ndarray | None = None, skip_uns: bool = False, res_scale: float = 0.0,
                nthreads: int | None = None) -> np.ndarray:
    """Requantize s32 [..., K] into packed codes of format y_uns, optionally with
    the residual add of reading 15 (skip codes of format skip_uns) -- reading 16."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    K = acc.shape[-1]
    ss = np.ascontiguousarray(scale_shift, dtype=np.float32)
    assert ss.size == 2 * K and K <= 8192
    M = acc.size // K
    sk = None if skip is None else np.ascontiguousarray(skip, dtype=np.uint8).reshape(M, K * bits // 8)
    out = np.empty((M, K * bits // 8), dtype=np.uint8)
    _load().oracle_requant_fmt(_ptr(acc), M, K, _ptr(ss), None if sk is None else _ptr(sk), int(bool(skip_uns)),
                               float(np.float32(res_scale)), int(bool(relu)), bits, int(bool(y_uns)), _ptr(out),
                               nthreads or default_threads())
    return out.reshape(*acc.shape[:-1], K * bits // 8)


def conv_q(x: np.ndarray, w: np.ndarray, C: int, stride: int, pad: int, bits: int,
           scale_shift: np.ndarray, relu: bool, pix: np.ndarray | None = None,
           nthreads: int | None = None, skip: np.ndarray | None = None, res_scale: float = 0.0,
           x_uns: bool = False, y_uns: bool = False, skip_uns: bool = False) -> np.ndarray:
    """One whole layer: conv_s32 -> requant -> pack; with
    `skip` (packed, the output's shape; rows `pix` only when pix is given) the
    residual epilogue of reading 15; x_uns / y_uns / skip_uns: unsigned code
    formats of the input, output and skip tensors (reading 16)."""
    acc = conv_s32(x, w, C, stride, pad, bits, pix=pix, nthreads=nthreads, x_uns=x_uns)
    if x_uns or y_uns or skip_uns:
        sk = None
        if skip is not None:
            sk = skip.reshape(-1, skip.shape[-1])
            if pix is not None:
                sk = sk[pix]
        return requant_fmt(acc, scale_shift, relu, bits, y_uns, skip=sk, skip_uns=skip_uns, res_scale=res_scale,
                           nthreads=nthreads)
    if skip is not None:
        sk = skip.reshape(-1, skip.shape[-1])
        if pix is not None:
            sk = sk[pix]
        return requant_res(acc, scale_shift, sk, res_scale, relu, bits, nthreads=nthreads)
    return requant(acc, scale_shift, relu, bits, nthreads=nthreads)


def maxpool(x: np.ndarray, C: int, R: int, stride: int, pad: int, bits: int,
            nthreads: int | None = None, uns: bool = False) -> np.ndarray:
    """R x R max pooling of packed NHWC codes, padding never wins (the ResNet
    stem's 3x3/2 pool; section 1); uns: the codes
    are unsigned (reading 16)."""
    x = np.ascontiguousarray(x, dtype=np.uint8)
    N, H, W, nb = x.shape
    assert nb == C * bits // 8 and C <= 4096
    P, Q = out_dim(H, R, stride, pad), out_dim(W, R, stride, pad)
    y = np.empty((N, P, Q, nb), dtype=np.uint8)
    rc = _load().oracle_maxpool_fmt(_ptr(x), N, H, W, C, R, stride, pad, bits, int(bool(uns)), _ptr(y),
                                    nthreads or default_threads())
    if rc != 0:
        raise ValueError("oracle_maxpool: a window has no in-range tap")
    return y
