"""B200-native quantized INT8/INT4 implicit-GEMM convolution (arXiv 2202.06819).

Thin Python binding over the C ABI of ``libconvq.so`` (``include/convq.h``):
argument marshalling only.  Every step of the path -- quantize/pack, the
implicit-GEMM convolution on tcgen05 tensor cores, the fused requantize +
repack epilogue -- runs in the CUDA kernels of ``csrc/``.  PyTorch is used only
for device memory and streams (``Tensor.data_ptr()``,
``torch.cuda.current_stream()``).  There is no CPU fallback: if the extension
is missing or no B200 is present, calls raise ``ConvQError``.

Names follow the paper's problem statement (section 2.1): N, H, W,
C (= I, input channels), K (= O, output channels), R, S, stride, pad, bits.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

__all__ = [
    "ConvQError", "ConvPlan", "PlanInfo", "load", "quantize", "pack_weights", "padded_channels",
    "int8_peak", "out_dim", "OUT_PACKED", "OUT_S32", "StemPlan", "maxpool", "requant",
    "SearchOpts", "search",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CONV_Q_LIB") or os.path.join(_HERE, "libconvq.so")  # CONV_Q_LIB: A/B measurement of another build

OK, EINVAL, EUNSUPPORTED, EOVERFLOW, ECUDA, ENOMEM = 0, -1, -2, -3, -4, -5
OUT_PACKED, OUT_S32 = 0, 1
_CODE_NAMES = {EINVAL: "EINVAL", EUNSUPPORTED: "EUNSUPPORTED", EOVERFLOW: "EOVERFLOW",
               ECUDA: "ECUDA", ENOMEM: "ENOMEM"}


class ConvQError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODE_NAMES.get(code, code)}: {msg}")
        self.code = code


class _Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("N", "H", "W", "C", "K", "R", "S", "stride", "pad", "bits", "P", "Q")] + [
        ("M", ctypes.c_int64), ("Kg", ctypes.c_int64), ("x_bytes", ctypes.c_int64), ("w_bytes", ctypes.c_int64),
        ("y_bytes", ctypes.c_int64), ("y_s32_bytes", ctypes.c_int64), ("relu", ctypes.c_int),
        ("out_mode", ctypes.c_int), ("num_candidates", ctypes.c_int), ("config_index", ctypes.c_int),
        ("config", ctypes.c_char * 64), ("tuned_us", ctypes.c_float), ("macs", ctypes.c_int64),
        ("s2d", ctypes.c_int), ("x_dims", ctypes.c_int * 4), ("w_dims", ctypes.c_int * 4)]


class SearchOpts(ctypes.Structure):
    """conv_q_search_opts_t (include/convq.h, NEXT-4: PAPER.md:309-314 defaults)."""
    _fields_ = [("trials", ctypes.c_int), ("batch", ctypes.c_int), ("sa_iters", ctypes.c_int),
                ("sa_early_stop", ctypes.c_int), ("sa_points", ctypes.c_int), ("diversity", ctypes.c_int),
                ("sa_temp0", ctypes.c_float), ("sa_cool", ctypes.c_float), ("seed", ctypes.c_ulonglong)]

    @classmethod
    def make(cls, **kw) -> "SearchOpts":
        o = cls()
        load().conv_q_search_opts_default(ctypes.byref(o))
        for k, v in kw.items():
            if not hasattr(o, k):
                raise ConvQError(EINVAL, f"unknown search option {k}")
            setattr(o, k, v)
        return o


_VALID_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int))
_COST_FN = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int))


@dataclass
class PlanInfo:
    N: int; H: int; W: int; C: int; K: int; R: int; S: int; stride: int; pad: int; bits: int
    P: int; Q: int; M: int; Kg: int
    x_bytes: int; w_bytes: int; y_bytes: int; y_s32_bytes: int
    relu: int; out_mode: int; num_candidates: int; config_index: int; config: str; tuned_us: float; macs: int
    s2d: int; x_dims: tuple; w_dims: tuple


_lib = None


def load(build_if_missing: bool = False) -> ctypes.CDLL:
    """Load libconvq.so (in-tree).  Raises if it is absent: no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if build_if_missing:
            from . import _build
            _build.build()
        else:
            raise ConvQError(ECUDA, f"{LIB_PATH} not built; run `python __graft_entry__.py build` "
                                    "(or paper_2202_06819_b200/_build.py)")
    lib = ctypes.CDLL(LIB_PATH)
    i, vp, f = ctypes.c_int, ctypes.c_void_p, ctypes.c_float
    lib.conv_q_plan.restype = vp
    lib.conv_q_plan.argtypes = [i] * 10
    lib.conv_q_run.restype = i
    lib.conv_q_run.argtypes = [vp, vp, vp, vp, vp]
    lib.conv_q_plan_set_stream.restype = i
    lib.conv_q_plan_set_stream.argtypes = [vp, vp]
    lib.conv_q_plan_set_epilogue.restype = i
    lib.conv_q_plan_set_epilogue.argtypes = [vp, i, i]
    lib.conv_q_plan_num_candidates.restype = i
    lib.conv_q_plan_num_candidates.argtypes = [vp]
    lib.conv_q_plan_candidate_name.restype = i
    lib.conv_q_plan_candidate_name.argtypes = [vp, i, ctypes.c_char_p, i]
    lib.conv_q_plan_set_config.restype = i
    lib.conv_q_plan_set_config.argtypes = [vp, i]
    lib.conv_q_plan_tune.restype = i
    lib.conv_q_plan_tune.argtypes = [vp, vp, vp, vp, vp, i, i]
    lib.conv_q_plan_info.restype = i
    lib.conv_q_plan_info.argtypes = [vp, ctypes.POINTER(_Info)]
    lib.conv_q_plan_destroy.restype = None
    lib.conv_q_plan_destroy.argtypes = [vp]
    lib.conv_q_quantize.restype = i
    lib.conv_q_quantize.argtypes = [vp, i, i, i, i, f, i, vp, vp]
    lib.conv_q_padded_channels.restype = i
    lib.conv_q_padded_channels.argtypes = [i, i]
    lib.conv_q_pack_weights.restype = i
    lib.conv_q_pack_weights.argtypes = [vp, i, i, i, i, i, vp, vp]
    lib.conv_q_plan_s2d.restype = vp
    lib.conv_q_plan_s2d.argtypes = [i] * 9
    lib.conv_q_s2d_quantize.restype = i
    lib.conv_q_s2d_quantize.argtypes = [vp, vp, f, vp, vp]
    lib.conv_q_s2d_pack_weights.restype = i
    lib.conv_q_s2d_pack_weights.argtypes = [vp, vp, vp, vp]
    lib.conv_q_last_status.restype = i
    lib.conv_q_last_status.argtypes = []
    lib.conv_q_last_error.restype = ctypes.c_char_p
    lib.conv_q_last_error.argtypes = []
    lib.conv_q_version.restype = i
    lib.conv_q_version.argtypes = []
    lib.conv_q_plan_time_candidates.restype = i
    lib.conv_q_plan_time_candidates.argtypes = [vp, vp, vp, vp, vp, i, i, ctypes.POINTER(ctypes.c_float)]
    lib.conv_q_requant.restype = i
    lib.conv_q_requant.argtypes = [vp, ctypes.c_int64, i, vp, i, i, vp, vp]
    lib.conv_q_plan_set_residual.restype = i
    lib.conv_q_plan_set_residual.argtypes = [vp, vp, f]
    lib.conv_q_maxpool.restype = i
    lib.conv_q_maxpool.argtypes = [vp, i, i, i, i, i, i, i, i, vp, vp]
    lib.conv_q_maxpool_fmt.restype = i
    lib.conv_q_maxpool_fmt.argtypes = [vp, i, i, i, i, i, i, i, i, i, vp, vp]
    lib.conv_q_plan_set_formats.restype = i
    lib.conv_q_plan_set_formats.argtypes = [vp, i, i, i]
    lib.conv_q_plan_set_deps.restype = i
    lib.conv_q_plan_set_deps.argtypes = [vp, vp, vp, vp]
    lib.conv_q_int8_peak.restype = i
    lib.conv_q_int8_peak.argtypes = [i, ctypes.POINTER(ctypes.c_double)]
    lib.conv_q_search_opts_default.restype = None
    lib.conv_q_search_opts_default.argtypes = [ctypes.POINTER(SearchOpts)]
    lib.conv_q_search.restype = i
    lib.conv_q_search.argtypes = [i, ctypes.POINTER(ctypes.c_int), _VALID_FN, _COST_FN, vp, ctypes.POINTER(SearchOpts),
                                  ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_int)]
    lib.conv_q_plan_space.restype = i
    lib.conv_q_plan_space.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_longlong)]
    lib.conv_q_plan_time.restype = i
    lib.conv_q_plan_time.argtypes = [vp, vp, vp, vp, vp, i, i, ctypes.POINTER(ctypes.c_float)]
    lib.conv_q_plan_set_point.restype = i
    lib.conv_q_plan_get_point.restype = i
    lib.conv_q_plan_get_point.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    lib.conv_q_plan_set_point.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    lib.conv_q_plan_search.restype = i
    lib.conv_q_plan_search.argtypes = [vp, vp, vp, vp, vp, ctypes.POINTER(SearchOpts), i, i,
                                       ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]
    _lib = lib
    return lib


def _check(rc: int) -> int:
    if rc < 0:
        raise ConvQError(rc, load().conv_q_last_error().decode())
    return rc


def _ptr(t) -> int:
    """Device address of a torch tensor (or a raw int address)."""
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def out_dim(H: int, R: int, stride: int, pad: int) -> int:
    return (H + 2 * pad - R) // stride + 1


def padded_channels(C: int, bits: int) -> int:
    return _check(load().conv_q_padded_channels(C, bits))


class ConvPlan:
    """conv_q_plan(N,H,W,C,K,R,S,stride,pad,bits) + conv_q_run(plan,x,w,scale,y)."""

    def __init__(self, N, H, W, C, K, R, S, stride, pad, bits, relu=False, out_mode=OUT_PACKED,
                 x_uns=False, y_uns=False):
        lib = load()
        h = lib.conv_q_plan(N, H, W, C, K, R, S, stride, pad, bits)
        if not h:
            raise ConvQError(lib.conv_q_last_status(), lib.conv_q_last_error().decode())
        self._h = ctypes.c_void_p(h)
        self.N, self.H, self.W, self.C, self.K = N, H, W, C, K
        self.R, self.S, self.stride, self.pad, self.bits = R, S, stride, pad, bits
        self.P, self.Q = out_dim(H, R, stride, pad), out_dim(W, S, stride, pad)
        self._need = None
        self.x_uns = self.y_uns = self.skip_uns = False
        if x_uns or y_uns:
            self.set_formats(x_uns, y_uns)
        self.set_epilogue(relu, out_mode)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.conv_q_plan_destroy(h)
            self._h = None

    # -- configuration
    def set_epilogue(self, relu: bool, out_mode: int = OUT_PACKED):
        _check(load().conv_q_plan_set_epilogue(self._h, int(bool(relu)), out_mode))
        self.relu, self.out_mode = bool(relu), out_mode
        self._need = None

    def set_stream(self, stream):
        _check(load().conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))

    def set_formats(self, x_uns: bool = False, y_uns: bool = False, skip_uns: bool = False):
        """Unsigned code formats of x / y / the residual skip (conv_q_plan_set_formats,
        DESIGN reading 16)."""
        _check(load().conv_q_plan_set_formats(self._h, int(bool(x_uns)), int(bool(y_uns)), int(bool(skip_uns))))
        self.x_uns, self.y_uns, self.skip_uns = bool(x_uns), bool(y_uns), bool(skip_uns)

    def set_residual(self, skip, res_scale: float = 0.0):
        """Fused residual add (conv_q_plan_set_residual, DESIGN reading 15): skip is a
        packed tensor in y's layout (kept alive by the caller), or None to disable."""
        if skip is not None and not isinstance(skip, int):
            if skip.numel() * skip.element_size() < self.N * self.P * self.Q * self.K * self.bits // 8:
                raise ConvQError(EINVAL, "skip: smaller than the output tensor")
        self._skip = skip
        ptr = None if skip is None else _ptr(skip)
        _check(load().conv_q_plan_set_residual(self._h, ctypes.c_void_p(ptr), float(res_scale)))

    def set_deps(self, in_done=None, skip_done=None, out_done=None):
        """Cross-launch completion counters (conv_q_plan_set_deps): one-element int32
        device tensors (zeroed before each chain run), or None."""
        ptr = lambda t: ctypes.c_void_p(None if t is None else _ptr(t))  # noqa: E731
        _check(load().conv_q_plan_set_deps(self._h, ptr(in_done), ptr(skip_done), ptr(out_done)))
        self._deps = (in_done, skip_done, out_done)

    def candidates(self) -> list[str]:
        lib = load()
        n = _check(lib.conv_q_plan_num_candidates(self._h))
        out = []
        for i in range(n):
            buf = ctypes.create_string_buffer(64)
            _check(lib.conv_q_plan_candidate_name(self._h, i, buf, 64))
            out.append(buf.value.decode())
        return out

    def set_config(self, index: int):
        _check(load().conv_q_plan_set_config(self._h, index))

    def _check_buffers(self, x, w, scale, y):
        """Sizes / dtypes / contiguity of torch tensors against the plan (raw
        integer addresses are passed through unchecked)."""
        if self._need is None:
            inf = self.info()
            self._need = (inf.x_bytes, inf.w_bytes, inf.y_s32_bytes if self.out_mode == OUT_S32 else inf.y_bytes,
                          2 * inf.K)
        nx, nw, ny, nss = self._need
        for name, t, n in (("x", x, nx), ("w", w, nw), ("y", y, ny)):
            if isinstance(t, int):
                continue
            if not t.is_contiguous() or t.numel() * t.element_size() < n:
                raise ConvQError(EINVAL, f"{name}: need a contiguous buffer of >= {n} bytes, got "
                                         f"{t.numel() * t.element_size()} (contiguous={t.is_contiguous()})")
        if not isinstance(scale, int):
            import torch
            if scale.dtype != torch.float32 or not scale.is_contiguous() or scale.numel() < nss:
                raise ConvQError(EINVAL, f"scale: need {nss} contiguous float32 values (scale then shift)")

    def info(self) -> PlanInfo:
        inf = _Info()
        _check(load().conv_q_plan_info(self._h, ctypes.byref(inf)))
        d = {n: getattr(inf, n) for n, _ in _Info._fields_}
        d["config"] = inf.config.decode()
        d["x_dims"], d["w_dims"] = tuple(inf.x_dims), tuple(inf.w_dims)
        return PlanInfo(**d)

    # -- sizes (bytes)
    @property
    def x_bytes(self):
        return self.N * self.H * self.W * self.C * self.bits // 8

    @property
    def w_bytes(self):
        return self.K * self.R * self.S * self.C * self.bits // 8

    @property
    def y_bytes(self):
        return self.N * self.P * self.Q * self.K * self.bits // 8

    @property
    def macs(self):
        return self.N * self.P * self.Q * self.K * self.R * self.S * self.C

    # -- execution
    def run(self, x, w, scale, y, stream=None):
        """y <- requant(conv(x, w)) on `stream` (default: torch's current stream)."""
        self._check_buffers(x, w, scale, y)
        lib = load()
        _check(lib.conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))
        _check(lib.conv_q_run(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)),
                              ctypes.c_void_p(_ptr(scale)), ctypes.c_void_p(_ptr(y))))
        return y

    def time_candidates(self, x, w, scale, y, warmup=3, reps=10, stream=None) -> list[float]:
        """Per-candidate launch time in us (conv_q_plan_time_candidates); selection unchanged."""
        self._check_buffers(x, w, scale, y)
        lib = load()
        _check(lib.conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))
        n = _check(lib.conv_q_plan_num_candidates(self._h))
        arr = (ctypes.c_float * n)()
        _check(lib.conv_q_plan_time_candidates(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)),
                                               ctypes.c_void_p(_ptr(scale)), ctypes.c_void_p(_ptr(y)),
                                               warmup, reps, arr))
        return list(arr)

    def time(self, x, w, scale, y, warmup=2, reps=20, stream=None) -> float:
        """Graph-timed microseconds per launch of the current selection (conv_q_plan_time)."""
        self._check_buffers(x, w, scale, y)
        lib = load()
        _check(lib.conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))
        us = ctypes.c_float(0)
        _check(lib.conv_q_plan_time(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)),
                                    ctypes.c_void_p(_ptr(scale)), ctypes.c_void_p(_ptr(y)), warmup, reps,
                                    ctypes.byref(us)))
        return us.value

    def space(self) -> tuple[list[int], int]:
        """(knob sizes, number of valid points) of the plan's enlarged schedule space (NEXT-4)."""
        n = ctypes.c_int(0)
        sizes = (ctypes.c_int * 16)()
        nv = ctypes.c_longlong(0)
        _check(load().conv_q_plan_space(self._h, ctypes.byref(n), sizes, ctypes.byref(nv)))
        return list(sizes[:n.value]), nv.value

    def set_point(self, knobs):
        """Select one point of space() (conv_q_plan_set_point)."""
        _check(load().conv_q_plan_set_point(self._h, (ctypes.c_int * len(knobs))(*knobs)))

    def get_point(self) -> list[int]:
        """The current selection as a point of space() (conv_q_plan_get_point)."""
        k = (ctypes.c_int * 16)()
        _check(load().conv_q_plan_get_point(self._h, k))
        return list(k[:len(self.space()[0])])

    def search(self, x, w, scale, y, warmup=2, reps=10, stream=None, **opts) -> dict:
        """Learned, diversity-aware search over space() on the device (conv_q_plan_search):
        selects the fastest measured point; returns {best_us, history_us, config}."""
        self._check_buffers(x, w, scale, y)
        lib = load()
        _check(lib.conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))
        o = SearchOpts.make(**opts)
        hist = (ctypes.c_double * max(o.trials, 1))()
        best = ctypes.c_float(0)
        n = _check(lib.conv_q_plan_search(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)),
                                          ctypes.c_void_p(_ptr(scale)), ctypes.c_void_p(_ptr(y)), ctypes.byref(o),
                                          warmup, reps, ctypes.byref(best), hist))
        return {"best_us": best.value, "history_us": list(hist[:n]), "config": self.info().config}

    def tune(self, x, w, scale, y, warmup=3, reps=10, stream=None) -> int:
        self._check_buffers(x, w, scale, y)
        lib = load()
        _check(lib.conv_q_plan_set_stream(self._h, ctypes.c_void_p(_stream(stream))))
        return _check(lib.conv_q_plan_tune(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(w)),
                                           ctypes.c_void_p(_ptr(scale)), ctypes.c_void_p(_ptr(y)),
                                           warmup, reps))


class StemPlan(ConvPlan):
    """conv_q_plan_s2d: a stride-2 stem conv (C <= 4 s8 / 8 s4, e.g. ResNet conv1
    7x7/2 over RGB) run as a stride-1 conv over a space-to-depth(2) view.
    Same output as ConvPlan(N,H,W,C',K,R,S,2,pad,bits) on the channel-padded
    input; inputs come from quantize() / pack_weights() of this class."""

    def __init__(self, N, H, W, C, K, R, S, pad, bits, relu=False, out_mode=OUT_PACKED, y_uns=False):
        lib = load()
        h = lib.conv_q_plan_s2d(N, H, W, C, K, R, S, pad, bits)
        if not h:
            raise ConvQError(lib.conv_q_last_status(), lib.conv_q_last_error().decode())
        self._h = ctypes.c_void_p(h)
        self.N, self.H, self.W, self.C, self.K = N, H, W, C, K
        self.R, self.S, self.stride, self.pad, self.bits = R, S, 2, pad, bits
        self.P, self.Q = out_dim(H, R, 2, pad), out_dim(W, S, 2, pad)
        self._need = None
        self.x_uns = self.y_uns = self.skip_uns = False
        if y_uns:
            self.set_formats(False, True)
        self.set_epilogue(relu, out_mode)
        inf = self.info()
        self.x_dims, self.w_dims = inf.x_dims, inf.w_dims

    @property
    def x_bytes(self):
        d = self.x_dims
        return d[0] * d[1] * d[2] * d[3]

    @property
    def w_bytes(self):
        d = self.w_dims
        return d[0] * d[1] * d[2] * d[3]

    def quantize(self, x_fp16, inv_scale: float, out=None, stream=None):
        """fp16 NHWC image [N,H,W,C] -> the s2d tensor (uint8, x_dims)."""
        import torch
        assert x_fp16.dtype == torch.float16 and x_fp16.is_contiguous()
        assert tuple(x_fp16.shape) == (self.N, self.H, self.W, self.C)
        if out is None:
            out = torch.empty(self.x_dims, dtype=torch.uint8, device=x_fp16.device)
        _check(load().conv_q_s2d_quantize(self._h, ctypes.c_void_p(x_fp16.data_ptr()), float(inv_scale),
                                          ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream(stream))))
        return out

    def pack_weights(self, w_codes, out=None, stream=None):
        """int8 KRSC codes [K,R,S,C] (device) -> window weights (uint8, w_dims)."""
        import torch
        assert w_codes.dtype == torch.int8 and w_codes.is_contiguous()
        assert tuple(w_codes.shape) == (self.K, self.R, self.S, self.C)
        if out is None:
            out = torch.empty(self.w_dims, dtype=torch.uint8, device=w_codes.device)
        _check(load().conv_q_s2d_pack_weights(self._h, ctypes.c_void_p(w_codes.data_ptr()),
                                              ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream(stream))))
        return out


def quantize(x_fp16, inv_scale: float, bits: int, out=None, stream=None):
    """fp16 NHWC torch tensor -> packed NHWC uint8 tensor with C' channels."""
    import torch
    N, H, W, C = x_fp16.shape
    assert x_fp16.dtype == torch.float16 and x_fp16.is_contiguous()
    Cp = padded_channels(C, bits)
    if out is None:
        out = torch.empty((N, H, W, Cp * bits // 8), dtype=torch.uint8, device=x_fp16.device)
    _check(load().conv_q_quantize(ctypes.c_void_p(x_fp16.data_ptr()), N, H, W, C, float(inv_scale), bits,
                                  ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream(stream))))
    return out


def pack_weights(w_codes, bits: int, out=None, stream=None):
    """int8 KRSC codes (torch, device) -> packed KRSC uint8 [K,R,S,C*bits/8]."""
    import torch
    K, R, S, C = w_codes.shape
    assert w_codes.dtype == torch.int8 and w_codes.is_contiguous()
    if out is None:
        out = torch.empty((K, R, S, C * bits // 8), dtype=torch.uint8, device=w_codes.device)
    _check(load().conv_q_pack_weights(ctypes.c_void_p(w_codes.data_ptr()), K, R, S, C, bits,
                                      ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream(stream))))
    return out


def requant(acc, scale, relu: bool, bits: int, out=None, stream=None):
    """Unfused epilogue (conv_q_requant): int32 [..., K] accumulators -> packed uint8 [..., K*bits/8]."""
    import torch
    assert acc.dtype == torch.int32 and acc.is_contiguous()
    K = acc.shape[-1]
    M = acc.numel() // K
    assert scale.dtype == torch.float32 and scale.is_contiguous() and scale.numel() >= 2 * K
    if out is None:
        out = torch.empty(tuple(acc.shape[:-1]) + (K * bits // 8,), dtype=torch.uint8, device=acc.device)
    assert out.dtype == torch.uint8 and out.is_contiguous() and out.numel() >= M * K * bits // 8
    _check(load().conv_q_requant(ctypes.c_void_p(acc.data_ptr()), M, K, ctypes.c_void_p(scale.data_ptr()),
                                 int(bool(relu)), bits, ctypes.c_void_p(out.data_ptr()),
                                 ctypes.c_void_p(_stream(stream))))
    return out


def maxpool(x, C: int, R: int, stride: int, pad: int, bits: int, out=None, stream=None, uns: bool = False):
    """R x R max pooling of packed NHWC codes (conv_q_maxpool_fmt): uint8 [N,H,W,C*bits/8];
    uns: the codes are unsigned (DESIGN reading 16)."""
    import torch
    N, H, W, nb = x.shape
    assert x.dtype == torch.uint8 and x.is_contiguous() and nb == C * bits // 8
    P, Q = out_dim(H, R, stride, pad), out_dim(W, R, stride, pad)
    if out is None:
        out = torch.empty((N, P, Q, nb), dtype=torch.uint8, device=x.device)
    assert out.dtype == torch.uint8 and out.is_contiguous() and tuple(out.shape) == (N, P, Q, nb)
    _check(load().conv_q_maxpool_fmt(ctypes.c_void_p(x.data_ptr()), N, H, W, C, R, stride, pad, bits, int(bool(uns)),
                                     ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(_stream(stream))))
    return out


def int8_peak(iters: int = 200000) -> float:
    """Measured dense tcgen05 kind::i8 rate (ops/s) with operands in smem."""
    v = ctypes.c_double(0.0)
    _check(load().conv_q_int8_peak(iters, ctypes.byref(v)))
    return v.value


def search(knob_sizes, cost, valid=None, **opts) -> dict:
    """conv_q_search over a generic knob space (host only; NEXT-4 engine):
    cost(knobs) -> float > 0 (lower is better; <= 0 = failed), valid(knobs) -> bool.
    Returns {best, n, history_cost, history_knobs}."""
    lib = load()
    nk = len(knob_sizes)
    sizes = (ctypes.c_int * nk)(*knob_sizes)
    o = SearchOpts.make(**opts)
    err = []

    def _c(_ctx, k):
        try:
            return float(cost([k[i] for i in range(nk)]))
        except Exception as e:   # noqa: BLE001 -- surfaced after the call
            err.append(e)
            return -1.0

    def _v(_ctx, k):
        return 1 if valid([k[i] for i in range(nk)]) else 0

    cf = _COST_FN(_c)
    vf = _VALID_FN(_v) if valid is not None else _VALID_FN()
    best = (ctypes.c_int * nk)()
    hc = (ctypes.c_double * max(o.trials, 1))()
    hk = (ctypes.c_int * (max(o.trials, 1) * nk))()
    n = _check(lib.conv_q_search(nk, sizes, vf, cf, None, ctypes.byref(o), best, hc, hk))
    if err:
        raise err[0]
    return {"best": list(best), "n": n, "history_cost": list(hc[:n]),
            "history_knobs": [list(hk[i * nk:(i + 1) * nk]) for i in range(n)]}
