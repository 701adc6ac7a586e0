"""Batched 2-D convolution (mirror of pkg/src/dnnp/conv.py) on B200.

Same names, argument meaning and error behaviour as the reference; every
engine value routes to the one implicit-GEMM kernel family (tcgen05 BF16x3
for fp32 by default, SIMT DFMA for fp64) through the C ABI.
"""
from __future__ import annotations

import enum
import functools
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import AllocTooLarge, EmptyOutput, ShapeMismatch, ZeroExtent
from .tensor import (TensorDesc, TensorView, _is_torch, as_dtype, bind_stream, buf_info,
                     elem_code, empty_view, make_desc, scalar_ptr)


class ConvMode(enum.Enum):
    CONVOLUTION = "convolution"
    CROSS_CORRELATION = "cross_correlation"


class Engine(enum.Enum):
    DIRECT = "direct"
    EXPLICIT = "explicit_lowering"
    IMPLICIT = "implicit_gemm"


_ENGINE_ALIASES = {"direct": Engine.DIRECT, "explicit": Engine.EXPLICIT,
                   "explicit_lowering": Engine.EXPLICIT, "implicit": Engine.IMPLICIT,
                   "implicit_gemm": Engine.IMPLICIT}
_ENGINE_CODE = {Engine.DIRECT: 0, Engine.EXPLICIT: 1, Engine.IMPLICIT: 2}


def as_engine(engine) -> Engine:
    if isinstance(engine, Engine):
        return engine
    try:
        return _ENGINE_ALIASES[str(engine).lower()]
    except KeyError:
        raise ShapeMismatch(f"unknown engine {engine!r}") from None


def as_mode(mode) -> ConvMode:
    if isinstance(mode, ConvMode):
        return mode
    try:
        return ConvMode(str(mode).lower())
    except ValueError:
        raise ShapeMismatch(f"unknown convolution mode {mode!r}") from None


@dataclass(frozen=True)
class FilterDesc:
    """Filter shape (k, c, r, s), dense KCRS layout (conv.py:72-97)."""

    k: int
    c: int
    r: int
    s: int
    dtype: np.dtype

    def __hash__(self):
        h = self.__dict__.get("_hash")
        if h is None:
            h = hash((self.k, self.c, self.r, self.s, self.dtype))
            object.__setattr__(self, "_hash", h)
        return h

    def __post_init__(self):
        for e in (self.k, self.c, self.r, self.s):
            if e < 1:
                raise ZeroExtent(f"filter extents must be >= 1: {self}")

    @property
    def extents(self):
        return (self.k, self.c, self.r, self.s)

    @property
    def strides(self):
        return (self.c * self.r * self.s, self.r * self.s, self.s, 1)

    @property
    def size(self) -> int:
        return self.k * self.c * self.r * self.s

    def c_desc(self):
        return _c_filter(elem_code(self.dtype), self.k, self.c, self.r, self.s).h


_filter_cache = {}


def _c_filter(elem, k, c, r, s):
    key = (elem, k, c, r, s)
    h = _filter_cache.get(key)
    if h is None:
        h = _filter_cache[key] = _lib.FilterDescHandle(elem, k, c, r, s)
    return h


def make_filter_desc(k, c, r, s, elem_type="f32") -> FilterDesc:
    return FilterDesc(k, c, r, s, as_dtype(elem_type))


class FilterView:
    """A filter descriptor bound to a dense buffer (numpy or torch)."""

    def __init__(self, desc: FilterDesc, buf):
        if not _is_torch(buf):
            buf = np.asarray(buf)
        ptr, count, dt, cuda = buf_info(buf)
        if dt != desc.dtype:
            raise ShapeMismatch(f"filter buffer dtype {dt} does not match {desc.dtype}")
        if count < desc.size:
            raise ShapeMismatch(f"filter buffer of {count} elements, need {desc.size}")
        self.desc = desc
        self.buf = buf
        self.is_cuda = cuda
        self._torch = _is_torch(buf)
        self._dev = buf.device.index if cuda else None

    @property
    def ptr(self):
        b = self.buf
        return b.data_ptr() if self._torch else b.ctypes.data

    @property
    def array(self):
        return self.buf[: self.desc.size].reshape(self.desc.extents)

    @classmethod
    def from_array(cls, arr, device=None) -> "FilterView":
        if _is_torch(arr):
            device = device or arr.device
            arr = arr.detach().cpu().numpy()
        arr = np.asarray(arr)
        if arr.ndim != 4:
            raise ShapeMismatch("expected a 4-D (k, c, r, s) array")
        desc = FilterDesc(*arr.shape, dtype=as_dtype(arr.dtype))
        flat = np.ascontiguousarray(arr).reshape(-1)
        if device is not None:
            import torch
            flat = torch.from_numpy(flat.copy()).to(device)
        return cls(desc, flat)


@dataclass(frozen=True)
class ConvDesc:
    """Strides, padding, mode, and gradient-accumulation flag (conv.py:133-150)."""

    u: int = 1
    v: int = 1
    pad_h: int = 0
    pad_w: int = 0
    mode: ConvMode = ConvMode.CONVOLUTION
    accumulate: bool = False

    def __hash__(self):
        h = self.__dict__.get("_hash")
        if h is None:
            h = hash((self.u, self.v, self.pad_h, self.pad_w, self.mode, self.accumulate))
            object.__setattr__(self, "_hash", h)
        return h

    def __post_init__(self):
        if self.u < 1 or self.v < 1:
            raise ShapeMismatch(f"strides must be >= 1: u={self.u}, v={self.v}")
        if self.pad_h < 0 or self.pad_w < 0:
            raise ShapeMismatch(f"padding must be >= 0: {self.pad_h}, {self.pad_w}")
        object.__setattr__(self, "mode", as_mode(self.mode))

    def c_desc(self):
        key = (self.u, self.v, self.pad_h, self.pad_w, self.mode, self.accumulate)
        h = _conv_cache.get(key)
        if h is None:
            h = _conv_cache[key] = _lib.ConvDescHandle(
                self.u, self.v, self.pad_h, self.pad_w,
                0 if self.mode is ConvMode.CONVOLUTION else 1, self.accumulate)
        return h.h


_conv_cache = {}


def pad_preset(preset: str, r: int, s: int):
    """MATLAB-style padding presets: valid, same, full (conv.py:153-162)."""
    preset = preset.lower()
    if preset == "valid":
        return (0, 0)
    if preset == "same":
        return (r // 2, s // 2)
    if preset == "full":
        return (r - 1, s - 1)
    raise ShapeMismatch(f"unknown padding preset {preset!r}")


def output_extent(in_extent: int, filt_extent: int, stride: int, pad: int) -> int:
    """ceil((H - R + 1 + 2*pad) / u); empty output is an error (conv.py:165-179)."""
    if in_extent < 1 or filt_extent < 1 or stride < 1 or pad < 0:
        raise ShapeMismatch(f"bad window parameters ({in_extent}, {filt_extent}, {stride}, {pad})")
    numer = in_extent - filt_extent + 1 + 2 * pad
    if numer < 1:
        raise EmptyOutput(f"window of {filt_extent} over extent {in_extent} with pad {pad} "
                          "produces no output")
    return -(-numer // stride)


def access(p, stride, filt_extent, tap, pad, mode=ConvMode.CONVOLUTION) -> int:
    """Input index read by output position p at filter tap (conv.py:182-192)."""
    if as_mode(mode) is ConvMode.CONVOLUTION:
        return p * stride + filt_extent - tap - 1 - pad
    return p * stride + tap - pad


def conv_out_shape(x: TensorDesc, f: FilterDesc, conv: ConvDesc):
    """(N, K, P, Q); validates channel agreement (conv.py:195-201)."""
    if x.c != f.c:
        raise ShapeMismatch(f"input channels {x.c} vs filter channels {f.c}")
    p = output_extent(x.h, f.r, conv.u, conv.pad_h)
    q = output_extent(x.w, f.s, conv.v, conv.pad_w)
    return (x.n, f.k, p, q)


def _check_triplet(x: TensorView, f: FilterView, conv: ConvDesc):
    if x.desc.dtype != f.desc.dtype:
        raise ShapeMismatch(f"element types {x.desc.dtype} vs {f.desc.dtype}")
    return conv_out_shape(x.desc, f.desc, conv)


def _check_out(out: TensorView, extents, dtype, what):
    if out.desc.extents != tuple(extents):
        raise ShapeMismatch(f"{what} extents {out.desc.extents}, expected {tuple(extents)}")
    if out.desc.dtype != dtype:
        raise ShapeMismatch(f"{what} element type {out.desc.dtype}, expected {dtype}")


def _lowered_guard(engine, x_desc: TensorDesc, f_desc: FilterDesc, out_shape, max_bytes):
    """The explicit engine's C R S x N P Q lowered matrix limit (reference
    conv.py:507-511 / 615-618 / 701): AllocTooLarge above max_lowered_bytes
    (the library itself refuses anything above the 4 GiB default)."""
    if engine is not Engine.EXPLICIT:
        return
    n, _k, p, q = out_shape
    need = x_desc.c * f_desc.r * f_desc.s * n * p * q * x_desc.dtype.itemsize
    if need > max_bytes:
        raise AllocTooLarge(f"lowered matrix needs {need} bytes, limit {max_bytes}")


def _ws(workspace):
    """(pointer, bytes) of a caller workspace: a CUDA tensor (any dtype)."""
    return workspace.data_ptr(), workspace.numel() * workspace.element_size()


def convolution_workspace_size(pass_, x_desc, f_desc, conv: ConvDesc, y_desc,
                               engine="implicit") -> int:
    """Device workspace bytes of one pass (0 / "fwd", 1 / "bwd_data", 2 /
    "bwd_filter") for these descriptors (additive, dnnp_get_convolution_
    workspace_size: exact, measured by running the pass once on scratch
    tensors -- a setup-time call)."""
    import ctypes
    code = {"fwd": 0, "bwd_data": 1, "bwd_filter": 2}.get(pass_, pass_)
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().dnnp_get_convolution_workspace_size(
        _lib.handle(), int(code), x_desc.c_desc(), f_desc.c_desc(), conv.c_desc(),
        y_desc.c_desc(), _ENGINE_CODE[as_engine(engine)], ctypes.byref(out)),
        "get_convolution_workspace_size")
    return int(out.value)


@functools.lru_cache(maxsize=1024)
def _plan(pass_, in_desc, f_desc, conv, out_desc, engine, max_lowered_bytes):
    """Validated call plan, cached per (pass, descriptors, engine, limit):
    the checks the reference makes (same order and exceptions) and the native
    descriptor handles, so a repeated call does no Python-side work beyond
    reading pointers.  pass_: 0 forward (in = x, out = y), 1 backward-data
    (in = dx, out = dy), 2 backward-filter (in = x, out = dy, f = df)."""
    engine = as_engine(engine)
    if in_desc.dtype != f_desc.dtype:
        raise ShapeMismatch(f"element types {in_desc.dtype} vs {f_desc.dtype}")
    out_shape = conv_out_shape(in_desc, f_desc, conv)
    what = "output" if pass_ == 0 else "output gradient"
    if out_desc.extents != tuple(out_shape):
        raise ShapeMismatch(f"{what} extents {out_desc.extents}, expected {tuple(out_shape)}")
    if out_desc.dtype != in_desc.dtype:
        raise ShapeMismatch(f"{what} element type {out_desc.dtype}, expected {in_desc.dtype}")
    _lowered_guard(engine, in_desc, f_desc, out_shape, max_lowered_bytes)
    return (in_desc.c_desc(), f_desc.c_desc(), conv.c_desc(), out_desc.c_desc(),
            _ENGINE_CODE[engine])


def conv_forward(x: TensorView, f: FilterView, conv: ConvDesc, engine, y: TensorView,
                 alpha: float = 1.0, beta: float = 0.0, *, tile=None, threads: int = 1,
                 max_lowered_bytes: int = 4 << 30, workspace=None) -> None:
    """y := alpha * conv(x, f) + beta * y (accumulate forces beta=1).
    workspace: optional CUDA tensor the pass takes its scratch from."""
    xd, fd, cd, yd, ecode = _plan(0, x.desc, f.desc, conv, y.desc, engine, max_lowered_bytes)
    bind_stream(x, f, y)
    a_keep, a = scalar_ptr(alpha, y.desc.dtype)
    b_keep, b = scalar_ptr(beta, y.desc.dtype)
    if workspace is not None:
        _lib.check(_lib.lib().dnnp_convolution_forward_ex(
            _lib.handle(), a, xd, x.ptr, fd, f.ptr, cd, ecode, b, yd, y.ptr, *_ws(workspace)),
            "convolution_forward_ex")
        return
    _lib.check(_lib.lib().dnnp_convolution_forward(
        _lib.handle(), a, xd, x.ptr, fd, f.ptr, cd, ecode, b, yd, y.ptr), "convolution_forward")


def conv_backward_data(dy: TensorView, f: FilterView, conv: ConvDesc, engine, dx: TensorView,
                       *, tile=None, threads: int = 1, max_lowered_bytes: int = 4 << 30,
                       workspace=None) -> None:
    """Gradient with respect to the input; accumulate mode adds into dx."""
    dxd, fd, cd, dyd, ecode = _plan(1, dx.desc, f.desc, conv, dy.desc, engine,
                                    max_lowered_bytes)
    bind_stream(dy, f, dx)
    if workspace is not None:
        _lib.check(_lib.lib().dnnp_convolution_backward_data_ex(
            _lib.handle(), fd, f.ptr, dyd, dy.ptr, cd, ecode, dxd, dx.ptr, *_ws(workspace)),
            "convolution_backward_data_ex")
        return
    _lib.check(_lib.lib().dnnp_convolution_backward_data(
        _lib.handle(), fd, f.ptr, dyd, dy.ptr, cd, ecode, dxd, dx.ptr),
        "convolution_backward_data")


def conv_backward_filter(dy: TensorView, x: TensorView, conv: ConvDesc, engine, df: FilterView,
                         *, tile=None, threads: int = 1,
                         max_lowered_bytes: int = 4 << 30, workspace=None) -> None:
    """Gradient with respect to the filter; accumulate mode adds into df."""
    xd, fd, cd, dyd, ecode = _plan(2, x.desc, df.desc, conv, dy.desc, engine, max_lowered_bytes)
    bind_stream(dy, x, df)
    if workspace is not None:
        _lib.check(_lib.lib().dnnp_convolution_backward_filter_ex(
            _lib.handle(), xd, x.ptr, dyd, dy.ptr, cd, ecode, fd, df.ptr, *_ws(workspace)),
            "convolution_backward_filter_ex")
        return
    _lib.check(_lib.lib().dnnp_convolution_backward_filter(
        _lib.handle(), xd, x.ptr, dyd, dy.ptr, cd, ecode, fd, df.ptr),
        "convolution_backward_filter")


def conv_backward(dy: TensorView, f: FilterView, x: TensorView, conv: ConvDesc, engine,
                  dx: TensorView, df: FilterView) -> None:
    """Additive fused backward of one layer: dx and df in one call (dy packed
    once for both tensor-core GEMMs); same results as conv_backward_data +
    conv_backward_filter."""
    engine = as_engine(engine)
    out_shape = _check_triplet(x, f, conv)
    _check_out(dy, out_shape, x.desc.dtype, "output gradient")
    bind_stream(dy, f, x, dx, df)
    _lib.check(_lib.lib().dnnp_convolution_backward(
        _lib.handle(), f.desc.c_desc(), f.ptr, dy.desc.c_desc(), dy.ptr, x.desc.c_desc(), x.ptr,
        conv.c_desc(), _ENGINE_CODE[engine], dx.desc.c_desc(), dx.ptr, df.desc.c_desc(), df.ptr),
        "convolution_backward")


def conv_backward_bias(dy: TensorView, db: TensorView | None = None) -> TensorView:
    """Per-output-map sum of dy, shape (1, K, 1, 1) (conv.py:754-760)."""
    d = dy.desc
    if db is None:
        db = empty_view(make_desc(1, d.c, 1, 1, elem_type=d.dtype),
                        device=dy.buf.device if dy.is_cuda else None)
    if db.desc.extents != (1, d.c, 1, 1):
        raise ShapeMismatch(f"bias gradient must be (1, {d.c}, 1, 1)")
    bind_stream(dy, db)
    _lib.check(_lib.lib().dnnp_convolution_backward_bias(
        _lib.handle(), dy.desc.c_desc(), dy.ptr, db.desc.c_desc(), db.ptr),
        "convolution_backward_bias")
    return db
