"""Activation, softmax and pooling (mirror of pkg/src/dnnp/nnops.py) on B200."""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .conv import output_extent
from .errors import EmptyWindow, MissingArgmax, ShapeMismatch
from .tensor import TensorView, _is_torch, bind_stream


class ActivationKind(enum.Enum):
    SIGMOID = "sigmoid"
    RELU = "relu"
    TANH = "tanh"


class SoftmaxMode(enum.Enum):
    PER_IMAGE = "per_image"
    PER_SPATIAL = "per_spatial"


class PoolKind(enum.Enum):
    MAX = "max"
    AVERAGE = "average"


_ACT = {ActivationKind.SIGMOID: 0, ActivationKind.RELU: 1, ActivationKind.TANH: 2}
_SOFTMAX = {SoftmaxMode.PER_IMAGE: 0, SoftmaxMode.PER_SPATIAL: 1}


def _as_enum(cls, value):
    if isinstance(value, cls):
        return value
    try:
        return cls(str(value).lower())
    except ValueError:
        raise ShapeMismatch(f"unknown {cls.__name__} {value!r}") from None


def _check_like(a: TensorView, b: TensorView, what: str):
    if a.desc.extents != b.desc.extents:
        raise ShapeMismatch(f"{what}: extents {a.desc.extents} vs {b.desc.extents}")
    if a.desc.dtype != b.desc.dtype:
        raise ShapeMismatch(f"{what}: element types {a.desc.dtype} vs {b.desc.dtype}")


def activation_forward(kind, x: TensorView, y: TensorView) -> None:
    """y = activation(x), elementwise (nnops.py:60-70)."""
    kind = _as_enum(ActivationKind, kind)
    _check_like(x, y, "activation")
    bind_stream(x, y)
    _lib.check(_lib.lib().dnnp_activation_forward(_lib.handle(), _ACT[kind], x.desc.c_desc(),
                                                  x.ptr, y.desc.c_desc(), y.ptr),
               "activation_forward")


def activation_backward(kind, y: TensorView, dy: TensorView, dx: TensorView) -> None:
    """dx = dy * activation'(x) written in y (nnops.py:73-88)."""
    kind = _as_enum(ActivationKind, kind)
    _check_like(y, dy, "activation backward")
    _check_like(y, dx, "activation backward")
    bind_stream(y, dy, dx)
    _lib.check(_lib.lib().dnnp_activation_backward(
        _lib.handle(), _ACT[kind], y.desc.c_desc(), y.ptr, dy.desc.c_desc(), dy.ptr,
        dx.desc.c_desc(), dx.ptr), "activation_backward")


def softmax_forward(mode, x: TensorView, y: TensorView) -> None:
    """Numerically stable softmax over the mode's group (nnops.py:95-104)."""
    mode = _as_enum(SoftmaxMode, mode)
    _check_like(x, y, "softmax")
    bind_stream(x, y)
    _lib.check(_lib.lib().dnnp_softmax_forward(_lib.handle(), _SOFTMAX[mode], x.desc.c_desc(),
                                               x.ptr, y.desc.c_desc(), y.ptr),
               "softmax_forward")


def softmax_backward(mode, y: TensorView, dy: TensorView, dx: TensorView) -> None:
    """dx_i = y_i * (dy_i - sum_group(dy * y)) (nnops.py:107-117)."""
    mode = _as_enum(SoftmaxMode, mode)
    _check_like(y, dy, "softmax backward")
    _check_like(y, dx, "softmax backward")
    bind_stream(y, dy, dx)
    _lib.check(_lib.lib().dnnp_softmax_backward(
        _lib.handle(), _SOFTMAX[mode], y.desc.c_desc(), y.ptr, dy.desc.c_desc(), dy.ptr,
        dx.desc.c_desc(), dx.ptr), "softmax_backward")


@dataclass(frozen=True)
class PoolingDesc:
    """Window, stride and padding of a pooling op (nnops.py:120-139)."""

    kind: PoolKind = PoolKind.MAX
    window_h: int = 2
    window_w: int = 2
    stride_h: int = 1
    stride_w: int = 1
    pad_h: int = 0
    pad_w: int = 0

    def __post_init__(self):
        object.__setattr__(self, "kind", _as_enum(PoolKind, self.kind))
        if self.window_h < 1 or self.window_w < 1:
            raise ShapeMismatch(f"pooling window must be >= 1: {self}")
        if self.stride_h < 1 or self.stride_w < 1:
            raise ShapeMismatch(f"pooling stride must be >= 1: {self}")
        if self.pad_h < 0 or self.pad_w < 0:
            raise ShapeMismatch(f"pooling padding must be >= 0: {self}")

    def c_desc(self):
        key = (self.kind, self.window_h, self.window_w, self.stride_h, self.stride_w,
               self.pad_h, self.pad_w)
        h = _pool_cache.get(key)
        if h is None:
            h = _pool_cache[key] = _lib.PoolDescHandle(
                0 if self.kind is PoolKind.MAX else 1, self.window_h, self.window_w,
                self.stride_h, self.stride_w, self.pad_h, self.pad_w)
        return h.h


_pool_cache = {}


def pool_out_shape(pd: PoolingDesc, x):
    d = x.desc if isinstance(x, TensorView) else x
    p = output_extent(d.h, pd.window_h, pd.stride_h, pd.pad_h)
    q = output_extent(d.w, pd.window_w, pd.stride_w, pd.pad_w)
    return (d.n, d.c, p, q)


def _check_windows(pd: PoolingDesc, h, w, p_ext, q_ext):
    for p in range(p_ext):
        hs = p * pd.stride_h - pd.pad_h
        if max(0, hs) >= min(h, hs + pd.window_h):
            raise EmptyWindow(f"pooling window at row {p} lies entirely in padding")
    for q in range(q_ext):
        ws = q * pd.stride_w - pd.pad_w
        if max(0, ws) >= min(w, ws + pd.window_w):
            raise EmptyWindow(f"pooling window at col {q} lies entirely in padding")


def _argmax_ptr(argmax, shape):
    if argmax is None:
        return None
    if _is_torch(argmax):
        import torch
        if tuple(argmax.shape) != tuple(shape) or argmax.dtype != torch.int64 or \
                not argmax.is_contiguous():
            raise ShapeMismatch("argmax buffer must be int64 and output-shaped")
        return argmax.data_ptr()
    if argmax.shape != tuple(shape) or argmax.dtype != np.int64 or \
            not argmax.flags.c_contiguous:
        raise ShapeMismatch("argmax buffer must be int64 and output-shaped")
    return argmax.ctypes.data


def pool_forward(pd: PoolingDesc, x: TensorView, y: TensorView, argmax_out=None) -> None:
    """Max or average over each window's in-image elements (nnops.py:157-200).
    argmax_out (int64, output-shaped) receives the logical NCHW index of the
    first maximum in (h, w) scan order."""
    n, c, p_ext, q_ext = pool_out_shape(pd, x)
    if y.desc.extents != (n, c, p_ext, q_ext) or y.desc.dtype != x.desc.dtype:
        raise ShapeMismatch(f"pooled output must be {(n, c, p_ext, q_ext)} {x.desc.dtype}, "
                            f"got {y.desc.extents} {y.desc.dtype}")
    am = _argmax_ptr(argmax_out, (n, c, p_ext, q_ext))
    _check_windows(pd, x.desc.h, x.desc.w, p_ext, q_ext)
    bind_stream(x, y)
    _lib.check(_lib.lib().dnnp_pooling_forward(
        _lib.handle(), pd.c_desc(), x.desc.c_desc(), x.ptr, y.desc.c_desc(), y.ptr,
        ctypes.c_void_p(am) if am else None), "pooling_forward")


def pool_backward(pd: PoolingDesc, y: TensorView, dy: TensorView, x: TensorView, dx: TensorView,
                  argmax=None) -> None:
    """Route output gradients back through the windows (nnops.py:203-246)."""
    n, c, p_ext, q_ext = pool_out_shape(pd, x)
    _check_like(x, dx, "pool backward")
    for t in (y, dy):
        if t.desc.extents != (n, c, p_ext, q_ext) or t.desc.dtype != x.desc.dtype:
            raise ShapeMismatch("pooled gradient shape mismatch")
    am = None
    if pd.kind is PoolKind.MAX:
        if argmax is None:
            raise MissingArgmax("max pooling backward needs the forward argmax")
        am = _argmax_ptr(argmax, (n, c, p_ext, q_ext))
    else:
        _check_windows(pd, x.desc.h, x.desc.w, p_ext, q_ext)
    bind_stream(y, dy, x, dx)
    _lib.check(_lib.lib().dnnp_pooling_backward(
        _lib.handle(), pd.c_desc(), y.desc.c_desc(), y.ptr, dy.desc.c_desc(), dy.ptr,
        x.desc.c_desc(), x.ptr, dx.desc.c_desc(), dx.ptr,
        ctypes.c_void_p(am) if am else None), "pooling_backward")


# ---------------------------------------------------------- fused epilogues
# Additive: the Caffe layer sequence conv -> bias -> act
# and its backward conv_bwd_data -> act_bwd in one pass over the output
# (include/dnnp.h dnnp_convolution_bias_activation_forward /
# dnnp_convolution_backward_data_activation).

def conv_bias_activation_forward(x: TensorView, f, conv, engine, y: TensorView, bias=None,
                                 activation=None, alpha: float = 1.0, beta: float = 0.0) -> None:
    """y := act(alpha * conv(x, f) + beta * y + bias[k]); bias (1, K, 1, 1) or None,
    activation an ActivationKind / name or None."""
    from .conv import _ENGINE_CODE, _check_out, _check_triplet, as_engine
    from .tensor import scalar_ptr
    engine = as_engine(engine)
    out_shape = _check_triplet(x, f, conv)
    _check_out(y, out_shape, x.desc.dtype, "output")
    act = -1 if activation is None else _ACT[_as_enum(ActivationKind, activation)]
    if bias is not None and bias.desc.extents != (1, out_shape[1], 1, 1):
        raise ShapeMismatch(f"bias must be (1, {out_shape[1]}, 1, 1)")
    views = (x, f, y) if bias is None else (x, f, y, bias)
    bind_stream(*views)
    a_keep, a = scalar_ptr(alpha, y.desc.dtype)
    b_keep, b = scalar_ptr(beta, y.desc.dtype)
    _lib.check(_lib.lib().dnnp_convolution_bias_activation_forward(
        _lib.handle(), a, x.desc.c_desc(), x.ptr, f.desc.c_desc(), f.ptr, conv.c_desc(),
        _ENGINE_CODE[engine], b, None if bias is None else bias.desc.c_desc(),
        None if bias is None else bias.ptr, act, y.desc.c_desc(), y.ptr),
        "convolution_bias_activation_forward")


def conv_backward_data_activation(dy: TensorView, f, conv, engine, dx: TensorView, activation,
                                  y: TensorView) -> None:
    """dx (+)= act'(y) * conv_backward_data(dy, f); y = the activation output
    that was this convolution's input (extents of dx)."""
    from .conv import _ENGINE_CODE, _check_out, _check_triplet, as_engine
    engine = as_engine(engine)
    kind = _as_enum(ActivationKind, activation)
    out_shape = _check_triplet(dx, f, conv)
    _check_out(dy, out_shape, dx.desc.dtype, "output gradient")
    _check_like(y, dx, "convolution backward-data activation")
    bind_stream(dy, f, dx, y)
    _lib.check(_lib.lib().dnnp_convolution_backward_data_activation(
        _lib.handle(), f.desc.c_desc(), f.ptr, dy.desc.c_desc(), dy.ptr, conv.c_desc(),
        _ENGINE_CODE[engine], _ACT[kind], y.desc.c_desc(), y.ptr, dx.desc.c_desc(), dx.ptr),
        "convolution_backward_data_activation")
