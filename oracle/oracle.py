"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the C oracle (liboracle.so).

Imported by tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / --impl reference legs.  The product never imports this.
Buffers are flat numpy arrays with 8-int64 geometry {n,c,h,w,sn,sc,sh,sw}.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.oracle_output_extent_c.restype = ctypes.c_int64
        _lib.oracle_output_extent_c.argtypes = [ctypes.c_int64] * 4
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _g(g):
    return np.ascontiguousarray(np.asarray(g, dtype=np.int64))


def _sfx(dt):
    return "f64" if np.dtype(dt) == np.float64 else "f32"


def _call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise ValueError(f"{name} rejected the problem (status {rc})")


def divider_constants(d):
    out = np.zeros(3, dtype=np.uint32)
    lib().oracle_divider_constants(ctypes.c_uint32(d), _p(out))
    return tuple(int(v) for v in out)


def divide_many(d, n):
    n = np.ascontiguousarray(n, dtype=np.uint32)
    q = np.empty_like(n)
    lib().oracle_divide_many(ctypes.c_uint32(d), _p(n), _p(q), ctypes.c_int64(n.size))
    return q


def output_extent(in_ext, filt, stride, pad):
    return int(lib().oracle_output_extent_c(in_ext, filt, stride, pad))


def conv_forward(xg, x, fg, f, cg, yg, y, alpha=1.0, beta=0.0, threads=1):
    """In place on y (flat buffer)."""
    xg, fg, cg, yg = _g(xg), _g(fg), _g(cg), _g(yg)
    _call(f"oracle_conv_forward_{_sfx(x.dtype)}", _p(xg), _p(x), _p(fg), _p(f), _p(cg), _p(yg),
          _p(y), ctypes.c_double(alpha), ctypes.c_double(beta), ctypes.c_int(threads))


def conv_backward_data(fg, f, dyg, dy, cg, dxg, dx):
    fg, dyg, cg, dxg = _g(fg), _g(dyg), _g(cg), _g(dxg)
    _call(f"oracle_conv_backward_data_{_sfx(f.dtype)}", _p(fg), _p(f), _p(dyg), _p(dy), _p(cg),
          _p(dxg), _p(dx))


def conv_backward_filter(xg, x, dyg, dy, cg, fg, df, threads=1):
    xg, dyg, cg, fg = _g(xg), _g(dyg), _g(cg), _g(fg)
    _call(f"oracle_conv_backward_filter_{_sfx(x.dtype)}", _p(xg), _p(x), _p(dyg), _p(dy), _p(cg),
          _p(fg), _p(df), ctypes.c_int(threads))


def conv_backward_bias(dyg, dy):
    dyg = _g(dyg)
    db = np.zeros(int(dyg[1]), dtype=dy.dtype)
    _call(f"oracle_conv_backward_bias_{_sfx(dy.dtype)}", _p(dyg), _p(dy), _p(db))
    return db


def activation_forward(kind, xg, x, yg, y):
    _call(f"oracle_activation_forward_{_sfx(x.dtype)}", ctypes.c_int(kind), _p(_g(xg)), _p(x),
          _p(_g(yg)), _p(y))


def activation_backward(kind, yg, y, dyg, dy, dxg, dx):
    _call(f"oracle_activation_backward_{_sfx(y.dtype)}", ctypes.c_int(kind), _p(_g(yg)), _p(y),
          _p(_g(dyg)), _p(dy), _p(_g(dxg)), _p(dx))


def softmax_forward(mode, xg, x, yg, y):
    _call(f"oracle_softmax_forward_{_sfx(x.dtype)}", ctypes.c_int(mode), _p(_g(xg)), _p(x),
          _p(_g(yg)), _p(y))


def softmax_backward(mode, yg, y, dyg, dy, dxg, dx):
    _call(f"oracle_softmax_backward_{_sfx(y.dtype)}", ctypes.c_int(mode), _p(_g(yg)), _p(y),
          _p(_g(dyg)), _p(dy), _p(_g(dxg)), _p(dx))


def pool_forward(pg, xg, x, yg, y, argmax=None):
    _call(f"oracle_pool_forward_{_sfx(x.dtype)}", _p(_g(pg)), _p(_g(xg)), _p(x), _p(_g(yg)),
          _p(y), _p(argmax) if argmax is not None else None)


def pool_backward(pg, dyg, dy, dxg, dx, argmax=None):
    _call(f"oracle_pool_backward_{_sfx(dy.dtype)}", _p(_g(pg)), _p(_g(dyg)), _p(dy), _p(_g(dxg)),
          _p(dx), _p(argmax) if argmax is not None else None)


def transform(sg, s, dg, d, alpha, beta):
    _call(f"oracle_transform_{_sfx(s.dtype)}", _p(_g(sg)), _p(s), _p(_g(dg)), _p(d),
          ctypes.c_double(alpha), ctypes.c_double(beta))


def add_broadcast(bg, b, og, o, alpha, beta):
    _call(f"oracle_add_broadcast_{_sfx(b.dtype)}", _p(_g(bg)), _p(b), _p(_g(og)), _p(o),
          ctypes.c_double(alpha), ctypes.c_double(beta))


def rel_err(a, b):
    """Normalised max error max|a-b| / max|b| (reference test_acceptance.py:91-96)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.abs(b).max()) if b.size else 0.0, 1e-30)
    return float(np.abs(a - b).max()) / scale if a.size else 0.0
