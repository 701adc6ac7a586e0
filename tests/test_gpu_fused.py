"""Fused conv epilogues (additive API) against the
unfused sequence of reference-API calls on the same inputs:
  forward:   conv_forward -> add_broadcast(bias) -> activation_forward
  bwd-data:  conv_backward_data -> activation_backward(y = the layer input)
Covers the tensor-core epilogue (channel columns, scattered super-pixel /
space-to-depth / blocked columns, CTA pairs, reduction segments), the
unfused fallbacks (fp64, SIMT fp32, gate with other strides, accumulate over
segments) and host buffers."""
import os
from contextlib import contextmanager

import numpy as np
import pytest

import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu
TOL = {"f32": 2e-6, "f64": 1e-13}


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    dp._lib.reload_tuning()  # the library caches the switches
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        dp._lib.reload_tuning()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def view(rng, n, c, h, w, dt="f32", layout="nchw", lo=-0.5):
    import torch
    d = dp.make_desc(n, c, h, w, layout=layout, elem_type=dt)
    npdt = np.float32 if dt == "f32" else np.float64
    buf = rng.uniform(lo, 0.5, d.max_offset() + 1).astype(npdt)
    return dp.TensorView(d, torch.from_numpy(buf).cuda())


def clone(v):
    return dp.TensorView(v.desc, v.buf.clone())


#        N   C   H   W   K  R  S  u  v ph pw
SHAPES = [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1),     # unit stride, channel columns
          (2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2),   # space-to-depth (conv1-like)
          (2, 16, 15, 15, 24, 5, 5, 2, 2, 2, 2),    # strided: super-pixel bwd-data
          (3, 64, 15, 15, 96, 5, 5, 1, 1, 2, 2),    # conv2-like: blocked bwd-data columns
          (2, 32, 13, 13, 256, 3, 3, 1, 1, 1, 1)]   # wide K: CTA pairs


def fwd_pair(shape, act, with_bias, dt="f32", alpha=1.0, beta=0.0, accumulate=False,
             layout="nchw", host=False, seed=0):
    import torch
    rng = np.random.default_rng(seed)
    N, C, H, W, K, R, S, u, v, ph, pw = shape
    cd = dp.ConvDesc(u, v, ph, pw, "convolution", accumulate)
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    x = view(rng, N, C, H, W, dt)
    npdt = np.float32 if dt == "f32" else np.float64
    f = dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt),
                      torch.from_numpy(rng.uniform(-0.5, 0.5, K * C * R * S).astype(npdt)).cuda())
    b = view(rng, 1, K, 1, 1, dt) if with_bias else None
    y0 = view(rng, N, K, P, Q, dt, layout)
    yf, yu = clone(y0), clone(y0)
    if host:
        x = dp.TensorView(x.desc, x.buf.cpu().numpy())
        f = dp.FilterView(f.desc, f.buf.cpu().numpy())
        b = None if b is None else dp.TensorView(b.desc, b.buf.cpu().numpy())
        yf = dp.TensorView(yf.desc, yf.buf.cpu().numpy())
    dp.conv_bias_activation_forward(x, f, cd, "implicit", yf, bias=b, activation=act,
                                    alpha=alpha, beta=beta)
    xs = x if not host else dp.TensorView(x.desc, torch.from_numpy(x.buf).cuda())
    fs = f if not host else dp.FilterView(f.desc, torch.from_numpy(f.buf).cuda())
    bs = b if (b is None or not host) else dp.TensorView(b.desc, torch.from_numpy(b.buf).cuda())
    dp.conv_forward(xs, fs, cd, "implicit", yu, alpha=alpha, beta=beta)
    if bs is not None:
        dp.add_broadcast(bs, yu, 1.0, 1.0)
    if act is not None:
        dp.activation_forward(act, yu, yu)
    torch.cuda.synchronize()
    out = yf.buf if host else yf.buf.cpu().numpy()
    return rel(out, yu.buf.cpu().numpy())


def bwd_pair(shape, act, dt="f32", accumulate=False, gate_layout="nchw", host=False, seed=0):
    import torch
    rng = np.random.default_rng(seed)
    N, C, H, W, K, R, S, u, v, ph, pw = shape
    cd = dp.ConvDesc(u, v, ph, pw, "convolution", accumulate)
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    dy = view(rng, N, K, P, Q, dt)
    npdt = np.float32 if dt == "f32" else np.float64
    f = dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt),
                      torch.from_numpy(rng.uniform(-0.5, 0.5, K * C * R * S).astype(npdt)).cuda())
    # the activation output feeding the conv: relu outputs have exact zeros
    g = view(rng, N, C, H, W, dt, gate_layout, lo=-0.5 if act != "relu" else -0.3)
    if act == "relu":
        g.buf.clamp_(min=0)
    elif act == "sigmoid":
        g.buf.add_(0.5)
    dx0 = view(rng, N, C, H, W, dt)
    dxf, dxu = clone(dx0), clone(dx0)
    if host:
        args = [dp.TensorView(dy.desc, dy.buf.cpu().numpy()), dp.FilterView(f.desc, f.buf.cpu().numpy())]
        dxh = dp.TensorView(dxf.desc, dxf.buf.cpu().numpy())
        gh = dp.TensorView(g.desc, g.buf.cpu().numpy())
        dp.conv_backward_data_activation(args[0], args[1], cd, "implicit", dxh, act, gh)
        out = dxh.buf
    else:
        dp.conv_backward_data_activation(dy, f, cd, "implicit", dxf, act, g)
        out = None
    tmp = dp.empty_view(dp.make_desc(N, C, H, W, elem_type=dt), device="cuda")
    dp.conv_backward_data(dy, f, dp.ConvDesc(u, v, ph, pw), "implicit", tmp)
    dp.activation_backward(act, g, tmp, tmp)
    dp.transform(tmp, dxu, 1.0, 1.0 if accumulate else 0.0)
    torch.cuda.synchronize()
    return rel(out if host else dxf.buf.cpu().numpy(), dxu.buf.cpu().numpy())


@pytest.mark.parametrize("shape", SHAPES, ids=[f"s{i}" for i in range(len(SHAPES))])
@pytest.mark.parametrize("act", [None, "relu", "sigmoid", "tanh"])
def test_forward_fused(shape, act):
    assert fwd_pair(shape, act, with_bias=True) <= TOL["f32"]
    if act == "relu":
        assert fwd_pair(shape, act, with_bias=False) <= TOL["f32"]


@pytest.mark.parametrize("alpha,beta,accumulate", [(0.5, -1.25, False), (1.0, 0.0, True)])
def test_forward_scalars(alpha, beta, accumulate):
    for shape in SHAPES[:3]:
        assert fwd_pair(shape, "relu", True, alpha=alpha, beta=beta,
                        accumulate=accumulate) <= TOL["f32"]


def test_forward_segments_layout_host():
    with env(DNNP_TC_CHAIN=128):
        assert fwd_pair(SHAPES[0], "tanh", True, beta=0.5) <= TOL["f32"]
        assert fwd_pair(SHAPES[1], "relu", True) <= TOL["f32"]
    assert fwd_pair(SHAPES[0], "relu", True, layout="nhwc") <= TOL["f32"]
    assert fwd_pair(SHAPES[2], "sigmoid", True, host=True) <= TOL["f32"]


def test_forward_fallbacks():
    assert fwd_pair(SHAPES[0], "relu", True, dt="f64") <= TOL["f64"]
    dp.set_math(dp.MATH_SIMT_FP32)
    try:
        assert fwd_pair(SHAPES[2], "sigmoid", True) <= TOL["f32"]
    finally:
        dp.set_math(dp.MATH_DEFAULT)


@pytest.mark.parametrize("shape", SHAPES, ids=[f"s{i}" for i in range(len(SHAPES))])
@pytest.mark.parametrize("act", ["relu", "sigmoid", "tanh"])
def test_backward_data_fused(shape, act):
    assert bwd_pair(shape, act) <= TOL["f32"]


@pytest.mark.parametrize("shape", SHAPES[:4], ids=[f"s{i}" for i in range(4)])
def test_backward_data_accumulate(shape):
    assert bwd_pair(shape, "relu", accumulate=True) <= TOL["f32"]


def test_backward_data_segments_and_fallbacks():
    with env(DNNP_TC_CHAIN=128):
        assert bwd_pair(SHAPES[0], "relu") <= TOL["f32"]            # fused, segmented
        assert bwd_pair(SHAPES[2], "tanh") <= TOL["f32"]
        assert bwd_pair(SHAPES[0], "relu", accumulate=True) <= TOL["f32"]  # unfused fallback
    assert bwd_pair(SHAPES[0], "relu", gate_layout="nhwc") <= TOL["f32"]  # other strides
    assert bwd_pair(SHAPES[2], "sigmoid", dt="f64") <= TOL["f64"]
    assert bwd_pair(SHAPES[0], "relu", dt="f64", accumulate=True) <= TOL["f64"]
    assert bwd_pair(SHAPES[3], "relu", host=True) <= TOL["f32"]


def test_fused_status_contract():
    import torch
    x = dp.TensorView(dp.make_desc(1, 2, 5, 5), torch.zeros(50, device="cuda"))
    f = dp.FilterView(dp.make_filter_desc(3, 2, 3, 3), torch.zeros(54, device="cuda"))
    y = dp.TensorView(dp.make_desc(1, 3, 3, 3), torch.zeros(27, device="cuda"))
    bad = dp.TensorView(dp.make_desc(1, 4, 1, 1), torch.zeros(4, device="cuda"))
    with pytest.raises(dp.ShapeMismatch):
        dp.conv_bias_activation_forward(x, f, dp.ConvDesc(), "implicit", y, bias=bad)
    g = dp.TensorView(dp.make_desc(1, 2, 4, 5), torch.zeros(40, device="cuda"))
    with pytest.raises(dp.ShapeMismatch):
        dp.conv_backward_data_activation(y, f, dp.ConvDesc(), "implicit", x, "relu", g)


def test_fused_runs_in_the_epilogue():
    """The tensor-core path applies the ops in its epilogue: the fused call
    launches fewer kernels than the unfused sequence (no separate bias /
    activation kernels)."""
    import torch
    counts = {}
    for fused in (True, False):
        before = dp.kernel_launch_count()
        if fused:
            fwd_pair(SHAPES[0], "relu", True)
        else:
            fwd_pair(SHAPES[0], None, False)
        counts[fused] = dp.kernel_launch_count() - before
    torch.cuda.synchronize()
    # fused pair = fused call + (conv, bias, act) ; unfused pair = 2 x conv
    assert counts[True] == counts[False] + 2, counts
