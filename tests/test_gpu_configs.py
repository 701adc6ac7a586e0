"""Oracle parity at the BASELINE.json configurations themselves.

The CUDA path (through the reference-shaped Python API) against the C oracle
(oracle/, pinned to golden vectors produced by the reference package) on the
reference bench generator's inputs: uniform(-0.5, 0.5) from
np.random.default_rng([2014, layer_index]) in layer order x, f (then dy),
reference pkg/src/dnnp/bench.py:151-157.

* configs[0]  C1: N=16 C=64 56x56 K=64 3x3 pad 1 (fp32 and fp64);
* configs[1]  AlexNet conv1-5 at N=128, every pass (the benchmarked step);
* Table-2 layers (pkg/src/dnnp/suites/table2.suite) at N=16;
* configs[4]  the bandwidth primitives on 128x64x55x55 (activation, 3x3/2
  max/avg pooling), 1024x1000x1x1 per-image and 16x21x64x64 per-spatial
  softmax, on dense NCHW, NHWC and a channel slice [16:48) of a 64-channel
  parent, fp32 and fp64.

Bars (north_star): fp32 <= 1e-4, fp64 <= 1e-12 normalised error
max|gpu - oracle| / max|oracle|; argmax, max-pool values and pooling /
activation backward bit-exact.
"""
import os

import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1
TOL = {np.float32: 1e-4, np.float64: 1e-12}


def _torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def bench_inputs(n, c, h, w, k, r, s, p, q, index, dt):
    """Reference bench generator (bench.py:151-157) plus dy as the next draw."""
    g = np.random.default_rng([2014, index])
    x = g.uniform(-0.5, 0.5, n * c * h * w)
    f = g.uniform(-0.5, 0.5, k * c * r * s)
    dy = g.uniform(-0.5, 0.5, n * k * p * q)
    return x.astype(dt), f.astype(dt), dy.astype(dt)


def conv_vs_oracle(n, c, h, w, k, r, s, u, v, ph, pw, index, dt):
    """GPU fwd / bwd-data / bwd-filter vs the oracle; returns the errors."""
    torch = _torch()
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    x, f, dy = bench_inputs(n, c, h, w, k, r, s, p, q, index, dt)
    et = "f32" if dt == np.float32 else "f64"
    cd = dp.ConvDesc(u, v, ph, pw, "convolution")
    xt, ft, dyt = (torch.from_numpy(a).cuda() for a in (x, f, dy))
    xv = dp.TensorView(dp.make_desc(n, c, h, w, elem_type=et), xt)
    fv = dp.FilterView(dp.make_filter_desc(k, c, r, s, elem_type=et), ft)
    dyv = dp.TensorView(dp.make_desc(n, k, p, q, elem_type=et), dyt)
    yv = dp.empty_view(dp.make_desc(n, k, p, q, elem_type=et), device="cuda")
    dxv = dp.empty_view(dp.make_desc(n, c, h, w, elem_type=et), device="cuda")
    dft = torch.empty(k * c * r * s, device="cuda", dtype=xt.dtype)
    dfv = dp.FilterView(dp.make_filter_desc(k, c, r, s, elem_type=et), dft)
    dp.conv_forward(xv, fv, cd, "implicit", yv)
    dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
    dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
    torch.cuda.synchronize()
    xg = [n, c, h, w, c * h * w, h * w, w, 1]
    yg = [n, k, p, q, k * p * q, p * q, q, 1]
    fg, cg = [k, c, r, s], [u, v, ph, pw, 0, 0]
    ry = np.zeros(n * k * p * q, dt)
    orc.conv_forward(xg, x, fg, f, cg, yg, ry, threads=THREADS)
    rdx = np.zeros(n * c * h * w, dt)
    orc.conv_backward_data(fg, f, yg, dy, cg, xg, rdx)
    rdf = np.zeros(k * c * r * s, dt)
    orc.conv_backward_filter(xg, x, yg, dy, cg, fg, rdf, threads=THREADS)
    return {"fwd": orc.rel_err(yv.buf.cpu().numpy(), ry),
            "bwd_data": orc.rel_err(dxv.buf.cpu().numpy(), rdx),
            "bwd_filter": orc.rel_err(dft.cpu().numpy(), rdf)}


@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=["f32", "f64"])
def test_c1_vs_oracle(dt):
    """configs[0]: the reference's CPU-runnable case (layer index 0)."""
    errs = conv_vs_oracle(16, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1, 0, dt)
    assert max(errs.values()) <= TOL[dt], errs


ALEXNET = [  # torchvision shapes: name, C, H, K, R, stride, pad
    ("conv1", 3, 224, 64, 11, 4, 2),
    ("conv2", 64, 27, 192, 5, 1, 2),
    ("conv3", 192, 13, 384, 3, 1, 1),
    ("conv4", 384, 13, 256, 3, 1, 1),
    ("conv5", 256, 13, 256, 3, 1, 1),
]


@pytest.mark.parametrize("li", range(5), ids=[a[0] for a in ALEXNET])
def test_alexnet_n128_vs_oracle(li):
    """configs[1] at full size: the benchmarked step's inputs (bench.py
    make_inputs draws the same arrays), every pass, fp32."""
    _, c, h, k, r, u, pad = ALEXNET[li]
    errs = conv_vs_oracle(128, c, h, h, k, r, r, u, u, pad, pad, li, np.float32)
    assert max(errs.values()) <= TOL[np.float32], errs


@pytest.mark.parametrize("li", range(5), ids=[a[0] for a in ALEXNET])
def test_alexnet_f64_vs_oracle(li):
    """The fp64 (DFMA) path on the AlexNet shapes at N=8."""
    _, c, h, k, r, u, pad = ALEXNET[li]
    errs = conv_vs_oracle(8, c, h, h, k, r, r, u, u, pad, pad, li, np.float64)
    assert max(errs.values()) <= TOL[np.float64], errs


TABLE2 = [  # pkg/src/dnnp/suites/table2.suite:3-7 (C, H=W, K, R=S; unit stride, no pad)
    ("layer1", 3, 128, 96, 11),
    ("layer2", 96, 64, 128, 9),
    ("layer3", 128, 32, 128, 9),
    ("layer4", 128, 16, 128, 7),
    ("layer5", 384, 13, 384, 3),
]


@pytest.mark.parametrize("li", range(5), ids=[t[0] for t in TABLE2])
def test_table2_n16_vs_oracle(li):
    """Table-2 layers at the reference verify batch (16): long reductions
    (layer1 dW sums 16*118*118 products per weight)."""
    _, c, h, k, r = TABLE2[li]
    errs = conv_vs_oracle(16, c, h, h, k, r, r, 1, 1, 0, 0, li, np.float32)
    assert max(errs.values()) <= TOL[np.float32], errs


# ---------------------------------------------------------------- configs[4]

LAYOUTS = ("nchw", "nhwc", "slice")


def bw_view(rng, n, c, h, w, dt, layout):
    """(TensorView on cuda, host buffer from the view's base, oracle geometry,
    device buffer).  'slice' = channels [16:48) of a 64-channel NCHW parent,
    with the parent's strides and an offset base pointer."""
    torch = _torch()
    et = "f32" if dt == np.float32 else "f64"
    if layout == "slice":
        pc = 64
        buf = rng.uniform(-0.5, 0.5, n * pc * h * w).astype(dt)
        strides = (pc * h * w, h * w, w, 1)
        base = 16 * h * w
        desc = dp.make_desc(n, 32, h, w, layout="custom", strides=strides, elem_type=et)
        t = torch.from_numpy(buf).cuda()
        g = [n, 32, h, w, *strides]
        return dp.TensorView(desc, t[base:]), buf[base:], g, t[base:]
    desc = dp.make_desc(n, c, h, w, layout=layout, elem_type=et)
    buf = rng.uniform(-0.5, 0.5, desc.max_offset() + 1).astype(dt)
    t = torch.from_numpy(buf).cuda()
    return dp.TensorView(desc, t), buf, [n, c, h, w, *desc.strides], t


ACT_SHAPE = (128, 64, 55, 55)


def _ids(dt):
    return "f32" if dt == np.float32 else "f64"


@pytest.mark.parametrize("kind", ["sigmoid", "relu", "tanh"])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=_ids)
@pytest.mark.parametrize("layout", LAYOUTS)
def test_activation_bshape_vs_oracle(layout, dt, kind):
    rng = np.random.default_rng(6100)
    kcode = {"sigmoid": 0, "relu": 1, "tanh": 2}[kind]
    n, c, h, w = ACT_SHAPE
    xv, x, xg, _ = bw_view(rng, n, c, h, w, dt, layout)
    x *= 8.0  # exercise saturation of sigmoid / tanh
    xv.buf.copy_(_torch().from_numpy(x))
    yv, _, yg, yt = bw_view(rng, n, c, h, w, dt, layout)
    dp.activation_forward(kind, xv, yv)
    yref = np.zeros_like(yt.cpu().numpy())
    yref[:] = yt.cpu().numpy()  # gaps of a slice view keep their values
    orc.activation_forward(kcode, xg, x, yg, yref)
    assert orc.rel_err(yt.cpu().numpy(), yref) <= TOL[dt]
    ydev = yt.cpu().numpy()
    dyv, dy, dyg, _ = bw_view(rng, n, c, h, w, dt, layout)
    dxv, _, dxg, dxt = bw_view(rng, n, c, h, w, dt, layout)
    dxref = dxt.cpu().numpy().copy()
    dp.activation_backward(kind, yv, dyv, dxv)
    orc.activation_backward(kcode, yg, ydev, dyg, dy, dxg, dxref)
    assert np.array_equal(dxt.cpu().numpy(), dxref)


@pytest.mark.parametrize("kind", ["max", "average"])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=_ids)
@pytest.mark.parametrize("layout", LAYOUTS)
def test_pool_bshape_vs_oracle(layout, dt, kind):
    """AlexNet pool1: 128x64x55x55, 3x3 stride 2 -> 27x27."""
    torch = _torch()
    rng = np.random.default_rng(6200)
    n, c, h, w = ACT_SHAPE
    pd = dp.PoolingDesc(kind, 3, 3, 2, 2, 0, 0)
    pg = [0 if kind == "max" else 1, 3, 3, 2, 2, 0, 0]
    xv, x, xg, _ = bw_view(rng, n, c, h, w, dt, layout)
    _, cc, P, Q = dp.pool_out_shape(pd, xv)
    yv, _, yg, yt = bw_view(rng, n, cc, P, Q, dt, layout)
    am = torch.full((n, cc, P, Q), -1, dtype=torch.int64, device="cuda") if kind == "max" else None
    dp.pool_forward(pd, xv, yv, am)
    yref = yt.cpu().numpy().copy()
    amref = np.full(n * cc * P * Q, -1, dtype=np.int64)
    orc.pool_forward(pg, xg, x, yg, yref, amref if kind == "max" else None)
    if kind == "max":
        assert np.array_equal(am.cpu().numpy().reshape(-1), amref)
        assert np.array_equal(yt.cpu().numpy(), yref)
    else:
        assert orc.rel_err(yt.cpu().numpy(), yref) <= TOL[dt]
    dyv, dy, dyg, _ = bw_view(rng, n, cc, P, Q, dt, layout)
    dxv, _, dxg, dxt = bw_view(rng, n, cc, h, w, dt, layout)
    dxref = dxt.cpu().numpy().copy()
    dp.pool_backward(pd, yv, dyv, xv, dxv, am)
    orc.pool_backward(pg, dyg, dy, dxg, dxref, amref if kind == "max" else None)
    assert np.array_equal(dxt.cpu().numpy(), dxref)


@pytest.mark.parametrize("case", ["per_image_1024x1000", "per_spatial_16x21x64x64"])
@pytest.mark.parametrize("dt", [np.float32, np.float64], ids=_ids)
@pytest.mark.parametrize("layout", LAYOUTS)
def test_softmax_bshape_vs_oracle(layout, dt, case):
    mode = "per_image" if case.startswith("per_image") else "per_spatial"
    shape = (1024, 1000, 1, 1) if mode == "per_image" else (16, 21, 64, 64)
    rng = np.random.default_rng(6300)
    n, c, h, w = shape
    mcode = 0 if mode == "per_image" else 1
    xv, x, xg, _ = bw_view(rng, n, c, h, w, dt, layout)
    x *= 8.0
    xv.buf.copy_(_torch().from_numpy(x))
    yv, _, yg, yt = bw_view(rng, n, c, h, w, dt, layout)
    dp.softmax_forward(mode, xv, yv)
    yref = yt.cpu().numpy().copy()
    orc.softmax_forward(mcode, xg, x, yg, yref)
    assert orc.rel_err(yt.cpu().numpy(), yref) <= TOL[dt]
    ydev = yt.cpu().numpy()
    dyv, dy, dyg, _ = bw_view(rng, n, c, h, w, dt, layout)
    dxv, _, dxg, dxt = bw_view(rng, n, c, h, w, dt, layout)
    dxref = dxt.cpu().numpy().copy()
    dp.softmax_backward(mode, yv, dyv, dxv)
    orc.softmax_backward(mcode, yg, ydev, dyg, dy, dxg, dxref)
    assert orc.rel_err(dxt.cpu().numpy(), dxref) <= TOL[dt]
