"""Additive fused backward (dnnp_convolution_backward): dx and dw of one
layer in one call, dy packed once for both tensor-core GEMMs; bit-identical
to the two separate calls (same kernels, same packed operands), including
accumulate, host buffers, and the fallbacks (K not a multiple of 64, fp64,
SIMT fp32, x / dx with different layouts)."""
import numpy as np
import pytest

import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

SHAPES = [(4, 64, 27, 27, 192, 5, 5, 1, 1, 2, 2),      # conv2-like (row-blocked dgrad)
          (2, 3, 40, 44, 64, 11, 11, 4, 4, 2, 2),      # space-to-depth
          (4, 96, 13, 13, 128, 3, 3, 1, 1, 1, 1),
          (2, 16, 15, 15, 40, 3, 3, 1, 1, 1, 1)]       # K % 64 != 0: two plain calls


def run(shape, dt="f32", acc=False, host=False, dx_layout="nchw", fused=True, seed=0):
    import torch
    n, c, h, w, k, r, s, u, v, ph, pw = shape
    rng = np.random.default_rng(seed)
    npdt = np.float32 if dt == "f32" else np.float64
    cd = dp.ConvDesc(u, v, ph, pw, "convolution", acc)
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    mk = lambda cnt: rng.uniform(-0.5, 0.5, cnt).astype(npdt)
    x, f, dy, dx0, df0 = mk(n * c * h * w), mk(k * c * r * s), mk(n * k * p * q), mk(n * c * h * w), mk(k * c * r * s)
    conv = (lambda a: a.copy()) if host else (lambda a: torch.from_numpy(a.copy()).cuda())
    xd = dp.make_desc(n, c, h, w, elem_type=dt)
    dxd = dp.make_desc(n, c, h, w, layout=dx_layout, elem_type=dt)
    yd = dp.make_desc(n, k, p, q, elem_type=dt)
    fd = dp.make_filter_desc(k, c, r, s, elem_type=dt)
    xv, dyv = dp.TensorView(xd, conv(x)), dp.TensorView(yd, conv(dy))
    fv = dp.FilterView(fd, conv(f))
    dxv, dfv = dp.TensorView(dxd, conv(dx0)), dp.FilterView(fd, conv(df0))
    if fused:
        dp.conv_backward(dyv, fv, xv, cd, "implicit", dxv, dfv)
    else:
        dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
        dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
    torch.cuda.synchronize()
    get = (lambda b: b) if host else (lambda b: b.cpu().numpy())
    return get(dxv.buf), get(dfv.buf)


@pytest.mark.parametrize("shape", SHAPES, ids=[f"s{i}" for i in range(len(SHAPES))])
@pytest.mark.parametrize("acc", [False, True])
def test_fused_backward_matches_separate(shape, acc):
    a = run(shape, acc=acc, fused=True)
    b = run(shape, acc=acc, fused=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_fused_backward_fallbacks():
    for kw in ({"dt": "f64"}, {"host": True}, {"dx_layout": "nhwc"}):
        a = run(SHAPES[2], fused=True, **kw)
        b = run(SHAPES[2], fused=False, **kw)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), kw
    dp.set_math(dp.MATH_SIMT_FP32)
    try:
        a = run(SHAPES[2], fused=True)
        b = run(SHAPES[2], fused=False)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    finally:
        dp.set_math(dp.MATH_DEFAULT)
