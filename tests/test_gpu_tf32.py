"""3xTF32 tensor-core mode (DNNP_MATH_TC_TF32X3, north_star's named fp32
split): every operand a = big + small with big = tf32(a), small =
tf32(a - big); each 8-deep k-step issues big.small + small.big + big.big
with tcgen05.mma.kind::tf32 into one fp32 TMEM accumulator.  Checked
against the C oracle like BF16x3, on the benchmark layers and on every
kernel variant the planner selects (space-to-depth, tap folding, row /
column blocking, super-pixel backward-data, CTA pairs, stream-K,
reduction segments, NHWC / strided views), plus the SIMT fallback for
geometries outside the TMA kernels."""
import os

import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north_star fp32 bar (normalised)


@pytest.fixture(autouse=True)
def _tf32_mode():
    dp.set_math(dp.MATH_TC_TF32X3)
    yield
    dp.set_math(dp.MATH_DEFAULT)


def run_all(n, c, h, w, k, r, s, u, v, ph, pw, seed, layout="nchw",
            mode="convolution", acc=False):
    import torch
    rng = np.random.default_rng(seed)
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    xd = dp.make_desc(n, c, h, w, layout=layout)
    yd = dp.make_desc(n, k, p, q, layout=layout)
    x = rng.uniform(-0.5, 0.5, xd.max_offset() + 1).astype(np.float32)
    dy = rng.uniform(-0.5, 0.5, yd.max_offset() + 1).astype(np.float32)
    f = rng.uniform(-0.5, 0.5, k * c * r * s).astype(np.float32)
    y0 = rng.uniform(-0.5, 0.5, yd.max_offset() + 1).astype(np.float32)
    dx0 = rng.uniform(-0.5, 0.5, xd.max_offset() + 1).astype(np.float32)
    df0 = rng.uniform(-0.5, 0.5, k * c * r * s).astype(np.float32)
    cd = dp.ConvDesc(u, v, ph, pw, mode, acc)
    cu = lambda a: torch.from_numpy(a.copy()).cuda()  # noqa: E731
    xv, dyv = dp.TensorView(xd, cu(x)), dp.TensorView(yd, cu(dy))
    fv = dp.FilterView(dp.make_filter_desc(k, c, r, s), cu(f))
    yv, dxv = dp.TensorView(yd, cu(y0)), dp.TensorView(xd, cu(dx0))
    dfv = dp.FilterView(dp.make_filter_desc(k, c, r, s), cu(df0))
    dp.conv_forward(xv, fv, cd, "implicit", yv)
    dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
    dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
    torch.cuda.synchronize()
    xg, yg = [n, c, h, w, *xd.strides], [n, k, p, q, *yd.strides]
    fg = [k, c, r, s]
    cg = [u, v, ph, pw, 0 if mode == "convolution" else 1, int(acc)]
    ry, rdx, rdf = y0.copy(), dx0.copy(), df0.copy()
    orc.conv_forward(xg, x, fg, f, cg, yg, ry, beta=1.0 if acc else 0.0,
                     threads=os.cpu_count() or 1)
    orc.conv_backward_data(fg, f, yg, dy, cg, xg, rdx)
    orc.conv_backward_filter(xg, x, yg, dy, cg, fg, rdf, threads=os.cpu_count() or 1)
    return {"fwd": orc.rel_err(yv.buf.cpu().numpy(), ry),
            "bwd_data": orc.rel_err(dxv.buf.cpu().numpy(), rdx),
            "bwd_filter": orc.rel_err(dfv.buf.cpu().numpy(), rdf)}


ALEXNET = [("conv1", 3, 224, 64, 11, 4, 2), ("conv2", 64, 27, 192, 5, 1, 2),
           ("conv3", 192, 13, 384, 3, 1, 1), ("conv4", 384, 13, 256, 3, 1, 1),
           ("conv5", 256, 13, 256, 3, 1, 1)]


@pytest.mark.parametrize("li", range(5), ids=[a[0] for a in ALEXNET])
def test_tf32x3_alexnet_vs_oracle(li):
    _, c, h, k, r, u, pad = ALEXNET[li]
    errs = run_all(32, c, h, h, k, r, r, u, u, pad, pad, 100 + li)
    assert max(errs.values()) <= TOL, errs


#        N   C   H   W   K   R   S  u  v ph pw
SHAPES = [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1),      # channel columns, padding
          (2, 3, 40, 44, 64, 11, 11, 4, 4, 2, 2),    # space-to-depth
          (2, 3, 40, 44, 96, 11, 11, 1, 1, 0, 0),    # tap folding / wide column blocking
          (2, 16, 15, 15, 24, 5, 5, 2, 2, 2, 2),     # super-pixel bwd-data
          (3, 64, 15, 15, 96, 5, 5, 1, 1, 2, 2),     # row-blocked bwd-data
          (2, 32, 13, 13, 256, 3, 3, 1, 1, 1, 1),    # CTA pairs
          (8, 64, 13, 13, 192, 3, 3, 1, 1, 1, 1),    # stream-K last wave
          (1, 256, 14, 14, 96, 7, 7, 1, 1, 3, 3),    # long reduction (segments), small grid
          (2, 5, 9, 7, 7, 2, 3, 3, 2, 1, 0)]         # odd everything


@pytest.mark.parametrize("layout", ["nchw", "nhwc"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_tf32x3_variants_vs_oracle(si, layout):
    mode = "convolution" if si % 2 == 0 else "cross_correlation"
    errs = run_all(*SHAPES[si], 200 + si, layout=layout, mode=mode)
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("si", [0, 1, 5])
def test_tf32x3_accumulate(si):
    errs = run_all(*SHAPES[si], 300 + si, acc=True)
    assert max(errs.values()) <= TOL, errs


def test_tf32x3_mode_reported():
    assert dp.get_math() == dp.MATH_TC_TF32X3
