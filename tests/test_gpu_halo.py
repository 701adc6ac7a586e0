"""Halo-tile tensor-core kernels (csrc/conv_halo.cuh, csrc/wgrad_halo.cuh):
the space-to-depth forward, backward-data and backward-filter of strided
few-channel convolutions (AlexNet conv1) read one halo of packed pixel rows
per tile and address every filter tap by the UMMA descriptor start row (and,
for backward-filter, a second tap by the descriptor's leading byte offset).  Checked against the C oracle: AlexNet
conv1 itself (default selection), and -- with DNNP_TC_HALO forcing the kernel
past its 80% useful-grid threshold -- the channel-block widths 16 / 32 / 64,
48- and 64-column tiles, ragged last tiles, both modes, NHWC and strided
views, alpha / beta and accumulate; DNNP_TC_NO_HALO gives the im2col kernel
on the same inputs."""
import os

import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp
from test_gpu_tc_paths import env

pytestmark = pytest.mark.gpu

TOL = 1e-4


def run(n, c, h, w, k, r, s, u, v, ph, pw, seed, passes=("fwd", "bwd_data", "bwd_filter"), layout="nchw",
        mode="convolution", acc=False, alpha=1.0, beta=0.0):
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
    cd = dp.ConvDesc(u, v, ph, pw, mode, acc)
    cu = lambda a: torch.from_numpy(a.copy()).cuda()  # noqa: E731
    fv = dp.FilterView(dp.make_filter_desc(k, c, r, s), cu(f))
    xg, yg, fg = [n, c, h, w, *xd.strides], [n, k, p, q, *yd.strides], [k, c, r, s]
    cg = [u, v, ph, pw, 0 if mode == "convolution" else 1, int(acc)]
    errs = {}
    if "fwd" in passes:
        yv = dp.TensorView(yd, cu(y0))
        dp.conv_forward(dp.TensorView(xd, cu(x)), fv, cd, "implicit", yv, alpha=alpha, beta=beta)
        ref = y0.copy()
        orc.conv_forward(xg, x, fg, f, cg, yg, ref, alpha=alpha, beta=beta)
        errs["fwd"] = orc.rel_err(yv.buf.cpu().numpy(), ref)
    if "bwd_data" in passes:
        dxv = dp.TensorView(xd, cu(dx0))
        dp.conv_backward_data(dp.TensorView(yd, cu(dy)), fv, cd, "implicit", dxv)
        ref = dx0.copy()
        orc.conv_backward_data(fg, f, yg, dy, cg, xg, ref)
        errs["bwd_data"] = orc.rel_err(dxv.buf.cpu().numpy(), ref)
    if "bwd_filter" in passes:
        df0 = rng.uniform(-0.5, 0.5, k * c * r * s).astype(np.float32)
        dfv = dp.FilterView(dp.make_filter_desc(k, c, r, s), cu(df0))
        dp.conv_backward_filter(dp.TensorView(yd, cu(dy)), dp.TensorView(xd, cu(x)), cd, "implicit", dfv)
        ref = df0.copy()
        orc.conv_backward_filter(xg, x, yg, dy, cg, fg, ref, threads=os.cpu_count() or 1)
        errs["bwd_filter"] = orc.rel_err(dfv.buf.cpu().numpy(), ref)
    torch.cuda.synchronize()
    return errs


def check(errs):
    assert max(errs.values()) <= TOL, errs


def test_alexnet_conv1_default():
    """conv1 at N=8 (the 93%-useful grid selects the halo kernel by default)."""
    check(run(8, 3, 224, 224, 64, 11, 11, 4, 4, 2, 2, 1))


@pytest.mark.parametrize("n", [1, 5])
def test_alexnet_conv1_small_and_odd_batches(n):
    """Single image (a partial tile per CTA pair, fewer chunks than clusters
    in the backward-filter split) and an odd batch, default selection; plus
    alpha / beta and accumulate on the default path."""
    check(run(n, 3, 224, 224, 64, 11, 11, 4, 4, 2, 2, 50 + n))
    check(run(n, 3, 224, 224, 64, 11, 11, 4, 4, 2, 2, 60 + n, alpha=-0.5, beta=2.0, passes=("fwd",)))
    check(run(n, 3, 224, 224, 64, 11, 11, 4, 4, 2, 2, 70 + n, acc=True, passes=("bwd_data", "bwd_filter")))


#        N   C   H   W   K   R   S  u  v ph pw
SHAPES = [(2, 3, 40, 44, 64, 11, 11, 4, 4, 2, 2),    # conv1-like: 48 channels (16-wide blocks), 64 cols
          (3, 3, 61, 57, 40, 11, 11, 4, 4, 2, 2),    # ragged: 40 output channels (48-column tile)
          (2, 4, 33, 35, 24, 6, 6, 2, 2, 1, 1),      # 16 s2d channels, 3 x 3 taps
          (2, 8, 30, 26, 64, 4, 4, 2, 2, 0, 1),      # 32 s2d channels (32-wide blocks)
          (2, 16, 22, 20, 48, 4, 4, 2, 2, 1, 1),     # 64 s2d channels (64-wide blocks)
          (1, 3, 19, 23, 16, 5, 7, 3, 2, 2, 3)]      # odd strides / pads, tiny grid


@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_halo_forced_vs_oracle(si):
    mode = "convolution" if si % 2 == 0 else "cross_correlation"
    with env(DNNP_TC_HALO=1):
        check(run(*SHAPES[si], 10 + si, mode=mode))
    with env(DNNP_TC_NO_HALO=1):
        check(run(*SHAPES[si], 10 + si, mode=mode))


@pytest.mark.parametrize("si", [0, 1])
def test_halo_nhwc_and_blend(si):
    with env(DNNP_TC_HALO=1):
        check(run(*SHAPES[si], 20 + si, layout="nhwc"))
        check(run(*SHAPES[si], 30 + si, alpha=0.75, beta=0.5, passes=("fwd",)))
        check(run(*SHAPES[si], 40 + si, acc=True, passes=("bwd_data", "bwd_filter")))
