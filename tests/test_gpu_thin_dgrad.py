"""fp64 / SIMT-fp32 special tiles.  Backward-data for thin outputs (C <= 4 channels, csrc/conv_simt.cu
thin::dgrad_thin_kernel): the fp64 and SIMT-fp32 paths run AlexNet conv1 /
Table-2 layer1 backward-data as a direct convolution over a shared-memory dy
halo.  Checked against the C oracle on strided phases (u, v > 1 with phases
that own fewer taps), both modes (filter flip), NHWC and channel-slice
views, accumulate, C = 1..4 and every phase-tap bucket (nSp 3 / 5 / 7 / 11 /
16); DNNP_SIMT_NO_THIN runs the same cases through the GEMM tiles."""
import os

import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

TOL = {np.float32: 1e-5, np.float64: 1e-12}


def run(n, c, h, w, k, r, s, u, v, ph, pw, dt, seed, layout="nchw", mode="convolution",
        acc=False):
    import torch
    rng = np.random.default_rng(seed)
    et = "f32" if dt == np.float32 else "f64"
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    xd = dp.make_desc(n, c, h, w, layout=layout, elem_type=et)
    yd = dp.make_desc(n, k, p, q, layout=layout, elem_type=et)
    dy = rng.uniform(-0.5, 0.5, yd.max_offset() + 1).astype(dt)
    f = rng.uniform(-0.5, 0.5, k * c * r * s).astype(dt)
    dx0 = rng.uniform(-0.5, 0.5, xd.max_offset() + 1).astype(dt)
    cd = dp.ConvDesc(u, v, ph, pw, mode, acc)
    cu = lambda a: torch.from_numpy(a.copy()).cuda()  # noqa: E731
    dxv = dp.TensorView(xd, cu(dx0))
    dp.conv_backward_data(dp.TensorView(yd, cu(dy)),
                          dp.FilterView(dp.make_filter_desc(k, c, r, s, elem_type=et), cu(f)),
                          cd, "implicit", dxv)
    torch.cuda.synchronize()
    ref = dx0.copy()
    orc.conv_backward_data([k, c, r, s], f, [n, k, p, q, *yd.strides], dy,
                           [u, v, ph, pw, 0 if mode == "convolution" else 1, int(acc)],
                           [n, c, h, w, *xd.strides], ref)
    return orc.rel_err(dxv.buf.cpu().numpy(), ref)


#        N  C   H   W   K   R   S  u  v ph pw
SHAPES = [(8, 3, 128, 124, 16, 11, 11, 4, 4, 2, 2),   # AlexNet conv1: 16 phases, 2-3 taps each
          (2, 3, 70, 66, 8, 11, 11, 1, 1, 0, 0),    # Table-2 layer1: nSp = 11
          (2, 1, 64, 80, 5, 3, 3, 1, 1, 1, 1),      # C = 1, nSp = 3
          (4, 2, 50, 47, 7, 5, 5, 2, 1, 2, 2),      # C = 2, mixed strides
          (2, 4, 48, 72, 6, 7, 7, 1, 1, 3, 3),      # C = 4, nSp = 7
          (2, 3, 40, 90, 4, 9, 16, 1, 1, 4, 5),     # nSp = 16 bucket, rectangular filter
          (6, 3, 100, 41, 3, 5, 9, 3, 2, 1, 0)]     # odd everything


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_thin_dgrad_vs_oracle(si, dt):
    if dt == np.float32:
        dp.set_math(dp.MATH_SIMT_FP32)
    try:
        mode = "convolution" if si % 2 == 0 else "cross_correlation"
        err = run(*SHAPES[si], dt, 700 + si, mode=mode)
        assert err <= TOL[dt], err
    finally:
        dp.set_math(dp.MATH_DEFAULT)


@pytest.mark.parametrize("si", [0, 1, 4])
def test_thin_dgrad_nhwc_and_accumulate_f64(si):
    assert run(*SHAPES[si], np.float64, 800 + si, layout="nhwc") <= 1e-12
    assert run(*SHAPES[si], np.float64, 810 + si, acc=True) <= 1e-12


@pytest.mark.parametrize("si", [0, 3])
def test_thin_dgrad_matches_gemm_tiles(si):
    """The GEMM tiles (DNNP_SIMT_NO_THIN) on the same case: both at the fp64 bar."""
    from test_gpu_tc_paths import env
    assert run(*SHAPES[si], np.float64, 900 + si) <= 1e-12
    with env(DNNP_SIMT_NO_THIN=1):
        assert run(*SHAPES[si], np.float64, 900 + si) <= 1e-12


# ---- fp64 128 x 128 tiles (SimtCfgBig64) --------------------------------------

BIG_SHAPES = [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1),     # ragged rows / columns / reduction
              (3, 130, 9, 10, 136, 3, 3, 2, 2, 1, 1),   # > 128 columns, strided phases
              (2, 16, 15, 15, 256, 5, 5, 1, 1, 2, 2)]   # two full column tiles


@pytest.mark.parametrize("si", range(len(BIG_SHAPES)))
def test_f64_big_tiles_forced(si):
    """DNNP_SIMT_BIG forces the 8 x 8-per-thread fp64 tile on every pass
    (by default it needs a full wave of tiles, which test-sized problems
    do not reach); fwd / bwd-data / bwd-filter against the oracle."""
    import torch
    from test_gpu_tc_paths import env
    n, c, h, w, k, r, s, u, v, ph, pw = BIG_SHAPES[si]
    rng = np.random.default_rng(950 + si)
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    xd = dp.make_desc(n, c, h, w, elem_type="f64")
    yd = dp.make_desc(n, k, p, q, elem_type="f64")
    fdsc = dp.make_filter_desc(k, c, r, s, elem_type="f64")
    x = rng.uniform(-0.5, 0.5, xd.max_offset() + 1)
    dy = rng.uniform(-0.5, 0.5, yd.max_offset() + 1)
    f = rng.uniform(-0.5, 0.5, k * c * r * s)
    cd = dp.ConvDesc(u, v, ph, pw)
    cu = lambda a: torch.from_numpy(a.copy()).cuda()  # noqa: E731
    xg, yg, fg = [n, c, h, w, *xd.strides], [n, k, p, q, *yd.strides], [k, c, r, s]
    cg = [u, v, ph, pw, 0, 0]
    ry, rdx, rdf = np.zeros(yd.max_offset() + 1), np.zeros(xd.max_offset() + 1), np.zeros(f.size)
    orc.conv_forward(xg, x, fg, f, cg, yg, ry, threads=os.cpu_count() or 1)
    orc.conv_backward_data(fg, f, yg, dy, cg, xg, rdx)
    orc.conv_backward_filter(xg, x, yg, dy, cg, fg, rdf, threads=os.cpu_count() or 1)
    with env(DNNP_SIMT_BIG=1):
        yv, dxv = dp.empty_view(yd, device="cuda"), dp.empty_view(xd, device="cuda")
        dfv = dp.FilterView(fdsc, torch.empty(f.size, dtype=torch.float64, device="cuda"))
        xv, fv, dyv = dp.TensorView(xd, cu(x)), dp.FilterView(fdsc, cu(f)), dp.TensorView(yd, cu(dy))
        dp.conv_forward(xv, fv, cd, "implicit", yv)
        dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
        dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
        torch.cuda.synchronize()
    errs = [orc.rel_err(yv.buf.cpu().numpy(), ry), orc.rel_err(dxv.buf.cpu().numpy(), rdx),
            orc.rel_err(dfv.buf.cpu().numpy(), rdf)]
    assert max(errs) <= 1e-12, errs
