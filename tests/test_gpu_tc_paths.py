"""GPU parity of every variant of the tensor-core convolution path against the
C oracle (fp32, normalised error <= 1e-4, the test_acceptance.py:91-96
metric).  Variants are selected per call through the library's environment
switches (read on every call):

  space-to-depth (strided, few channels)   DNNP_TC_NO_S2D
  CTA pairs / single CTAs                  DNNP_TC_NC=2 / DNNP_TC_NC=1
  stream-K last wave                       DNNP_TC_SK=1 (+ DNNP_TC_NC / DNNP_TC_BN)
  column blocking (unit-stride small N)    DNNP_TC_NO_BLOCK
  cp.async gather kernel (no TMA)          DNNP_TC_NO_TMA
and through the problem shape: 16/32/64-channel TMA blocks, super-pixel
strided bwd-data, strided output views with alpha/beta/accumulate."""
import contextlib
import os

import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

TOL = 1e-4


@contextlib.contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    try:
        for k, v in kv.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
        dp._lib.reload_tuning()  # the library caches the switches
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        dp._lib.reload_tuning()


def rand_view(rng, n, c, h, w, layout="nchw", fill=None):
    import torch
    desc = dp.make_desc(n, c, h, w, layout=layout)
    buf = rng.uniform(-0.5, 0.5, desc.max_offset() + 1).astype(np.float32)
    if fill is not None:
        buf[:] = fill
    g = np.array([n, c, h, w, *desc.strides], dtype=np.int64)
    t = torch.from_numpy(buf.copy()).cuda()
    return dp.TensorView(desc, t), buf, g, t


def run_case(shape, passes=("fwd", "bwd_data", "bwd_filter"), layout_in="nchw",
             layout_out="nchw", mode="convolution", seed=0, alpha=1.0, beta=0.0,
             accumulate=False):
    import torch
    rng = np.random.default_rng(seed)
    N, C, H, W, K, R, S, u, v, ph, pw = shape
    cd = dp.ConvDesc(u, v, ph, pw, mode, accumulate)
    cg = [u, v, ph, pw, 0 if mode == "convolution" else 1, 1 if accumulate else 0]
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    f = rng.uniform(-0.5, 0.5, K * C * R * S).astype(np.float32)
    fv = dp.FilterView(dp.make_filter_desc(K, C, R, S), torch.from_numpy(f).cuda())
    errs = {}
    if "fwd" in passes:
        xv, x, xg, _ = rand_view(rng, N, C, H, W, layout_in)
        yv, y0, yg, yt = rand_view(rng, N, K, P, Q, layout_out)
        dp.conv_forward(xv, fv, cd, "implicit", yv, alpha=alpha, beta=beta)
        ref = y0.copy()
        orc.conv_forward(xg, x, [K, C, R, S], f, cg, yg, ref, alpha=alpha, beta=beta, threads=8)
        errs["fwd"] = orc.rel_err(yt.cpu().numpy(), ref)
    if "bwd_data" in passes:
        dyv, dy, dyg, _ = rand_view(rng, N, K, P, Q, layout_in)
        dxv, dx0, dxg, dxt = rand_view(rng, N, C, H, W, layout_out)
        dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
        ref = dx0.copy()
        orc.conv_backward_data([K, C, R, S], f, dyg, dy, cg, dxg, ref)
        errs["bwd_data"] = orc.rel_err(dxt.cpu().numpy(), ref)
    if "bwd_filter" in passes:
        xv, x, xg, _ = rand_view(rng, N, C, H, W, layout_in)
        dyv, dy, dyg, _ = rand_view(rng, N, K, P, Q, layout_out)
        df0 = rng.uniform(-0.5, 0.5, K * C * R * S).astype(np.float32)
        dft = torch.from_numpy(df0.copy()).cuda()
        dfv = dp.FilterView(dp.make_filter_desc(K, C, R, S), dft)
        dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
        ref = df0.copy()
        orc.conv_backward_filter(xg, x, dyg, dy, cg, [K, C, R, S], ref, threads=8)
        errs["bwd_filter"] = orc.rel_err(dft.cpu().numpy(), ref)
    return errs


def check(errs):
    bad = {k: v for k, v in errs.items() if not v <= TOL}
    assert not bad, errs


#       N  C   H   W   K   R   S  u  v ph pw
S2D_SHAPES = [
    (2, 3, 31, 31, 16, 11, 11, 4, 4, 2, 2),    # ragged width (per-pixel space-to-depth pack)
    (2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2),    # W % 4 == 0
    (3, 4, 20, 20, 24, 5, 5, 2, 2, 2, 2),      # stride 2, 16 phase channels
    (2, 2, 17, 23, 40, 7, 5, 3, 2, 1, 2),      # anisotropic stride / filter / padding
]


@pytest.mark.parametrize("shape", S2D_SHAPES)
@pytest.mark.parametrize("mode", ["convolution", "cross_correlation"])
def test_space_to_depth(shape, mode):
    check(run_case(shape, mode=mode, seed=1))
    with env(DNNP_TC_NO_S2D=1):
        check(run_case(shape, mode=mode, seed=1))


@pytest.mark.parametrize("shape", [
    (2, 32, 13, 13, 48, 3, 3, 2, 2, 1, 1),     # super-pixel bwd-data, 4 phases
    (1, 40, 15, 14, 24, 5, 4, 3, 2, 2, 1),     # 6 phases, ragged image
])
def test_strided_super_pixel(shape):
    check(run_case(shape, seed=2))


@pytest.mark.parametrize("block", [None, 1])
@pytest.mark.parametrize("shape", [
    (2, 64, 15, 15, 96, 5, 5, 1, 1, 2, 2),     # conv2-like bwd-data, N = 64 -> blocked 128
    (3, 16, 9, 11, 32, 3, 3, 1, 1, 1, 1),      # odd output width: ragged last block
])
def test_column_blocking(shape, block):
    with env(DNNP_TC_NO_BLOCK=block):
        check(run_case(shape, seed=3))


@pytest.mark.parametrize("nc", [1, 2])
@pytest.mark.parametrize("shape", [
    (4, 64, 14, 14, 192, 3, 3, 1, 1, 1, 1),
    (2, 96, 13, 13, 256, 3, 3, 1, 1, 1, 1),
])
def test_cta_pairs(shape, nc):
    with env(DNNP_TC_NC=nc):
        check(run_case(shape, seed=4))


@pytest.mark.parametrize("cin", [16, 24, 40])  # 16 / 32 / 64-channel TMA blocks (40 -> OOB fill)
def test_channel_blocks(cin):
    check(run_case((2, cin, 10, 12, 32, 3, 3, 1, 1, 1, 1), seed=5))


def test_stream_k_last_wave():
    # 160 row tiles of 128 on 148 persistent CTAs: 12-tile last wave split along K
    shape = (20, 32, 32, 32, 64, 3, 3, 1, 1, 1, 1)
    with env(DNNP_TC_SK=1, DNNP_TC_NC=1, DNNP_TC_BN=64):
        check(run_case(shape, passes=("fwd", "bwd_data"), seed=6))
    with env(DNNP_TC_SK=1, DNNP_TC_NC=2, DNNP_TC_BN=64):
        check(run_case(shape, passes=("fwd",), seed=6))


@pytest.mark.parametrize("shape", [
    (2, 3, 31, 31, 16, 11, 11, 4, 4, 2, 2),
    (2, 16, 15, 15, 24, 5, 5, 1, 1, 2, 2),
    (2, 32, 13, 13, 48, 3, 3, 2, 2, 1, 1),
])
def test_cp_async_fallback(shape):
    with env(DNNP_TC_NO_TMA=1):
        check(run_case(shape, seed=7))


@pytest.mark.parametrize("lin,lout", [("nhwc", "nchw"), ("nchw", "nhwc"), ("nhwc", "nhwc")])
def test_layouts(lin, lout):
    check(run_case((2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1), layout_in=lin, layout_out=lout, seed=8))
    check(run_case((2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2), layout_in=lin, layout_out=lout, seed=8))


@pytest.mark.parametrize("alpha,beta", [(0.5, 0.0), (2.0, -1.5), (1.0, 1.0)])
def test_alpha_beta(alpha, beta):
    check(run_case((2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1), passes=("fwd",), alpha=alpha, beta=beta,
                   seed=9))
    check(run_case((2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2), passes=("fwd",), alpha=alpha,
                   beta=beta, seed=9))


def test_accumulate_all_passes():
    check(run_case((2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1), accumulate=True, seed=10))
    check(run_case((2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2), accumulate=True, seed=10))
    check(run_case((2, 64, 15, 15, 96, 5, 5, 1, 1, 2, 2), passes=("bwd_data",), accumulate=True,
                   seed=10))


@pytest.mark.parametrize("tma", [1, 0], ids=["tma", "cp_async"])
@pytest.mark.parametrize("alpha,beta,accumulate", [(1.0, 0.0, False), (0.5, -0.75, False),
                                                   (1.0, 0.0, True)])
def test_reduction_segments(tma, alpha, beta, accumulate):
    """Reductions split into k-block segments chained through the output
    (DNNP_TC_CHAIN forces several segments on a small problem; the wgrad
    analogue DNNP_WG_CHAIN forces more splits)."""
    kv = dict(DNNP_TC_CHAIN=128, DNNP_WG_CHAIN=64)
    if not tma:
        kv["DNNP_TC_NO_TMA"] = 1
    with env(**kv):
        check(run_case((2, 40, 11, 9, 24, 3, 3, 1, 1, 1, 1), alpha=alpha, beta=beta,
                       accumulate=accumulate, seed=11))
        check(run_case((2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2), passes=("fwd", "bwd_data"),
                       alpha=alpha, beta=beta, accumulate=accumulate, seed=11))


def test_long_reduction_accuracy():
    """C*R*S = 512*49 = 25088 products per output: past the single-accumulator
    truncation budget, so the forward / bwd-data run segmented (vs fp64)."""
    check(run_case((2, 512, 9, 9, 64, 7, 7, 1, 1, 3, 3), passes=("fwd",), seed=12))
    check(run_case((2, 64, 9, 9, 512, 7, 7, 1, 1, 3, 3), passes=("bwd_data",), seed=12))


#        N  C   H   W   K   R   S  u  v ph pw
FOLD_SHAPES = [
    (2, 3, 40, 44, 96, 11, 11, 1, 1, 0, 0),   # paper Table-2 layer1-like (C=3, 11x11, stride 1)
    (2, 3, 17, 19, 24, 5, 7, 1, 1, 2, 3),     # anisotropic filter / padding
    (2, 8, 23, 21, 16, 5, 5, 4, 4, 2, 2),     # strided, C*u*v > 64 (no space-to-depth)
    (2, 4, 15, 15, 32, 3, 9, 2, 1, 1, 4),     # vertical stride only
]


@pytest.mark.parametrize("shape", FOLD_SHAPES)
@pytest.mark.parametrize("mode", ["convolution", "cross_correlation"])
def test_tap_folding(shape, mode):
    """Horizontal taps folded into channels (forward, backward-filter) vs the
    oracle, and the unfolded path for comparison (DNNP_TC_NO_FOLD)."""
    check(run_case(shape, mode=mode, seed=13))
    with env(DNNP_TC_NO_FOLD=1):
        check(run_case(shape, passes=("fwd", "bwd_filter"), mode=mode, seed=13))


def test_tap_folding_layouts_and_scalars():
    check(run_case(FOLD_SHAPES[0], layout_in="nhwc", layout_out="nchw", seed=14))
    check(run_case(FOLD_SHAPES[1], passes=("fwd",), alpha=0.5, beta=-1.0, seed=14))
    check(run_case(FOLD_SHAPES[2], accumulate=True, seed=14))


@pytest.mark.parametrize("shape", [(2, 3, 40, 44, 96, 11, 11, 1, 1, 0, 0),
                                   (2, 5, 19, 23, 24, 5, 7, 1, 1, 2, 3),
                                   (3, 12, 17, 15, 40, 3, 3, 1, 1, 1, 1)])
def test_wide_column_blocking(shape):
    """Narrow unit-stride bwd-data outputs block 4 or 8 output columns per
    GEMM row (DNNP_TC_BW2 pins the factor to 2)."""
    check(run_case(shape, passes=("bwd_data",), seed=15))
    check(run_case(shape, passes=("bwd_data",), accumulate=True, seed=15))
    with env(DNNP_TC_BW2=1):
        check(run_case(shape, passes=("bwd_data",), seed=15))
    with env(DNNP_TC_NO_2D=1):  # columns only (the default adds 2 rows: a 2 x bw block)
        check(run_case(shape, passes=("bwd_data",), seed=15))


@pytest.mark.parametrize("shape", [(2, 3, 40, 44, 24, 11, 11, 1, 1, 0, 0),
                                   (2, 5, 33, 31, 16, 5, 5, 2, 2, 2, 2),
                                   (3, 12, 30, 30, 8, 3, 3, 1, 1, 1, 1),
                                   (8, 3, 96, 96, 4, 11, 11, 4, 4, 2, 2)])
def test_simt_narrow_tiles(shape):
    """Thin GEMMs on the SIMT fp32 path: <= 4 output columns take the tiny
    tile, <= 16 the narrow one (DNNP_SIMT_NO_TINY / DNNP_SIMT_NO_NARROW step
    back to the wider tiles); fp64 is covered by test_gpu_parity's thin
    shapes."""
    dp.set_math(dp.MATH_SIMT_FP32)
    try:
        check(run_case(shape, seed=16))
        with env(DNNP_SIMT_NO_TINY=1):
            check(run_case(shape, passes=("fwd", "bwd_data"), seed=16))
        with env(DNNP_SIMT_NO_TINY=1, DNNP_SIMT_NO_NARROW=1):
            check(run_case(shape, passes=("fwd", "bwd_data"), seed=16))
    finally:
        dp.set_math(dp.MATH_DEFAULT)


@pytest.mark.parametrize("shape", [(2, 24, 11, 9, 192, 3, 3, 1, 1, 1, 1),
                                   (2, 16, 13, 13, 64, 5, 5, 1, 1, 2, 2),
                                   (3, 3, 32, 36, 192, 11, 11, 4, 4, 2, 2)])
def test_wgrad_pairs_32_channel_dy_blocks(shape):
    """Backward-filter on CTA pairs with 32-channel dy blocks (64-byte
    swizzle, MN-major): bn = 192 by default, bn = 64 forced."""
    check(run_case(shape, passes=("bwd_filter",), seed=17))
    with env(DNNP_WG_BW32_64=1):
        check(run_case(shape, passes=("bwd_filter",), seed=17))
    with env(DNNP_WG_NO_BW32=1):
        check(run_case(shape, passes=("bwd_filter",), seed=17))


def test_row_staged_filter_pack_variant():
    """The opt-in row-staged forward filter pack (DNNP_PACK_ROWS) across the
    plain, space-to-depth, folded and row-blocked forward geometries."""
    with env(DNNP_PACK_ROWS=1):
        for shape in [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1), (2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2),
                      (2, 3, 17, 19, 24, 5, 7, 1, 1, 2, 3), (2, 32, 13, 13, 256, 3, 3, 1, 1, 1, 1)]:
            check(run_case(shape, passes=("fwd",), seed=18))
