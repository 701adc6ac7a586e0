"""SURVEY 8(f) rows checked against the C oracle (not only against another
path of this library):

* rank 3, fused epilogues: forward + bias + activation is compared with the
  oracle's conv_forward -> add_broadcast -> activation_forward chain
  (reference conv.py:565-582, tensor.py:260-271, nnops.py:54-72);
  backward-data + activation-backward with conv_backward_data ->
  activation_backward (conv.py:720-734, nnops.py:75-88);
* rank 4, the explicit-lowering engine (conv.py:494-535) on every pass;
* rank 1, the CLI's --verify kernel (the device loop nest) against the oracle.

Bars: fp32 <= 1e-4, fp64 <= 1e-12 normalised (north_star)."""
import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "f64": 1e-12}
ACT = {"sigmoid": 0, "relu": 1, "tanh": 2}

#        N   C   H   W   K  R  S  u  v ph pw
SHAPES = [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1),
          (2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2),   # space-to-depth
          (2, 16, 15, 15, 24, 5, 5, 2, 2, 2, 2),    # super-pixel bwd-data
          (3, 64, 15, 15, 96, 5, 5, 1, 1, 2, 2),    # blocked bwd-data columns
          (2, 32, 13, 13, 256, 3, 3, 1, 1, 1, 1)]   # CTA pairs


def _geom(n, c, h, w):
    return [n, c, h, w, c * h * w, h * w, w, 1]


def _np(dt):
    return np.float32 if dt == "f32" else np.float64


def _cuda(a):
    import torch
    return torch.from_numpy(a.copy()).cuda()


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("act", [None, "relu", "sigmoid", "tanh"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_fused_forward_vs_oracle(si, act, dt):
    import torch
    N, C, H, W, K, R, S, u, v, ph, pw = SHAPES[si]
    rng = np.random.default_rng(700 + si)
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    mk = lambda cnt: rng.uniform(-0.5, 0.5, cnt).astype(_np(dt))  # noqa: E731
    x, f, b, y0 = mk(N * C * H * W), mk(K * C * R * S), mk(K), mk(N * K * P * Q)
    alpha, beta = 0.75, -0.5
    yv = dp.TensorView(dp.make_desc(N, K, P, Q, elem_type=dt), _cuda(y0))
    dp.conv_bias_activation_forward(
        dp.TensorView(dp.make_desc(N, C, H, W, elem_type=dt), _cuda(x)),
        dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt), _cuda(f)),
        dp.ConvDesc(u, v, ph, pw), "implicit", yv,
        bias=dp.TensorView(dp.make_desc(1, K, 1, 1, elem_type=dt), _cuda(b)),
        activation=act, alpha=alpha, beta=beta)
    torch.cuda.synchronize()
    ref = y0.copy()
    yg = _geom(N, K, P, Q)
    orc.conv_forward(_geom(N, C, H, W), x, [K, C, R, S], f, [u, v, ph, pw, 0, 0], yg, ref,
                     alpha=alpha, beta=beta)
    orc.add_broadcast(_geom(1, K, 1, 1), b, yg, ref, 1.0, 1.0)
    if act is not None:
        orc.activation_forward(ACT[act], yg, ref.copy(), yg, ref)
    assert orc.rel_err(yv.buf.cpu().numpy(), ref) <= TOL[dt]


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("acc", [False, True])
@pytest.mark.parametrize("act", ["relu", "sigmoid", "tanh"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_fused_backward_data_vs_oracle(si, act, acc, dt):
    import torch
    N, C, H, W, K, R, S, u, v, ph, pw = SHAPES[si]
    rng = np.random.default_rng(800 + si)
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    mk = lambda cnt: rng.uniform(-0.5, 0.5, cnt).astype(_np(dt))  # noqa: E731
    dy, f, dx0 = mk(N * K * P * Q), mk(K * C * R * S), mk(N * C * H * W)
    g = mk(N * C * H * W)  # the activation output that fed the convolution
    if act == "relu":
        g = np.maximum(g, 0).astype(_np(dt))
    elif act == "sigmoid":
        g = (g + 0.5).astype(_np(dt))
    dxv = dp.TensorView(dp.make_desc(N, C, H, W, elem_type=dt), _cuda(dx0))
    dp.conv_backward_data_activation(
        dp.TensorView(dp.make_desc(N, K, P, Q, elem_type=dt), _cuda(dy)),
        dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt), _cuda(f)),
        dp.ConvDesc(u, v, ph, pw, "convolution", acc), "implicit", dxv, act,
        dp.TensorView(dp.make_desc(N, C, H, W, elem_type=dt), _cuda(g)))
    torch.cuda.synchronize()
    xg = _geom(N, C, H, W)
    tmp = np.zeros(N * C * H * W, _np(dt))
    orc.conv_backward_data([K, C, R, S], f, _geom(N, K, P, Q), dy, [u, v, ph, pw, 0, 0], xg, tmp)
    gated = np.zeros_like(tmp)
    orc.activation_backward(ACT[act], xg, g, xg, tmp, xg, gated)
    ref = gated + dx0 if acc else gated
    assert orc.rel_err(dxv.buf.cpu().numpy(), ref) <= TOL[dt]


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("r,stride,pad", [(1, 1, 0), (3, 1, 1), (5, 2, 2), (4, 3, 0)])
def test_explicit_engine_vs_oracle(r, stride, pad, dt):
    import torch
    n, c, h, k = 4, 8, 24, 16
    rng = np.random.default_rng(900 + r)
    p = dp.output_extent(h, r, stride, pad)
    mk = lambda cnt: rng.uniform(-0.5, 0.5, cnt).astype(_np(dt))  # noqa: E731
    x, f, dy = mk(n * c * h * h), mk(k * c * r * r), mk(n * k * p * p)
    cd = dp.ConvDesc(stride, stride, pad, pad)
    xv = dp.TensorView(dp.make_desc(n, c, h, h, elem_type=dt), _cuda(x))
    fv = dp.FilterView(dp.make_filter_desc(k, c, r, r, elem_type=dt), _cuda(f))
    dyv = dp.TensorView(dp.make_desc(n, k, p, p, elem_type=dt), _cuda(dy))
    yv = dp.empty_view(dp.make_desc(n, k, p, p, elem_type=dt), device="cuda")
    dxv = dp.empty_view(dp.make_desc(n, c, h, h, elem_type=dt), device="cuda")
    dfv = dp.FilterView(dp.make_filter_desc(k, c, r, r, elem_type=dt),
                        torch.empty(k * c * r * r, device="cuda", dtype=xv.buf.dtype))
    dp.conv_forward(xv, fv, cd, "explicit", yv)
    dp.conv_backward_data(dyv, fv, cd, "explicit", dxv)
    dp.conv_backward_filter(dyv, xv, cd, "explicit", dfv)
    torch.cuda.synchronize()
    xg, yg, fg, cg = _geom(n, c, h, h), _geom(n, k, p, p), [k, c, r, r], [stride, stride, pad, pad, 0, 0]
    ry, rdx, rdf = (np.zeros(n * k * p * p, _np(dt)), np.zeros(n * c * h * h, _np(dt)),
                    np.zeros(k * c * r * r, _np(dt)))
    orc.conv_forward(xg, x, fg, f, cg, yg, ry)
    orc.conv_backward_data(fg, f, yg, dy, cg, xg, rdx)
    orc.conv_backward_filter(xg, x, yg, dy, cg, fg, rdf)
    assert orc.rel_err(yv.buf.cpu().numpy(), ry) <= TOL[dt]
    assert orc.rel_err(dxv.buf.cpu().numpy(), rdx) <= TOL[dt]
    assert orc.rel_err(dfv.buf.cpu().numpy(), rdf) <= TOL[dt]


def test_explicit_max_lowered_bytes_every_pass():
    """AllocTooLarge from max_lowered_bytes on all three passes (reference
    conv.py:507-511, 615-618, 701; test_lowering.py:87-90)."""
    import torch
    n, c, h, k, r = 2, 4, 10, 3, 3
    p = h - r + 1
    xv = dp.TensorView(dp.make_desc(n, c, h, h), torch.zeros(n * c * h * h, device="cuda"))
    fv = dp.FilterView(dp.make_filter_desc(k, c, r, r), torch.zeros(k * c * r * r, device="cuda"))
    dyv = dp.TensorView(dp.make_desc(n, k, p, p), torch.zeros(n * k * p * p, device="cuda"))
    need = c * r * r * n * p * p * 4
    cd = dp.ConvDesc()
    with pytest.raises(dp.AllocTooLarge):
        dp.conv_forward(xv, fv, cd, "explicit", dp.empty_view(dyv.desc, device="cuda"),
                        max_lowered_bytes=need - 1)
    with pytest.raises(dp.AllocTooLarge):
        dp.conv_backward_data(dyv, fv, cd, "explicit", dp.empty_view(xv.desc, device="cuda"),
                              max_lowered_bytes=need - 1)
    with pytest.raises(dp.AllocTooLarge):
        dp.conv_backward_filter(dyv, xv, cd, "explicit", fv, max_lowered_bytes=need - 1)
    # at exactly the limit all three run
    dp.conv_forward(xv, fv, cd, "explicit", dp.empty_view(dyv.desc, device="cuda"),
                    max_lowered_bytes=need)
    dp.conv_backward_data(dyv, fv, cd, "explicit", dp.empty_view(xv.desc, device="cuda"),
                          max_lowered_bytes=need)
    dp.conv_backward_filter(dyv, xv, cd, "explicit", fv, max_lowered_bytes=need)


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_cli_verify_reference_vs_oracle(si, dt):
    """The CLI's --verify reference (device fp64 loop nests) against the
    oracle, every pass; NHWC operands and cross-correlation on odd shapes."""
    import ctypes
    import torch
    from paper_1410_0759_b200 import _lib
    N, C, H, W, K, R, S, u, v, ph, pw = SHAPES[si]
    mode = "convolution" if si % 2 == 0 else "cross_correlation"
    layout = "nhwc" if si % 2 else "nchw"
    rng = np.random.default_rng(950 + si)
    P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
    xd = dp.make_desc(N, C, H, W, layout=layout, elem_type=dt)
    yd = dp.make_desc(N, K, P, Q, layout=layout, elem_type=dt)
    fd = dp.make_filter_desc(K, C, R, S, elem_type=dt)
    cd = dp.ConvDesc(u, v, ph, pw, mode)
    x = rng.uniform(-0.5, 0.5, xd.max_offset() + 1).astype(_np(dt))
    dy = rng.uniform(-0.5, 0.5, yd.max_offset() + 1).astype(_np(dt))
    f = rng.uniform(-0.5, 0.5, K * C * R * S).astype(_np(dt))
    xt, dyt, ft = _cuda(x), _cuda(dy), _cuda(f)
    cg = [u, v, ph, pw, 0 if mode == "convolution" else 1, 0]
    xg, yg, fg = [N, C, H, W, *xd.strides], [N, K, P, Q, *yd.strides], [K, C, R, S]
    outs = {}
    for code, (a, b, cnt) in enumerate(((xt, ft, N * K * P * Q), (dyt, ft, N * C * H * W),
                                        (dyt, xt, K * C * R * S))):
        out = torch.empty(cnt, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().dnnp_convolution_verify_reference(
            _lib.handle(), code, xd.c_desc(), fd.c_desc(), cd.c_desc(), yd.c_desc(),
            ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
            ctypes.c_void_p(out.data_ptr())))
        outs[code] = out.cpu().numpy()
    dense_y, dense_x = _geom(N, K, P, Q), _geom(N, C, H, W)
    ry = np.zeros(N * K * P * Q, np.float64)
    orc.conv_forward(xg, x.astype(np.float64), fg, f.astype(np.float64), cg, dense_y, ry)
    rdx = np.zeros(N * C * H * W, np.float64)
    orc.conv_backward_data(fg, f.astype(np.float64), yg, dy.astype(np.float64), cg, dense_x, rdx)
    rdf = np.zeros(K * C * R * S, np.float64)
    orc.conv_backward_filter(xg, x.astype(np.float64), yg, dy.astype(np.float64), cg, fg, rdf)
    for code, ref in enumerate((ry, rdx, rdf)):
        assert orc.rel_err(outs[code], ref) <= 1e-12, code
