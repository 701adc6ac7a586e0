"""GPU parity: libdnnp.so (through the reference-shaped Python API and the
C ABI) against the reference's golden vectors and the C oracle.

Tolerances (north_star): fp32 <= 1e-4 and fp64 <= 1e-12 normalised error
max|a-b|/max|ref| (the test_acceptance.py:91-96 metric); argmax, pooling
backward, activation backward, transform and add_broadcast bit-exact."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

F32_TOL, F64_TOL = 1e-4, 1e-12
MATHS = [0, 1]  # default (tensor cores when eligible), SIMT fp32


def tol(dt):
    return F32_TOL if np.dtype(dt) == np.float32 else F64_TOL


@pytest.fixture(autouse=True)
def _reset_math():
    yield
    dp.set_math(0)


def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def view(geom, buf, base, device=None):
    g = [int(v) for v in geom]
    desc = dp.make_desc(*g[:4], layout="custom", strides=g[4:], elem_type=buf.dtype)
    if device is None:
        return dp.TensorView(desc, buf[base:])
    torch = torch_cuda()
    t = torch.from_numpy(buf).to(device)
    return dp.TensorView(desc, t[base:]), t


def to_host(t):
    return t.detach().cpu().numpy()


def _conv_case(g, i):
    p = f"c{i}_"
    return {k[len(p):]: g[k] for k in g.files if k.startswith(p)}


def _mode(cg):
    return "convolution" if int(cg[4]) == 0 else "cross_correlation"


def _cd(cg):
    return dp.ConvDesc(int(cg[0]), int(cg[1]), int(cg[2]), int(cg[3]), _mode(cg), bool(cg[5]))


@pytest.mark.parametrize("device", [None, "cuda"])
@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("i", range(16))
def test_conv_golden(golden_conv, i, math, device):
    dp.set_math(math)
    c = _conv_case(golden_conv, i)
    b = c["bases"]
    dt = c["x"].dtype
    fd = dp.make_filter_desc(*[int(v) for v in c["fg"]], elem_type=dt)
    keep = []

    def mk(geom, buf, base):
        if device is None:
            return view(geom, buf, base), None
        v, t = view(geom, buf, base, device)
        keep.append(t)
        return v, t

    def fview(buf):
        if device is None:
            return dp.FilterView(fd, buf), buf
        torch = torch_cuda()
        t = torch.from_numpy(buf).to(device)
        keep.append(t)
        return dp.FilterView(fd, t), t

    # forward: alpha/beta into a strided y (gaps untouched)
    xv, _ = mk(c["xg"], c["x"].copy(), b[0])
    y = c["y_in"].copy()
    yv, yt = mk(c["yg"], y, b[1])
    f = c["f"].copy()
    fv, _ = fview(f)
    dp.conv_forward(xv, fv, _cd(c["cg"]), "implicit", yv, alpha=float(c["scal"][0]),
                    beta=float(c["scal"][1]))
    yo = y if device is None else to_host(yt)
    assert orc.rel_err(yo, c["y_out"]) <= tol(dt)
    # backward data (accumulate where the golden case does)
    dyv, _ = mk(c["yg"], c["dy"].copy(), b[2])
    dx = c["dx_in"].copy()
    dxv, dxt = mk(c["xg"], dx, b[3])
    dp.conv_backward_data(dyv, fv, _cd(c["cg_acc"]), "direct", dxv)
    dxo = dx if device is None else to_host(dxt)
    assert orc.rel_err(dxo, c["dx_out"]) <= tol(dt)
    # backward filter
    df = c["df_in"].copy()
    dfv, dft = fview(df)
    dp.conv_backward_filter(dyv, xv, _cd(c["cg_acc"]), "explicit", dfv)
    dfo = df if device is None else to_host(dft)
    assert orc.rel_err(dfo, c["df_out"]) <= tol(dt)
    # bias
    db = dp.conv_backward_bias(dyv)
    dbo = db.numpy().reshape(-1)
    assert orc.rel_err(dbo, c["db"]) <= tol(dt)


def _nn(g, key):
    p = key + "_"
    return {k[len(p):]: g[k] for k in g.files if k.startswith(p)}


SENTINEL = 7.0


@pytest.mark.parametrize("device", [None, "cuda"])
def test_nnops_golden(golden_nnops, device):
    g = golden_nnops
    keys = sorted({k.split("_")[0] for k in g.files})
    torch = torch_cuda() if device else None

    def mk(geom, buf, base):
        if device is None:
            return view(geom, buf, base), buf
        v, t = view(geom, buf, base, device)
        return v, t

    def host(t):
        return t if device is None else to_host(t)

    for key in keys:
        c = _nn(g, key)
        kind, bs = key[0], c["bases"]
        dt = (c.get("x") if "x" in c else c.get("s", c.get("b"))).dtype
        if kind == "a":
            act = ["sigmoid", "relu", "tanh"][int(c["meta"][0])]
            xv, _ = mk(c["xg"], c["x"].copy(), bs[0])
            yv, yt = mk(c["yg"], np.full_like(c["y"], SENTINEL), bs[1])
            dp.activation_forward(act, xv, yv)
            e = orc.rel_err(host(yt), c["y"])
            assert e <= (1e-6 if dt == np.float32 else 1e-14), (key, e)
            if act == "relu":
                assert np.array_equal(host(yt), c["y"]), key
            yv2, _ = mk(c["yg"], c["y"].copy(), bs[1])
            dyv, _ = mk(c["dyg"], c["dy"].copy(), bs[2])
            dxv, dxt = mk(c["dxg"], np.full_like(c["dx"], SENTINEL), bs[3])
            dp.activation_backward(act, yv2, dyv, dxv)
            assert np.array_equal(host(dxt), c["dx"]), key
        elif kind == "s":
            mode = ["per_image", "per_spatial"][int(c["meta"][0])]
            xv, _ = mk(c["xg"], c["x"].copy(), bs[0])
            yv, yt = mk(c["yg"], np.full_like(c["y"], SENTINEL), bs[1])
            dp.softmax_forward(mode, xv, yv)
            assert orc.rel_err(host(yt), c["y"]) <= tol(dt), key
            yv2, _ = mk(c["yg"], c["y"].copy(), bs[1])
            dyv, _ = mk(c["dyg"], c["dy"].copy(), bs[2])
            dxv, dxt = mk(c["dxg"], np.full_like(c["dx"], SENTINEL), bs[3])
            dp.softmax_backward(mode, yv2, dyv, dxv)
            assert orc.rel_err(host(dxt), c["dx"]) <= tol(dt), key
        elif kind == "p":
            m = [int(v) for v in c["meta"]]
            pd = dp.PoolingDesc("max" if m[0] == 0 else "average", *m[1:])
            xv, _ = mk(c["xg"], c["x"].copy(), bs[0])
            yv, yt = mk(c["yg"], np.full_like(c["y"], SENTINEL), bs[1])
            shape = tuple(int(v) for v in c["yg"][:4])
            am = np.full(shape, -1, dtype=np.int64)
            if device is not None:
                am = torch.from_numpy(am).to(device)
            dp.pool_forward(pd, xv, yv, am if m[0] == 0 else None)
            amh = am if device is None else to_host(am)
            assert np.array_equal(amh.reshape(-1), c["argmax"]), key
            if m[0] == 0:
                assert np.array_equal(host(yt), c["y"]), key
            else:
                assert orc.rel_err(host(yt), c["y"]) <= tol(dt) / 100, key
            dyv, _ = mk(c["dyg"], c["dy"].copy(), bs[2])
            dxv, dxt = mk(c["dxg"], np.full_like(c["dx"], SENTINEL), bs[3])
            dp.pool_backward(pd, yv, dyv, xv, dxv, am if m[0] == 0 else None)
            assert np.array_equal(host(dxt), c["dx"]), key
        elif kind == "t":
            sv, _ = mk(c["sg"], c["s"].copy(), bs[0])
            dv, dt_ = mk(c["dg"], c["d_in"].copy(), bs[1])
            dp.transform(sv, dv, alpha=1.5, beta=-0.5)
            assert np.array_equal(host(dt_), c["d_out"]), key
        elif kind == "b":
            bv, _ = mk(c["bg"], c["b"].copy(), bs[0])
            ov, ot = mk(c["og"], c["o_in"].copy(), bs[1])
            dp.add_broadcast(bv, ov, alpha=2.0, beta=0.5)
            assert np.array_equal(host(ot), c["o_out"]), key


# ---- random problems vs the C oracle ----------------------------------------

LAYOUTS = ("nchw", "nhwc")

RANDOM_SHAPES = [
    # N C H W K R S u v ph pw
    (2, 3, 31, 29, 16, 11, 11, 4, 4, 2, 2),   # AlexNet conv1-like
    (2, 16, 15, 15, 24, 5, 5, 1, 1, 2, 2),    # conv2-like
    (3, 24, 9, 9, 40, 3, 3, 1, 1, 1, 1),      # conv3-5-like
    (2, 8, 12, 10, 8, 3, 3, 2, 2, 1, 1),
    (1, 64, 8, 8, 72, 3, 3, 1, 1, 1, 1),      # channel counts past one k-block
    (4, 32, 7, 7, 130, 1, 1, 1, 1, 0, 0),     # 1x1, ragged K
    (4, 3, 40, 40, 8, 5, 5, 1, 1, 2, 2),      # thin GEMMs (narrow SIMT tiles: fwd N=8, dgrad N=3)
    (4, 2, 80, 72, 12, 3, 3, 2, 2, 1, 1),     # thin + strided bwd-data phases
    (2, 12, 48, 48, 3, 3, 3, 1, 1, 1, 1),     # <= 4 output columns (tiny SIMT tile: fwd N=3)
]


def _rand_view(rng, n, c, h, w, dt, layout, device):
    desc = dp.make_desc(n, c, h, w, layout=layout, elem_type=dt)
    buf = rng.uniform(-0.5, 0.5, desc.max_offset() + 1).astype(dt)
    g = np.array([n, c, h, w, *desc.strides], dtype=np.int64)
    if device is None:
        return dp.TensorView(desc, buf), buf, g, None
    torch = torch_cuda()
    t = torch.from_numpy(buf.copy()).to(device)
    return dp.TensorView(desc, t), buf, g, t


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("si", range(len(RANDOM_SHAPES)))
def test_conv_random_vs_oracle(si, dt, math):
    dp.set_math(math)
    rng = np.random.default_rng(1000 + si)
    N, C, H, W, K, R, S, u, v, ph, pw = RANDOM_SHAPES[si]
    for mode in ("convolution", "cross_correlation"):
        lay = LAYOUTS[si % 2]
        cd = dp.ConvDesc(u, v, ph, pw, mode)
        cg = [u, v, ph, pw, 0 if mode == "convolution" else 1, 0]
        P, Q = dp.output_extent(H, R, u, ph), dp.output_extent(W, S, v, pw)
        xv, x, xg, _ = _rand_view(rng, N, C, H, W, dt, lay, "cuda")
        f = rng.uniform(-0.5, 0.5, K * C * R * S).astype(dt)
        import torch
        ft = torch.from_numpy(f.copy()).cuda()
        fv = dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt), ft)
        yv, _, yg, yt = _rand_view(rng, N, K, P, Q, dt, "nchw", "cuda")
        dp.conv_forward(xv, fv, cd, "implicit", yv)
        ref = np.zeros(N * K * P * Q, dtype=dt)
        orc.conv_forward(xg, x, [K, C, R, S], f, cg, yg, ref, threads=4)
        assert orc.rel_err(to_host(yt), ref) <= tol(dt), ("fwd", mode)
        dyv, dy, dyg, _ = _rand_view(rng, N, K, P, Q, dt, lay, "cuda")
        dxv, _, dxg, dxt = _rand_view(rng, N, C, H, W, dt, "nchw", "cuda")
        dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
        ref = np.zeros(N * C * H * W, dtype=dt)
        orc.conv_backward_data([K, C, R, S], f, dyg, dy, cg, dxg, ref)
        assert orc.rel_err(to_host(dxt), ref) <= tol(dt), ("dgrad", mode)
        dft = torch.zeros(K * C * R * S, dtype=ft.dtype, device="cuda")
        dfv = dp.FilterView(dp.make_filter_desc(K, C, R, S, elem_type=dt), dft)
        dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
        ref = np.zeros(K * C * R * S, dtype=dt)
        orc.conv_backward_filter(xg, x, dyg, dy, cg, [K, C, R, S], ref)
        assert orc.rel_err(to_host(dft), ref) <= tol(dt), ("wgrad", mode)


POOL_SHAPES = [
    # N C H W wh ww sh sw ph pw
    (2, 24, 17, 15, 3, 3, 2, 2, 0, 0),    # AlexNet pool-like, channels past the NHWC threshold
    (3, 16, 12, 13, 2, 3, 2, 1, 1, 1),    # padded, overlapping along w only
    (2, 5, 11, 9, 3, 2, 1, 2, 1, 0),      # few channels (plane kernels in both layouts)
    (1, 40, 9, 9, 4, 4, 3, 3, 2, 2),      # window > stride + 1, padding on both sides
    (2, 18, 10, 10, 3, 3, 2, 2, 1, 1),    # NHWC without 16-byte channel vectors in fp32
    (2, 32, 29, 29, 3, 3, 2, 2, 0, 0),    # NHWC 3x3/2: fast and generic forward threads in one block
]


@pytest.mark.parametrize("kind", ["max", "average"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("si", range(len(POOL_SHAPES)))
def test_pool_random_vs_oracle(si, layout, dt, kind):
    """Pooling forward/backward on random NCHW and NHWC views against the C
    oracle: argmax, max-pool outputs and both backward passes bit-exact."""
    import torch
    N, C, H, W, wh, ww, sh, sw, ph, pw = POOL_SHAPES[si]
    rng = np.random.default_rng(3000 + si)
    pd = dp.PoolingDesc(kind, wh, ww, sh, sw, ph, pw)
    pg = [0 if kind == "max" else 1, wh, ww, sh, sw, ph, pw]
    xv, x, xg, _ = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    _, _, P, Q = dp.pool_out_shape(pd, xv)
    yv, _, yg, yt = _rand_view(rng, N, C, P, Q, dt, layout, "cuda")
    am = torch.full((N, C, P, Q), -1, dtype=torch.int64, device="cuda") if kind == "max" else None
    dp.pool_forward(pd, xv, yv, am)
    yref = np.zeros(yt.numel(), dtype=dt)
    amref = np.full(N * C * P * Q, -1, dtype=np.int64)
    orc.pool_forward(pg, xg, x, yg, yref, amref if kind == "max" else None)
    ydev = to_host(yt)
    if kind == "max":
        assert np.array_equal(to_host(am).reshape(-1), amref)
        assert np.array_equal(ydev, yref)
    else:
        assert orc.rel_err(ydev, yref) <= tol(dt) / 100
    dyv, dy, dyg, _ = _rand_view(rng, N, C, P, Q, dt, layout, "cuda")
    dxv, _, dxg, dxt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    dp.pool_backward(pd, yv, dyv, xv, dxv, am)
    dxref = np.zeros(dxt.numel(), dtype=dt)
    orc.pool_backward(pg, dyg, dy, dxg, dxref, amref if kind == "max" else None)
    assert np.array_equal(to_host(dxt), dxref)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("pad", [0, 1])
def test_pool_max_ties_and_nan_vs_oracle(pad, layout, dt):
    """Max pooling with many ties and scattered NaNs (first max / first NaN
    in window scan order, nnops.py:157-200): argmax, y and dx bit-exact."""
    import torch
    N, C, H, W = 2, 32, 23, 21
    rng = np.random.default_rng(4000 + pad)
    pd = dp.PoolingDesc("max", 3, 3, 2, 2, pad, pad)
    pg = [0, 3, 3, 2, 2, pad, pad]
    xv, x, xg, xt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    x[:] = rng.integers(-2, 3, x.size).astype(dt)
    x[rng.random(x.size) < 0.02] = np.nan
    xt.copy_(torch.from_numpy(x))
    _, _, P, Q = dp.pool_out_shape(pd, xv)
    yv, _, yg, yt = _rand_view(rng, N, C, P, Q, dt, layout, "cuda")
    am = torch.full((N, C, P, Q), -1, dtype=torch.int64, device="cuda")
    dp.pool_forward(pd, xv, yv, am)
    yref = np.zeros(yt.numel(), dtype=dt)
    amref = np.full(N * C * P * Q, -1, dtype=np.int64)
    orc.pool_forward(pg, xg, x, yg, yref, amref)
    assert np.array_equal(to_host(am).reshape(-1), amref)
    assert np.array_equal(to_host(yt), yref, equal_nan=True)
    dyv, dy, dyg, _ = _rand_view(rng, N, C, P, Q, dt, layout, "cuda")
    dxv, _, dxg, dxt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    dp.pool_backward(pd, yv, dyv, xv, dxv, am)
    dxref = np.zeros(dxt.numel(), dtype=dt)
    orc.pool_backward(pg, dyg, dy, dxg, dxref, amref)
    assert np.array_equal(to_host(dxt), dxref)


SOFTMAX_SHAPES = [(5, 1000, 1, 1), (3, 10, 3, 3), (4, 7, 6, 6), (2, 3, 13, 13), (2, 5, 16, 16)]


@pytest.mark.parametrize("mode", ["per_image", "per_spatial"])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("si", range(len(SOFTMAX_SHAPES)))
def test_softmax_random_vs_oracle(si, layout, dt, mode):
    """Softmax forward / backward against the C oracle across the group
    sizes of every per-image kernel variant (warp-per-image 4..32 values per
    lane, and the two-phase form past 1024 elements)."""
    N, C, H, W = SOFTMAX_SHAPES[si]
    rng = np.random.default_rng(5000 + si)
    mcode = 0 if mode == "per_image" else 1
    import torch
    xv, x, xg, xt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    x *= 8
    xt.copy_(torch.from_numpy(x))
    yv, _, yg, yt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    dp.softmax_forward(mode, xv, yv)
    yref = np.zeros(yt.numel(), dtype=dt)
    orc.softmax_forward(mcode, xg, x, yg, yref)
    assert orc.rel_err(to_host(yt), yref) <= tol(dt)
    dyv, dy, dyg, _ = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    dxv, _, dxg, dxt = _rand_view(rng, N, C, H, W, dt, layout, "cuda")
    dp.softmax_backward(mode, yv, dyv, dxv)
    dxref = np.zeros(dxt.numel(), dtype=dt)
    orc.softmax_backward(mcode, yg, to_host(yt), dyg, dy, dxg, dxref)
    assert orc.rel_err(to_host(dxt), dxref) <= tol(dt)


def test_accumulate_and_beta_semantics():
    torch = torch_cuda()
    rng = np.random.default_rng(3)
    xv, x, xg, _ = _rand_view(rng, 2, 4, 6, 6, np.float32, "nchw", "cuda")
    f = torch.from_numpy(rng.uniform(-1, 1, 5 * 4 * 9).astype(np.float32)).cuda()
    fv = dp.FilterView(dp.make_filter_desc(5, 4, 3, 3), f)
    y = torch.full((2 * 5 * 4 * 4,), float("nan"), device="cuda")
    yv = dp.TensorView(dp.make_desc(2, 5, 4, 4), y)
    dp.conv_forward(xv, fv, dp.ConvDesc(), "implicit", yv, alpha=1.0, beta=0.0)
    assert torch.isfinite(y).all()  # beta == 0 never reads y
    y0 = y.clone()
    dp.conv_forward(xv, fv, dp.ConvDesc(accumulate=True), "implicit", yv, alpha=1.0, beta=0.0)
    assert torch.allclose(y, 2 * y0, rtol=1e-5, atol=1e-6)  # accumulate forces beta = 1


def test_capi_conformance_full(tmp_path):
    exe = tmp_path / "conformance"
    lib = os.path.join(ROOT, "paper_1410_0759_b200")
    subprocess.run(["gcc", "-O2", "-I" + os.path.join(ROOT, "include"), "-o", str(exe),
                    os.path.join(ROOT, "tests", "capi", "conformance.c"), "-L" + lib, "-ldnnp",
                    "-Wl,-rpath," + lib, "-lpthread", "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:]


def test_native_kernels_launched():
    before = dp.kernel_launch_count()
    x = dp.TensorView.from_array(np.ones((1, 1, 4, 4), dtype=np.float32), device="cuda")
    y = dp.empty_view(x.desc, device="cuda")
    dp.activation_forward("relu", x, y)
    assert dp.kernel_launch_count() > before


REF_DIR = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_DIR, "test_capi_ref")),
                    reason="reference C test not built (oracle/build_ref.sh)")
def test_reference_capi_program_unchanged():
    """The reference's own pkg/capi/tests/test_capi.c, compiled unchanged
    against include/dnnp.h and linked to libdnnp.so: all 58 checks pass."""
    r = subprocess.run([os.path.join(REF_DIR, "test_capi_ref")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "58 passed, 0 failed" in r.stdout


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_DIR, "conv_example_ref")),
                    reason="reference example not built (oracle/build_ref.sh)")
def test_reference_example_golden_bytes(tmp_path):
    """pkg/capi/examples/conv_example.c unchanged: its raw f32 output equals
    the reference native golden bytes (Makefile:36-41 `cmp`)."""
    out = tmp_path / "example.bin"
    r = subprocess.run([os.path.join(REF_DIR, "conv_example_ref"), str(out)], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    golden = np.array([7, -36, 10, -11, -5, 5, 25, -9], dtype=np.float32).tobytes()
    assert out.read_bytes() == golden
