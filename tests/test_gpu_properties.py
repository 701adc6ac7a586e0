"""The reference's property suite, re-run against the GPU library through its
drop-in Python API (the same call shapes the reference tests make).

Each test restates one reference property (cited per test) with its own
generator and seed; the inputs are host numpy arrays, so every call also goes
through the C ABI's host-buffer staging.  Where the GPU arithmetic cannot
give the reference's exact CPU result the bar is stated and justified:

* fp32 engine agreement: the reference asks 1e-5 between its CPU engines
  (test_acceptance.py:81-101); here every engine runs the BF16x3 tensor-core
  kernels (EXPLICIT through the lowered matrix, a different reduction order),
  each ~4e-6 from exact, so engines are held to the north_star 1e-4 against
  the C oracle and 2e-5 pairwise.  fp64 keeps the reference's 1e-12.
* layout invariance and stride subsampling are exact in fp64 (the DFMA
  kernels reduce over (c, r, s) in one fixed order whatever the strides), as
  in the reference (test_acceptance.py:339-458, test_conv_forward.py:109-120).
"""
import numpy as np
import pytest

import oracle as orc
import paper_1410_0759_b200 as dp

pytestmark = pytest.mark.gpu

ENGINES = ("direct", "explicit", "implicit")


def _et(dt):
    return "f32" if np.dtype(dt) == np.float32 else "f64"


def fwd(xa, fa, conv, engine="implicit", layout="nchw"):
    x = dp.TensorView.from_array(xa, layout=layout)
    f = dp.FilterView.from_array(fa)
    shape = dp.conv_out_shape(x.desc, f.desc, conv)
    y = dp.empty_view(dp.make_desc(*shape, layout=layout, elem_type=_et(xa.dtype)))
    dp.conv_forward(x, f, conv, engine, y)
    return y.numpy()


def bwd_data(dya, fa, conv, engine, xshape, layout="nchw"):
    dy = dp.TensorView.from_array(dya, layout=layout)
    f = dp.FilterView.from_array(fa)
    dx = dp.empty_view(dp.make_desc(*xshape, layout=layout, elem_type=_et(dya.dtype)))
    dp.conv_backward_data(dy, f, conv, engine, dx)
    return dx.numpy()


def bwd_filter(dya, xa, conv, engine, fshape, layout="nchw"):
    dy = dp.TensorView.from_array(dya, layout=layout)
    x = dp.TensorView.from_array(xa, layout=layout)
    df = dp.FilterView.from_array(np.zeros(fshape, dtype=xa.dtype))
    dp.conv_backward_filter(dy, x, conv, engine, df)
    return np.asarray(df.array).copy()


def oracle_fwd(xa, fa, conv):
    n, c, h, w = xa.shape
    k, _, r, s = fa.shape
    p, q = dp.output_extent(h, r, conv.u, conv.pad_h), dp.output_extent(w, s, conv.v, conv.pad_w)
    y = np.zeros(n * k * p * q, dtype=xa.dtype)
    mode = 0 if conv.mode == dp.ConvMode.CONVOLUTION else 1
    orc.conv_forward([n, c, h, w, c * h * w, h * w, w, 1], np.ascontiguousarray(xa).ravel(),
                     [k, c, r, s], np.ascontiguousarray(fa).ravel(),
                     [conv.u, conv.v, conv.pad_h, conv.pad_w, mode, 0],
                     [n, k, p, q, k * p * q, p * q, q, 1], y)
    return y.reshape(n, k, p, q)


def random_conv(rng, dtype, hi=7):
    """Instance generator with the reference's ranges (test_acceptance.py:58-69):
    extents 1..6, filters 1..4, strides 1..3, padding 0..2, either mode."""
    while True:
        n, c, h, w, k = (int(v) for v in rng.integers(1, hi, 5))
        r, s = (int(v) for v in rng.integers(1, 5, 2))
        u, v = (int(a) for a in rng.integers(1, 4, 2))
        ph, pw = (int(a) for a in rng.integers(0, 3, 2))
        if h - r + 1 + 2 * ph >= 1 and w - s + 1 + 2 * pw >= 1:
            break
    mode = "convolution" if rng.integers(2) == 0 else "cross_correlation"
    xa = rng.standard_normal((n, c, h, w)).astype(dtype)
    fa = rng.standard_normal((k, c, r, s)).astype(dtype)
    return xa, fa, dp.ConvDesc(u, v, ph, pw, mode)


def test_engine_equivalence_200():
    """test_acceptance.py:81-101: 200 random instances, alternating f32 / f64,
    every engine against the oracle and pairwise."""
    rng = np.random.default_rng(1001)
    for trial in range(200):
        dtype = np.float32 if trial % 2 == 0 else np.float64
        xa, fa, conv = random_conv(rng, dtype)
        ref = oracle_fwd(xa, fa, conv)
        outs = [fwd(xa, fa, conv, e) for e in ENGINES]
        scale = max(float(np.abs(ref).max()), 1e-30)
        bar_ref, bar_pair = (1e-4, 2e-5) if dtype == np.float32 else (1e-12, 1e-12)
        for e, o in zip(ENGINES, outs):
            assert np.abs(o - ref).max() / scale <= bar_ref, (trial, e)
        for i in range(3):
            for j in range(i + 1, 3):
                assert np.abs(outs[i] - outs[j]).max() / scale <= bar_pair, (trial, i, j)


def fd_gradient(func, arr, eps=1e-5):
    """Central differences of a scalar function of arr (modified in place)."""
    g = np.zeros_like(arr)
    flat, gf = arr.reshape(-1), g.reshape(-1)
    for i in range(flat.size):
        old = flat[i]
        flat[i] = old + eps
        up = func()
        flat[i] = old - eps
        dn = func()
        flat[i] = old
        gf[i] = (up - dn) / (2 * eps)
    return g


def assert_fd(got, ref, what):
    """The reference's closeness rule (tests/oracles.py:149-157): per element
    |a - e| <= max(1e-4 * max(|a|, |e|), 1e-7)."""
    got = np.asarray(got, dtype=np.float64)
    tol = np.maximum(1e-4 * np.maximum(np.abs(got), np.abs(ref)), 1e-7)
    bad = np.abs(got - ref) > tol
    assert not bad.any(), (what, float(np.abs(got - ref).max()))


def test_gradient_suite_conv():
    """test_acceptance.py:163-216: backward data / filter against central
    differences of <conv(x, f), dy>, 50 instances rotating the engines."""
    rng = np.random.default_rng(2002)
    for i in range(50):
        while True:
            n, c, h, w = (int(v) for v in rng.integers(1, 4, 4))
            k, r, s = (int(v) for v in rng.integers(1, 4, 3))
            u, v = (int(a) for a in rng.integers(1, 3, 2))
            ph, pw = (int(a) for a in rng.integers(0, 2, 2))
            if h - r + 1 + 2 * ph >= 1 and w - s + 1 + 2 * pw >= 1:
                break
        conv = dp.ConvDesc(u, v, ph, pw, "convolution" if rng.integers(2) == 0
                           else "cross_correlation")
        xa = rng.standard_normal((n, c, h, w))
        fa = rng.standard_normal((k, c, r, s))
        dya = rng.standard_normal(fwd(xa, fa, conv).shape)
        engine = ENGINES[i % 3]
        scalar = lambda: float((fwd(xa, fa, conv, "direct") * dya).sum())  # noqa: E731
        assert_fd(bwd_data(dya, fa, conv, engine, xa.shape), fd_gradient(scalar, xa),
                  f"bwd data {i}")
        assert_fd(bwd_filter(dya, xa, conv, engine, fa.shape), fd_gradient(scalar, fa),
                  f"bwd filter {i}")


def test_gradient_suite_bias():
    """test_acceptance.py:219-235: conv_backward_bias vs differences of
    <add_broadcast(b, y), dy>."""
    rng = np.random.default_rng(2003)
    for _ in range(50):
        n, k, p, q = (int(v) for v in rng.integers(1, 4, 4))
        dya = rng.standard_normal((n, k, p, q))
        db = np.asarray(dp.conv_backward_bias(dp.TensorView.from_array(dya)).array)[0, :, 0, 0]
        ba = np.zeros((1, k, 1, 1))
        ya = rng.standard_normal((n, k, p, q))

        def scalar():
            out = dp.TensorView.from_array(ya.copy())
            dp.add_broadcast(dp.TensorView.from_array(ba), out)
            return float((out.numpy() * dya).sum())

        assert_fd(db.reshape(1, k, 1, 1), fd_gradient(scalar, ba), "bias")


def test_gradient_suite_activations():
    """test_acceptance.py:238-261 (relu inputs kept off the kink)."""
    rng = np.random.default_rng(2004)
    kinds = ["sigmoid", "relu", "tanh"]
    for i in range(50):
        kind = kinds[i % 3]
        shape = tuple(int(v) for v in rng.integers(1, 4, 4))
        xa = rng.standard_normal(shape)
        if kind == "relu":
            xa[np.abs(xa) < 0.05] += 0.2
        dya = rng.standard_normal(shape)

        def run(arr=xa):
            y = dp.empty_view(dp.make_desc(*shape, elem_type="f64"))
            dp.activation_forward(kind, dp.TensorView.from_array(arr), y)
            return y

        y = run()
        dx = dp.empty_view(dp.make_desc(*shape, elem_type="f64"))
        dp.activation_backward(kind, y, dp.TensorView.from_array(dya), dx)
        assert_fd(dx.numpy(), fd_gradient(lambda: float((run().numpy() * dya).sum()), xa), kind)


def test_gradient_suite_softmax():
    """test_acceptance.py:264-281, both modes."""
    rng = np.random.default_rng(2005)
    for i in range(50):
        mode = "per_image" if i % 2 == 0 else "per_spatial"
        shape = tuple(int(v) for v in rng.integers(1, 4, 4))
        xa = rng.standard_normal(shape)
        dya = rng.standard_normal(shape)

        def run(arr=xa):
            y = dp.empty_view(dp.make_desc(*shape, elem_type="f64"))
            dp.softmax_forward(mode, dp.TensorView.from_array(arr), y)
            return y

        dx = dp.empty_view(dp.make_desc(*shape, elem_type="f64"))
        dp.softmax_backward(mode, run(), dp.TensorView.from_array(dya), dx)
        assert_fd(dx.numpy(), fd_gradient(lambda: float((run().numpy() * dya).sum()), xa), mode)


def test_gradient_suite_pooling():
    """test_acceptance.py:284-318: max pooling on distinct values (argsort
    permutation, no ties) and average pooling."""
    rng = np.random.default_rng(2006)
    for i in range(50):
        kind = "max" if i % 2 == 0 else "average"
        n, c = (int(v) for v in rng.integers(1, 3, 2))
        h, w = (int(v) for v in rng.integers(2, 5, 2))
        wh, ww = int(rng.integers(1, h + 1)), int(rng.integers(1, w + 1))
        sh, sw = (int(a) for a in rng.integers(1, 3, 2))
        pd = dp.PoolingDesc(kind, wh, ww, sh, sw, 0, 0)
        if kind == "max":
            xa = np.argsort(rng.standard_normal(n * c * h * w)).astype(np.float64)
            xa = xa.reshape(n, c, h, w)
        else:
            xa = rng.standard_normal((n, c, h, w))
        x = dp.TensorView.from_array(xa)
        oshape = dp.pool_out_shape(pd, x)
        dya = rng.standard_normal(oshape)

        def run(arr=xa):
            y = dp.empty_view(dp.make_desc(*oshape, elem_type="f64"))
            am = np.empty(oshape, dtype=np.int64)
            dp.pool_forward(pd, dp.TensorView.from_array(arr), y, am)
            return y, am

        y, am = run()
        dx = dp.empty_view(dp.make_desc(n, c, h, w, elem_type="f64"))
        dp.pool_backward(pd, y, dp.TensorView.from_array(dya), x, dx, am)
        assert_fd(dx.numpy(), fd_gradient(lambda: float((run()[0].numpy() * dya).sum()), xa),
                  kind)


def test_adjoint_identity_small():
    """test_conv_backward.py:152-165: <conv(x), dy> = <x, bwd_data(dy)> =
    <f, bwd_filter(dy, x)> to 1e-10 for every engine (fp64)."""
    rng = np.random.default_rng(5150)
    for _ in range(8):
        xa, fa, conv = random_conv(rng, np.float64)
        y = fwd(xa, fa, conv)
        dya = rng.standard_normal(y.shape)
        lhs = float((y * dya).sum())
        for e in ENGINES:
            m_data = float((xa * bwd_data(dya, fa, conv, e, xa.shape)).sum())
            m_filt = float((fa * bwd_filter(dya, xa, conv, e, fa.shape)).sum())
            scale = max(abs(lhs), 1.0)
            assert abs(lhs - m_data) <= 1e-10 * scale, e
            assert abs(lhs - m_filt) <= 1e-10 * scale, e


@pytest.mark.parametrize("engine", ENGINES)
def test_stride_subsamples_unit_output(engine):
    """test_conv_forward.py:109-114, exact (fp64)."""
    rng = np.random.default_rng(109)
    xa = rng.standard_normal((2, 3, 7, 9))
    fa = rng.standard_normal((2, 3, 3, 3))
    dense = fwd(xa, fa, dp.ConvDesc(1, 1, 1, 1), engine)
    strided = fwd(xa, fa, dp.ConvDesc(2, 2, 1, 1), engine)
    assert np.array_equal(strided, dense[:, :, ::2, ::2])


@pytest.mark.parametrize("engine", ENGINES)
def test_layout_invariance_exact_conv(engine):
    """test_conv_forward.py:116-120 and test_acceptance.py:339-386: fp64
    forward / backward-data / backward-filter identical on NCHW and NHWC."""
    rng = np.random.default_rng(4001)
    for _ in range(4):
        xa, fa, conv = random_conv(rng, np.float64)
        dya = rng.standard_normal(fwd(xa, fa, conv).shape)
        assert np.array_equal(fwd(xa, fa, conv, engine, "nchw"), fwd(xa, fa, conv, engine, "nhwc"))
        assert np.array_equal(bwd_data(dya, fa, conv, engine, xa.shape, "nchw"),
                              bwd_data(dya, fa, conv, engine, xa.shape, "nhwc"))
        assert np.array_equal(bwd_filter(dya, xa, conv, engine, fa.shape, "nchw"),
                              bwd_filter(dya, xa, conv, engine, fa.shape, "nhwc"))


def test_layout_invariance_full_op_set():
    """test_acceptance.py:387-458: bias, transform, broadcast add,
    activations, softmax and pooling give identical fp64 results on NCHW and
    NHWC views."""
    rng = np.random.default_rng(4002)
    xa = rng.standard_normal((2, 3, 6, 7))
    dy_full = rng.standard_normal(xa.shape)

    def both(apply):
        a, b = apply("nchw"), apply("nhwc")
        assert np.array_equal(a, b)

    dya = rng.standard_normal((2, 4, 3, 7))
    both(lambda lay: np.asarray(dp.conv_backward_bias(
        dp.TensorView.from_array(dya, layout=lay)).array).copy())

    def via_transform(lay):
        dst = dp.empty_view(dp.make_desc(*xa.shape, elem_type="f64"))
        dp.transform(dp.TensorView.from_array(xa, layout=lay), dst, alpha=1.5, beta=0.0)
        return dst.numpy()

    both(via_transform)
    ba = rng.standard_normal((1, 3, 1, 1))

    def via_bias(lay):
        out = dp.TensorView.from_array(xa, layout=lay)
        dp.add_broadcast(dp.TensorView.from_array(ba), out, alpha=2.0, beta=0.5)
        return out.numpy()

    both(via_bias)
    for kind in ("sigmoid", "relu", "tanh"):
        def act(lay, kind=kind):
            y = dp.empty_view(dp.make_desc(*xa.shape, layout=lay, elem_type="f64"))
            dp.activation_forward(kind, dp.TensorView.from_array(xa, layout=lay), y)
            dx = dp.empty_view(dp.make_desc(*xa.shape, layout=lay, elem_type="f64"))
            dp.activation_backward(kind, y, dp.TensorView.from_array(dy_full, layout=lay), dx)
            return np.concatenate([y.numpy().ravel(), dx.numpy().ravel()])
        both(act)
    for mode in ("per_image", "per_spatial"):
        def smax(lay, mode=mode):
            y = dp.empty_view(dp.make_desc(*xa.shape, layout=lay, elem_type="f64"))
            dp.softmax_forward(mode, dp.TensorView.from_array(xa, layout=lay), y)
            dx = dp.empty_view(dp.make_desc(*xa.shape, layout=lay, elem_type="f64"))
            dp.softmax_backward(mode, y, dp.TensorView.from_array(dy_full, layout=lay), dx)
            return np.concatenate([y.numpy().ravel(), dx.numpy().ravel()])
        both(smax)
    for kind in ("max", "average"):
        pd = dp.PoolingDesc(kind, 2, 3, 2, 1, 1, 1)
        pshape = dp.pool_out_shape(pd, dp.TensorView.from_array(xa))
        pdy = rng.standard_normal(pshape)

        def pool(lay, pd=pd, pshape=pshape, pdy=pdy):
            x = dp.TensorView.from_array(xa, layout=lay)
            y = dp.empty_view(dp.make_desc(*pshape, layout=lay, elem_type="f64"))
            am = np.empty(pshape, dtype=np.int64)
            dp.pool_forward(pd, x, y, am)
            dx = dp.empty_view(dp.make_desc(*xa.shape, layout=lay, elem_type="f64"))
            dp.pool_backward(pd, y, dp.TensorView.from_array(pdy, layout=lay), x, dx, am)
            parts = [y.numpy().ravel(), dx.numpy().ravel()]
            if pd.kind == dp.PoolKind.MAX:  # argmax is only written by max pooling
                parts.append(am.ravel().astype(np.float64))
            return np.concatenate(parts)
        both(pool)


def test_zero_auxiliary_memory_fp64():
    """test_acceptance.py:309-337: the implicit engine's scratch stays bounded
    by the output size and does not move while the filter area r*s grows
    25x (fp64: the DFMA kernels gather straight from the caller's tensor)."""
    rng = np.random.default_rng(3001)
    xa = rng.standard_normal((2, 3, 8, 8))
    totals = {}
    for r in (1, 3, 5):
        fa = rng.standard_normal((4, 3, r, r))
        conv = dp.ConvDesc(1, 1, r // 2, r // 2)
        x = dp.TensorView.from_array(xa, device="cuda")
        f = dp.FilterView.from_array(fa, device="cuda")
        shape = dp.conv_out_shape(x.desc, f.desc, conv)
        y = dp.empty_view(dp.make_desc(*shape, elem_type="f64"), device="cuda")
        dp.scratch_high_water(reset=True)
        dp.conv_forward(x, f, conv, "implicit", y)
        totals[r] = dp.scratch_high_water()
        assert totals[r] <= int(np.prod(shape)) * 8, totals
    assert totals[1] == totals[3] == totals[5], totals
