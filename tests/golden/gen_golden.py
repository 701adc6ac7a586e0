#!/usr/bin/env python3
"""Generate golden input/output vectors from the REFERENCE implementation.

Run once in the build container, where the reference package is readable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

It imports the unmodified reference `dnnp` package (pure numpy CPU code),
runs it on small seeded problems covering every hot-path operation, layout
(NCHW, NHWC, channel-slice sub-tensor views, padded rows), both convolution
modes, strides, padding, alpha/beta and accumulate, and writes the flat
buffers in and out to tests/golden/*.npz.  Nothing at test time reads the
reference; the fixtures travel with the repo.
"""
import json
import os
import sys

import numpy as np

import dnnp  # the reference package (PYTHONPATH=/root/reference/pkg/src)
from dnnp import (ConvDesc, Engine, FilterView, PoolingDesc, TensorView, make_desc,
                  make_filter_desc)

HERE = os.path.dirname(os.path.abspath(__file__))


def layout_strides(kind, n, c, h, w):
    """(strides, buffer length) for a named layout."""
    if kind == "nchw":
        return (c * h * w, h * w, w, 1), n * c * h * w
    if kind == "nhwc":
        return (h * w * c, 1, w * c, c), n * c * h * w
    if kind == "slice":  # channel slice [2, 2+c) of a (c+5)-channel NCHW parent
        pc = c + 5
        return (pc * h * w, h * w, w, 1), n * pc * h * w  # base offset applied by caller
    if kind == "padrow":  # NCHW with each row padded by 3 elements
        wp = w + 3
        return (c * h * wp, h * wp, wp, 1), n * c * h * wp
    raise ValueError(kind)


def make_view(rng, kind, n, c, h, w, dt):
    strides, length = layout_strides(kind, n, c, h, w)
    base = 2 * h * w if kind == "slice" else 0
    buf = rng.uniform(-0.5, 0.5, length + base).astype(dt)
    sub = buf[base:]
    desc = make_desc(n, c, h, w, layout="custom", strides=strides, elem_type=dt)
    return buf, base, TensorView(desc, sub), strides


def geom(n, c, h, w, strides):
    return np.array([n, c, h, w, *strides], dtype=np.int64)


def conv_cases():
    rng = np.random.default_rng(20141003)
    out = {}
    meta = []
    shapes = [
        # N C H W K R S u v ph pw mode
        (1, 3, 3, 3, 2, 2, 2, 1, 1, 0, 0, "convolution"),       # Fig. 1 sized
        (2, 3, 7, 6, 4, 3, 3, 1, 1, 1, 1, "convolution"),
        (2, 4, 9, 8, 5, 3, 2, 2, 1, 1, 0, "cross_correlation"),
        (1, 5, 11, 11, 3, 5, 5, 2, 2, 2, 2, "convolution"),
        (3, 2, 8, 10, 6, 1, 1, 1, 1, 0, 0, "cross_correlation"),
        (2, 3, 13, 12, 4, 4, 3, 3, 2, 1, 2, "convolution"),
        (1, 6, 6, 6, 7, 3, 3, 1, 1, 2, 2, "cross_correlation"),
        (2, 8, 10, 10, 16, 3, 3, 1, 1, 1, 1, "convolution"),
    ]
    layouts = ["nchw", "nhwc", "slice", "padrow"]
    idx = 0
    for si, (N, C, H, W, K, R, S, u, v, ph, pw, mode) in enumerate(shapes):
        for dt in (np.float32, np.float64):
            lay_x = layouts[(si + (dt == np.float64)) % 4]
            lay_y = layouts[(si + 1) % 4]
            conv = ConvDesc(u, v, ph, pw, mode, accumulate=False)
            P = dnnp.output_extent(H, R, u, ph)
            Q = dnnp.output_extent(W, S, v, pw)
            # forward with alpha/beta
            xb, xbase, xv, xs = make_view(rng, lay_x, N, C, H, W, dt)
            fa = rng.uniform(-0.5, 0.5, K * C * R * S).astype(dt)
            fv = FilterView(make_filter_desc(K, C, R, S, elem_type=dt), fa)
            yb, ybase, yv, ys = make_view(rng, lay_y, N, K, P, Q, dt)
            y_in = yb.copy()
            alpha, beta = (1.0, 0.0) if si % 3 == 0 else ((0.75, 0.5) if si % 3 == 1 else (-1.25, 1.0))
            dnnp.conv_forward(xv, fv, conv, Engine.IMPLICIT, yv, alpha=alpha, beta=beta)
            # backward data (accumulate on odd shapes) into a fresh dx view
            acc = si % 2 == 1
            conv_acc = ConvDesc(u, v, ph, pw, mode, accumulate=acc)
            dyb, dybase, dyv, dys = make_view(rng, lay_y, N, K, P, Q, dt)
            dxb, dxbase, dxv, dxs = make_view(rng, lay_x, N, C, H, W, dt)
            dx_in = dxb.copy()
            dnnp.conv_backward_data(dyv, fv, conv_acc, Engine.IMPLICIT, dxv)
            # backward filter
            dfa = rng.uniform(-0.5, 0.5, K * C * R * S).astype(dt)
            df_in = dfa.copy()
            dfv = FilterView(make_filter_desc(K, C, R, S, elem_type=dt), dfa)
            dnnp.conv_backward_filter(dyv, xv, conv_acc, Engine.IMPLICIT, dfv)
            # bias
            db = dnnp.conv_backward_bias(dyv)
            p = f"c{idx}_"
            out[p + "xg"] = geom(N, C, H, W, xs)
            out[p + "yg"] = geom(N, K, P, Q, ys)
            out[p + "fg"] = np.array([K, C, R, S], dtype=np.int64)
            out[p + "cg"] = np.array([u, v, ph, pw, 0 if mode == "convolution" else 1, 0],
                                     dtype=np.int64)
            out[p + "cg_acc"] = np.array([u, v, ph, pw, 0 if mode == "convolution" else 1,
                                          int(acc)], dtype=np.int64)
            out[p + "bases"] = np.array([xbase, ybase, dybase, dxbase], dtype=np.int64)
            out[p + "scal"] = np.array([alpha, beta])
            out[p + "x"] = xb
            out[p + "f"] = fa
            out[p + "y_in"] = y_in
            out[p + "y_out"] = yb
            out[p + "dy"] = dyb
            out[p + "dx_in"] = dx_in
            out[p + "dx_out"] = dxb
            out[p + "df_in"] = df_in
            out[p + "df_out"] = dfa
            out[p + "db"] = np.ascontiguousarray(db.array).reshape(-1)
            meta.append({"case": idx, "shape": [N, C, H, W, K, R, S, u, v, ph, pw], "mode": mode,
                         "dtype": np.dtype(dt).name, "x_layout": lay_x, "y_layout": lay_y,
                         "alpha": alpha, "beta": beta, "accumulate": acc})
            idx += 1
    out["count"] = np.array([idx])
    return out, meta


SENTINEL = 7.0


def out_view(rng, kind, n, c, h, w, dt):
    """Output view whose whole buffer (gaps included) starts at SENTINEL."""
    buf, base, view, strides = make_view(rng, kind, n, c, h, w, dt)
    buf[:] = SENTINEL
    return buf, base, view, strides


def nnops_cases():
    rng = np.random.default_rng(19410)
    out = {}
    meta = []
    idx = 0
    for dt in (np.float32, np.float64):
        for lay in ("nchw", "nhwc", "slice"):
            N, C, H, W = 2, 3, 7, 6
            for kind in ("sigmoid", "relu", "tanh"):
                xb, xbase, xv, xs = make_view(rng, lay, N, C, H, W, dt)
                xb[xbase] = 0.0
                xb *= 8.0
                yb, ybase, yv, ys = out_view(rng, "nchw", N, C, H, W, dt)
                dnnp.activation_forward(kind, xv, yv)
                dyb, dybase, dyv, dys = make_view(rng, lay, N, C, H, W, dt)
                dxb, dxbase, dxv, dxs = out_view(rng, "nhwc", N, C, H, W, dt)
                dnnp.activation_backward(kind, yv, dyv, dxv)
                p = f"a{idx}_"
                out[p + "meta"] = np.array([["sigmoid", "relu", "tanh"].index(kind)])
                out[p + "xg"], out[p + "yg"] = geom(N, C, H, W, xs), geom(N, C, H, W, ys)
                out[p + "dyg"], out[p + "dxg"] = geom(N, C, H, W, dys), geom(N, C, H, W, dxs)
                out[p + "bases"] = np.array([xbase, ybase, dybase, dxbase])
                out[p + "x"], out[p + "y"], out[p + "dy"], out[p + "dx"] = xb, yb, dyb, dxb
                meta.append({"case": p, "op": "activation", "kind": kind, "layout": lay,
                             "dtype": np.dtype(dt).name})
                idx += 1
            for mode in ("per_image", "per_spatial"):
                xb, xbase, xv, xs = make_view(rng, lay, N, C, H, W, dt)
                xb *= 6.0
                yb, ybase, yv, ys = out_view(rng, "nchw", N, C, H, W, dt)
                dnnp.softmax_forward(mode, xv, yv)
                dyb, dybase, dyv, dys = make_view(rng, lay, N, C, H, W, dt)
                dxb, dxbase, dxv, dxs = out_view(rng, "padrow", N, C, H, W, dt)
                dnnp.softmax_backward(mode, yv, dyv, dxv)
                p = f"s{idx}_"
                out[p + "meta"] = np.array([0 if mode == "per_image" else 1])
                out[p + "xg"], out[p + "yg"] = geom(N, C, H, W, xs), geom(N, C, H, W, ys)
                out[p + "dyg"], out[p + "dxg"] = geom(N, C, H, W, dys), geom(N, C, H, W, dxs)
                out[p + "bases"] = np.array([xbase, ybase, dybase, dxbase])
                out[p + "x"], out[p + "y"], out[p + "dy"], out[p + "dx"] = xb, yb, dyb, dxb
                meta.append({"case": p, "op": "softmax", "mode": mode, "layout": lay,
                             "dtype": np.dtype(dt).name})
                idx += 1
            for (kind, wh, ww, sh, sw, ph, pw) in (("max", 3, 3, 2, 2, 0, 0), ("max", 2, 3, 1, 2, 1, 1),
                                                  ("average", 3, 3, 2, 2, 1, 1), ("average", 2, 2, 2, 2, 0, 0)):
                N, C, H, W = 2, 3, 9, 8
                xb, xbase, xv, xs = make_view(rng, lay, N, C, H, W, dt)
                # quantised values force ties (argmax must take the first)
                xb[:] = np.round(xb * 4) / 4
                pd = PoolingDesc(kind, wh, ww, sh, sw, ph, pw)
                n_, c_, P, Q = dnnp.pool_out_shape(pd, xv)
                yb, ybase, yv, ys = out_view(rng, "nchw", N, C, P, Q, dt)
                am = np.full((N, C, P, Q), -1, dtype=np.int64)
                dnnp.pool_forward(pd, xv, yv, am if kind == "max" else None)
                dyb, dybase, dyv, dys = make_view(rng, lay, N, C, P, Q, dt)
                dxb, dxbase, dxv, dxs = out_view(rng, "nhwc", N, C, H, W, dt)
                dnnp.pool_backward(pd, yv, dyv, xv, dxv, am if kind == "max" else None)
                p = f"p{idx}_"
                out[p + "meta"] = np.array([0 if kind == "max" else 1, wh, ww, sh, sw, ph, pw])
                out[p + "xg"], out[p + "yg"] = geom(N, C, H, W, xs), geom(N, C, P, Q, ys)
                out[p + "dyg"], out[p + "dxg"] = geom(N, C, P, Q, dys), geom(N, C, H, W, dxs)
                out[p + "bases"] = np.array([xbase, ybase, dybase, dxbase])
                out[p + "x"], out[p + "y"], out[p + "dy"], out[p + "dx"] = xb, yb, dyb, dxb
                out[p + "argmax"] = am.reshape(-1)
                meta.append({"case": p, "op": "pool", "kind": kind, "layout": lay,
                             "dtype": np.dtype(dt).name})
                idx += 1
            # transform + add_broadcast
            N, C, H, W = 2, 4, 5, 3
            sb, sbase, sv, ss = make_view(rng, lay, N, C, H, W, dt)
            db_, dbase, dv, ds = make_view(rng, "padrow", N, C, H, W, dt)
            d_in = db_.copy()
            dnnp.transform(sv, dv, alpha=1.5, beta=-0.5)
            p = f"t{idx}_"
            out[p + "sg"], out[p + "dg"] = geom(N, C, H, W, ss), geom(N, C, H, W, ds)
            out[p + "bases"] = np.array([sbase, dbase])
            out[p + "s"], out[p + "d_in"], out[p + "d_out"] = sb, d_in, db_
            meta.append({"case": p, "op": "transform", "layout": lay, "dtype": np.dtype(dt).name})
            idx += 1
            bb, bbase, bv, bs = make_view(rng, "nchw", 1, C, 1, W, dt)
            ob, obase, ov, os_ = make_view(rng, lay, N, C, H, W, dt)
            o_in = ob.copy()
            dnnp.add_broadcast(bv, ov, alpha=2.0, beta=0.5)
            p = f"b{idx}_"
            out[p + "bg"], out[p + "og"] = geom(1, C, 1, W, bs), geom(N, C, H, W, os_)
            out[p + "bases"] = np.array([bbase, obase])
            out[p + "b"], out[p + "o_in"], out[p + "o_out"] = bb, o_in, ob
            meta.append({"case": p, "op": "add_broadcast", "layout": lay, "dtype": np.dtype(dt).name})
            idx += 1
    return out, meta


def intdiv_cases():
    cases = {}
    for d in [1, 2, 3, 5, 7, 9, 11, 12, 24, 56, 121, 384, 1023, 3136, 13924, 65536, 2**31 - 1,
              2**31 + 1, 2**32 - 1]:
        md = dnnp.make_divider(d)
        cases[str(d)] = [md.multiplier, md.shift, int(md.add_indicator)]
    return cases


def fig1_example():
    # pkg/capi/tools/gen_golden.py problem: N=1 C=3 3x3, K=2 2x2, valid, unit stride
    N, C, H, W, K, R, S = 1, 3, 3, 3, 2, 2, 2
    x = np.array([(i % 11) - 5 for i in range(N * C * H * W)], dtype=np.float32).reshape(N, C, H, W)
    f = np.array([((i * 3) % 7) - 3 for i in range(K * C * R * S)], dtype=np.float32).reshape(K, C, R, S)
    xv, fv = TensorView.from_array(x), FilterView.from_array(f)
    conv = ConvDesc()
    y = dnnp.empty_view(make_desc(*dnnp.conv_out_shape(xv.desc, fv.desc, conv)))
    dnnp.conv_forward(xv, fv, conv, Engine.IMPLICIT, y)
    return np.ascontiguousarray(y.array).ravel().tolist()


def main():
    conv, conv_meta = conv_cases()
    np.savez_compressed(os.path.join(HERE, "conv.npz"), **conv)
    nn, nn_meta = nnops_cases()
    np.savez_compressed(os.path.join(HERE, "nnops.npz"), **nn)
    info = {"generator": "tests/golden/gen_golden.py", "reference": "pkg/src/dnnp (numpy)",
            "numpy": np.__version__, "conv_cases": conv_meta, "nnops_cases": nn_meta,
            "intdiv": intdiv_cases(), "fig1_example": fig1_example()}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(info, fh, indent=1)
    print("wrote", len(conv_meta), "conv cases and", len(nn_meta), "nnops cases;",
          "fig1 =", info["fig1_example"], file=sys.stderr)


if __name__ == "__main__":
    main()
