"""Bandwidth-bound primitives (SURVEY.md section 8(d) "B"): achieved GB/s of
activation / softmax / pooling forward and backward on dense NCHW, dense NHWC
and a channel-slice sub-tensor view ([16:48) of a 64-channel NCHW parent),
fp32 and fp64, against the measured HBM copy bandwidth (MEASURED_PEAKS.json).

Algorithmic bytes (section 8(d)): eb = element bytes, E = input elements,
E' = pooled elements; activation fwd 2 eb E, bwd 3 eb E; softmax fwd 2 eb E,
bwd 3 eb E; max-pool fwd eb E + (eb + 8) E', bwd (eb + 8) E' + eb E; avg-pool
fwd / bwd eb E + eb E'.  L2 is flushed (256 MiB write) before every timed
call; CUDA events on torch's current stream (the library's stream).

    python tools/bench_bw.py [--quick] [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def make_view(n, c, h, w, layout, dt, fill="rand"):
    """(TensorView, torch storage) for layout nchw / nhwc / slice."""
    tdt = torch.float32 if dt == "f32" else torch.float64
    if layout == "slice":
        parent_c = 64
        buf = torch.rand(n * parent_c * h * w, dtype=tdt, device="cuda") - 0.5
        desc = dp.make_desc(n, c, h, w, layout="custom",
                            strides=[parent_c * h * w, h * w, w, 1], elem_type=dt)
        return dp.TensorView(desc, buf[16 * h * w:]), buf
    desc = dp.make_desc(n, c, h, w, layout=layout, elem_type=dt)
    buf = torch.rand(desc.max_offset() + 1, dtype=tdt, device="cuda") - 0.5
    return dp.TensorView(desc, buf), buf


def timed(op, flush, reps):
    """Kernel time of op: a 1 GiB L2-flushing write is queued first, so the
    op's launch is already waiting behind it when the start event records
    (host dispatch is outside the window); events on the op's stream."""
    op()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        flush.fill_(1.0)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        op()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    peak, basis = hbm_peak()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
    results = []
    dts = ["f32"] if args.quick else ["f32", "f64"]
    layouts = ["nchw", "nhwc", "slice"]
    N, C, H = 128, 64, 55
    for dt in dts:
        eb = 4 if dt == "f32" else 8
        for lay in layouts:
            c = 32 if lay == "slice" else C
            E = N * c * H * H
            x, _ = make_view(N, c, H, H, lay, dt)
            y, _ = make_view(N, c, H, H, lay, dt)
            dy, _ = make_view(N, c, H, H, lay, dt)
            dx, _ = make_view(N, c, H, H, lay, dt)
            for kind in ("relu", "tanh", "sigmoid"):
                ms = timed(lambda: dp.activation_forward(kind, x, y), flush, args.reps)
                results.append((f"act_fwd_{kind}", dt, lay, 2 * eb * E, ms))
                ms = timed(lambda: dp.activation_backward(kind, y, dy, dx), flush, args.reps)
                results.append((f"act_bwd_{kind}", dt, lay, 3 * eb * E, ms))
            for pk in ("max", "average"):
                pd = dp.PoolingDesc(pk, 3, 3, 2, 2, 0, 0)
                _, _, P, Q = dp.pool_out_shape(pd, x)
                Ep = N * c * P * Q
                py, _ = make_view(N, c, P, Q, lay, dt)
                pdy, _ = make_view(N, c, P, Q, lay, dt)
                am = torch.empty((N, c, P, Q), dtype=torch.int64, device="cuda") if pk == "max" else None
                ms = timed(lambda: dp.pool_forward(pd, x, py, am), flush, args.reps)
                fb = eb * E + (eb + 8) * Ep if pk == "max" else eb * E + eb * Ep
                results.append((f"pool_fwd_{pk}", dt, lay, fb, ms))
                ms = timed(lambda: dp.pool_backward(pd, py, pdy, x, dx, am), flush, args.reps)
                bb = (eb + 8) * Ep + eb * E if pk == "max" else eb * Ep + eb * E
                results.append((f"pool_bwd_{pk}", dt, lay, bb, ms))
        # softmax shapes of section 8(d)
        for (mode, shp) in (("per_image", (1024, 1000, 1, 1)), ("per_spatial", (16, 21, 64, 64))):
            for lay in layouts:
                n, c, h, w = shp
                if lay == "slice":
                    if c < 48:
                        continue
                    c = 32
                E = n * c * h * w
                x, _ = make_view(n, c, h, w, lay, dt)
                y, _ = make_view(n, c, h, w, lay, dt)
                dy, _ = make_view(n, c, h, w, lay, dt)
                dx, _ = make_view(n, c, h, w, lay, dt)
                ms = timed(lambda: dp.softmax_forward(mode, x, y), flush, args.reps)
                results.append((f"softmax_fwd_{mode}", dt, lay, 2 * eb * E, ms))
                ms = timed(lambda: dp.softmax_backward(mode, y, dy, dx), flush, args.reps)
                results.append((f"softmax_bwd_{mode}", dt, lay, 3 * eb * E, ms))
    out = []
    for name, dt, lay, byt, ms in results:
        gbs = byt / (ms / 1e3) / 1e9
        out.append({"op": name, "dtype": dt, "layout": lay, "bytes": int(byt), "ms": round(ms, 4),
                    "GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 3)})
        print(f"{name:24s} {dt} {lay:6s} {byt / 1e6:9.1f} MB {ms * 1e3:8.1f} us "
              f"{gbs:7.0f} GB/s  {100 * gbs / peak:5.1f}% of {basis} HBM {peak:.0f}", flush=True)
    if args.json:
        json.dump({"hbm_peak_gbs": peak, "peak_basis": basis, "results": out}, open(args.json, "w"),
                  indent=1)


if __name__ == "__main__":
    main()
