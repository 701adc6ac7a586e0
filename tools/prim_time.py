"""Kernel-time probe for the bandwidth primitives: each op timed (a) back to
back, 20 launches captured in a CUDA graph (no host dispatch, L2 warm when
the working set fits), (b) cold: one launch after a 1 GiB write + 256 MiB
read flush (L2 clean and empty), events around the launch only.

    python tools/prim_time.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402


def view(shape, dt=torch.float32, layout="nchw"):
    d = dp.make_desc(*shape, layout=layout, elem_type="f32" if dt == torch.float32 else "f64")
    return dp.TensorView(d, torch.rand(d.max_offset() + 1, dtype=dt, device="cuda") - 0.5)


def graph_time(op, reps=20):
    op()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                op()
    torch.cuda.synchronize()
    g.replay()  # the first launch of a graph uploads it: not timed
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (3 * reps)


def cold_time(op, wflush, rflush, reps=5):
    op()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        wflush.fill_(1.0)
        rflush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


def main():
    wflush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rflush = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ops = []
    x, y = view((128, 64, 55, 55)), view((128, 64, 55, 55))
    ops.append(("act_fwd_relu", 2 * 4 * x.desc.size, lambda: dp.activation_forward("relu", x, y)))
    for kind in ("max", "average"):
        pd = dp.PoolingDesc(kind, 3, 3, 2, 2, 0, 0)
        py = view((128, 64, 27, 27))
        am = torch.empty((128, 64, 27, 27), dtype=torch.int64, device="cuda") if kind == "max" else None
        E, Ep = x.desc.size, py.desc.size
        fb = 4 * E + (12 if kind == "max" else 4) * Ep
        ops.append((f"pool_fwd_{kind}", fb, lambda pd=pd, py=py, am=am: dp.pool_forward(pd, x, py, am)))
        dpy = view((128, 64, 27, 27))
        if am is not None:
            dp.pool_forward(pd, x, py, am)
        ops.append((f"pool_bwd_{kind}", fb, lambda pd=pd, py=py, dpy=dpy, am=am:
                    dp.pool_backward(pd, py, dpy, x, y, am)))
    for mode, shp in (("per_image", (1024, 1000, 1, 1)), ("per_spatial", (16, 21, 64, 64))):
        a, b, c2 = view(shp), view(shp), view(shp)
        n = int(np.prod(shp))
        ops.append((f"softmax_fwd_{mode}", 8 * n, lambda a=a, b=b, mode=mode: dp.softmax_forward(mode, a, b)))
        ops.append((f"softmax_bwd_{mode}", 12 * n,
                    lambda a=a, b=b, c2=c2, mode=mode: dp.softmax_backward(mode, a, b, c2)))
    peak = 6555.8
    for name, byt, op in ops:
        g = graph_time(op)
        c = cold_time(op, wflush, rflush)
        print(f"{name:26s} {byt / 1e6:8.1f} MB  graph {g * 1e3:7.1f} us ({byt / g / 1e6:6.0f} GB/s "
              f"{100 * byt / g / 1e6 / peak:5.1f}%)  cold {c * 1e3:7.1f} us ({byt / c / 1e6:6.0f} GB/s "
              f"{100 * byt / c / 1e6 / peak:5.1f}%)", flush=True)


if __name__ == "__main__":
    main()
