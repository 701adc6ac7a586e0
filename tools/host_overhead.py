"""Host-side cost of one API call: wall clock of back-to-back submissions of
a tiny convolution (N=1: the GPU finishes each call faster than the host
submits it, so wall time per call = host cost), through the Python mirror and
through the C ABI directly (ctypes call with prebuilt descriptors).

    python tools/host_overhead.py
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import _lib  # noqa: E402


def per_call(op, n=100):
    for _ in range(20):
        op()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        op()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / n


def main():
    N, C, H, K, R = 1, 64, 13, 64, 3
    x = dp.TensorView(dp.make_desc(N, C, H, H), torch.rand(N * C * H * H, device="cuda"))
    f = dp.FilterView(dp.make_filter_desc(K, C, R, R), torch.rand(K * C * R * R, device="cuda"))
    y = dp.empty_view(dp.make_desc(N, K, H, H), device="cuda")
    dy = dp.TensorView(dp.make_desc(N, K, H, H), torch.rand(N * K * H * H, device="cuda"))
    dx = dp.empty_view(dp.make_desc(N, C, H, H), device="cuda")
    df = dp.FilterView(dp.make_filter_desc(K, C, R, R), torch.empty(K * C * R * R, device="cuda"))
    cd = dp.ConvDesc(1, 1, 1, 1)
    L = _lib.lib()
    h = _lib.handle()
    one, zero = ctypes.c_float(1.0), ctypes.c_float(0.0)
    xd, fd, yd, cdd = x.desc.c_desc(), f.desc.c_desc(), y.desc.c_desc(), cd.c_desc()
    dyd, dxd = dy.desc.c_desc(), dx.desc.c_desc()
    xp, fp, yp = x.ptr, f.ptr, y.ptr
    dyp, dxp, dfp = dy.ptr, dx.ptr, df.ptr
    _lib.set_stream(torch.cuda.current_stream().cuda_stream)
    rows = [
        ("python fwd", lambda: dp.conv_forward(x, f, cd, "implicit", y)),
        ("python bwd_data", lambda: dp.conv_backward_data(dy, f, cd, "implicit", dx)),
        ("python bwd_filter", lambda: dp.conv_backward_filter(dy, x, cd, "implicit", df)),
        ("C ABI fwd", lambda: L.dnnp_convolution_forward(h, ctypes.byref(one), xd, xp, fd, fp, cdd,
                                                         2, ctypes.byref(zero), yd, yp)),
        ("C ABI bwd_data", lambda: L.dnnp_convolution_backward_data(h, fd, fp, dyd, dyp, cdd, 2,
                                                                    dxd, dxp)),
        ("C ABI bwd_filter", lambda: L.dnnp_convolution_backward_filter(h, xd, xp, dyd, dyp, cdd,
                                                                        2, fd, dfp)),
        ("python relu fwd", lambda: dp.activation_forward("relu", y, y)),
    ]
    for name, op in rows:
        l0 = dp.kernel_launch_count()
        us = per_call(op)
        k = (dp.kernel_launch_count() - l0) / 120
        print(f"{name:22s} {us:7.1f} us/call  ({k:.1f} kernels/call)", flush=True)


if __name__ == "__main__":
    main()
