"""Where the end-to-end (host buffer) time goes: raw pinned H2D / D2H
bandwidth on this box, then each bench op through the C ABI with pinned host
buffers (wall time per call, bytes moved).

    python tools/e2e_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    n = 256 * 1024 * 1024
    h = torch.empty(n // 4, pin_memory=True)
    d = torch.empty(n // 4, device="cuda")
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)),
                     ("D2H", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"pinned {name}: {n / dt / 1e9:.1f} GB/s", flush=True)
    layers = bench.make_inputs(128, torch.device("cuda"), torch)
    bench.build_views(dp, layers, torch, torch.device("cuda"))
    for L in layers:
        nn, c, hh, k, r, p = L["n"], L["c"], L["h"], L["k"], L["r"], L["p"]
        hx = L["x"].cpu().pin_memory()
        hf = L["f"].cpu().pin_memory()
        hdy = L["dy"].cpu().pin_memory()
        hy = torch.empty(nn * k * p * p, pin_memory=True)
        hdx = torch.empty(nn * c * hh * hh, pin_memory=True)
        hdf = torch.empty(k * c * r * r, pin_memory=True)
        x = dp.TensorView(dp.make_desc(nn, c, hh, hh), hx.numpy())
        f = dp.FilterView(dp.make_filter_desc(k, c, r, r), hf.numpy())
        dy = dp.TensorView(dp.make_desc(nn, k, p, p), hdy.numpy())
        y = dp.TensorView(dp.make_desc(nn, k, p, p), hy.numpy())
        dx = dp.TensorView(dp.make_desc(nn, c, hh, hh), hdx.numpy())
        df = dp.FilterView(dp.make_filter_desc(k, c, r, r), hdf.numpy())
        ops = {"fwd": (lambda: dp.conv_forward(x, f, L["cd"], "implicit", y),
                       hx.numel() * 4 + hf.numel() * 4, hy.numel() * 4),
               "bwd_data": (lambda: dp.conv_backward_data(dy, f, L["cd"], "implicit", dx),
                            hdy.numel() * 4 + hf.numel() * 4, hdx.numel() * 4),
               "bwd_filter": (lambda: dp.conv_backward_filter(dy, x, L["cd"], "implicit", df),
                              hdy.numel() * 4 + hx.numel() * 4, hdf.numel() * 4)}
        for pas, (op, bin_, bout) in ops.items():
            op()
            t0 = time.perf_counter()
            for _ in range(3):
                op()
            dt = (time.perf_counter() - t0) / 3
            print(f"{L['name']}.{pas}: {dt * 1e3:7.2f} ms wall  in {bin_ / 1e6:6.1f} MB  out "
                  f"{bout / 1e6:6.1f} MB  -> {(bin_ + bout) / dt / 1e9:5.1f} GB/s", flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def bench_like():
    """The bench's e2e loop (run_e2e), step by step, wall clock per step."""
    import numpy as np
    dev = torch.device("cuda")
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)

    class A:
        steps = 5
    t0 = time.perf_counter()
    r = bench.run_e2e(dp, layers, torch, dev, 1, A(), 3 * sum(L["flops"] for L in layers))
    print("run_e2e:", r, f"total wall {time.perf_counter() - t0:.2f} s", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "bench":
    bench_like()
