"""Per-call time of the bench's end-to-end step (C ABI, pinned host buffers,
AlexNet N=128): each of the 15 calls timed alone with the bytes it moves
over PCIe and the rate that implies.

    python tools/e2e_calls.py
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
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    tot = 0.0
    for L in layers:
        n, c, h, k, r, p = L["n"], L["c"], L["h"], L["k"], L["r"], L["p"]
        hx, hf, hdy = (t.cpu().pin_memory() for t in (L["x"], L["f"], L["dy"]))
        hy = torch.empty(n * k * p * p, pin_memory=True)
        hdx = torch.empty(n * c * h * h, pin_memory=True)
        hdf = torch.empty(k * c * r * r, pin_memory=True)
        x = dp.TensorView(dp.make_desc(n, c, h, h), hx.numpy())
        f = dp.FilterView(dp.make_filter_desc(k, c, r, r), hf.numpy())
        dy = dp.TensorView(dp.make_desc(n, k, p, p), hdy.numpy())
        y = dp.TensorView(dp.make_desc(n, k, p, p), hy.numpy())
        dx = dp.TensorView(dp.make_desc(n, c, h, h), hdx.numpy())
        df = dp.FilterView(dp.make_filter_desc(k, c, r, r), hdf.numpy())
        xb, yb, fb = hx.numel() * 4, hy.numel() * 4, hf.numel() * 4
        calls = [("fwd", lambda: dp.conv_forward(x, f, L["cd"], "implicit", y), xb + fb, yb),
                 ("bwd_data", lambda: dp.conv_backward_data(dy, f, L["cd"], "implicit", dx), yb + fb, xb),
                 ("bwd_filter", lambda: dp.conv_backward_filter(dy, x, L["cd"], "implicit", df), xb + yb, fb)]
        for name, op, hin, hout in calls:
            op()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                op()
            ms = (time.perf_counter() - t0) / 5 * 1e3
            tot += ms
            lim = max(hin / 55e9, hout / 57e9) * 1e3
            print(f"{L['name']}.{name:10s} {ms:7.3f} ms  in {hin / 1e6:6.1f} MB out {hout / 1e6:6.1f} MB"
                  f"  PCIe floor {lim:6.3f} ms  ({100 * lim / ms:4.0f}%)", flush=True)
    print(f"step {tot:.2f} ms")


if __name__ == "__main__":
    main()
