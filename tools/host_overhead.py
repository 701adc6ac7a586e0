"""Host-side cost of one API call (wall clock of back-to-back submissions,
GPU work skipped with DNNP_TC_SKIP=6 so the queue never fills), split into
the Python layer and the C ABI.

    python tools/host_overhead.py
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    os.environ["DNNP_TC_SKIP"] = "6"
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    L = layers[4]
    ops = {
        "fwd": lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"]),
        "bwd_data": lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"]),
        "bwd_filter": lambda: dp.conv_backward_filter(L["dyv"], L["xv"], L["cd"], "implicit", L["dfv"]),
    }
    for name, op in ops.items():
        for _ in range(5):
            op()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(50):
            op()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{name}: host {1e6 * (t1 - t0) / 50:.1f} us/call, incl. drain {1e6 * (t2 - t0) / 50:.1f} us/call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        ops["fwd"]()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__":
    main()
