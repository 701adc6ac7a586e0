"""Profiling driver: run ONE AlexNet layer pass a few times (for ncu captures).

    python tools/prof_layer.py conv1 fwd [iters]

Same shapes and inputs as bench.py; no timing is reported here (numbers
taken under a profiler are never bench values).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "conv1"
    pas = sys.argv[2] if len(sys.argv) > 2 else "fwd"
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    n = int(os.environ.get("PROF_N", "128"))
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(n, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    L = [l for l in layers if l["name"] == name][0]
    op = {
        "fwd": lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"]),
        "bwd_data": lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"]),
        "bwd_filter": lambda: dp.conv_backward_filter(L["dyv"], L["xv"], L["cd"], "implicit", L["dfv"]),
    }[pas]
    for _ in range(iters):
        op()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
