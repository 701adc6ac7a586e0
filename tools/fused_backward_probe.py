"""Fused backward (one dy pack) vs the two separate calls on AlexNet
conv1-5 at N=128.

    python tools/fused_backward_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def timed(op, reps=10):
    op()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        op()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    tot = [0.0, 0.0]
    for lay in bc.load_suite("alexnet"):
        pr = bc._Problem(lay, "f32", 2014, 0)
        sep = timed(lambda: (pr.op("bwd_data", "implicit")(), pr.op("bwd_filter", "implicit")()))
        fus = timed(lambda: dp.conv_backward(pr.dy, pr.f, pr.x, pr.cd, "implicit", pr.dx, pr.df))
        tot[0] += sep
        tot[1] += fus
        print(f"{lay.name}: separate {sep:7.1f} us  fused {fus:7.1f} us  ({sep / fus:.2f}x)", flush=True)
    print(f"total: separate {tot[0]:.1f} us  fused {tot[1]:.1f} us  ({tot[0] / tot[1]:.2f}x)")


if __name__ == "__main__":
    main()
