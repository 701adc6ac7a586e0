"""Fused conv epilogues vs the unfused call sequence on AlexNet conv1-5 at
N=128 (fp32): forward + bias + ReLU, and bwd-data + ReLU-backward.

    python tools/fused_probe.py
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
    for lay in bc.load_suite("alexnet"):
        prob = bc._Problem(lay, "f32", 2014, 0)
        K = lay.k
        bias = dp.TensorView(dp.make_desc(1, K, 1, 1), torch.rand(K, device="cuda") - 0.5)
        g = dp.TensorView(prob.x.desc, prob.x.buf.clamp(min=0))
        tmp = dp.empty_view(prob.dx.desc, device="cuda")

        def fwd_unfused():
            dp.conv_forward(prob.x, prob.f, prob.cd, "implicit", prob.y)
            dp.add_broadcast(bias, prob.y, 1.0, 1.0)
            dp.activation_forward("relu", prob.y, prob.y)

        def fwd_fused():
            dp.conv_bias_activation_forward(prob.x, prob.f, prob.cd, "implicit", prob.y, bias=bias,
                                            activation="relu")

        def bwd_unfused():
            dp.conv_backward_data(prob.dy, prob.f, prob.cd, "implicit", tmp)
            dp.activation_backward("relu", g, tmp, prob.dx)

        def bwd_fused():
            dp.conv_backward_data_activation(prob.dy, prob.f, prob.cd, "implicit", prob.dx, "relu", g)

        t = [timed(fn) for fn in (fwd_unfused, fwd_fused, bwd_unfused, bwd_fused)]
        print(f"{lay.name}: fwd+bias+relu unfused {t[0]:7.1f} us fused {t[1]:7.1f} us "
              f"({t[0] / t[1]:.2f}x) | dgrad+relu' unfused {t[2]:7.1f} us fused {t[3]:7.1f} us "
              f"({t[2] / t[3]:.2f}x)", flush=True)


if __name__ == "__main__":
    main()
