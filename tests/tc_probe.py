"""Diagnostic: tensor-core conv vs the C oracle on a few shapes, with timing.
Run on the GPU box:  python tests/tc_probe.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as orc  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402

SHAPES = [
    # N C H W K R S u pad
    (1, 8, 8, 8, 32, 3, 3, 1, 1),
    (2, 3, 31, 31, 16, 11, 11, 4, 2),
    (2, 3, 32, 36, 64, 11, 11, 4, 2),
    (3, 3, 40, 40, 64, 11, 11, 4, 2),
    (2, 16, 15, 15, 24, 5, 5, 1, 2),
    (3, 24, 9, 9, 40, 3, 3, 1, 1),
    (1, 64, 8, 8, 72, 3, 3, 1, 1),
    (4, 32, 7, 7, 130, 1, 1, 1, 0),
    (2, 64, 14, 14, 256, 3, 3, 1, 1),
    (2, 96, 13, 13, 384, 3, 3, 1, 1),
]


def main():
    rng = np.random.default_rng(0)
    for (N, C, H, W, K, R, S, u, pad) in SHAPES:
        for mode in ("convolution", "cross_correlation"):
            cd = dp.ConvDesc(u, u, pad, pad, mode)
            cg = [u, u, pad, pad, 0 if mode == "convolution" else 1, 0]
            P, Q = dp.output_extent(H, R, u, pad), dp.output_extent(W, S, u, pad)
            x = rng.uniform(-0.5, 0.5, N * C * H * W).astype(np.float32)
            f = rng.uniform(-0.5, 0.5, K * C * R * S).astype(np.float32)
            dy = rng.uniform(-0.5, 0.5, N * K * P * Q).astype(np.float32)
            xv = dp.TensorView(dp.make_desc(N, C, H, W), torch.from_numpy(x).cuda())
            fv = dp.FilterView(dp.make_filter_desc(K, C, R, S), torch.from_numpy(f).cuda())
            yv = dp.empty_view(dp.make_desc(N, K, P, Q), device="cuda")
            dyv = dp.TensorView(dp.make_desc(N, K, P, Q), torch.from_numpy(dy).cuda())
            dxv = dp.empty_view(dp.make_desc(N, C, H, W), device="cuda")
            dp.set_math(0)
            dp.conv_forward(xv, fv, cd, "implicit", yv)
            torch.cuda.synchronize()
            xg = [N, C, H, W, C * H * W, H * W, W, 1]
            yg = [N, K, P, Q, K * P * Q, P * Q, Q, 1]
            ry = np.zeros(N * K * P * Q, np.float32)
            orc.conv_forward(xg, x, [K, C, R, S], f, cg, yg, ry, threads=8)
            ef = orc.rel_err(yv.buf.cpu().numpy(), ry)
            dp.conv_backward_data(dyv, fv, cd, "implicit", dxv)
            torch.cuda.synchronize()
            rdx = np.zeros(N * C * H * W, np.float32)
            orc.conv_backward_data([K, C, R, S], f, yg, dy, cg, xg, rdx)
            ed = orc.rel_err(dxv.buf.cpu().numpy(), rdx)
            dft = torch.zeros(K * C * R * S, device="cuda")
            dfv = dp.FilterView(dp.make_filter_desc(K, C, R, S), dft)
            dp.conv_backward_filter(dyv, xv, cd, "implicit", dfv)
            torch.cuda.synchronize()
            rdf = np.zeros(K * C * R * S, np.float32)
            orc.conv_backward_filter(xg, x, yg, dy, cg, [K, C, R, S], rdf, threads=8)
            ew = orc.rel_err(dft.cpu().numpy(), rdf)
            print(f"{(N, C, H, W, K, R, S, u, pad)} {mode[:4]} fwd_err={ef:.2e} "
                  f"dgrad_err={ed:.2e} wgrad_err={ew:.2e}", flush=True)


if __name__ == "__main__":
    main()
