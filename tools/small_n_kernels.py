"""Kernels of one small-batch forward call (OverFeat conv3, N=16) for ncu:
    ncu --metrics gpu__time_duration.sum ... python tools/small_n_kernels.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
c, h, k, r, pad = 256, 12, 512, 3, 1
x = dp.TensorView(dp.make_desc(n, c, h, h), torch.rand(n * c * h * h, device="cuda"))
f = dp.FilterView(dp.make_filter_desc(k, c, r, r), torch.rand(k * c * r * r, device="cuda"))
y = dp.empty_view(dp.make_desc(n, k, h, h), device="cuda")
cd = dp.ConvDesc(1, 1, pad, pad)
for _ in range(3):
    dp.conv_forward(x, f, cd, "implicit", y)
torch.cuda.synchronize()
