"""Debug: run one conv2-forward-sized problem with DNNP_TC_TRACE=1."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1410_0759_b200 as dp
N, C, H, K, R, u, pad = [int(v) for v in (sys.argv[1:] or [128, 64, 27, 192, 5, 1, 2])]
P = dp.output_extent(H, R, u, pad)
x = torch.rand(N * C * H * H, device="cuda") - 0.5
f = torch.rand(K * C * R * R, device="cuda") - 0.5
xv = dp.TensorView(dp.make_desc(N, C, H, H), x)
fv = dp.FilterView(dp.make_filter_desc(K, C, R, R), f)
yv = dp.empty_view(dp.make_desc(N, K, P, P), device="cuda")
cd = dp.ConvDesc(u, u, pad, pad)
for _ in range(3):
    dp.conv_forward(xv, fv, cd, "implicit", yv)
torch.cuda.synchronize()
