import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1410_0759_b200 as dp
for shape, pas in (((4, 16, 20, 20, 32, 3, 3, 1, 1, 1, 1), "fwd"), ((2, 3, 40, 44, 96, 11, 11, 1, 1, 0, 0), "bwd_data")):
    n, c, h, w, k, r, s, u, v, ph, pw = shape
    cd = dp.ConvDesc(u, v, ph, pw)
    p, q = dp.output_extent(h, r, u, ph), dp.output_extent(w, s, v, pw)
    xd, yd = dp.make_desc(n, c, h, w), dp.make_desc(n, k, p, q)
    fd = dp.make_filter_desc(k, c, r, s)
    for i in range(3):
        need = dp.convolution_workspace_size(pas, xd, fd, cd, yd)
        x = torch.rand(n*c*h*w, device="cuda"); dy = torch.rand(n*k*p*q, device="cuda"); f = torch.rand(k*c*r*s, device="cuda")
        dp.scratch_high_water(reset=True)
        if pas == "fwd":
            dp.conv_forward(dp.TensorView(xd, x), dp.FilterView(fd, f), cd, "implicit", dp.TensorView(yd, torch.zeros(n*k*p*q, device="cuda")))
        else:
            dp.conv_backward_data(dp.TensorView(yd, dy), dp.FilterView(fd, f), cd, "implicit", dp.TensorView(xd, torch.zeros(n*c*h*w, device="cuda")))
        torch.cuda.synchronize()
        print(shape, pas, "query", need, "arena high-water of a plain call", dp.scratch_high_water(), flush=True)
