"""Small invocations of the round's newer paths for compute-sanitizer
(memcheck): channels-innermost and pipelined pooling, row blocking, tap
folding, 32-channel dy pairs, 128-pixel wgrad stages, fused epilogues,
fused backward, caller workspace.

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(1, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from test_gpu_tc_paths import run_case  # noqa: E402


def main():
    for shape in [(2, 24, 11, 9, 40, 3, 3, 1, 1, 1, 1), (2, 3, 17, 19, 24, 5, 7, 1, 1, 2, 3),
                  (2, 3, 32, 36, 64, 11, 11, 4, 4, 2, 2), (2, 24, 11, 9, 192, 3, 3, 1, 1, 1, 1)]:
        errs = run_case(shape, seed=1)
        print(shape, {k: f"{v:.1e}" for k, v in errs.items()}, flush=True)
    for lay in ("nchw", "nhwc"):
        for dt in ("f32", "f64"):
            for kind in ("max", "average"):
                d = dp.make_desc(2, 32, 13, 13, layout=lay, elem_type=dt)
                tdt = torch.float32 if dt == "f32" else torch.float64
                x = dp.TensorView(d, torch.rand(d.max_offset() + 1, dtype=tdt, device="cuda"))
                pd = dp.PoolingDesc(kind, 3, 3, 2, 2, 0, 0)
                _, _, P, Q = dp.pool_out_shape(pd, x)
                y = dp.TensorView(dp.make_desc(2, 32, P, Q, layout=lay, elem_type=dt),
                                  torch.empty(2 * 32 * P * Q, dtype=tdt, device="cuda"))
                am = torch.empty((2, 32, P, Q), dtype=torch.int64, device="cuda") if kind == "max" else None
                dp.pool_forward(pd, x, y, am)
    n, c, h, k = 2, 64, 9, 64
    xd, yd, fd = dp.make_desc(n, c, h, h), dp.make_desc(n, k, h, h), dp.make_filter_desc(k, c, 3, 3)
    x = dp.TensorView(xd, torch.rand(n * c * h * h, device="cuda"))
    dy = dp.TensorView(yd, torch.rand(n * k * h * h, device="cuda"))
    f = dp.FilterView(fd, torch.rand(k * c * 9, device="cuda"))
    dx = dp.TensorView(xd, torch.empty(n * c * h * h, device="cuda"))
    df = dp.FilterView(fd, torch.empty(k * c * 9, device="cuda"))
    cd = dp.ConvDesc(1, 1, 1, 1)
    dp.conv_backward(dy, f, x, cd, "implicit", dx, df)
    need = dp.convolution_workspace_size("fwd", xd, fd, cd, yd)
    ws = torch.empty(need + 1024, dtype=torch.uint8, device="cuda")
    y = dp.TensorView(yd, torch.empty(n * k * h * h, device="cuda"))
    dp.conv_forward(x, f, cd, "implicit", y, workspace=ws)
    b = dp.TensorView(dp.make_desc(1, k, 1, 1), torch.rand(k, device="cuda"))
    dp.conv_bias_activation_forward(x, f, cd, "implicit", y, bias=b, activation="relu")
    dp.conv_backward_data_activation(dy, f, cd, "implicit", dx, "relu", x)
    torch.cuda.synchronize()
    print("sanitize smoke done", flush=True)


if __name__ == "__main__":
    main()
