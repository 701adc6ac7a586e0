"""One 3x3/2 max-pooling backward at the SURVEY 8(d) shape (128x64x55x55,
NCHW) in a loop: ncu target for the pooling kernels.

    python tools/pool_prof.py [max|average] [iters]      (POOL_FWD=1: the forward)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "max"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    d = dp.make_desc(128, 64, 55, 55)
    x = dp.TensorView(d, torch.rand(d.max_offset() + 1, device="cuda") - 0.5)
    dx = dp.TensorView(d, torch.empty(d.max_offset() + 1, device="cuda"))
    yd = dp.make_desc(128, 64, 27, 27)
    y = dp.TensorView(yd, torch.empty(yd.max_offset() + 1, device="cuda"))
    dy = dp.TensorView(yd, torch.rand(yd.max_offset() + 1, device="cuda") - 0.5)
    am = torch.empty((128, 64, 27, 27), dtype=torch.int64, device="cuda") if kind == "max" else None
    pd = dp.PoolingDesc(kind, 3, 3, 2, 2, 0, 0)
    dp.pool_forward(pd, x, y, am)
    for _ in range(iters):
        if os.environ.get("POOL_FWD"):
            dp.pool_forward(pd, x, y, am)
        else:
            dp.pool_backward(pd, y, dy, x, dx, am)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
