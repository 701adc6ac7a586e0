"""One max-pool forward + backward on the section-8(d) shape (ncu target).

    python tools/pool_one.py [nchw|nhwc]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_bw import make_view  # noqa: E402


def main():
    lay = sys.argv[1] if len(sys.argv) > 1 else "nchw"
    N, C, H = 128, 64, 55
    x, _ = make_view(N, C, H, H, lay, "f32")
    dx, _ = make_view(N, C, H, H, lay, "f32")
    pd = dp.PoolingDesc(os.environ.get("POOL_KIND", "max"), 3, 3, 2, 2, 0, 0)
    _, _, P, Q = dp.pool_out_shape(pd, x)
    y, _ = make_view(N, C, P, Q, lay, "f32")
    dy, _ = make_view(N, C, P, Q, lay, "f32")
    am = torch.empty((N, C, P, Q), dtype=torch.int64, device="cuda") if pd.kind.value == "max" else None
    for _ in range(2):
        dp.pool_forward(pd, x, y, am)
        dp.pool_backward(pd, y, dy, x, dx, am)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
