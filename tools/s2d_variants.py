"""conv1 forward / backward-filter under each space-to-depth pack variant:
whole-op time, the GEMM kernels' time (kernel-timing record) and the rest
(packing, filter pack, reduction).

    python tools/s2d_variants.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    lay = bc.load_suite("alexnet")[0]
    prob = bc._Problem(lay, "f32", 2014, 0)
    for var in ("", "DNNP_S2D_ROWS", "DNNP_S2D_TILE", "DNNP_S2D_DENSE"):
        for k in ("DNNP_S2D_ROWS", "DNNP_S2D_TILE", "DNNP_S2D_DENSE"):
            os.environ.pop(k, None)
        if var:
            os.environ[var] = "1"
        for pas in ("fwd", "bwd_filter"):
            op = prob.op(pas, "implicit")
            t = bc._time(op, 9)
            dp.kernel_timing(1)
            op()
            torch.cuda.synchronize()
            ks = dp.kernel_times()
            dp.kernel_timing(0)
            kt = sum(m for m, _ in ks) / 1e3
            print(f"{var or 'per-pixel':>15} {pas:<10}: op {t * 1e6:7.1f} us  gemm {kt * 1e6:7.1f} us  "
                  f"rest {(t - kt) * 1e6:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
