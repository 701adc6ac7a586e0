"""Backward-filter configuration and CTA-0 stage timeline (DNNP_TC_TRACE) of
one AlexNet layer at N=128.

    python tools/wg_trace.py conv1
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "conv1"
    lay = {l.name: l for l in bc.load_suite("alexnet")}[name]
    prob = bc._Problem(lay, "f32", 2014, 0)
    op = prob.op("bwd_filter", "implicit")
    op()
    torch.cuda.synchronize()
    os.environ["DNNP_TC_TRACE"] = "1"
    op()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
