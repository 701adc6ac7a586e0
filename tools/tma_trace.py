"""conv_tma configuration and CTA-0 timeline (DNNP_TC_TRACE) of one AlexNet
layer pass at N=128, optionally under env variants.

    python tools/tma_trace.py conv2 bwd_data [ENV=VAL ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    name, pas = sys.argv[1], sys.argv[2]
    for kv in sys.argv[3:]:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    lay = {l.name: l for l in bc.load_suite("alexnet")}[name]
    prob = bc._Problem(lay, "f32", 2014, 0)
    op = prob.op(pas, "implicit")
    op()
    torch.cuda.synchronize()
    os.environ["DNNP_TC_TRACE"] = "1"
    op()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
