"""CTA-0 epilogue timeline (DNNP_TC_TRACE) of a forward / backward-data
call with and without fused epilogue ops.

    python tools/epi_trace.py [layer]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "conv3"
    lay = {l.name: l for l in bc.load_suite("alexnet")}[name]
    prob = bc._Problem(lay, "f32", 2014, 0)
    g = dp.TensorView(prob.x.desc, prob.x.buf.clamp(min=0))
    calls = {
        "dgrad plain": prob.op("bwd_data", "implicit"),
        "dgrad gate": lambda: dp.conv_backward_data_activation(prob.dy, prob.f, prob.cd, "implicit",
                                                               prob.dx, "relu", g),
    }
    for fn in calls.values():
        fn()
    torch.cuda.synchronize()
    os.environ["DNNP_TC_TRACE"] = "1"
    for k, fn in calls.items():
        print("===", k, flush=True)
        fn()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
