"""Memory negative control: scratch footprint and time of the explicit-
lowering engine vs the implicit kernels, forward pass, suite layers at their
suite batch (layers whose lowered matrix exceeds the 4 GiB limit report
AllocTooLarge, as the reference does).

    python tools/explicit_control.py [suite ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    suites = sys.argv[1:] or ["table2", "alexnet"]
    for suite in suites:
        for lay in bc.load_suite(suite):
            prob = bc._Problem(lay, "f32", 2014, 0)
            line = f"{suite:>8} {lay.name:<8}"
            outs = {}
            for eng in ("implicit", "explicit"):
                try:
                    op = prob.op("fwd", eng)
                    op()
                    torch.cuda.synchronize()
                    dp.scratch_high_water(reset=True)
                    t = bc._time(op, 5)
                    hw = dp.scratch_high_water()
                    outs[eng] = prob.y.buf.clone()
                    line += f" | {eng} {t * 1e6:8.1f} us {lay.flops() / t / 1e12:6.1f} TF/s scratch {hw / 2**20:8.1f} MiB"
                except dp.AllocTooLarge:
                    line += f" | {eng} AllocTooLarge (lowered {lay.c * lay.r * lay.s * lay.n * lay.out_hw()[0] * lay.out_hw()[1] * 4 / 2**30:.1f} GiB > 4 GiB)"
            if len(outs) == 2:
                d = float((outs["explicit"] - outs["implicit"]).abs().max() / outs["implicit"].abs().max())
                line += f" | diff {d:.1e}"
            print(line, flush=True)


if __name__ == "__main__":
    main()
