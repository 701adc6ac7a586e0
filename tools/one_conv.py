"""Run one suite layer's pass a few times (for ncu captures).

    python tools/one_conv.py <suite> <layer> <pass> [N] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    suite, name, pas = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else None
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    lay = {l.name: l for l in bc.load_suite(suite)}[name]
    if n:
        lay = bc.replace(lay, n=n)
    prob = bc._Problem(lay, "f32", 2014, 0)
    op = prob.op(pas, "implicit")
    for _ in range(reps):
        op()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
