"""Where a small-minibatch call's time goes (of_conv3 N=1..16): host time per
call (no sync), pipelined device time per call (50 back-to-back calls), and
the synchronous single-call time the bench CLI reports.

    python tools/small_n_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    base = {l.name: l for l in bc.load_suite("overfeat_vgg")}["of_conv3"]
    for n in (1, 4, 16, 128):
        lay = bc.replace(base, n=n)
        prob = bc._Problem(lay, "f32", 2014, 0)
        for pas in ("fwd", "bwd_data", "bwd_filter"):
            op = prob.op(pas, "implicit")
            for _ in range(5):
                op()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(50):
                op()
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            single = bc._time(op, 9)
            print(f"N={n:<4} {pas:<10} host {1e6 * (t1 - t0) / 50:6.1f} us/call  pipelined "
                  f"{1e6 * (t2 - t0) / 50:7.1f} us/call  single {single * 1e6:7.1f} us", flush=True)


if __name__ == "__main__":
    main()
