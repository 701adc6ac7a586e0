"""Error of one long forward reduction (C*R*S = 25088) vs the segment cap
DNNP_TC_CHAIN, and its cost, at an N where time is measurable.

    python tools/chain_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    for lay in (bc.Layer("c512k7", 32, 512, 14, 14, 512, 7, 7, 1, 1, 3, 3),
                bc.Layer("table2_l3", 128, 128, 32, 32, 128, 9, 9)):
        prob = bc._Problem(lay, "f32", 2014, 0)
        refs = {pas: bc._reference(lay, prob, pas) for pas in ("fwd", "bwd_data")}
        for chain in ("1000000000", "16384", "8192", "4096"):
            os.environ["DNNP_TC_CHAIN"] = chain
            for pas in ("fwd", "bwd_data"):
                t = bc._time(prob.op(pas, "implicit"), 5)
                prob.op(pas, "implicit")()
                torch.cuda.synchronize()
                ref = refs[pas]
                e = float((prob.result(pas).double() - ref).abs().max() / ref.abs().max())
                print(f"{lay.name} {pas:<8} chain {chain:>10}: err {e:.2e}  {t * 1e6:8.1f} us  "
                      f"{lay.flops() / t / 1e12:6.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
