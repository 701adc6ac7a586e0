"""Backward-filter time vs the pixels-per-split cap (DNNP_WG_CHAIN) on the
AlexNet layers at N=128.

    python tools/wg_chain.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    for lay in bc.load_suite("alexnet"):
        prob = bc._Problem(lay, "f32", 2014, 0)
        ref = bc._reference(lay, prob, "bwd_filter") if lay.name in ("conv1", "conv2") else None
        for chain in ("1000000000", "32768", "16384", "8192", "4096"):
            os.environ["DNNP_WG_CHAIN"] = chain
            t = bc._time(prob.op("bwd_filter", "implicit"), 7)
            e = ""
            if ref is not None:
                prob.op("bwd_filter", "implicit")()
                torch.cuda.synchronize()
                e = f"err {float((prob.df.buf.double() - ref).abs().max() / ref.abs().max()):.2e}"
            print(f"{lay.name} chain {chain:>10}: {t * 1e6:7.1f} us {lay.flops() / t / 1e12:6.1f} TF/s {e}",
                  flush=True)


if __name__ == "__main__":
    main()
