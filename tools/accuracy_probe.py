"""Normalised error (max|err| / max|ref|) of the fp32 tensor-core path against
the fp64 path for every pass of the bundled suites, and for the wgrad
reduction-chain cap (DNNP_WG_CHAIN) on table2 layer1.

    python tools/accuracy_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def errs(layer):
    prob = bc._Problem(layer, "f32", 2014, 0)
    out = {}
    for pas in bc.PASSES:
        ref = bc._reference(layer, prob, pas)
        prob.op(pas, "implicit")()
        torch.cuda.synchronize()
        out[pas] = float((prob.result(pas).double() - ref).abs().max() / ref.abs().max())
    return out


def main():
    for suite in ("table2", "alexnet", "overfeat_vgg"):
        for base in bc.load_suite(suite):
            lay = bc.replace(base, n=16)
            e = errs(lay)
            print(f"{suite:>12} {lay.name:<10} " + "  ".join(f"{k} {v:.2e}" for k, v in e.items()),
                  flush=True)
    lay = bc.replace(bc.load_suite("table2")[0], n=16)
    for chain in ("1000000000", "65536", "16384", "8192", "2048"):
        os.environ["DNNP_WG_CHAIN"] = chain
        prob = bc._Problem(lay, "f32", 2014, 0)
        ref = bc._reference(lay, prob, "bwd_filter")
        t = bc._time(prob.op("bwd_filter", "implicit"), 5)
        prob.op("bwd_filter", "implicit")()
        torch.cuda.synchronize()
        e = float((prob.result("bwd_filter").double() - ref).abs().max() / ref.abs().max())
        print(f"layer1 N=16 bwd_filter chain {chain:>10}: err {e:.2e}  {t * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
