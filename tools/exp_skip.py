"""Experiment: time one layer pass with parts of the TMA conv kernel disabled
(DNNP_TC_SKIP: 1 = no A loads, 2 = no loads, 4 = no MMAs) to find the
limiter.  Results are garbage numerically; only the timing matters.

    python tools/exp_skip.py conv1 fwd
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    layers_sel = sys.argv[1].split(",") if len(sys.argv) > 1 else ["conv1"]
    passes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fwd"]
    skips = [int(s) for s in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "4", "6"])]
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    for L in layers:
        if L["name"] not in layers_sel:
            continue
        for pas in passes:
            op = {
                "fwd": lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"]),
                "bwd_data": lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"]),
                "bwd_filter": lambda: dp.conv_backward_filter(L["dyv"], L["xv"], L["cd"], "implicit", L["dfv"]),
            }[pas]
            for sk in skips:
                os.environ["DNNP_TC_SKIP"] = str(sk % 8)
                os.environ["DNNP_TC_SPIN"] = str(sk // 8)
                for _ in range(3):
                    op()
                torch.cuda.synchronize()
                ts = []
                for _ in range(10):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record()
                    op()
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                ts.sort()
                print(f"{L['name']}.{pas} skip={sk}: median {ts[5]*1e3:.1f} us  min {ts[0]*1e3:.1f} us",
                      flush=True)
    os.environ.pop("DNNP_TC_SKIP", None)


if __name__ == "__main__":
    main()
