"""Stream-K check: every AlexNet layer's fwd / bwd-data at the bench size with
and without the stream-K last wave (DNNP_TC_NO_SK), normalised difference
and timing of both.

    python tools/sk_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def timed(op, reps=10):
    for _ in range(2):
        op()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        op()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    for L in layers:
        for pas in ("fwd", "bwd_data"):
            if pas == "fwd":
                op = lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"])
                out = L["yv"].buf
            else:
                op = lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"])
                out = L["dxv"].buf
            os.environ.pop("DNNP_TC_SK", None)
            t_dp = timed(op)
            op()
            torch.cuda.synchronize()
            ref = out.clone()
            os.environ["DNNP_TC_SK"] = "1"
            t_sk = timed(op)
            op()
            torch.cuda.synchronize()
            os.environ.pop("DNNP_TC_SK", None)
            d = (out - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
            print(f"{L['name']}.{pas}: no-SK {t_dp:7.1f} us  SK {t_sk:7.1f} us  max|diff|/max|ref| {d:.2e}",
                  flush=True)


if __name__ == "__main__":
    main()
