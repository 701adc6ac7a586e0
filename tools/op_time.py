"""Per-op time of the AlexNet benchmark layers (N=128, the bench's inputs):
every op (packs + GEMM + reductions of one API call) captured 10x into a CUDA
graph and replayed back to back; CUDA events around the replay.

    python tools/op_time.py [layer ...]        # default: all five layers
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def graph_ms(op, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        op()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                op()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (3 * reps)


def main():
    want = sys.argv[1:] or [a[0] for a in bench.ALEXNET]
    n = int(os.environ.get("OP_N", "128"))
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(n, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    for L in layers:
        if L["name"] not in want:
            continue
        fl = bench.layer_flops(n, L["c"], L["h"], L["k"], L["r"], L["u"], L["pad"])
        ops = {
            "fwd": lambda: dp.conv_forward(L["xv"], L["fv"], L["cd"], "implicit", L["yv"]),
            "bwd_data": lambda: dp.conv_backward_data(L["dyv"], L["fv"], L["cd"], "implicit", L["dxv"]),
            "bwd_filter": lambda: dp.conv_backward_filter(L["dyv"], L["xv"], L["cd"], "implicit",
                                                          L["dfv"]),
        }
        for pas, op in ops.items():
            ms = graph_ms(op)
            print(f"{L['name']}.{pas:10s} {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
