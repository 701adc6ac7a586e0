"""Can a bench step (15 library calls) be captured into a CUDA graph and
replayed?  Compares outputs with eager calls and times both.

    python tools/graph_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(128, dev, torch)
    bench.build_views(dp, layers, torch, dev)
    for _ in range(3):
        bench.run_step(dp, layers, torch)
    torch.cuda.synchronize()
    ref = [(L["yv"].buf.clone(), L["dxv"].buf.clone(), L["dfv"].buf.clone()) for L in layers]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            bench.run_step(dp, layers, torch)
    torch.cuda.synchronize()
    for L in layers:
        L["yv"].buf.zero_(); L["dxv"].buf.zero_(); L["dfv"].buf.zero_()
    g.replay()
    torch.cuda.synchronize()
    for L, (y, dx, df) in zip(layers, ref):
        print(L["name"], "max|diff| y", float((L["yv"].buf - y).abs().max()), "dx",
              float((L["dxv"].buf - dx).abs().max()), "df", float((L["dfv"].buf - df).abs().max()),
              flush=True)
    flush = torch.empty(64 * 1024 * 1024, device=dev)
    for name, fn in (("eager", lambda: bench.run_step(dp, layers, torch)), ("graph", g.replay)):
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{name}: median {ts[5]:.3f} ms/step  min {ts[0]:.3f}", flush=True)


if __name__ == "__main__":
    main()
