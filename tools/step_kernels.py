"""One AlexNet training step (N=128, the bench's inputs and call sequence)
between cudaProfilerStart / Stop, for a per-kernel launch list:

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum --csv python tools/step_kernels.py > step.csv
    python tools/step_kernels.py --summary step.csv
"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
    agg = {}
    for d in per.values():
        name = d["name"].split("(")[0].replace("void ", "").split("::")[-1]
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0) / 1e3
        a[2] += (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{len(per)} kernels, {tot / 1e3:.1f} us serialised")
    for name, (n, us, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{us:8.1f} us {100 * us * 1e3 / tot:5.1f}%  x{n:<3d} {mb:8.1f} MB  {mb / us if us else 0:5.2f} TB/s  {name}")


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--summary":
        return summary(sys.argv[2])
    import torch
    import bench
    import paper_1410_0759_b200 as dp
    dev = torch.device("cuda", 0)
    layers = bench.make_inputs(int(os.environ.get("STEP_N", "128")), dev, torch)
    bench.build_views(dp, layers, torch, dev)
    for _ in range(2):
        bench.run_step(dp, layers, torch)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    bench.run_step(dp, layers, torch)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
