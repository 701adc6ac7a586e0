"""fp64 convolution throughput (AlexNet conv2-5 shapes at a reduced batch),
fwd / bwd-data / bwd-filter, algorithmic FLOP/s.

    python tools/bench_f64.py [N]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1410_0759_b200 as dp  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    for (name, c, h, k, r, u, pad) in bench.ALEXNET:
        p = bench.out_extent(h, r, u, pad)
        fl = bench.layer_flops(n, c, h, k, r, u, pad)
        x = dp.TensorView(dp.make_desc(n, c, h, h, elem_type="f64"),
                          torch.rand(n * c * h * h, dtype=torch.float64, device="cuda") - 0.5)
        f = dp.FilterView(dp.make_filter_desc(k, c, r, r, elem_type="f64"),
                          torch.rand(k * c * r * r, dtype=torch.float64, device="cuda") - 0.5)
        y = dp.empty_view(dp.make_desc(n, k, p, p, elem_type="f64"), device="cuda")
        dy = dp.TensorView(dp.make_desc(n, k, p, p, elem_type="f64"),
                           torch.rand(n * k * p * p, dtype=torch.float64, device="cuda") - 0.5)
        dx = dp.empty_view(dp.make_desc(n, c, h, h, elem_type="f64"), device="cuda")
        df = dp.FilterView(dp.make_filter_desc(k, c, r, r, elem_type="f64"),
                           torch.empty(k * c * r * r, dtype=torch.float64, device="cuda"))
        cd = dp.ConvDesc(u, u, pad, pad)
        ops = {"fwd": lambda: dp.conv_forward(x, f, cd, "implicit", y),
               "bwd_data": lambda: dp.conv_backward_data(dy, f, cd, "implicit", dx),
               "bwd_filter": lambda: dp.conv_backward_filter(dy, x, cd, "implicit", df)}
        for pas, op in ops.items():
            op()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                op()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 3
            print(f"{name}.{pas} N={n} f64: {ms:8.3f} ms  {fl / (ms / 1e3) / 1e12:6.2f} TFLOP/s",
                  flush=True)


if __name__ == "__main__":
    main()
