"""A/B of the tile choice for small-batch forward (OverFeat conv3 / conv2):
device time per call (20 calls replayed in a graph) for each forced (BN, NC,
split) against the planner's default.
    python tools/small_n_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402


def dev_us(op, reps=20):
    for _ in range(3):
        op()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                op()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def setenv(**kv):
    for k in ("DNNP_TC_BN", "DNNP_TC_NC", "DNNP_TC_SK", "DNNP_TC_NO_SK", "DNNP_TC_NO_SPLIT",
              "DNNP_TC_NO_VBLOCK", "DNNP_TC_NO_BLOCK"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in kv.items()})
    dp._lib.reload_tuning()


for name, c, h, k, r, pad in (("of_conv3", 256, 12, 512, 3, 1), ("of_conv2", 96, 24, 256, 5, 2)):
    for n in (4, 16, 32):
        x = dp.TensorView(dp.make_desc(n, c, h, h), torch.rand(n * c * h * h, device="cuda"))
        f = dp.FilterView(dp.make_filter_desc(k, c, r, r), torch.rand(k * c * r * r, device="cuda"))
        y = dp.empty_view(dp.make_desc(n, k, h, h), device="cuda")
        cd = dp.ConvDesc(1, 1, pad, pad)
        op = lambda: dp.conv_forward(x, f, cd, "implicit", y)  # noqa: E731
        res = []
        for cfg in ({}, {"DNNP_TC_NO_SPLIT": 1},
                    {"DNNP_TC_BN": 64, "DNNP_TC_NC": 1}, {"DNNP_TC_BN": 128, "DNNP_TC_NC": 1},
                    {"DNNP_TC_BN": 128, "DNNP_TC_NC": 2}, {"DNNP_TC_BN": 256, "DNNP_TC_NC": 1},
                    {"DNNP_TC_BN": 256, "DNNP_TC_NC": 2}, {"DNNP_TC_BN": 256, "DNNP_TC_NC": 2, "DNNP_TC_SK": 1},
                    {"DNNP_TC_BN": 128, "DNNP_TC_NC": 2, "DNNP_TC_SK": 1}):
            setenv(**cfg)
            res.append((dev_us(op), cfg))
        setenv()
        best = min(res, key=lambda t: t[0])
        print(f"{name} N={n}: default {res[0][0]:.1f} us; best {best[0]:.1f} us {best[1]}; all " +
              " | ".join(f"{t:.1f}" for t, _ in res), flush=True)
