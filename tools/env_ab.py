"""Time one AlexNet layer pass (N=128) under environment variants.

    python tools/env_ab.py conv1 fwd,bwd_data "" DNNP_TC_BLOCK_S2D=1 ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    name, passes = sys.argv[1], sys.argv[2].split(",")
    variants = sys.argv[3:] or [""]
    lay = {l.name: l for l in bc.load_suite("alexnet")}[name]
    prob = bc._Problem(lay, "f32", 2014, 0)
    refs = {}
    for var in variants:
        kv = dict(x.split("=", 1) for x in var.split() if x)
        old = {k: os.environ.get(k) for k in kv}
        os.environ.update(kv)
        for pas in passes:
            op = prob.op(pas, "implicit")
            t = bc._time(op, 9)
            dp.kernel_timing(1)
            op()
            torch.cuda.synchronize()
            kt = sum(m for m, _ in dp.kernel_times()) / 1e3
            dp.kernel_timing(0)
            out = prob.result(pas).clone()
            if pas not in refs:
                refs[pas] = out
            d = float((out - refs[pas]).abs().max() / refs[pas].abs().max())
            print(f"{name}.{pas:<10} [{var or 'default':<28}] op {t * 1e6:7.1f} us  gemm {kt * 1e6:7.1f} us "
                  f"({lay.flops() / kt / 1e12:6.1f} TF/s)  diff {d:.1e}", flush=True)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


if __name__ == "__main__":
    main()
