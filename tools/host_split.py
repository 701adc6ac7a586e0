"""Host cost of one convolution call split into the Python layer and the C
ABI (raw ctypes call with prebuilt arguments), GPU work skipped
(DNNP_TC_SKIP=6: kernels launch but do no loads / MMAs), of_conv3 N=1.

    python tools/host_split.py
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1410_0759_b200 as dp  # noqa: E402
from paper_1410_0759_b200 import _lib, bench_cli as bc  # noqa: E402
from paper_1410_0759_b200.conv import _ENGINE_CODE, as_engine  # noqa: E402
from paper_1410_0759_b200.tensor import scalar_ptr  # noqa: E402


def per_call(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / n


def main():
    lay = bc.replace({l.name: l for l in bc.load_suite("overfeat_vgg")}["of_conv3"], n=1)
    prob = bc._Problem(lay, "f32", 2014, 0)
    x, f, y, cd = prob.x, prob.f, prob.y, prob.cd
    a_keep, a = scalar_ptr(1.0, y.desc.dtype)
    b_keep, b = scalar_ptr(0.0, y.desc.dtype)
    L = _lib.lib()
    h = _lib.handle()
    args = (h, a, x.desc.c_desc(), x.ptr, f.desc.c_desc(), f.ptr, cd.c_desc(),
            _ENGINE_CODE[as_engine("implicit")], b, y.desc.c_desc(), y.ptr)
    _lib.set_stream(torch.cuda.current_stream().cuda_stream)
    for skip in ("0", "6"):
        os.environ["DNNP_TC_SKIP"] = skip
        full = per_call(lambda: dp.conv_forward(x, f, cd, "implicit", y))
        raw = per_call(lambda: L.dnnp_convolution_forward(*args))
        print(f"skip={skip}: python API {full:6.1f} us/call, raw C ABI {raw:6.1f} us/call", flush=True)
    os.environ["DNNP_TC_SKIP"] = "6"
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        dp.conv_forward(x, f, cd, "implicit", y)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(10)


if __name__ == "__main__":
    main()
