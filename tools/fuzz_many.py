"""Large one-off parity fuzz (tests/test_gpu_fuzz.py geometry generator,
more seeds): prints every failing case.

    python tools/fuzz_many.py [count] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # the oracle package before tests/ (conftest order)
sys.path.insert(1, os.path.join(ROOT, "tests"))

from test_gpu_fuzz import shapes  # noqa: E402
from test_gpu_tc_paths import TOL, run_case  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    bad = 0
    worst = 0.0
    for i, shp in enumerate(shapes(seed, count)):
        mode = "convolution" if i % 2 == 0 else "cross_correlation"
        lay = "nhwc" if i % 3 == 0 else "nchw"
        errs = run_case(shp, mode=mode, layout_in=lay, accumulate=(i % 5 == 2), seed=i)
        worst = max(worst, max(errs.values()))
        if not all(e <= TOL for e in errs.values()):
            bad += 1
            print("FAIL", shp, mode, lay, errs, flush=True)
    print(f"{count} cases, {bad} failures, worst normalised error {worst:.2e}", flush=True)


if __name__ == "__main__":
    main()
