"""Effective SM clock under a tensor-core kernel: CTA-0 cycles of one conv5
forward (DNNP_TC_TRACE, clock64) against its CUDA-event time inside a
back-to-back loop (GPU never idle), plus nvidia-smi's SM clock sampled
while the loop runs.

    python tools/clock_probe.py
"""
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1410_0759_b200 import bench_cli as bc  # noqa: E402


def main():
    lay = {l.name: l for l in bc.load_suite("alexnet")}["conv5"]
    prob = bc._Problem(lay, "f32", 2014, 0)
    op = prob.op("fwd", "implicit")
    for _ in range(3):
        op()
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                samples.append(out)
            except Exception:
                pass

    th = threading.Thread(target=sample)
    th.start()
    reps = 400
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        op()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    per = a.elapsed_time(b) / reps * 1e3
    print(f"conv5 fwd (pack + GEMM) back-to-back: {per:.1f} us per call; nvidia-smi clocks,power: {samples[:6]}",
          flush=True)
    os.environ["DNNP_TC_TRACE"] = "1"
    op()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
