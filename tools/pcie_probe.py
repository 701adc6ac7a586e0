"""Pinned host <-> device copy rates on this box: H2D alone, D2H alone, and
both directions at once on two streams (is the link full duplex?).

    python tools/pcie_probe.py
"""
import time

import torch


def main():
    n = 512 * 1024 * 1024
    h1 = torch.empty(n // 4, pin_memory=True)
    h2 = torch.empty(n // 4, pin_memory=True)
    d1 = torch.empty(n // 4, device="cuda")
    d2 = torch.empty(n // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, both in (("H2D", 0), ("D2H", 1), ("both", 2)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            if both in (0, 2):
                with torch.cuda.stream(s1):
                    d1.copy_(h1, non_blocking=True)
            if both in (1, 2):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        byt = n * (2 if both == 2 else 1)
        print(f"{name}: {byt / dt / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
