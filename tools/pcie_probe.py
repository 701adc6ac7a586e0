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


def multi():
    """H2D split over k streams (do several copy engines help one direction?)."""
    n = 512 * 1024 * 1024
    h = torch.empty(n // 4, pin_memory=True)
    d = torch.empty(n // 4, device="cuda")
    for k in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(k)]
        part = (n // 4) // k
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        print(f"H2D over {k} streams: {n / dt / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__" and len(__import__("sys").argv) > 1:
    multi()
