#!/usr/bin/env python
"""Pinned host <-> device copy bandwidth on this box (1 GiB copies, H2D alone,
D2H alone, both directions at once): the floor under bench.py's e2e line,
which moves every layer's x / y over PCIe."""
import time

import torch


def main():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(up):
                    d.copy_(h, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(down):
                    h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(mode, round(5 * n / dt / 1e9, 1), "GB/s per direction")


if __name__ == "__main__":
    main()
