#!/usr/bin/env python
"""PCIe copy rates on this box (pinned host <-> HBM): H2D alone, D2H alone,
both at once on two streams, and the chunked e2e step's phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    nb = 344 * 2**20
    h_in = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True)
    d_a = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
    d_b = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d_a.copy_(h_in, non_blocking=True)
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()

    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    t_both = timed(both)
    print(f"H2D {nb / t_h2d / 1e9:.1f} GB/s, D2H {nb / t_d2h / 1e9:.1f} GB/s, "
          f"concurrent {2 * nb / t_both / 1e9:.1f} GB/s total ({t_both * 1e3:.2f} ms for {nb / 2**20:.0f} MiB each way)")
    # pageable numpy source
    import numpy as np

    a = np.ones(nb // 8)
    t_pg = timed(lambda: d_a.copy_(torch.from_numpy(a), non_blocking=True))
    print(f"H2D from pageable numpy {nb / t_pg / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
