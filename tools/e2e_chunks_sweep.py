"""Chunk-count sweep of the host-array pipelined half step (C2, m = 4, 1024^2):
pinned and pageable numpy inputs, stepping._diss2d_host_pipelined(nchunks=...)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05246_b200 as hb  # noqa: E402
from paper_1802_05246_b200 import stepping as S  # noqa: E402

m, n = 4, 1024
grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
cfg = hb.SchemeConfig(m=m, lam=0.9)
bc = hb.BoundarySpec2D()
rng = np.random.default_rng(0)
u0, v0 = rng.standard_normal((n, n, m + 1, m + 1)), rng.standard_normal((n, n, m, m))
up, vp = torch.from_numpy(u0).pin_memory().numpy(), torch.from_numpy(v0).pin_memory().numpy()
dof = n * n * ((m + 1) ** 2 + m * m)
for rep in range(2):
    for name, (a, b) in (("pinned", (up, vp)), ("pageable", (u0, v0))):
        for nc in (8, 16, 24, 32, 48):
            for _ in range(2):
                S._diss2d_host_pipelined(a, b, grid, hb.PRIMAL, m, cfg, bc, nchunks=nc)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(5):
                S._diss2d_host_pipelined(a, b, grid, hb.PRIMAL, m, cfg, bc, nchunks=nc)
            dt = (time.perf_counter() - t) / 5
            print(f"{name} nchunks={nc}: {dof / dt / 1e9:.3f} GDOF/s ({dt * 1e3:.2f} ms)", flush=True)
