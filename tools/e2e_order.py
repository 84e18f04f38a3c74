"""A/B of the host-array pipelined half step (stepping._diss2d_host_pipelined):
pinned vs pageable inputs, uploads issued first vs launches interleaved, and
optionally an older copy of stepping.py (argv[1]) in the same process."""
import importlib.util
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05246_b200 as hb  # noqa: E402
from paper_1802_05246_b200 import stepping as S  # noqa: E402

variants = [("new", S)]
if len(sys.argv) > 1:
    spec = importlib.util.spec_from_file_location("paper_1802_05246_b200.stepping_old", sys.argv[1])
    old = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(old)
    variants.append(("old", old))
m, n = 4, 1024
grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
cfg = hb.SchemeConfig(m=m, lam=0.9)
bc = hb.BoundarySpec2D()
rng = np.random.default_rng(0)
u0 = rng.standard_normal((n, n, m + 1, m + 1))
v0 = rng.standard_normal((n, n, m, m))
up = torch.from_numpy(u0).pin_memory().numpy()
vp = torch.from_numpy(v0).pin_memory().numpy()
dof = n * n * ((m + 1) ** 2 + m * m)
for rep in range(2):
    for vname, mod in variants:
        for name, (a, b) in (("pinned", (up, vp)), ("pageable", (u0, v0))):
            for il in ((False, True) if vname == "new" else (None,)):
                kw = {} if il is None else {"_interleave": il}
                for _ in range(2):
                    mod._diss2d_host_pipelined(a, b, grid, hb.PRIMAL, m, cfg, bc, **kw)
                torch.cuda.synchronize()
                t = time.perf_counter()
                for _ in range(5):
                    mod._diss2d_host_pipelined(a, b, grid, hb.PRIMAL, m, cfg, bc, **kw)
                dtm = (time.perf_counter() - t) / 5
                tag = "" if il is None else (" interleave" if il else " uploads-first")
                print(f"{vname} {name}{tag}: {dof / dtm / 1e9:.3f} GDOF/s", flush=True)
