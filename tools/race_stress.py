#!/usr/bin/env python
"""Race / bounds stress of the 2D cell-map kernels (the pool has no
compute-sanitizer: SURVEY §5's racecheck/synccheck evidence is gathered this
way instead).

  HERMB200_LIB=build_var/debug/libhermb200.so python tools/race_stress.py --out a.npz
  python tools/race_stress.py --compare default.npz a.npz b.npz

The debug build (tools/build_variant.sh debug -DHW_CM_DEBUG=1) poisons every
ring slot with NaN between its consumption and its refill, sleeps a random
span before every producer stage and consumer chunk (so the mbarrier
handoffs, the dynamic tile claims and programmatic dependent launch see
orderings the product build rarely produces) and traps on out-of-window
global reads / output cells.  The kernels are deterministic (each output is a
fixed sum regardless of which CTA computes its tile), so every run — default
or debug, any timing — must give the same bits, with no NaN.
"""

import argparse
import hashlib
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = [("diss", m, n, False) for m, n in ((2, 400), (3, 384), (4, 512), (5, 320), (6, 256), (7, 200), (8, 160))] + \
          [("cons", m, n, True) for m, n in ((3, 300), (4, 300), (5, 256), (6, 160), (8, 128))] + \
          [("boot", 4, 200, True), ("boot", 6, 120, False), ("cons", 5, 200, False)]


def run(steps):
    import numpy as np
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import cons2d_into, diss2d_into

    out = {}
    for sch, m, n, walls in CONFIGS:
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, not walls)
        bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0", 0.2, -0.1),
                               hb.BoundarySpec("neumann0", "neumann0")) if walls else hb.BoundarySpec2D()
        cfg = hb.SchemeConfig(m=m, lam=0.9)
        g = torch.Generator(device="cpu").manual_seed(1000 * m + n)

        def rnd(par, k):
            shp = (grid.axis(0).n_nodes(par), grid.axis(1).n_nodes(par), k + 1, k + 1)
            return torch.randn(shp, generator=g, dtype=torch.float64).cuda()

        if sch == "diss":
            bufs = {hb.PRIMAL: (rnd(hb.PRIMAL, m), rnd(hb.PRIMAL, m - 1)),
                    hb.DUAL: (rnd(hb.DUAL, m), rnd(hb.DUAL, m - 1))}
            par = hb.PRIMAL
            for _ in range(steps):
                diss2d_into(*bufs[par], *bufs[hb.flip(par)], grid, par, m, cfg, bc)
                par = hb.flip(par)
            res = torch.cat([bufs[par][0].flatten(), bufs[par][1].flatten()])
        elif sch == "cons":
            lv = {hb.PRIMAL: rnd(hb.PRIMAL, m), hb.DUAL: rnd(hb.DUAL, m)}
            par = hb.PRIMAL
            for _ in range(steps):
                cons2d_into(lv[par], lv[hb.flip(par)], lv[hb.flip(par)], grid, par, m, cfg, bc)
                par = hb.flip(par)
            res = torch.cat([lv[hb.PRIMAL].flatten(), lv[hb.DUAL].flatten()])
        else:
            st = hb.bootstrap_first_half(hb.Field2D(grid, hb.PRIMAL, 0.0, rnd(hb.PRIMAL, m)),
                                         hb.Field2D(grid, hb.PRIMAL, 0.0, rnd(hb.PRIMAL, m)), cfg, bc)
            res = st.current.values.flatten()
        torch.cuda.synchronize()
        a = res.cpu().numpy()
        key = f"{sch}_m{m}_n{n}{'_walls' if walls else ''}"
        out[key] = a
        print(f"{key}: nan={int(np.isnan(a).sum())} sha={hashlib.sha1(a.tobytes()).hexdigest()[:12]}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--compare", nargs="+")
    args = ap.parse_args()
    import numpy as np

    if args.compare:
        ref = dict(np.load(args.compare[0]))
        bad = 0
        for other in args.compare[1:]:
            o = dict(np.load(other))
            for k, v in ref.items():
                same = np.array_equal(v, o[k]) and not np.isnan(o[k]).any()
                bad += not same
                print(f"{os.path.basename(other)} {k}: {'bitwise equal' if same else 'DIFFERS'}")
        print("race_stress:", "PASS" if bad == 0 else f"FAIL ({bad})")
        sys.exit(1 if bad else 0)
    res = run(args.steps)
    np.savez(args.out, **res)
    print("lib:", os.environ.get("HERMB200_LIB", "default"), "saved", args.out, math.fsum(len(v) for v in res.values()))


if __name__ == "__main__":
    main()
