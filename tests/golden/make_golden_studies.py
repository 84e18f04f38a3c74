"""Golden refinement studies / conservation traces produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_studies.py

Runs hermwave.driver (read-only from /root/reference/pkg/src) on small
configurations of each experiment and stores the per-level errors, fitted
rates and energy deltas in tests/golden/studies.npz (numpy version stamped).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import hermwave as hw  # noqa: E402
from hermwave.driver import make_config, run_experiment  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# name -> (experiment, overrides); kept small so the reference finishes in seconds
STUDIES = {
    "pw2d_diss_m3": ("planewave2d", dict(m=3, lam=0.9, levels=4, n0=6)),
    "pw2d_cons_m2_exact": ("planewave2d", dict(scheme="conservative", m=2, lam=0.9, levels=4, n0=6)),
    "pw2d_cons_m2_boot": ("planewave2d", dict(scheme="conservative", m=2, lam=0.7, levels=3, n0=6,
                                              init="bootstrap")),
    "g1d_diss_m3": ("gaussian1d", dict(m=3, levels=4, n0=10)),
    "g1d_cons_m2_boot": ("gaussian1d", dict(scheme="conservative", m=2, levels=4, n0=12, init="bootstrap",
                                            boundary="neumann0")),
    "g1d_diss_m2_per": ("gaussian1d", dict(m=2, levels=3, n0=12, boundary="periodic", lam=0.9)),
    "c1d_smooth_m2": ("conserve1d", dict(m=2, steps=300, sample_every=100)),
    # the driver's default ladders: observed orders in the asymptotic range
    "pw2d_default_m4": ("planewave2d", dict(m=4)),
    "g1d_default_m3": ("gaussian1d", dict(m=3)),
    "c1d_random_m3": ("conserve1d", dict(m=3, steps=200, sample_every=50, mode="random", seed=7)),
}


def main():
    arrays = {}
    for name, (exp, over) in STUDIES.items():
        cfg = make_config(exp, None, over)
        res = run_experiment(cfg)
        if exp == "conserve1d":
            steps, times, deltas, e0 = res
            arrays[f"{name}/steps"] = steps
            arrays[f"{name}/times"] = times
            arrays[f"{name}/deltas"] = deltas
            arrays[f"{name}/e0"] = np.array(e0)
        else:
            arrays[f"{name}/ns"] = res.ns
            arrays[f"{name}/err_u"] = res.err_u
            if res.err_dux is not None:
                arrays[f"{name}/err_dux"] = res.err_dux
                arrays[f"{name}/err_v"] = res.err_v
            if len(res.ns) >= 3:
                arrays[f"{name}/rate"] = np.array(res.rate())
        print(name, "done")
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "studies.npz")
    np.savez_compressed(path, **arrays, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
