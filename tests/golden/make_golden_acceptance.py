"""The reference's acceptance criteria 1-3 (refinement rates), as the
REFERENCE itself measures them (tests/test_acceptance.py:53-100 of hermwave).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_acceptance.py

Runs hermwave.driver's default ladders for gaussian1d (dissipative m=1..4,
conservative m=1..3) and planewave2d (both schemes, m=1..3) at lambda 0.8 and
1.0 and stores the per-level errors and fitted rates in
tests/golden/acceptance.npz (numpy version stamped).
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import replace

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import hermwave as hw  # noqa: E402
from hermwave.driver import default_config, run_gaussian_1d, run_planewave_2d  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = ([("gaussian1d", "dissipative", m, lam) for m in (1, 2, 3, 4) for lam in (0.8, 1.0)]
         + [("gaussian1d", "conservative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)]
         + [("planewave2d", "dissipative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)]
         + [("planewave2d", "conservative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)])


def key(exp, scheme, m, lam):
    return f"{exp}/{scheme[:4]}/m{m}/lam{lam}"


def main():
    A = {}
    for exp, scheme, m, lam in CASES:
        t0 = time.time()
        cfg = replace(default_config(exp), scheme=scheme, m=m, lam=lam).validate()
        rep = run_gaussian_1d(cfg) if exp == "gaussian1d" else run_planewave_2d(cfg)
        k = key(exp, scheme, m, lam)
        A[f"{k}/ns"], A[f"{k}/err_u"], A[f"{k}/rate"] = rep.ns, rep.err_u, np.array(rep.rate())
        print(k, f"rate {rep.rate():.3f}", f"{time.time() - t0:.1f}s", flush=True)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "acceptance.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
