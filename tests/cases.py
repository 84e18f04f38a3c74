"""Case tables shared by the oracle and GPU parity tests (mirror of
tests/golden/make_golden.py, which generated the fixtures from the reference)."""

PRIMAL, DUAL = "primal", "dual"

CASES_2D = [
    ("p_m1", 1, 6, 5, True, PRIMAL, None, None, 0.9, 1.0, None, 1),
    ("p_m2", 2, 6, 7, True, DUAL, None, None, 0.9, 1.0, None, 1),
    ("p_m3", 3, 5, 6, True, PRIMAL, None, None, 0.7, 1.3, None, 1),
    ("p_m4", 4, 7, 6, True, PRIMAL, None, None, 0.9, 1.0, None, 1),
    ("p_m5", 5, 5, 5, True, DUAL, None, None, 0.9, 1.0, None, 1),
    ("p_m6", 6, 4, 5, True, PRIMAL, None, None, 0.9, 1.0, None, 1),
    ("p_m7", 7, 4, 4, True, PRIMAL, None, None, 0.8, 1.0, None, 1),
    ("p_m8", 8, 4, 5, True, DUAL, None, None, 0.9, 1.0, None, 1),
    ("p_m4_cap", 4, 6, 6, True, PRIMAL, None, None, 0.9, 1.0, 5, 1),
    ("p_m4_rect", 4, 6, 8, True, PRIMAL, None, None, 0.9, 1.0, None, 1),
    ("p_m4_multi", 4, 10, 9, True, PRIMAL, None, None, 0.9, 1.0, None, 6),
    ("w_m3_primal", 3, 6, 5, False, PRIMAL, ("dirichlet0", "neumann0", 0.3, 0.0),
     ("neumann0", "dirichlet0", 0.0, -0.4), 0.9, 1.0, None, 1),
    ("w_m3_dual", 3, 6, 5, False, DUAL, ("dirichlet0", "neumann0", 0.3, 0.0),
     ("neumann0", "dirichlet0", 0.0, -0.4), 0.9, 1.0, None, 1),
    ("w_m5_dual", 5, 5, 6, False, DUAL, ("dirichlet0", "dirichlet0", 0.0, 0.0),
     ("neumann0", "neumann0", 0.0, 0.0), 0.9, 1.0, None, 1),
    ("w_m4_multi", 4, 8, 7, False, PRIMAL, ("dirichlet0", "dirichlet0", 0.2, -0.1),
     ("dirichlet0", "neumann0", 0.5, 0.0), 0.9, 1.0, None, 5),
    ("w_m8_dual", 8, 4, 4, False, DUAL, ("neumann0", "dirichlet0", 0.0, 0.7),
     ("dirichlet0", "neumann0", -0.2, 0.0), 0.9, 1.0, None, 1),
]

CASES_1D = [
    ("p_m1", 1, 7, True, PRIMAL, None, 0.9, 1.0, None, 1, False),
    ("p_m3", 3, 9, True, DUAL, None, 0.9, 1.0, None, 1, False),
    ("p_m3_multi", 3, 12, True, PRIMAL, None, 0.9, 1.0, None, 20, False),
    ("p_m6", 6, 8, True, PRIMAL, None, 0.5, 2.0, None, 1, False),
    ("p_m8_cap", 8, 6, True, DUAL, None, 0.9, 1.0, 7, 1, False),
    ("p_m12", 12, 5, True, PRIMAL, None, 0.9, 1.0, None, 1, False),
    ("w_m2_primal", 2, 7, False, PRIMAL, ("dirichlet0", "neumann0", 0.25, 0.0), 0.8, 1.0, None, 1, False),
    ("w_m4_dual", 4, 7, False, DUAL, ("neumann0", "dirichlet0", 0.0, -0.6), 0.8, 1.0, None, 1, False),
    ("w_m3_multi", 3, 10, False, PRIMAL, ("dirichlet0", "dirichlet0", 0.1, 0.2), 0.9, 1.0, None, 9, False),
    ("f_m3", 3, 9, True, PRIMAL, None, 0.9, 1.0, None, 2, True),
]

# Grid2D(0.0, 1.0, -0.5, 0.7, nx, ny, periodic) and Grid1D(-0.4, 1.1, n, periodic)
X2D = (0.0, 1.0, -0.5, 0.7)
X1D = (-0.4, 1.1)

PERIODIC_BC = ("periodic", "periodic", 0.0, 0.0)

# BASELINE config C3's setup (tests/golden/make_golden_c3.py -> c3walls.npz): conservative
# scheme, Dirichlet x / Neumann y walls on the unit square, odd orders from both parities.
# (name, m, n, parity of the current level, steps, kind)
C3_CASES = [
    ("wave_m5_primal", 5, 24, PRIMAL, 8, "wave"),
    ("wave_m5_dual", 5, 24, DUAL, 8, "wave"),
    ("wave_m3_primal", 3, 20, PRIMAL, 8, "wave"),
    ("wave_m3_dual", 3, 16, DUAL, 8, "wave"),
    ("wave_m7_primal", 7, 12, PRIMAL, 8, "wave"),
    ("wave_m7_dual", 7, 12, DUAL, 8, "wave"),
    ("rand_m5_primal", 5, 10, PRIMAL, 8, "rand"),
    ("rand_m5_dual", 5, 10, DUAL, 8, "rand"),
    ("rand_m7_primal", 7, 8, PRIMAL, 6, "rand"),
    ("rand_m7_dual", 7, 8, DUAL, 6, "rand"),
]
C3_LAM = 0.9
C3_WAVE_BC = (("dirichlet0", "dirichlet0", 0.0, 0.0), ("neumann0", "neumann0", 0.0, 0.0))
C3_RAND_BC = (("dirichlet0", "dirichlet0", 0.3, -0.2), ("neumann0", "neumann0", 0.0, 0.0))

# 2D steps at m = 9..12 (tests/golden/make_golden_high2d.py -> high2d.npz):
# (name, m, nx, ny, walls, parity); Grid2D(0, 1, -0.5, 0.7, nx, ny, not walls)
HIGH2D_CASES = [
    ("p_m9", 9, 4, 5, False, PRIMAL),
    ("w_m9_dual", 9, 4, 4, True, DUAL),
    ("p_m10", 10, 4, 4, False, DUAL),
    ("w_m11_primal", 11, 3, 4, True, PRIMAL),
    ("p_m12", 12, 4, 3, False, PRIMAL),
    ("w_m12_dual", 12, 3, 3, True, DUAL),
]


def forcing_fn(l, s, x, t):
    import numpy as np

    return np.cos(x + 0.3 * l - 0.2 * s) * (1.0 + 0.1 * t)


def exact2d(x, y):
    import numpy as np

    return np.sin(2.0 * x + 0.3) * np.cos(1.5 * y - 0.2)
