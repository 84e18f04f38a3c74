"""CPU oracle for the Hermite hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (hermwave, arXiv 1802.05246,
/root/reference/pkg/src/hermwave), written independently, step for step in
the reference's own operation order so that its outputs match the
reference's bit for bit on this container's numpy/OpenBLAS.  It is pinned by
tests/test_oracle.py against the golden vectors in tests/golden/, which
tests/golden/make_golden.py produced by importing the reference itself.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module — as the checker, never as the product path.
"""

from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import numpy as np

PRIMAL, DUAL = "primal", "dual"


def flip(p):
    return DUAL if p == PRIMAL else PRIMAL


def n_nodes(n, periodic, parity):
    """grid.py:48-51."""
    return n if (periodic or parity == DUAL) else n + 1


def nodes(x_left, h, n, periodic, parity):
    """grid.py:53-55."""
    off = 0.0 if parity == PRIMAL else 0.5
    return x_left + h * (np.arange(n_nodes(n, periodic, parity)) + off)


# ----------------------------------------------------------------- interp.py

def _rational_inverse(rows):
    """Gauss-Jordan over Fractions with partial pivoting (interp.py:33-48)."""
    n = len(rows)
    work = [list(r) + [Fraction(int(i == j)) for j in range(n)] for i, r in enumerate(rows)]
    for c in range(n):
        p = max(range(c, n), key=lambda r: abs(work[r][c]))
        work[c], work[p] = work[p], work[c]
        s = Fraction(1) / work[c][c]
        work[c] = [x * s for x in work[c]]
        for r in range(n):
            f = work[r][c]
            if r != c and f != 0:
                work[r] = [x - f * y for x, y in zip(work[r], work[c])]
    return [r[n:] for r in work]


@lru_cache(maxsize=None)
def hermite_matrix(mu):
    """interp.py:51-75: (2mu+2)^2 map from stacked (left, right) node data to
    cell-centred scaled coefficients, exact then rounded once."""
    n = 2 * mu + 2
    cond = []
    for xi in (Fraction(-1, 2), Fraction(1, 2)):
        for l in range(mu + 1):
            cond.append([Fraction(math.comb(j, l)) * xi ** (j - l) if j >= l else Fraction(0)
                         for j in range(n)])
    inv = _rational_inverse(cond)
    out = np.array([[float(x) for x in r] for r in inv])
    out.setflags(write=False)
    return out


def interp_1d(data):
    """interp.py:78-90: (..., 2, mu+1) -> (..., 2mu+2)."""
    data = np.asarray(data, dtype=float)
    mu = data.shape[-1] - 1
    return data.reshape(data.shape[:-2] + (2 * mu + 2,)) @ hermite_matrix(mu).T


def interp_2d(data):
    """interp.py:93-111: (..., 2, 2, mux+1, muy+1) -> (..., 2mux+2, 2muy+2)."""
    data = np.asarray(data, dtype=float)
    mux, muy = data.shape[-2] - 1, data.shape[-1] - 1
    stacked = np.moveaxis(data, -3, -2)
    stacked = stacked.reshape(stacked.shape[:-4] + (2 * mux + 2, 2 * muy + 2))
    return np.einsum("ai,...ij,bj->...ab", hermite_matrix(mux), stacked, hermite_matrix(muy),
                     optimize=True)


# ----------------------------------------------------------------- boundary.py

def refl_signs(kind, n):
    """boundary.py:56-62."""
    l = np.arange(n)
    return (-1.0) ** (l + 1) if kind == "dirichlet0" else (-1.0) ** l


def ghost_1d(block, kind, value=0.0):
    """boundary.py:65-76."""
    out = np.asarray(block, dtype=float) * refl_signs(kind, np.shape(block)[-1])
    if kind == "dirichlet0" and value != 0.0:
        out = out.copy()
        out[..., 0] += 2.0 * value
    return out


def ghost_2d(block, kind, normal_axis, value=0.0):
    """boundary.py:79-98: reflect only the normal-axis order index."""
    block = np.asarray(block, dtype=float)
    ax = -2 if normal_axis == 0 else -1
    shape = [1, 1]
    shape[ax] = block.shape[ax]
    out = block * refl_signs(kind, block.shape[ax]).reshape(shape)
    if kind == "dirichlet0" and value != 0.0:
        out = out.copy()
        out[..., 0, 0] += 2.0 * value
    return out


def gather(values, axis, coeff_axis, parity, periodic, kinds, vals):
    """boundary.py:101-132: replace `axis` (sources) by (targets, 2) flanking data."""
    v = np.moveaxis(values, axis, 0)
    two_d = v.ndim > 2

    def reflect(block, kind, value):
        if two_d:
            return ghost_2d(block, kind, 0 if coeff_axis == "x" else 1, value)
        return ghost_1d(block, kind, value)

    if periodic:
        if parity == PRIMAL:
            lo, hi = v, np.roll(v, -1, axis=0)
        else:
            lo, hi = np.roll(v, 1, axis=0), v
    elif parity == PRIMAL:
        lo, hi = v[:-1], v[1:]
    else:
        padded = np.concatenate([reflect(v[:1], kinds[0], vals[0]), v,
                                 reflect(v[-1:], kinds[1], vals[1])], axis=0)
        lo, hi = padded[:-1], padded[1:]
    out = np.stack([lo, hi], axis=1)
    return np.moveaxis(out, (0, 1), (axis, axis + 1))


def pair_data(values, parity, periodic, bc, override=None):
    """boundary.py:135-147 (data only).  bc = (left, right, left_value, right_value)."""
    vals = (bc[2], bc[3]) if override is None else override
    return gather(values, 0, "x", parity, periodic, bc[:2], vals)


def corner_data(values, parity, periodic, bcx, bcy, override=None):
    """boundary.py:150-168 (data only): x gather then y gather."""
    vx = (bcx[2], bcx[3]) if override is None else override
    vy = (bcy[2], bcy[3]) if override is None else override
    a = gather(values, 0, "x", parity, periodic, bcx[:2], vx)
    b = gather(a, 2, "y", parity, periodic, bcy[:2], vy)
    return np.moveaxis(b, 1, 2)


PERIODIC_BC = ("periodic", "periodic", 0.0, 0.0)


# ----------------------------------------------------------------- dissipative.py

def taylor_1d(cu, cv, dt, h, speed, smax, forcing=None, centers=None, t=0.0):
    """dissipative.py:77-106."""
    cu = np.asarray(cu, dtype=float)
    cv = np.asarray(cv, dtype=float)
    lu, lv = cu.shape[-1], cv.shape[-1]
    U = np.zeros(cu.shape + (smax + 1,))
    V = np.zeros(cv.shape + (smax + 1,))
    U[..., 0] = cu
    V[..., 0] = cv
    r = speed * speed * dt / (h * h)
    ns = min(lv, lu - 2)
    mul = np.arange(2, ns + 2) * np.arange(1, ns + 1)
    for s in range(1, smax + 1):
        U[..., :lv, s] = (dt / s) * V[..., :, s - 1]
        V[..., :ns, s] = (r / s) * mul * U[..., 2:ns + 2, s - 1]
        if forcing is not None:
            for l in range(lv):
                fac = h**l * dt**s / (_fact(l) * _fact(s))
                V[..., l, s] += fac * forcing(l, s - 1, centers, t)
    return U, V


def _fact(n):
    r = 1.0
    for k in range(2, n + 1):
        r *= k
    return r


def horner(table, theta):
    """dissipative.py:116-121."""
    out = table[..., -1].copy()
    for s in range(table.shape[-1] - 2, -1, -1):
        out = out * theta + table[..., s]
    return out


def half_step_1d(u, v, parity, n, periodic, x_left, h, m, lam, speed=1.0, bc=PERIODIC_BC,
                 stage_cap=None, forcing=None, t=0.0):
    """dissipative.py:160-181 on raw arrays; returns (u_new, v_new) on flip(parity)."""
    dt = lam * h / speed
    du = pair_data(u, parity, periodic, bc)
    dv = pair_data(v, parity, periodic, bc, override=(0.0, 0.0))
    centers = nodes(x_left, h, n, periodic, flip(parity))
    smax = 2 * m if stage_cap is None else stage_cap
    U, V = taylor_1d(interp_1d(du), interp_1d(dv), dt, h, speed, smax, forcing, centers, t)
    return horner(U, 0.5)[:, :m + 1], horner(V, 0.5)[:, :m]


def taylor_2d(c0, d0, dt, hx, hy, speed, smax, d1=None):
    """dissipative.py:184-212."""
    k = c0.shape[-1]
    lv = d0.shape[-1]
    U = np.zeros(c0.shape[:-2] + (k, k, smax + 1))
    V = np.zeros_like(U)
    U[..., 0] = c0
    V[..., :lv, :lv, 0] = d0
    rx = speed * speed * dt / (hx * hx)
    ry = speed * speed * dt / (hy * hy)
    mul = np.arange(2, k) * np.arange(1, k - 1)
    for s in range(1, smax + 1):
        U[..., s] = (dt / s) * V[..., s - 1]
        if s == 1 and d1 is not None:
            V[..., :k - 2, :k - 2, 1] = d1
            continue
        V[..., :k - 2, :, s] = (rx / s) * mul[:, None] * U[..., 2:, :, s - 1]
        V[..., :, :k - 2, s] += (ry / s) * mul[None, :] * U[..., :, 2:, s - 1]
    return U, V


def half_step_2d(u, v, parity, nx, ny, periodic, hx, hy, m, lam, speed=1.0, bcx=PERIODIC_BC,
                 bcy=PERIODIC_BC, stage_cap=None):
    """dissipative.py:215-247 on raw arrays; returns (u_new, v_new) contiguous."""
    dt = lam * min(hx, hy) / speed
    du = corner_data(u, parity, periodic, bcx, bcy)
    dv = corner_data(v, parity, periodic, bcx, bcy, override=(0.0, 0.0))
    cmm = interp_2d(du)
    cx = interp_2d(du[..., :, :m])
    cy = interp_2d(du[..., :m, :])
    d0 = interp_2d(dv)
    rx = speed**2 * dt / (hx * hx)
    ry = speed**2 * dt / (hy * hy)
    mul = np.arange(2, 2 * m + 2) * np.arange(1, 2 * m + 1)
    d1 = rx * mul[:, None] * cx[..., 2:, :] + ry * mul[None, :] * cy[..., :, 2:]
    smax = 4 * m + 4 if stage_cap is None else stage_cap
    U, V = taylor_2d(cmm, d0, dt, hx, hy, speed, smax, d1=d1)
    return (np.ascontiguousarray(horner(U, 0.5)[..., :m + 1, :m + 1]),
            np.ascontiguousarray(horner(V, 0.5)[..., :m, :m]))


def half_step_2d_chunked(u, v, parity, nx, ny, periodic, hx, hy, m, lam, rows=8, **kw):
    """Row-chunked half_step_2d for periodic grids larger than RAM allows
    (bitwise identical to the unchunked call)."""
    assert periodic
    n0 = u.shape[0]
    outs_u, outs_v = [], []
    off = 0 if parity == PRIMAL else -1
    for r0 in range(0, n0, rows):
        r1 = min(n0, r0 + rows)
        idx = np.arange(r0 + off, r1 + off + 1) % n0
        # the row window is "primal with walls" along x (no ghosts), periodic along y
        a = gather(u[idx], 0, "x", PRIMAL, False, None, None)
        b = gather(a, 2, "y", parity, True, None, None)
        du = np.moveaxis(b, 1, 2)
        a = gather(v[idx], 0, "x", PRIMAL, False, None, None)
        b = gather(a, 2, "y", parity, True, None, None)
        dv = np.moveaxis(b, 1, 2)
        uu, vv = _step_from_corners(du, dv, hx, hy, m, lam, **kw)
        outs_u.append(uu)
        outs_v.append(vv)
    return np.concatenate(outs_u), np.concatenate(outs_v)


def _step_from_corners(du, dv, hx, hy, m, lam, speed=1.0, stage_cap=None):
    dt = lam * min(hx, hy) / speed
    cmm = interp_2d(du)
    cx = interp_2d(du[..., :, :m])
    cy = interp_2d(du[..., :m, :])
    d0 = interp_2d(dv)
    rx = speed**2 * dt / (hx * hx)
    ry = speed**2 * dt / (hy * hy)
    mul = np.arange(2, 2 * m + 2) * np.arange(1, 2 * m + 1)
    d1 = rx * mul[:, None] * cx[..., 2:, :] + ry * mul[None, :] * cy[..., :, 2:]
    smax = 4 * m + 4 if stage_cap is None else stage_cap
    U, V = taylor_2d(cmm, d0, dt, hx, hy, speed, smax, d1=d1)
    return (np.ascontiguousarray(horner(U, 0.5)[..., :m + 1, :m + 1]),
            np.ascontiguousarray(horner(V, 0.5)[..., :m, :m]))


# ----------------------------------------------------------------- conservative.py

def pascal_base(m):
    """conservative.py:59-66: base[i, j] = C(i+j, i) for i+j <= 2m."""
    n = 2 * m + 1
    base = np.zeros((n, n), dtype=np.int64)
    for i in range(n):
        for j in range(n - i):
            base[i, j] = math.comb(i + j, i)
    return base


@lru_cache(maxsize=None)
def update_matrix_1d(m, rho):
    """conservative.py:77-84."""
    w = np.zeros((m + 1, 2 * m + 2))
    for k in range(m + 1):
        for j in range(k, 2 * m + 2, 2):
            w[k, j] = math.comb(j, k) * rho ** (j - k)
    return w


@lru_cache(maxsize=None)
def update_tensor_2d(m, rho_x, rho_y):
    """conservative.py:87-112."""
    kk = 2 * m + 2
    base = pascal_base(m)
    wt = np.zeros((m + 1, m + 1, kk, kk))
    for k in range(m + 1):
        for l in range(m + 1):
            for i in range(m + 1):
                a = k + 2 * i
                if a > 2 * m + 1:
                    break
                for j in range(m + 1):
                    b = l + 2 * j
                    if b > 2 * m + 1:
                        break
                    fr = Fraction(math.comb(a, k) * math.comb(b, l) * int(base[i, j]),
                                  math.comb(2 * i + 2 * j, 2 * i))
                    wt[k, l, a, b] = float(fr) * rho_x ** (2 * i) * rho_y ** (2 * j)
    return wt


def cons_step_1d(cur, prev, parity_cur, n, periodic, m, lam, bc=PERIODIC_BC):
    """conservative.py:139-157 (1D): returns the new level (on prev's grid)."""
    c = interp_1d(pair_data(cur, parity_cur, periodic, bc))
    return 2.0 * (c @ update_matrix_1d(m, 0.5 * lam).T) - np.asarray(prev, dtype=float)


def cons_step_2d(cur, prev, parity_cur, periodic, hx, hy, m, lam, speed=1.0, bcx=PERIODIC_BC,
                 bcy=PERIODIC_BC):
    """conservative.py:139-157 (2D)."""
    c = interp_2d(corner_data(cur, parity_cur, periodic, bcx, bcy))
    dt = lam * min(hx, hy) / speed
    wt = update_tensor_2d(m, 0.5 * speed * dt / hx, 0.5 * speed * dt / hy)
    return 2.0 * np.einsum("klab,...ab->...kl", wt, c, optimize=True) - np.asarray(prev, dtype=float)


def bootstrap_1d(g0, g1, parity, n, periodic, h, m, lam, speed=1.0, bc=PERIODIC_BC):
    """conservative.py:172-182."""
    dt = lam * h / speed
    du = pair_data(g0, parity, periodic, bc)
    dv = pair_data(g1, parity, periodic, bc, override=(0.0, 0.0))
    U, _ = taylor_1d(interp_1d(du), interp_1d(dv), dt, h, speed, 2 * m + 3)
    return horner(U, 0.5)[:, :m + 1]


def bootstrap_2d(g0, g1, parity, periodic, hx, hy, m, lam, speed=1.0, bcx=PERIODIC_BC, bcy=PERIODIC_BC):
    """conservative.py:185-193."""
    dt = lam * min(hx, hy) / speed
    du = corner_data(g0, parity, periodic, bcx, bcy)
    dv = corner_data(g1, parity, periodic, bcx, bcy, override=(0.0, 0.0))
    U, _ = taylor_2d(interp_2d(du), interp_2d(dv), dt, hx, hy, speed, 4 * m + 4)
    return np.ascontiguousarray(horner(U, 0.5)[..., :m + 1, :m + 1])


# ----------------------------------------------------------------- diagnostics.py

def l2_cells_2d(c, cx, cy, hx, hy, exact, npts):
    """Per-cell (hx hy / 4) sum_pq w_p w_q (I u - exact)^2 from the cells' interpolant
    coefficients c (..., 2mx+2, 2my+2) and centres cx, cy (diagnostics.py:118-135)."""
    xg, wg = np.polynomial.legendre.leggauss(npts)
    vx = np.vander(0.5 * xg, c.shape[-2], increasing=True)
    vy = np.vander(0.5 * xg, c.shape[-1], increasing=True)
    vals = np.einsum("ijab,pa,qb->ijpq", c, vx, vy, optimize=True)
    x = cx[:, None] + 0.5 * hx * xg[None, :]
    y = cy[:, None] + 0.5 * hy * xg[None, :]
    diff = vals - exact(x[:, None, :, None], y[None, :, None, :])
    return np.sum(diff * diff * (wg[:, None] * wg[None, :]), axis=(2, 3)) * (0.25 * hx * hy)


def l2_error_2d(values, parity, nx, ny, periodic, x_left, y_left, hx, hy, exact, npts=None,
                bcx=PERIODIC_BC, bcy=PERIODIC_BC):
    """diagnostics.py:118-135."""
    mx, my = values.shape[2] - 1, values.shape[3] - 1
    npts = npts or 2 * max(mx, my) + 2
    c = interp_2d(corner_data(values, parity, periodic, bcx, bcy))
    xg, wg = np.polynomial.legendre.leggauss(npts)
    vx = np.vander(0.5 * xg, c.shape[-2], increasing=True)
    vy = np.vander(0.5 * xg, c.shape[-1], increasing=True)
    vals = np.einsum("ijab,pa,qb->ijpq", c, vx, vy, optimize=True)
    cx = nodes(x_left, hx, nx, periodic, flip(parity))
    cy = nodes(y_left, hy, ny, periodic, flip(parity))
    x = cx[:, None] + 0.5 * hx * xg[None, :]
    y = cy[:, None] + 0.5 * hy * xg[None, :]
    diff = vals - exact(x[:, None, :, None], y[None, :, None, :])
    total = np.sum(diff * diff * (wg[:, None] * wg[None, :])) * (0.25 * hx * hy)
    return math.sqrt(total)


def _piece_eval(coeffs, xi):
    out = np.zeros_like(xi) + coeffs[-1]
    for a in coeffs[-2::-1]:
        out = out * xi + a
    return out


def l2_error_1d(values, parity, n, periodic, x_left, h, exact, npts=None, bc=PERIODIC_BC, deriv=0):
    """diagnostics.py:47-100 (field_interpolant + l2_error + clip)."""
    mu = values.shape[1] - 1
    npts = npts or 2 * mu + 2
    coeffs = interp_1d(pair_data(values, parity, periodic, bc))
    centers = nodes(x_left, h, n, periodic, flip(parity))
    bp = np.concatenate([centers - 0.5 * h, centers[-1:] + 0.5 * h])
    clip = None if periodic else (x_left, x_left + n * h)
    xg, wg = np.polynomial.legendre.leggauss(npts)
    total = 0.0
    for i, cc in enumerate(coeffs):
        if deriv:
            cc = cc[1:] * np.arange(1, len(cc)) / h
        a, b = bp[i], bp[i + 1]
        if clip is not None:
            a, b = max(a, clip[0]), min(b, clip[1])
            if b <= a:
                continue
        x = 0.5 * (a + b) + 0.5 * (b - a) * xg
        d = _piece_eval(cc, (x - centers[i]) / h) - exact(x)
        total += 0.5 * (b - a) * np.dot(wg, d * d)
    return math.sqrt(total)


# ----------------------------------------------------------------- energies (1D)

def _deriv(coeffs, order, h):
    """poly.py:56-74 CellPolynomial.derivative on a (pieces, L) coefficient array."""
    n = coeffs.shape[-1] - order
    if n <= 0:
        return np.zeros(coeffs.shape[:-1] + (1,))
    fall = np.array([math.factorial(j + order) // math.factorial(j) for j in range(n)], dtype=float)
    return coeffs[..., order:] * fall / h**order


def _horner_cols(d, xi):
    """Evaluate pieces d (P, L) at points xi (P, Q) or (Q,)."""
    out = np.zeros(np.broadcast(d[:, :1], xi).shape) + d[:, -1:]
    for j in range(d.shape[-1] - 2, -1, -1):
        out = out * xi + d[:, j:j + 1]
    return out


def seminorm_sq_1d(values, parity, n, periodic, h, order, bc=PERIODIC_BC):
    """diagnostics.py:201-212 over field_interpolant's pieces (diagnostics.py:47-59)."""
    d = _deriv(interp_1d(pair_data(values, parity, periodic, bc)), order, h)
    xg, wg = np.polynomial.legendre.leggauss(d.shape[-1])
    q = _horner_cols(d, 0.5 * xg[None, :])
    return float(np.sum(0.5 * h * (q * q) @ wg))


def dissipative_energy_1d(u, v, parity, n, periodic, h, speed, bc=PERIODIC_BC):
    """diagnostics.py:229-234."""
    m = u.shape[1] - 1
    return speed * speed * seminorm_sq_1d(u, parity, n, periodic, h, m + 1, bc) + \
        seminorm_sq_1d(v, parity, n, periodic, h, m, bc)


# ----------------------------------------------------------------- energy (2D, defined here)

def _monomial_gram(n):
    """G[a][b] = int_{-1/2}^{1/2} xi^(a+b) dxi, exactly."""
    k = np.add.outer(np.arange(n), np.arange(n))
    return np.where(k % 2 == 0, 2.0 * 0.5 ** (k + 1) / (k + 1), 0.0)


def seminorm_sq_2d(values, parity, hx, hy, dx, dy):
    """sum_cells int int (d_x^dx d_y^dy I u)^2 of the tensor interpolant on a
    periodic grid: cell coefficients from corner_data + interp_2d, derivative
    taken on the monomial coefficients, the square integrated in closed form
    (a Gram matrix of monomials — independent of the device's Gauss rule).
    No reference counterpart (the reference energies are 1D only)."""
    c = interp_2d(corner_data(values, parity, True, PERIODIC_BC, PERIODIC_BC))
    nxc, nyc = c.shape[-2] - dx, c.shape[-1] - dy
    if nxc <= 0 or nyc <= 0:
        return 0.0
    fx = np.array([math.factorial(a + dx) / math.factorial(a) for a in range(nxc)]) / hx**dx
    fy = np.array([math.factorial(b + dy) / math.factorial(b) for b in range(nyc)]) / hy**dy
    d = c[..., dx:, dy:] * fx[:, None] * fy[None, :]
    return float(hx * hy * np.einsum("ijab,ac,ijcd,bd->", d, _monomial_gram(nxc), d, _monomial_gram(nyc)))


def dissipative_energy_2d(u, v, parity, hx, hy, speed):
    """c^2 (|d_x^{m+1} I u|^2 + |d_y^{m+1} I u|^2) + |d_x^m I v|^2 + |d_y^m I v|^2
    (paper_1802_05246_b200.norms.dissipative_energy_2d's definition)."""
    m = u.shape[-1] - 1
    eu = seminorm_sq_2d(u, parity, hx, hy, m + 1, 0) + seminorm_sq_2d(u, parity, hx, hy, 0, m + 1)
    ev = seminorm_sq_2d(v, parity, hx, hy, m, 0) + seminorm_sq_2d(v, parity, hx, hy, 0, m)
    return speed * speed * eu + ev


def conservative_energy_1d(cur, prev, parity_cur, n, h, delta):
    """diagnostics.py:190-226 on a periodic grid, restated per union piece.

    Cur piece t spans its two source nodes; the prev pieces shifted by
    -/+delta that meet it are the ones centred on those nodes, split at
    xi = -/+delta/h (pp_subtract's merged breakpoints).  Both (m+1)-th
    derivatives are evaluated in their own scaled variables at m+1 Gauss
    points per union piece (exact for the degree-2m integrand)."""
    m = cur.shape[1] - 1
    off = 0 if parity_cur == PRIMAL else -1
    dc = _deriv(interp_1d(pair_data(cur, parity_cur, True, PERIODIC_BC)), m + 1, h)
    dp = _deriv(interp_1d(pair_data(prev, flip(parity_cur), True, PERIODIC_BC)), m + 1, h)
    t = np.arange(n)
    dl, dr = dp[(t + off) % n], dp[(t + off + 1) % n]
    xg, wg = np.polynomial.legendre.leggauss(m + 1)
    dx = delta / h
    total = 0.0
    for sgn in (1, -1):
        xs = -sgn * dx
        for lo, hi, dpp, shp in ((-0.5, xs, dl, sgn * dx + 0.5), (xs, 0.5, dr, sgn * dx - 0.5)):
            if hi <= lo:
                continue
            xi = 0.5 * (lo + hi) + 0.5 * (hi - lo) * xg
            q = _horner_cols(dc, xi[None, :]) - _horner_cols(dpp, xi[None, :] + shp)
            total += float(np.sum(0.5 * (hi - lo) * h * (q * q) @ wg))
    return total


# ----------------------------------------------------------------- conservative energy (2D, defined here)
#
# The reference's conservative energy is 1D and periodic only (diagnostics.py:190-226):
# E = |P+|^2 + |P-|^2, P± = I cur - S± I prev, S± the shifts by c dt/2, in the
# (m+1) seminorm.  Expanding the squares, with C = (S+ + S-)/2 self-adjoint:
#     E = 2 (|I a|^2 + |I b|^2 - 2 <I a, C I b>),   a = current, b = previous,
# and because Hermite interpolation is an orthogonal projection in that
# seminorm, <I a, C I b> = <I a, I T b>, where T b = R_A C I_B b is exactly the
# scheme's own update of b (conservative.py:115-136 with prev = 0, halved).
# That adjoint form needs no shifted pieces, so it carries over to 2D: the
# tensor interpolant I = Ix Iy is an orthogonal projection in the MIXED
# seminorm |d_x^{m+1} d_y^{m+1} .| (integrate by parts in x, then in y), the
# wave cosine C(tau) is self-adjoint and commutes with it, and C(tau)
# restricted to a cell (c tau <= h/2) is the update tensor — so
#     E2 = 2 (|I a|^2 + |I b|^2 - <I a, I (2 T b)>)   (mixed seminorm)
# is conserved exactly by full_step_conservative in exact arithmetic.  Walls:
# the Dirichlet / Neumann ghosts (boundary.py:56-98) are the odd / even
# reflections, so a wall grid is the quarter of a periodic doubled grid;
# integrating over the physical domain counts cells that straddle a wall
# (dual parity, ghost-padded) with weight 1/2 per axis.

def _cons_apply_2d(values, parity, periodic, hx, hy, m, speed, dt, bcx=PERIODIC_BC, bcy=PERIODIC_BC):
    """2 T b: conservative.py:130-136 with prev = 0 and an explicit dt."""
    c = interp_2d(corner_data(values, parity, periodic, bcx, bcy))
    wt = update_tensor_2d(m, 0.5 * speed * dt / hx, 0.5 * speed * dt / hy)
    return 2.0 * np.einsum("klab,...ab->...kl", wt, c, optimize=True)


def inner_cells_2d(cx, cy, hx, hy, dx, dy):
    """Per-cell int int (d_x^dx d_y^dy p)(d_x^dx d_y^dy q) of cell polynomials with
    coefficient arrays cx, cy (..., 2mx+2, 2my+2) in the cell variables, exactly
    (monomial Gram)."""
    nxc, nyc = cx.shape[-2] - dx, cx.shape[-1] - dy
    if nxc <= 0 or nyc <= 0:
        return np.zeros(cx.shape[:-2])
    fx = np.array([math.factorial(a + dx) / math.factorial(a) for a in range(nxc)]) / hx**dx
    fy = np.array([math.factorial(b + dy) / math.factorial(b) for b in range(nyc)]) / hy**dy
    dX = cx[..., dx:, dy:] * fx[:, None] * fy[None, :]
    dY = cy[..., dx:, dy:] * fx[:, None] * fy[None, :]
    return hx * hy * np.einsum("ijab,ac,ijcd,bd->ij", dX, _monomial_gram(nxc), dY, _monomial_gram(nyc))


def inner_2d(x, y, parity, periodic, hx, hy, dx, dy, bcx=PERIODIC_BC, bcy=PERIODIC_BC):
    """sum over the field's cells of w_cell * int int (d_x^dx d_y^dy I x)(d_x^dx d_y^dy I y),
    integrated in closed form (monomial Gram); w_cell = 1/2 per axis on which the
    cell straddles a wall (ghost-padded dual cells), else 1."""
    cx = interp_2d(corner_data(x, parity, periodic, bcx, bcy))
    cy = cx if y is x else interp_2d(corner_data(y, parity, periodic, bcx, bcy))
    per_cell = inner_cells_2d(cx, cy, hx, hy, dx, dy)
    if per_cell.ndim < 2:
        return 0.0
    wx = np.ones(per_cell.shape[0])
    wy = np.ones(per_cell.shape[1])
    if not periodic and parity == DUAL:
        wx[[0, -1]] = 0.5
        wy[[0, -1]] = 0.5
    return float(np.sum(per_cell * wx[:, None] * wy[None, :]))


SEMINORMS = {"mixed": lambda m: [(m + 1, m + 1)], "l2": lambda m: [(0, 0)], "h1": lambda m: [(1, 0), (0, 1)]}


def cons_energy_2d(cur, prev, parity_cur, periodic, hx, hy, speed, dt, bcx=PERIODIC_BC, bcy=PERIODIC_BC,
                   seminorm="mixed"):
    """E2 above (paper_1802_05246_b200.norms.conservative_energy_2d's definition);
    seminorm "mixed" is the exactly conserved one, "l2" / "h1" the same adjoint
    form in lower-order seminorms (conserved by the exact wave, by the scheme up
    to its projection error)."""
    m = cur.shape[-1] - 1
    pb = flip(parity_cur)
    tb2 = _cons_apply_2d(prev, pb, periodic, hx, hy, m, speed, dt, bcx, bcy)
    tot = 0.0
    for dx, dy in SEMINORMS[seminorm](m):
        ia = inner_2d(cur, cur, parity_cur, periodic, hx, hy, dx, dy, bcx, bcy)
        ib = inner_2d(prev, prev, pb, periodic, hx, hy, dx, dy, bcx, bcy)
        iab = inner_2d(cur, tb2, parity_cur, periodic, hx, hy, dx, dy, bcx, bcy)
        tot += ia + ib - iab
    return 2.0 * tot


def wall_compatible(values, bcx, bcy):
    """Project primal wall-node data onto the reflection symmetry the wall ghosts
    define (Dirichlet: f = g, even-order normal derivatives 0; Neumann: odd-order
    normal derivatives 0) — what a step from the dual grid produces and exact
    initial data satisfy.  Test-input helper for the energy checks."""
    d = np.array(values, dtype=float)
    k = np.arange(d.shape[-1])
    for axis, bc in ((0, bcx), (1, bcy)):
        if bc[0] == "periodic":
            continue
        for side, kind, g in ((0, bc[0], bc[2]), (-1, bc[1], bc[3])):
            node = d[side] if axis == 0 else d[:, side]
            bad = (k % 2 == 0) if kind == "dirichlet0" else (k % 2 == 1)
            if axis == 0:
                node[:, bad, :] = 0.0
            else:
                node[:, :, bad] = 0.0
            if kind == "dirichlet0":
                node[:, 0, 0] = g
    return d


def cons_energy_1d_adjoint(cur, prev, parity_cur, n, h, speed, dt):
    """The 1D reference energy (diagnostics.py:190-226) through the adjoint form
    2 (|I a|^2 + |I b|^2 - <I a, I (2 T b)>) in the (m+1) seminorm, periodic:
    the construction E2 generalises, pinned against the reference's
    conservative_energy in tests/test_energy.py."""
    m = cur.shape[1] - 1
    pb = flip(parity_cur)
    c = interp_1d(pair_data(prev, pb, True, PERIODIC_BC))
    tb2 = 2.0 * (c @ update_matrix_1d(m, 0.5 * speed * dt / h).T)
    xg, wg = np.polynomial.legendre.leggauss(m + 1)

    def inner(x, y, par):
        dxx = _deriv(interp_1d(pair_data(x, par, True, PERIODIC_BC)), m + 1, h)
        dyy = _deriv(interp_1d(pair_data(y, par, True, PERIODIC_BC)), m + 1, h)
        qx = _horner_cols(dxx, 0.5 * xg[None, :])
        qy = _horner_cols(dyy, 0.5 * xg[None, :])
        return float(np.sum(0.5 * h * (qx * qy) @ wg))

    return 2.0 * (inner(cur, cur, parity_cur) + inner(prev, prev, pb) - inner(cur, tb2, parity_cur))


# ----------------------------------------------------------------- driver.py data

def scale_cols(vals, h):
    """driver.py:195-200."""
    fac = np.ones(vals.shape[-1])
    for l in range(1, vals.shape[-1]):
        fac[l] = fac[l - 1] * h / l
    return vals * fac


def sine_derivs(x, kmax, t):
    """driver.py:234-238."""
    x = np.asarray(x, dtype=float)
    k = np.arange(kmax + 1)
    return np.sin(x[..., None] + 0.5 * np.pi * k) * math.cos(t)


def planewave_data(xn, yn, t, kx, ky, kappa, hx, hy, tder=0):
    """driver.py:241-256."""
    w = 2.0 * np.pi * kappa
    theta = w * (xn[:, None] + yn[None, :] + math.sqrt(2.0) * t)
    out = np.empty(theta.shape + (kx + 1, ky + 1))
    for k in range(kx + 1):
        for l in range(ky + 1):
            amp = w ** (k + l) * (math.sqrt(2.0) * w) ** tder
            amp *= hx**k / math.factorial(k) * hy**l / math.factorial(l)
            out[..., k, l] = amp * np.sin(theta + 0.5 * np.pi * (k + l + tder))
    return out


def fit_rate(hs, errors):
    """diagnostics.py:263-278."""
    hs = np.asarray(hs, dtype=float)
    errors = np.asarray(errors, dtype=float)
    k = (len(hs) + 1) // 2
    return float(np.polyfit(np.log(hs[-k:]), np.log(errors[-k:]), 1)[0])
