// Diagnostics on the device: 2D / 1D L2 error reductions, the finite check
// and the closed-form initial data generators.
#pragma once

#include "common.cuh"
#include "line1d.cuh"

namespace hw {

constexpr int kRedThreads = 256;

// Deterministic block reduction (fixed tree order).
__device__ inline double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void sum_partials_kernel(const double* part, int64_t n, double* out) {
  __shared__ double sh[kRedThreads];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  const double r = block_sum(s, sh);
  if (threadIdx.x == 0) *out = r;
}

struct L2Err2DArgs {
  Rows f;
  int64_t nx, ny, ntx, nty;
  int64_t trow0, ntrows;  // target (cell) rows reduced: [trow0, trow0 + ntrows) (slabs)
  int off, periodic;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;
  int mx, my, npts;
  const double* ex;   // Ex[p][sx*(mx+1)+k] = sum_a (xg_p/2)^a M_x[a][sx*(mx+1)+k]
  const double* ey;
  const double* gw;   // Gauss weights
  const double* gx;   // Gauss nodes on [-1,1]
  int exact_kind;
  const double* exact;  // [ci - trow0][cj][p][q]
  double prm[4];
  double x0, y0, hx, hy, coff;  // target node coordinates x0 + hx (i + coff)
  double* part;
};

__device__ inline double exact_builtin(int kind, const double* prm, double x, double y) {
  if (kind == 1) return sin(prm[0] * (x + y + sqrt(2.0) * prm[1]));  // driver.py:393-394
  return sin(prm[0] * x) * sin(prm[1] * y) * cos(prm[2] * prm[3]);
}

// diagnostics.py:118-135 l2_error_field_2d: one thread per target cell.
// exact_kind 3 (no exact solution) with derivative evaluation matrices Ex/Ey
// gives the squared seminorm sum of the 2D energy (hw_seminorm2d).
__global__ void l2err2d_kernel(L2Err2DArgs a) {
  __shared__ double sh[kRedThreads];
  const int64_t ncell = a.ntrows * a.nty;
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double local = 0.0;
  if (cell < ncell) {
    const int64_t tl = cell / a.nty, tj = cell - tl * a.nty, ti = a.trow0 + tl;
    const int mx = a.mx, my = a.my, wx = mx + 1, wy = my + 1, P = wx * wy;
    const RowRef r0 = resolve_row(a.f, ti + a.off, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
    const RowRef r1 = resolve_row(a.f, ti + a.off + 1, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
    const ColRef c0 = resolve_col(tj + a.off, a.ny, a.periodic, a.kyl, a.kyh, a.gyl, a.gyh);
    const ColRef c1 = resolve_col(tj + a.off + 1, a.ny, a.periodic, a.kyl, a.kyh, a.gyl, a.gyh);
    const RowRef* rr[2] = {&r0, &r1};
    const ColRef* cc[2] = {&c0, &c1};
    const double cx = a.x0 + a.hx * ((double)ti + a.coff);
    const double cy = a.y0 + a.hy * ((double)tj + a.coff);
    double T[2 * 13];
    for (int q = 0; q < a.npts; ++q) {
      // T[sx][k] = sum_{sy,l} Ey[q][sy,l] U[sx][sy][k][l]
      for (int sx = 0; sx < 2; ++sx)
        for (int k = 0; k < wx; ++k) {
          double s = 0.0;
          for (int sy = 0; sy < 2; ++sy)
            for (int l = 0; l < wy; ++l) {
              double val = rr[sx]->p[cc[sy]->c * P + k * wy + l];
              if (rr[sx]->kind | cc[sy]->kind)
                val = ghosted(val, k, l, rr[sx]->kind, rr[sx]->g, cc[sy]->kind, cc[sy]->g);
              s = fma(__ldg(a.ey + q * 2 * wy + sy * wy + l), val, s);
            }
          T[sx * wx + k] = s;
        }
      const double yq = cy + 0.5 * a.hy * a.gx[q];
      for (int p = 0; p < a.npts; ++p) {
        double val = 0.0;
        for (int e = 0; e < 2 * wx; ++e) val = fma(__ldg(a.ex + p * 2 * wx + e), T[e], val);
        double ex;
        if (a.exact_kind == 0) {
          ex = a.exact[((tl * a.nty + tj) * a.npts + p) * a.npts + q];
        } else if (a.exact_kind == 3) {  // seminorms: the derivative interpolant alone
          ex = 0.0;
        } else {
          const double xp = cx + 0.5 * a.hx * a.gx[p];
          ex = exact_builtin(a.exact_kind, a.prm, xp, yq);
        }
        const double d = val - ex;
        local = fma(a.gw[p] * a.gw[q], d * d, local);
      }
    }
  }
  const double bs = block_sum(local, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = bs;
}

// ---------------------------------------------------------------- bilinear seminorm (conservative energy)
// Compensated (double-double) accumulation: the 2D conservative energy is a
// difference of O(1) inner products that cancel to O((omega dt)^2), so the
// reduction itself must not add O(log N eps) relative error.
__device__ inline void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

__device__ inline void dd_add(double& hi, double& lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  hi = s;
  lo += e;
}

// Deterministic double-double block reduction (fixed tree order); sh holds 2 * blockDim doubles.
__device__ inline void block_sum_dd(double& hi, double& lo, double* sh) {
  sh[threadIdx.x] = hi;
  sh[blockDim.x + threadIdx.x] = lo;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      double h, e;
      two_sum(sh[threadIdx.x], sh[threadIdx.x + s], h, e);
      e += sh[blockDim.x + threadIdx.x] + sh[blockDim.x + threadIdx.x + s];
      double h2, e2;
      two_sum(h, e, h2, e2);
      sh[threadIdx.x] = h2;
      sh[blockDim.x + threadIdx.x] = e2;
    }
    __syncthreads();
  }
  hi = sh[0];
  lo = sh[blockDim.x];
  __syncthreads();
}

__global__ void sum_partials_dd_kernel(const double* part, int64_t n, double* out) {
  __shared__ double sh[2 * kRedThreads];
  double hi = 0.0, lo = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    dd_add(hi, lo, part[2 * i]);
    lo += part[2 * i + 1];
  }
  block_sum_dd(hi, lo, sh);
  if (threadIdx.x == 0) *out = hi + lo;
}

struct Inner2DArgs {
  Rows f, g;
  int same;  // g aliases f
  int64_t nx, ny, nty, trow0, ntrows;
  int off, periodic;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;
  int mx, my, npts, wall_half;
  const double* ex;  // as L2Err2DArgs (derivative evaluation matrices, 1/h^d folded in)
  const double* ey;
  const double* gw;
  double* part;      // (hi, lo) per block
};

// T[sx*wx + k] = sum_{sy,l} Ey[q][sy,l] U[sx][sy][k][l] for one field of one cell.
__device__ inline void cell_ycontract(const RowRef* const* rr, const ColRef* const* cc, int wx, int wy, int P,
                                      const double* ey, int q, double* T) {
  for (int sx = 0; sx < 2; ++sx)
    for (int k = 0; k < wx; ++k) {
      double s = 0.0;
      for (int sy = 0; sy < 2; ++sy)
        for (int l = 0; l < wy; ++l) {
          double val = rr[sx]->p[cc[sy]->c * P + k * wy + l];
          if (rr[sx]->kind | cc[sy]->kind)
            val = ghosted(val, k, l, rr[sx]->kind, rr[sx]->g, cc[sy]->kind, cc[sy]->g);
          s = fma(__ldg(ey + q * 2 * wy + sy * wy + l), val, s);
        }
      T[sx * wx + k] = s;
    }
}

// sum_cells w_cell int int (D I f)(D I g), D = d_x^dx d_y^dy folded into Ex/Ey,
// over target rows [trow0, trow0 + ntrows) of the field's corner gather.
// wall_half: cells whose gather used a wall ghost (dual parity) straddle the
// wall and count 1/2 per such axis (the integral over the physical domain of
// the reflected extension the ghosts define, boundary.py:56-98).
__global__ void inner2d_kernel(Inner2DArgs a) {
  __shared__ double sh[2 * kRedThreads];
  const int64_t ncell = a.ntrows * a.nty;
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double hi = 0.0, lo = 0.0;
  if (cell < ncell) {
    const int64_t ti = a.trow0 + cell / a.nty, tj = cell % a.nty;
    const int mx = a.mx, my = a.my, wx = mx + 1, wy = my + 1, P = wx * wy;
    const int64_t sx0 = ti + a.off, sy0 = tj + a.off;
    RowRef fr[2], gr[2];
    ColRef cl[2];
    for (int s = 0; s < 2; ++s) {
      fr[s] = resolve_row(a.f, sx0 + s, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
      gr[s] = resolve_row(a.g, sx0 + s, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
      cl[s] = resolve_col(sy0 + s, a.ny, a.periodic, a.kyl, a.kyh, a.gyl, a.gyh);
    }
    const RowRef* frp[2] = {&fr[0], &fr[1]};
    const RowRef* grp[2] = {&gr[0], &gr[1]};
    const ColRef* clp[2] = {&cl[0], &cl[1]};
    double wcell = 1.0;
    if (a.wall_half && !a.periodic) {
      if (sx0 < 0 || sx0 + 1 > a.nx - 1) wcell *= 0.5;
      if (sy0 < 0 || sy0 + 1 > a.ny - 1) wcell *= 0.5;
    }
    double Tf[2 * 13], Tg[2 * 13];
    for (int q = 0; q < a.npts; ++q) {
      cell_ycontract(frp, clp, wx, wy, P, a.ey, q, Tf);
      if (!a.same) cell_ycontract(grp, clp, wx, wy, P, a.ey, q, Tg);
      const double* tg = a.same ? Tf : Tg;
      for (int p = 0; p < a.npts; ++p) {
        double vf = 0.0, vg = 0.0;
        for (int e = 0; e < 2 * wx; ++e) {
          const double x = __ldg(a.ex + p * 2 * wx + e);
          vf = fma(x, Tf[e], vf);
          vg = fma(x, tg[e], vg);
        }
        dd_add(hi, lo, wcell * a.gw[p] * a.gw[q] * vf * vg);
      }
    }
  }
  block_sum_dd(hi, lo, sh);
  if (threadIdx.x == 0) {
    a.part[2 * blockIdx.x] = hi;
    a.part[2 * blockIdx.x + 1] = lo;
  }
}

struct L2Err1DArgs {
  const double* f;
  int64_t n, nt;
  int off, periodic, kl, kh;
  double gl, gh;
  int mu, deriv, npts;
  double h;
  const double* hl;
  const double* xi;
  const double* w;
  const double* ex;
  double* part;
};

// diagnostics.py:66-85 l2_error per piece (+ CellPolynomial eval/derivative).
__global__ void l2err1d_kernel(L2Err1DArgs a) {
  __shared__ double sh[kRedThreads];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double local = 0.0;
  if (t < a.nt) {
    const int mu = a.mu;
    double L[13], R[13], c[26];
    for (int side = 0; side < 2; ++side) {
      int64_t s = t + a.off + side;
      int kind = 0;
      double g = 0.0;
      if (s < 0 || s >= a.n) {
        if (a.periodic) s = pmod(s, a.n);
        else if (s < 0) { s = 0; kind = a.kl; g = a.gl; }
        else { s = a.n - 1; kind = a.kh; g = a.gh; }
      }
      double* dst = side ? R : L;
      for (int l = 0; l <= mu; ++l) {
        double val = a.f[s * (mu + 1) + l];
        if (kind) {
          val *= refl_sign(kind, l);
          if (l == 0 && kind == HW_DIRICHLET0) val += 2.0 * g;
        }
        dst[l] = val;
      }
    }
    const int nc = 2 * mu + 2;
    for (int q = 0; q < nc; ++q) {
      double s = 0.0;
      for (int k = 0; k <= mu; ++k) {
        const double comb = ((q + k) & 1) ? L[k] - R[k] : L[k] + R[k];
        s = fma(a.hl[q * (mu + 1) + k], comb, s);
      }
      c[q] = s;
    }
    int deg = nc - 1;
    if (a.deriv == 1) {  // poly.py:56-74 derivative(1): a[1:] * j / h
      for (int j = 0; j < nc - 1; ++j) c[j] = c[j + 1] * (double)(j + 1) / a.h;
      deg = nc - 2;
    }
    for (int p = 0; p < a.npts; ++p) {
      const double x = a.xi[t * a.npts + p];
      double v = c[deg];
      for (int j = deg - 1; j >= 0; --j) v = v * x + c[j];  // poly.py:47-54 Horner
      const double d = v - a.ex[t * a.npts + p];
      local = fma(a.w[t * a.npts + p], d * d, local);
    }
  }
  const double bs = block_sum(local, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = bs;
}

__global__ void nonfinite_kernel(const double* x, int64_t n, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) ++c;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// driver.py:241-256 planewave_data / standing wave, one thread per node.
struct Init2DArgs {
  double* out;
  int64_t nx, ny;
  int64_t row0;  // global index of local row 0 (slabs): x = x0 + hx (row0 + i + off)
  int kx, ky;
  double x0, y0, off, t, hx, hy;
  int kind;  // 1 plane wave, 2 standing wave
  double w;  // plane wave: 2 pi kappa
  double ax, ay, px, py, om;
  int tder;
};

// driver.py:195-238 closed-form 1D initial data, one thread per node:
// derivative columns d^k/dx^k (k = 0..kmax) of
//   kind 0  G(x) = exp(a x^2)                          (gaussian_derivs)
//   kind 1  (G(x+t) + G(x-t)) / 2, tder 1: its u_t     (gaussian_box_u / _v)
//   kind 2  sin(x) cos(t)                              (sine_derivs)
// optionally scaled by h^k / k! (_scale_cols).  Gaussian derivatives by the
// Leibniz recurrence G^(k+1) = 2a (x G^(k) + k G^(k-1)) (G' = 2 a x G).
struct Init1DArgs {
  double* out;
  const double* xs;  // node coordinates (NULL: x = x0 + h (i + off))
  int64_t n;
  int kmax, kind, tder, scaled;
  double x0, h, off, t, a;
};

__device__ inline void gauss_cols(double x, double a, int kmax, double* d) {
  const double g = exp(a * x * x);
  d[0] = g;
  if (kmax >= 1) d[1] = 2.0 * a * x * g;
  for (int k = 1; k < kmax; ++k) d[k + 1] = 2.0 * a * (x * d[k] + (double)k * d[k - 1]);
}

__global__ void init1d_kernel(Init1DArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double x = a.xs ? a.xs[i] : a.x0 + a.h * ((double)i + a.off);
  double col[kMax1D + 3];
  if (a.kind == 0) {
    gauss_cols(x, a.a, a.kmax, col);
  } else if (a.kind == 1) {
    double gp[kMax1D + 3], gm[kMax1D + 3];
    gauss_cols(x + a.t, a.a, a.kmax + 1, gp);
    gauss_cols(x - a.t, a.a, a.kmax + 1, gm);
    // u = (G(x+t) + G(x-t)) / 2, u_t = (G'(x+t) - G'(x-t)) / 2
    for (int k = 0; k <= a.kmax; ++k)
      col[k] = a.tder ? 0.5 * (gp[k + 1] - gm[k + 1]) : 0.5 * (gp[k] + gm[k]);
  } else {
    const double ct = cos(a.t);
    for (int k = 0; k <= a.kmax; ++k) col[k] = sin(x + 0.5 * 3.141592653589793 * (double)k) * ct;
  }
  double fac = 1.0;
  for (int k = 0; k <= a.kmax; ++k) {
    if (k > 0 && a.scaled) fac = fac * a.h / (double)k;  // driver.py:195-200 running factor
    a.out[i * (a.kmax + 1) + k] = a.scaled ? col[k] * fac : col[k];
  }
}

__global__ void init2d_kernel(Init2DArgs a) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= a.nx * a.ny) return;
  const int64_t i = node / a.ny, j = node - i * a.ny;
  const double x = a.x0 + a.hx * ((double)(a.row0 + i) + a.off);
  const double y = a.y0 + a.hy * ((double)j + a.off);
  const int wx = a.kx + 1, wy = a.ky + 1;
  double* o = a.out + node * wx * wy;
  const double hpi = 0.5 * 3.141592653589793;
  if (a.kind == 1) {
    const double th = a.w * (x + y + sqrt(2.0) * a.t);
    for (int k = 0; k < wx; ++k) {
      double fk = 1.0;
      for (int q = 2; q <= k; ++q) fk *= q;
      for (int l = 0; l < wy; ++l) {
        double fl = 1.0;
        for (int q = 2; q <= l; ++q) fl *= q;
        double amp = pow(a.w, (double)(k + l)) * pow(sqrt(2.0) * a.w, (double)a.tder);
        amp *= pow(a.hx, (double)k) / fk * pow(a.hy, (double)l) / fl;
        o[k * wy + l] = amp * sin(th + hpi * (double)(k + l + a.tder));
      }
    }
  } else {
    for (int k = 0; k < wx; ++k) {
      double fk = 1.0;
      for (int q = 2; q <= k; ++q) fk *= q;
      const double dx = pow(a.ax, (double)k) * sin(a.ax * x + a.px + hpi * k) * pow(a.hx, (double)k) / fk;
      for (int l = 0; l < wy; ++l) {
        double fl = 1.0;
        for (int q = 2; q <= l; ++q) fl *= q;
        const double dy = pow(a.ay, (double)l) * sin(a.ay * y + a.py + hpi * l) * pow(a.hy, (double)l) / fl;
        const double dt = pow(a.om, (double)a.tder) * cos(a.om * a.t + hpi * a.tder);
        o[k * wy + l] = dx * dy * dt;
      }
    }
  }
}

}  // namespace hw

namespace hw {

// ------------------------------------------------------------------ 1D energies
// diagnostics.py:201-234.  Pieces are the cells of the field's own gather
// (field_interpolant, diagnostics.py:47-59): piece t interpolates the flanking
// source nodes of target t, centred at the target node, width h.
struct Energy1DArgs {
  const double* f;       // field (order mu) / kCons: current level (order m)
  const double* g;       // kCons: previous level (opposite parity, order m)
  int64_t n, nt;         // source nodes, pieces
  int off, offg;         // gather offsets of f's and g's parities
  int periodic, kl, kh;
  double gl, gh;
  int mu, order;         // interpolation order, derivative order
  double h, scale, delta;
  int npts;
  const double* gx;      // Gauss nodes / weights on [-1, 1]
  const double* gw;
  const double* hl;      // HL_mu
  double* part;
};

// Coefficients of the order-th derivative of the piece polynomial in its
// scaled variable xi = (x - centre)/h, including the 1/h^order factor
// (poly.py:56-74): d_j = c_{j+r} (j+r)!/j! / h^r.
__host__ __device__ inline int deriv_coeffs(const double* c, int ncoef, int r, double h, double* d) {
  const int nd = ncoef - r;
  double hr = 1.0;
  for (int q = 0; q < r; ++q) hr *= h;
  for (int j = 0; j < nd; ++j) {
    double fall = 1.0;
    for (int q = j + 1; q <= j + r; ++q) fall *= q;
    d[j] = c[j + r] * fall / hr;
  }
  return nd;
}

__host__ __device__ inline double horner(const double* d, int nd, double x) {
  double v = d[nd - 1];
  for (int j = nd - 2; j >= 0; --j) v = v * x + d[j];
  return v;
}

__host__ __device__ inline void piece_coeffs(const double* f, int mu, int64_t t, int off, const Energy1DArgs& a, double* c) {
  Line1DArgs la;
  la.n = a.n;
  la.off = off;
  la.periodic = a.periodic;
  la.kl = a.kl;
  la.kh = a.kh;
  double L[kMax1D + 1], R[kMax1D + 1];
  load_pair(f, mu, t, la, a.gl, a.gh, L, R);
  interp1d(a.hl, mu, L, R, c);
}

// seminorm_sq (diagnostics.py:201-212): sum over pieces of the Gauss integral
// of the squared order-th derivative over [centre - h/2, centre + h/2].
__global__ void seminorm1d_kernel(Energy1DArgs a) {
  __shared__ double sh[kRedThreads];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double local = 0.0;
  if (t < a.nt) {
    double c[2 * kMax1D + 2], d[2 * kMax1D + 2];
    piece_coeffs(a.f, a.mu, t, a.off, a, c);
    const int nd = deriv_coeffs(c, 2 * a.mu + 2, a.order, a.h, d);
    if (nd > 0) {
      for (int p = 0; p < a.npts; ++p) {
        const double q = horner(d, nd, 0.5 * a.gx[p]);
        local += 0.5 * a.h * a.gw[p] * q * q;
      }
    }
  }
  const double bs = block_sum(local * a.scale, sh);
  if (threadIdx.x == 0) a.part[blockIdx.x] = bs;
}

// conservative_energy (diagnostics.py:190-226) on a periodic grid:
// E = |P+|^2_{m+1} + |P-|^2_{m+1}, P± = cur - S± prev, S± w(x) = w(x ± delta).
// Within cur piece t (edges at its flanking source nodes) the shifted prev
// pieces are the ones centred on those two nodes, split at xi_s = -/+ delta/h:
// every union piece (pp_subtract's merged breakpoints) lies in one cur and one
// prev piece, and both derivatives are evaluated in their own scaled
// variables at the union piece's Gauss points (npts = m + 1: exact).
__host__ __device__ inline double cons_energy_piece(const Energy1DArgs& a, int64_t t) {
  const int m = a.mu, K = 2 * m + 2;
  double cc[2 * kMax1D + 2], cl[2 * kMax1D + 2], cr[2 * kMax1D + 2];
  double dc[2 * kMax1D + 2], dl[2 * kMax1D + 2], dr[2 * kMax1D + 2];
  // prev pieces centred on cur piece t's left / right source nodes
  const int64_t sl = pmod(t + a.off, a.n), sr = pmod(t + a.off + 1, a.n);
  piece_coeffs(a.f, m, t, a.off, a, cc);
  piece_coeffs(a.g, m, sl, a.offg, a, cl);
  piece_coeffs(a.g, m, sr, a.offg, a, cr);
  const int nd = deriv_coeffs(cc, K, m + 1, a.h, dc);
  deriv_coeffs(cl, K, m + 1, a.h, dl);
  deriv_coeffs(cr, K, m + 1, a.h, dr);
  const double dx = a.delta / a.h;
  double local = 0.0;
  for (int sgn = 1; sgn >= -1; sgn -= 2) {  // P+ evaluates prev at x + delta, P- at x - delta
    const double xs = -sgn * dx;            // split point in cur's scaled variable
    for (int piece = 0; piece < 2; ++piece) {
      const double lo = piece ? xs : -0.5, hi = piece ? 0.5 : xs;
      if (hi <= lo) continue;
      const double* dp = piece ? dr : dl;
      const double sh_p = sgn * dx + (piece ? -0.5 : 0.5);  // xi_prev = xi + sh_p
      for (int p = 0; p < a.npts; ++p) {
        const double xi = 0.5 * (lo + hi) + 0.5 * (hi - lo) * a.gx[p];
        const double q = horner(dc, nd, xi) - horner(dp, nd, xi + sh_p);
        local += 0.5 * (hi - lo) * a.h * a.gw[p] * q * q;
      }
    }
  }
  return local;
}

__global__ void cons_energy1d_kernel(Energy1DArgs a) {
  __shared__ double sh[kRedThreads];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double local = t < a.nt ? cons_energy_piece(a, t) : 0.0;
  const double bs = block_sum(local, sh);

  if (threadIdx.x == 0) a.part[blockIdx.x] = bs;
}

}  // namespace hw
