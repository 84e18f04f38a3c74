// The reference's lower-level batched building blocks (the
// functions hermwave re-exports beside the steps): interpolation, the
// Taylor recursions, Horner summation, the conservative update, the
// boundary gathers and ghost reflections.  The fused step kernels
// (cellmap.cuh, line1d.cuh) never call these; they exist so code written
// against hermwave's lower-level API runs on the device too.
//
// Element-wise arithmetic follows the reference's numpy expressions operation
// by operation with explicitly rounded multiplies and adds (no FMA
// contraction), so expand_taylor(_2d), eval_series, the ghosts and gathers
// are bit-identical to the reference; the contractions (interpolation,
// conservative update) run in a fixed sequential order where numpy calls
// BLAS, so they agree to rounding.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace hw {

constexpr int kLLMaxN = 26;  // 2 mu + 2 for mu <= 12

__device__ inline double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ inline double add_rn(double a, double b) { return __dadd_rn(a, b); }

// interp.py:78-90 apply_interp: out[b][a] = sum_i M[a][i] data[b][i].
__global__ void apply_interp_kernel(const double* data, double* out, int64_t batch, int n, const double* M) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * n) return;
  const int64_t b = idx / n;
  const int a = (int)(idx - b * n);
  const double* d = data + b * n;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = fma(M[a * n + i], d[i], s);
  out[idx] = s;
}

// interp.py:93-111 apply_interp_2d: out = M_x D M_y^T with D[i][j],
// i = sx (mux+1) + k, j = sy (muy+1) + l stacked from data[sx][sy][k][l].
// One thread per (batch element, output row a).
__global__ void apply_interp2d_kernel(const double* data, double* out, int64_t batch, int mux, int muy,
                                      const double* Mx, const double* My) {
  const int nx = 2 * mux + 2, ny = 2 * muy + 2, wx = mux + 1, wy = muy + 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * nx) return;
  const int64_t b = idx / nx;
  const int a = (int)(idx - b * nx);
  const double* d = data + b * 4 * wx * wy;  // [sx][sy][k][l]
  double t[kLLMaxN];
  for (int j = 0; j < ny; ++j) {
    const int sy = j / wy, l = j % wy;
    double s = 0.0;
    for (int i = 0; i < nx; ++i) {
      const int sx = i / wx, k = i % wx;
      s = fma(Mx[a * nx + i], d[((sx * 2 + sy) * wx + k) * wy + l], s);
    }
    t[j] = s;
  }
  double* o = out + (b * nx + a) * ny;
  for (int c = 0; c < ny; ++c) {
    double s = 0.0;
    for (int j = 0; j < ny; ++j) s = fma(t[j], My[c * ny + j], s);
    o[c] = s;
  }
}

// dissipative.py:77-106 expand_taylor, one thread per batch element.  Tables
// are (batch, L, smax + 1).  `fterm` (nullable): (batch, lv, smax) with the
// reference's forcing terms fac * forcing(l, s-1, centers, t) already formed.
__global__ void expand_taylor_kernel(const double* cu, const double* cv, double* cut, double* cvt, int64_t batch,
                                     int lu, int lv, double dt, double r, int smax, const double* fterm) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int S = smax + 1;
  double* U = cut + b * lu * S;
  double* V = cvt + b * lv * S;
  for (int l = 0; l < lu; ++l) {
    U[l * S] = cu[b * lu + l];
    for (int s = 1; s < S; ++s) U[l * S + s] = 0.0;
  }
  for (int l = 0; l < lv; ++l) {
    V[l * S] = cv[b * lv + l];
    for (int s = 1; s < S; ++s) V[l * S + s] = 0.0;
  }
  const int nsrc = lv < lu - 2 ? lv : lu - 2;
  for (int s = 1; s <= smax; ++s) {
    const double ds = dt / (double)s, rs = r / (double)s;
    for (int l = 0; l < lv; ++l) U[l * S + s] = mul_rn(ds, V[l * S + s - 1]);
    for (int l = 0; l < nsrc; ++l)  // (r/s) * mul * c, left to right
      V[l * S + s] = mul_rn(mul_rn(rs, (double)((l + 2) * (l + 1))), U[(l + 2) * S + s - 1]);
    if (fterm)
      for (int l = 0; l < lv; ++l) V[l * S + s] = add_rn(V[l * S + s], fterm[(b * lv + l) * smax + s - 1]);
  }
}

// dissipative.py:184-212 expand_taylor_2d, one thread per batch element.
// Tables (batch, K, K, smax + 1); d0 is (batch, lv, lv); d1 (nullable) is
// (batch, K-2, K-2).
__global__ void expand_taylor2d_kernel(const double* c0, const double* d0, const double* d1, double* ct, double* dtb,
                                       int64_t batch, int K, int lv, double dt, double rx, double ry, int smax) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int S = smax + 1;
  double* C = ct + b * K * K * S;
  double* D = dtb + b * K * K * S;
  auto at = [&](int k, int l, int s) { return (k * K + l) * S + s; };
  for (int k = 0; k < K; ++k)
    for (int l = 0; l < K; ++l) {
      C[at(k, l, 0)] = c0[(b * K + k) * K + l];
      D[at(k, l, 0)] = (k < lv && l < lv) ? d0[(b * lv + k) * lv + l] : 0.0;
      for (int s = 1; s < S; ++s) C[at(k, l, s)] = D[at(k, l, s)] = 0.0;
    }
  for (int s = 1; s <= smax; ++s) {
    const double ds = dt / (double)s;
    for (int k = 0; k < K; ++k)
      for (int l = 0; l < K; ++l) C[at(k, l, s)] = mul_rn(ds, D[at(k, l, s - 1)]);
    if (s == 1 && d1) {
      for (int k = 0; k < K - 2; ++k)
        for (int l = 0; l < K - 2; ++l) D[at(k, l, 1)] = d1[(b * (K - 2) + k) * (K - 2) + l];
      continue;
    }
    const double rxs = rx / (double)s, rys = ry / (double)s;
    for (int k = 0; k < K - 2; ++k) {
      const double fx = mul_rn(rxs, (double)((k + 2) * (k + 1)));
      for (int l = 0; l < K; ++l) D[at(k, l, s)] = mul_rn(fx, C[at(k + 2, l, s - 1)]);
    }
    for (int k = 0; k < K; ++k)
      for (int l = 0; l < K - 2; ++l) {
        const double fy = mul_rn(rys, (double)((l + 2) * (l + 1)));
        D[at(k, l, s)] = add_rn(D[at(k, l, s)], mul_rn(fy, C[at(k, l + 2, s - 1)]));
      }
  }
}

// dissipative.py:116-121 eval_series: out = table[-1]; out = out * theta + table[s].
__global__ void eval_series_kernel(const double* tab, double* out, int64_t batch, int S, double theta) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double* t = tab + b * S;
  double o = t[S - 1];
  for (int s = S - 2; s >= 0; --s) o = add_rn(mul_rn(o, theta), t[s]);
  out[b] = o;
}

// conservative.py:115-136: out[b][q] = 2 (sum_j W[q][j] c[b][j]) - prev[b][q]
// (1D: W is (m+1) x (2m+2); 2D: WT flattened to (m+1)^2 x (2m+2)^2).
__global__ void cons_update_kernel(const double* coeffs, const double* prev, double* out, int64_t batch, int nq,
                                   int nj, const double* W) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * nq) return;
  const int64_t b = idx / nq;
  const int q = (int)(idx - b * nq);
  const double* c = coeffs + b * nj;
  double s = 0.0;
  for (int j = 0; j < nj; ++j) s = fma(W[q * nj + j], c[j], s);
  out[idx] = add_rn(mul_rn(2.0, s), -prev[idx]);
}

// boundary.py:101-168 pair_sources / corner_sources (data part): for every
// target node the flanking source blocks, with periodic wrap or wall ghosts.
// 1D: out (nt, 2, w0); 2D: out (ntx, nty, 2, 2, w0, w1), x gathered first.
struct GatherArgs {
  const double* src;
  double* out;
  int64_t nx, ny, ntx, nty;  // ny = nty = 1 in 1D
  int w0, w1;                // block widths (w1 = 1 in 1D)
  int off, periodic, dims;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;
};

__global__ void gather_kernel(GatherArgs a) {
  const int64_t per = (int64_t)(a.dims == 2 ? 4 : 2) * a.w0 * a.w1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.ntx * a.nty * per) return;
  const int64_t cell = idx / per;
  int64_t r = idx - cell * per;
  const int l = (int)(r % a.w1);
  r /= a.w1;
  const int k = (int)(r % a.w0);
  r /= a.w0;
  const int sy = a.dims == 2 ? (int)(r % 2) : 0;
  const int sx = a.dims == 2 ? (int)(r / 2) : (int)r;
  const int64_t tx = cell / a.nty, ty = cell - tx * a.nty;
  const Rows rows{a.src, nullptr, nullptr, 0, a.nx};
  const RowRef rr = resolve_row(rows, tx + a.off + sx, a.nx, a.ny * a.w0 * a.w1, a.periodic, a.kxl, a.kxh, a.gxl,
                                a.gxh);
  ColRef cc{0, 0, 0.0};
  if (a.dims == 2) cc = resolve_col(ty + a.off + sy, a.ny, a.periodic, a.kyl, a.kyh, a.gyl, a.gyh);
  double v = rr.p[(cc.c * a.w0 + k) * a.w1 + l];
  // boundary.py:65-98: x reflection (ghost_data / ghost_data_2d along k),
  // then, in 2D, y reflection along l; a Dirichlet datum shifts c_0 (c_00)
  // only when it is nonzero
  if (rr.kind) {
    v *= refl_sign(rr.kind, k);
    if (k == 0 && l == 0 && rr.kind == HW_DIRICHLET0 && rr.g != 0.0) v += 2.0 * rr.g;
  }
  if (cc.kind) {
    v *= refl_sign(cc.kind, l);
    if (k == 0 && l == 0 && cc.kind == HW_DIRICHLET0 && cc.g != 0.0) v += 2.0 * cc.g;
  }
  a.out[idx] = v;
}

// boundary.py:65-98 ghost_data / ghost_data_2d on (batch, n0, n1) blocks:
// signs along axis `axis` (0: k, 1: l); the Dirichlet datum shifts [0][0].
__global__ void ghost_kernel(const double* in, double* out, int64_t batch, int n0, int n1, int axis, int kind,
                             double value) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * n0 * n1) return;
  const int e = (int)(idx % (n0 * n1)), k = e / n1, l = e % n1;
  double v = in[idx] * refl_sign(kind, axis == 0 ? k : l);
  if (kind == HW_DIRICHLET0 && value != 0.0 && k == 0 && l == 0) v += 2.0 * value;
  out[idx] = v;
}

// driver.py:195-200 _scale_cols: column l of every row times h^l / l!, the
// factor built by the same running product fac[l] = fac[l-1] * h / l.
__global__ void scale_cols_kernel(const double* in, double* out, int64_t rows, int cols, double h) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int l = (int)(idx % cols);
  double fac = 1.0;
  for (int q = 1; q <= l; ++q) fac = fac * h / (double)q;
  out[idx] = in[idx] * fac;
}

}  // namespace hw
