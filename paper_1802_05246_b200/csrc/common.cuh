// Shared device-side helpers: boundary reflection signs, source row/column
// resolution (periodic wrap, wall ghosts, slab halos) and error plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hermb200.h"

namespace hw {

constexpr int kMaxFast = 8;  // templated fast paths exist for m = 1..kMaxFast

// boundary.py:56-62 _signs: dirichlet0 -> (-1)^(l+1), neumann0 -> (-1)^l.
__host__ __device__ inline double refl_sign(int kind, int l) {
  const bool odd = (l & 1) != 0;
  if (kind == HW_DIRICHLET0) return odd ? 1.0 : -1.0;
  return odd ? -1.0 : 1.0;  // HW_NEUMANN0
}

__host__ __device__ inline int64_t pmod(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// One resolved source row: pointer to its first node plus the x-ghost
// reflection to apply (kind 0 = none) and its Dirichlet datum.
struct RowRef {
  const double* p;
  int kind;
  double g;
};

// Plain-struct mirror of hw_rows2d usable inside kernels.
struct Rows {
  const double* base;
  const double* lo;
  const double* hi;
  int64_t row0, nrows;
};

// Resolution of global source row s (boundary.py:101-132 _gather_axis along
// x): local rows, then slab halos, then periodic wrap / wall ghost.
__device__ inline RowRef resolve_row(const Rows& r, int64_t s, int64_t nx,
                                     int64_t row_len, int periodic, int klo,
                                     int khi, double glo, double ghi) {
  if (s >= r.row0 && s < r.row0 + r.nrows) return {r.base + (s - r.row0) * row_len, 0, 0.0};
  if (s == r.row0 - 1 && r.lo) return {r.lo, 0, 0.0};
  if (s == r.row0 + r.nrows && r.hi) return {r.hi, 0, 0.0};
  if (periodic) {
    const int64_t w = pmod(s, nx);
    return {r.base + (w - r.row0) * row_len, 0, 0.0};
  }
  if (s < 0) return {r.base + (0 - r.row0) * row_len, klo, glo};
  return {r.base + (nx - 1 - r.row0) * row_len, khi, ghi};
}

// Column resolution along y: returns the source column and the y-ghost kind.
struct ColRef {
  int64_t c;
  int kind;
  double g;
};

__device__ inline ColRef resolve_col(int64_t c, int64_t ny, int periodic, int klo, int khi,
                                     double glo, double ghi) {
  if (c >= 0 && c < ny) return {c, 0, 0.0};
  if (periodic) return {pmod(c, ny), 0, 0.0};
  if (c < 0) return {0, klo, glo};
  return {ny - 1, khi, ghi};
}

// Value of coefficient (k,l) of a 2D node after x- then y-reflection
// (boundary.py:79-98 ghost_data_2d applied by corner_sources x first, then y;
// boundary.py:150-168).  `gx_scale` is 1 for u and 0 for v (the velocity
// reflects around zero: dissipative.py:229, boundary.py:109-111).
__device__ inline double ghosted(double val, int k, int l, int xkind, double gx, int ykind,
                                 double gy) {
  if (xkind) {
    val *= refl_sign(xkind, k);
    if (k == 0 && l == 0 && xkind == HW_DIRICHLET0) val += 2.0 * gx;
  }
  if (ykind) {
    val *= refl_sign(ykind, l);
    if (k == 0 && l == 0 && ykind == HW_DIRICHLET0) val += 2.0 * gy;
  }
  return val;
}

// Source node index offset of target t: from PRIMAL (t, t+1), from DUAL
// (t-1, t) (boundary.py:119-130).
__host__ __device__ inline int src_offset(int parity_src) { return parity_src == HW_PRIMAL ? 0 : -1; }

inline int64_t target_count(int64_t n_src, int parity_src, int periodic) {
  if (periodic) return n_src;
  return parity_src == HW_PRIMAL ? n_src - 1 : n_src + 1;
}

}  // namespace hw
