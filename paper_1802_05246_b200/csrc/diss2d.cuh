// Fused 2D dissipative half step (dissipative.py:215-247 half_step_2d):
// corner gather + four tensor-product Hermite interpolants + the stabilised
// Taylor recursion evaluated at theta = 1/2, in one kernel.
//
// Algebra (see DESIGN.md §3 for the derivation):
//  * Parity split.  The right block of every Hermite matrix is (-1)^(a+k) times
//    the left block HL, so for output rows a of parity PA and columns b of
//    parity PB the 2x2 corner blocks U_sxsy collapse to one signed sum
//        G[k][l] = U00 + (-1)^(PA+k) U10 + (-1)^(PB+l) U01 + (-1)^(PA+k+PB+l) U11
//    and C[a][b] = sum_kl HL_x[a][k] HL_y[b][l] G[k][l].
//  * Closed-form recursion.  With the stabilised first stage d1 the recursion
//    of expand_taylor_2d (dissipative.py:184-212) sums to
//        u = cmm + sum_ij C(i+j,i) rx^i ry^j (k+2i)!/k! (l+2j)!/l!
//                    [A_{i+j} d0 + B_{i+j} d1][k+2i][l+2j]
//        v =       (same taps with Gamma_{i+j}, Delta_{i+j})
//    A_p = th^(2p+1) dt^(p+1)/(2p+1)!, B_p = th^(2p+2) dt^(p+1)/(2p+2)!,
//    Gamma_p = th^(2p) dt^p/(2p)!,     Delta_p = th^(2p+1) dt^p/(2p+1)!,
//    each zeroed when its stage exceeds the cap.  Writing phi(a) = a! r^floor(a/2)
//    the tap weight factors as g(i,j) phi_x(a) phi_y(b) / (phi_x(k) phi_y(l)),
//    so the phi's fold into the interpolation matrices (the tables below are
//    phi-scaled) and the taps use the tiny g(i,j) tables.  The stabilised
//    d1 = rx mul c_x[a+2] + ry mul c_y[.,b+2] becomes
//        phi_x(a)phi_y(b) d1[a][b] = c~_x[a+2][b] + c~_y[a][b+2]
//    because phi(a) r (a+2)(a+1) = phi(a+2).
//  * Each warp owns one parity class (PA,PB) for 32 consecutive target cells
//    (one per lane); all table reads are warp-uniform compile-time offsets, so
//    they are constant-bank operands of DFMA.  Intermediates never leave
//    registers: columns b of d0 / d1 are produced one at a time and scattered
//    straight into the class's output accumulators.
#pragma once

#include "common.cuh"

namespace hw {

template <int M>
struct Diss2DTables {
  static constexpr int K = 2 * M + 2;
  double mx[K][M + 1];    // phi_x(a) HL_m[a][k]
  double my[K][M + 1];    // phi_y(b) HL_m[b][l]
  double mx1[2 * M][M];   // phi_x(a) HL_{m-1}[a][k]
  double my1[2 * M][M];   // phi_y(b) HL_{m-1}[b][l]
  double gA[M][M], gB[M][M], gG[M][M], gD[M][M];
  double inv[M + 1][M + 1];  // 1 / (phi_x(k) phi_y(l))
};

struct Step2DArgs {
  Rows u, v;
  double* ud;
  double* vd;
  int64_t nx, ny;      // global source counts
  int64_t trow0, ntrows, nty;
  int off;             // source offset of target index (0 primal, -1 dual)
  int periodic;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;
};

template <int M>
struct Diss2DParams {
  Step2DArgs a;
  Diss2DTables<M> t;
};

constexpr int kTileJ = 32;  // target cells per CTA along y (one per lane)

template <int M>
struct Diss2DSmem {
  static constexpr int PU = (M + 1) * (M + 1);
  static constexpr int PV = M * M;
  static constexpr int PUP = PU | 1;  // odd stride: conflict-free 8B lane access
  static constexpr int PVP = PV | 1;
  static constexpr int NQ = kTileJ + 1;
  static constexpr int bytes = (2 * NQ * PUP + 2 * NQ * PVP) * 8;
};

// Stage two source rows x 33 source columns of one field into shared memory
// with ghost reflection applied.  Coalesced: consecutive threads read
// consecutive doubles of the (contiguous) row segment.
template <int P, int PP, int NL>
__device__ inline void stage_rows(double* __restrict__ dst, const RowRef& r0, const RowRef& r1,
                                  int64_t c0, const Step2DArgs& a, bool is_u) {
  constexpr int NQ = kTileJ + 1;
  constexpr int TOT = 2 * NQ * P;
  for (int idx = threadIdx.x; idx < TOT; idx += blockDim.x) {
    const int r = idx / (NQ * P);
    const int rem = idx - r * (NQ * P);
    const int q = rem / P;
    const int e = rem - q * P;
    const RowRef& R = r ? r1 : r0;
    const ColRef C = resolve_col(c0 + q, a.ny, a.periodic, a.kyl, a.kyh, is_u ? a.gyl : 0.0,
                                 is_u ? a.gyh : 0.0);
    double val = R.p[C.c * P + e];
    if (R.kind | C.kind) val = ghosted(val, e / NL, e % NL, R.kind, R.g, C.kind, C.g);
    dst[(r * NQ + q) * PP + e] = val;
  }
}

// Scatter one column b of a scaled d-array (rows a = PA + 2*ia) into the
// class accumulators with the g tables gu (u outputs) and gv (v outputs).
template <int M, int PA, int PB>
__device__ __forceinline__ void taps(const double (&d)[M], const int b, const double (&gu)[M][M],
                                     const double (&gv)[M][M],
                                     double (&au)[(M - PA) / 2 + 1][(M - PB) / 2 + 1],
                                     double (&av)[(M - 1 - PA) / 2 + 1][(M - 1 - PB) / 2 + 1]) {
#pragma unroll
  for (int ia = 0; ia < M; ++ia) {
    const int arow = PA + 2 * ia;
    if (arow >= 2 * M) continue;
#pragma unroll
    for (int i = 0; i <= ia; ++i) {
      const int k = arow - 2 * i;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const int l = b - 2 * j;
        if (l < 0) continue;
        if (k <= M && l <= M) au[(k - PA) / 2][(l - PB) / 2] = fma(gu[i][j], d[ia], au[(k - PA) / 2][(l - PB) / 2]);
        if (k < M && l < M) av[(k - PA) / 2][(l - PB) / 2] = fma(gv[i][j], d[ia], av[(k - PA) / 2][(l - PB) / 2]);
      }
    }
  }
}

template <int M, int PA, int PB>
__device__ __forceinline__ void diss2d_class(const Diss2DTables<M>& T, const double* __restrict__ u00,
                                             const double* __restrict__ u10, const double* __restrict__ v00,
                                             const double* __restrict__ v10, double* __restrict__ ou,
                                             double* __restrict__ ov) {
  using S = Diss2DSmem<M>;
  const double* u01 = u00 + S::PUP;
  const double* u11 = u10 + S::PUP;
  const double* v01 = v00 + S::PVP;
  const double* v11 = v10 + S::PVP;
  constexpr int NKU = (M - PA) / 2 + 1, NLU = (M - PB) / 2 + 1;
  constexpr int NKV = (M - 1 - PA) / 2 + 1, NLV = (M - 1 - PB) / 2 + 1;
  constexpr int NA = M;  // rows a = PA + 2 ia of the 2M-row arrays
  double au[NKU][NLU];
  double av[NKV][NLV];
#pragma unroll
  for (int x = 0; x < NKU; ++x)
#pragma unroll
    for (int y = 0; y < NLU; ++y) au[x][y] = 0.0;
#pragma unroll
  for (int x = 0; x < NKV; ++x)
#pragma unroll
    for (int y = 0; y < NLV; ++y) av[x][y] = 0.0;

  // ---- sweep V: d0 = I_{m-1,m-1} v (phi-scaled), taps A (u) and Gamma (v)
  {
    double G[M][M];
#pragma unroll
    for (int k = 0; k < M; ++k)
#pragma unroll
      for (int l = 0; l < M; ++l) {
        const int e = k * M + l;
        const bool sx = ((PA + k) & 1) == 0, sy = ((PB + l) & 1) == 0;
        const double A = sx ? v00[e] + v10[e] : v00[e] - v10[e];
        const double B = sx ? v01[e] + v11[e] : v01[e] - v11[e];
        G[k][l] = sy ? A + B : A - B;
      }
#pragma unroll
    for (int b = PB; b < 2 * M; b += 2) {
      double Y[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < M; ++l) s = fma(T.my1[b][l], G[k][l], s);
        Y[k] = s;
      }
      double d[M];
#pragma unroll
      for (int ia = 0; ia < NA; ++ia) {
        const int arow = PA + 2 * ia;
        double s = 0.0;
        if (arow < 2 * M) {
#pragma unroll
          for (int k = 0; k < M; ++k) s = fma(T.mx1[arow][k], Y[k], s);
        }
        d[ia] = s;
      }
      taps<M, PA, PB>(d, b, T.gA, T.gG, au, av);
    }
  }

  // ---- sweep U: cmm (low block), c_x = I_{m,m-1} u, c_y = I_{m-1,m} u
  {
    double G[M + 1][M + 1];
#pragma unroll
    for (int k = 0; k <= M; ++k)
#pragma unroll
      for (int l = 0; l <= M; ++l) {
        const int e = k * (M + 1) + l;
        const bool sx = ((PA + k) & 1) == 0, sy = ((PB + l) & 1) == 0;
        const double A = sx ? u00[e] + u10[e] : u00[e] - u10[e];
        const double B = sx ? u01[e] + u11[e] : u01[e] - u11[e];
        G[k][l] = sy ? A + B : A - B;
      }
    double cx[M];  // c~_x[a+2][b] of the previous column (held for d1)
#pragma unroll
    for (int ia = 0; ia < M; ++ia) cx[ia] = 0.0;
#pragma unroll
    for (int b = PB; b < 2 * M + 2; b += 2) {
      // Yu[k] = sum_l phi_y(b) HL_m[b][l] G[k][l]
      double Y[M + 1];
#pragma unroll
      for (int k = 0; k <= M; ++k) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l <= M; ++l) s = fma(T.my[b][l], G[k][l], s);
        Y[k] = s;
      }
      if (b <= M) {  // scaled cmm low block feeds u directly
#pragma unroll
        for (int ia = 0; ia < NKU; ++ia) {
          const int arow = PA + 2 * ia;
          double s = au[ia][(b - PB) / 2];
#pragma unroll
          for (int k = 0; k <= M; ++k) s = fma(T.mx[arow][k], Y[k], s);
          au[ia][(b - PB) / 2] = s;
        }
      }
      if (b >= 2) {  // c~_y[a][b] completes d1 column b-2
        double d[M];
#pragma unroll
        for (int ia = 0; ia < M; ++ia) {
          const int arow = PA + 2 * ia;
          double s = cx[ia];
          if (arow < 2 * M) {
#pragma unroll
            for (int k = 0; k < M; ++k) s = fma(T.mx1[arow][k], Y[k], s);
          }
          d[ia] = s;
        }
        taps<M, PA, PB>(d, b - 2, T.gB, T.gD, au, av);
      }
      if (b < 2 * M) {  // c~_x[a+2][b] from I_{m,m-1}
        double Yp[M + 1];
#pragma unroll
        for (int k = 0; k <= M; ++k) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < M; ++l) s = fma(T.my1[b][l], G[k][l], s);
          Yp[k] = s;
        }
#pragma unroll
        for (int ia = 0; ia < M; ++ia) {
          const int arow = PA + 2 * ia;
          double s = 0.0;
          if (arow < 2 * M) {
#pragma unroll
            for (int k = 0; k <= M; ++k) s = fma(T.mx[arow + 2][k], Yp[k], s);
          }
          cx[ia] = s;
        }
      }
    }
  }

  // ---- unscale and store this class's coefficients (straight to global)
  if (ou == nullptr) return;
#pragma unroll
  for (int x = 0; x < NKU; ++x)
#pragma unroll
    for (int y = 0; y < NLU; ++y) {
      const int k = PA + 2 * x, l = PB + 2 * y;
      ou[k * (M + 1) + l] = T.inv[k][l] * au[x][y];
    }
#pragma unroll
  for (int x = 0; x < NKV; ++x)
#pragma unroll
    for (int y = 0; y < NLV; ++y) {
      const int k = PA + 2 * x, l = PB + 2 * y;
      if (k < M && l < M) ov[k * M + l] = T.inv[k][l] * av[x][y];
    }
}

// Async 8-byte global->shared copy (LDGSTS); completion tracked per thread
// with commit/wait groups.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Target rows per tile (= warps per CTA, one row per warp).  The staged
// source block is double buffered, so large orders use fewer rows to fit.
template <int M>
constexpr int tile_rows() {
  return M <= 4 ? 4 : (M <= 6 ? 2 : 1);
}

// Issue the async copies of one tile's source block (kTileRows+1 rows x 33
// nodes) of one field into shared memory.  Ghost/wrapped nodes are copied
// from their mirror source; reflection signs are applied after arrival.
template <int P, int PP, int TR>
__device__ inline void issue_tile(double* __restrict__ dst, const Rows& R, int64_t s_first, int64_t c_first,
                                  const Step2DArgs& a) {
  constexpr int NQ = kTileJ + 1;
  const bool contiguous = c_first >= 0 && c_first + NQ <= a.ny;
  for (int r = 0; r <= TR; ++r) {
    const RowRef rr = resolve_row(R, s_first + r, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, 0.0, 0.0);
    double* d = dst + r * NQ * PP;
    if (contiguous) {
      // interior columns: the row segment is one contiguous block
      const double* src = rr.p + c_first * P;
      int q = threadIdx.x / P, e = threadIdx.x - (threadIdx.x / P) * P;
      const int dq = blockDim.x / P, de = blockDim.x - dq * P;
      for (int idx = threadIdx.x; idx < NQ * P; idx += blockDim.x) {
        cp_async8(d + q * PP + e, src + idx);
        q += dq;
        e += de;
        if (e >= P) {
          e -= P;
          ++q;
        }
      }
    } else {
      for (int idx = threadIdx.x; idx < NQ * P; idx += blockDim.x) {
        const int q = idx / P;
        const int e = idx - q * P;
        const ColRef cc = resolve_col(c_first + q, a.ny, a.periodic, a.kyl, a.kyh, 0.0, 0.0);
        cp_async8(d + q * PP + e, rr.p + cc.c * P + e);
      }
    }
  }
}

// Apply wall reflections to the ghost nodes of a staged tile (walls only).
template <int P, int PP, int NL, int TR>
__device__ inline void fix_ghosts(double* __restrict__ dst, int64_t s_first, int64_t c_first, const Step2DArgs& a,
                                  bool is_u) {
  constexpr int NQ = kTileJ + 1;
  for (int idx = threadIdx.x; idx < (TR + 1) * NQ * P; idx += blockDim.x) {
    const int r = idx / (NQ * P);
    const int rem = idx - r * (NQ * P);
    const int q = rem / P;
    const int e = rem - q * P;
    const int64_t s = s_first + r, c = c_first + q;
    int xk = 0, yk = 0;
    double gx = 0.0, gy = 0.0;
    if (s < 0) { xk = a.kxl; gx = a.gxl; }
    else if (s >= a.nx) { xk = a.kxh; gx = a.gxh; }
    if (c < 0) { yk = a.kyl; gy = a.gyl; }
    else if (c >= a.ny) { yk = a.kyh; gy = a.gyh; }
    if (xk | yk) {
      double* p = dst + (r * NQ + q) * PP + e;
      *p = ghosted(*p, e / NL, e % NL, xk, is_u ? gx : 0.0, yk, is_u ? gy : 0.0);
    }
  }
}

// Persistent kernel: each CTA walks tiles of kTileRows x 32 target cells,
// prefetching the next tile's source rows with cp.async while its four warps
// compute the current one.  All warps run the same parity class at the same
// time (warp w = tile row w), which keeps the instruction working set to one
// class's code.
template <int M>
__global__ void __launch_bounds__(32 * tile_rows<M>(), M <= 4 ? 2 : 1)
    diss2d_kernel(const __grid_constant__ Diss2DParams<M> P) {
  using S = Diss2DSmem<M>;
  constexpr int kTileRows = tile_rows<M>();
  constexpr int PU = S::PU, PV = S::PV, NQ = S::NQ;
  constexpr int BU = (kTileRows + 1) * NQ * S::PUP;  // doubles per u buffer
  constexpr int BV = (kTileRows + 1) * NQ * S::PVP;
  extern __shared__ __align__(16) double smem[];
  const Step2DArgs& a = P.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tcols = (a.nty + kTileJ - 1) / kTileJ;
  const int64_t trows = (a.ntrows + kTileRows - 1) / kTileRows;
  const int64_t ntiles = tcols * trows;
  const bool walls = !a.periodic;

  auto tile_origin = [&](int64_t tile, int64_t& tr0, int64_t& j0) {
    const int64_t ti = tile / tcols;
    tr0 = ti * kTileRows;
    j0 = (tile - ti * tcols) * kTileJ;
  };
  auto issue = [&](int64_t tile, int b) {
    int64_t tr0, j0;
    tile_origin(tile, tr0, j0);
    const int64_t s_first = a.trow0 + tr0 + a.off, c_first = j0 + a.off;
    issue_tile<PU, S::PUP, kTileRows>(smem + b * (BU + BV), a.u, s_first, c_first, a);
    issue_tile<PV, S::PVP, kTileRows>(smem + b * (BU + BV) + BU, a.v, s_first, c_first, a);
    cp_async_commit();
  };

  int b = 0;
  int64_t tile = blockIdx.x;
  if (tile < ntiles) issue(tile, 0);
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t next = tile + gridDim.x;
    if (next < ntiles) {
      issue(next, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    int64_t tr0, j0;
    tile_origin(tile, tr0, j0);
    double* su = smem + b * (BU + BV);
    double* sv = su + BU;
    if (walls) {
      const int64_t s_first = a.trow0 + tr0 + a.off, c_first = j0 + a.off;
      const bool edge = s_first < 0 || s_first + kTileRows >= a.nx || c_first < 0 || c_first + kTileJ >= a.ny;
      if (edge) {
        fix_ghosts<PU, S::PUP, M + 1, kTileRows>(su, s_first, c_first, a, true);
        fix_ghosts<PV, S::PVP, M, kTileRows>(sv, s_first, c_first, a, false);
        __syncthreads();
      }
    }
    const int64_t tr = tr0 + warp;
    const int64_t j = j0 + lane;
    const bool valid = tr < a.ntrows && j < a.nty;
    double* ou = valid ? a.ud + (tr * a.nty + j) * PU : nullptr;
    double* ov = valid ? a.vd + (tr * a.nty + j) * PV : nullptr;
    if (tr < a.ntrows) {
      const double* u0 = su + (warp * NQ + lane) * S::PUP;
      const double* u1 = u0 + NQ * S::PUP;
      const double* v0 = sv + (warp * NQ + lane) * S::PVP;
      const double* v1 = v0 + NQ * S::PVP;
      // one class at a time (the __syncwarp fences stop the scheduler from
      // interleaving classes, which would multiply live registers)
      diss2d_class<M, 0, 0>(P.t, u0, u1, v0, v1, ou, ov);
      __syncwarp();
      diss2d_class<M, 0, 1>(P.t, u0, u1, v0, v1, ou, ov);
      __syncwarp();
      diss2d_class<M, 1, 0>(P.t, u0, u1, v0, v1, ou, ov);
      __syncwarp();
      diss2d_class<M, 1, 1>(P.t, u0, u1, v0, v1, ou, ov);
    }
    __syncthreads();  // buffer b is refilled by the issue() of the next iteration
    b ^= 1;
  }
}

template <int M>
constexpr int diss2d_smem_bytes() {
  using S = Diss2DSmem<M>;
  return 2 * (tile_rows<M>() + 1) * S::NQ * (S::PUP + S::PVP) * 8;
}

}  // namespace hw
