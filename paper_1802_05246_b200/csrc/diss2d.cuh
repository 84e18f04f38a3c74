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
__device__ __forceinline__ void diss2d_class(const Diss2DTables<M>& T, const double* __restrict__ su,
                                             const double* __restrict__ sv, double* __restrict__ ou,
                                             double* __restrict__ ov, int lane) {
  using S = Diss2DSmem<M>;
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
    const double* v00 = sv + (0 * S::NQ + lane) * S::PVP;
    const double* v01 = sv + (0 * S::NQ + lane + 1) * S::PVP;
    const double* v10 = sv + (1 * S::NQ + lane) * S::PVP;
    const double* v11 = sv + (1 * S::NQ + lane + 1) * S::PVP;
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
    const double* u00 = su + (0 * S::NQ + lane) * S::PUP;
    const double* u01 = su + (0 * S::NQ + lane + 1) * S::PUP;
    const double* u10 = su + (1 * S::NQ + lane) * S::PUP;
    const double* u11 = su + (1 * S::NQ + lane + 1) * S::PUP;
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

  // ---- unscale and store this class's coefficients
#pragma unroll
  for (int x = 0; x < NKU; ++x)
#pragma unroll
    for (int y = 0; y < NLU; ++y) {
      const int k = PA + 2 * x, l = PB + 2 * y;
      ou[lane * (M + 1) * (M + 1) + k * (M + 1) + l] = T.inv[k][l] * au[x][y];
    }
#pragma unroll
  for (int x = 0; x < NKV; ++x)
#pragma unroll
    for (int y = 0; y < NLV; ++y) {
      const int k = PA + 2 * x, l = PB + 2 * y;
      if (k < M && l < M) ov[lane * M * M + k * M + l] = T.inv[k][l] * av[x][y];
    }
}

template <int M>
__global__ void __launch_bounds__(128) diss2d_kernel(const __grid_constant__ Diss2DParams<M> P) {
  using S = Diss2DSmem<M>;
  extern __shared__ __align__(16) double smem[];
  double* su = smem;
  double* sv = smem + 2 * S::NQ * S::PUP;
  const Step2DArgs& a = P.a;
  const int64_t j0 = (int64_t)blockIdx.x * kTileJ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int PU = S::PU, PV = S::PV;

  for (int64_t tr = blockIdx.y; tr < a.ntrows; tr += gridDim.y) {
    const int64_t t = a.trow0 + tr;
    const int64_t s0 = t + a.off;
    const RowRef ru0 = resolve_row(a.u, s0, a.nx, a.ny * PU, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
    const RowRef ru1 = resolve_row(a.u, s0 + 1, a.nx, a.ny * PU, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
    const RowRef rv0 = resolve_row(a.v, s0, a.nx, a.ny * PV, a.periodic, a.kxl, a.kxh, 0.0, 0.0);
    const RowRef rv1 = resolve_row(a.v, s0 + 1, a.nx, a.ny * PV, a.periodic, a.kxl, a.kxh, 0.0, 0.0);
    __syncthreads();  // previous iteration's output copy-out done
    stage_rows<PU, S::PUP, M + 1>(su, ru0, ru1, j0 + a.off, a, true);
    stage_rows<PV, S::PVP, M>(sv, rv0, rv1, j0 + a.off, a, false);
    __syncthreads();

    // outputs staged in registers, then written through smem for coalescing
    double* ou = smem;                       // reuse after the barrier below
    double* ov = smem + kTileJ * PU;
    // compute into registers first (sources are read inside); we need the raw
    // rows intact until every warp is done, so results go to a second region.
    double* ou2 = smem + 2 * S::NQ * S::PUP + 2 * S::NQ * S::PVP;
    double* ov2 = ou2 + kTileJ * PU;
    switch (warp) {
      case 0: diss2d_class<M, 0, 0>(P.t, su, sv, ou2, ov2, lane); break;
      case 1: diss2d_class<M, 0, 1>(P.t, su, sv, ou2, ov2, lane); break;
      case 2: diss2d_class<M, 1, 0>(P.t, su, sv, ou2, ov2, lane); break;
      default: diss2d_class<M, 1, 1>(P.t, su, sv, ou2, ov2, lane); break;
    }
    (void)ou;
    (void)ov;
    __syncthreads();
    const int64_t ncols = (a.nty - j0) < kTileJ ? (a.nty - j0) : kTileJ;
    double* gu = a.ud + (tr * a.nty + j0) * PU;
    double* gv = a.vd + (tr * a.nty + j0) * PV;
    for (int idx = threadIdx.x; idx < ncols * PU; idx += blockDim.x) gu[idx] = ou2[idx];
    for (int idx = threadIdx.x; idx < ncols * PV; idx += blockDim.x) gv[idx] = ov2[idx];
  }
}

}  // namespace hw
