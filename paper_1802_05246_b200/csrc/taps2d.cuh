// Full-order 2D tap kernels: the conservative update (conservative.py:130-157)
// and the conservative bootstrap (conservative.py:185-195).  Both are
// "interpolate I_{m,m} per input field, then a fixed even-offset stencil over
// the (2m+2)^2 interpolant":
//   conservative: new[k][l] = 2 sum_ij WT[k,l,k+2i,l+2j] c[k+2i][l+2j] - prev[k][l]
//                 WT = (a!/k!)(b!/l!) C(i+j,i)/(2i+2j)! rho_x^2i rho_y^2j
//                 (conservative.py:87-112), phi(a) = a! rho^a
//   bootstrap:    u[k][l] = sum_ij C(i+j,i) rx^i ry^j (a!/k!)(b!/l!)
//                      [th^2p dt^p/(2p)! c0 + th^(2p+1) dt^(p+1)/(2p+1)! d0][a][b]
//                 (closed form of expand_taylor_2d without d1), phi(a) = a! r^floor(a/2)
// Same parity-class / constant-operand organisation as diss2d.cuh.
#pragma once

#include "common.cuh"
#include "diss2d.cuh"

namespace hw {

template <int M, int NIN>
struct Taps2DTables {
  static constexpr int K = 2 * M + 2;
  double mx[K][M + 1];  // phi_x(a) HL_m[a][k]
  double my[K][M + 1];  // phi_y(b) HL_m[b][l]
  double g[NIN][M + 1][M + 1];
  double inv[M + 1][M + 1];  // scale / (phi_x(k) phi_y(l))
};

struct Taps2DArgs {
  Rows f0, f1;           // input fields (f1 used when NIN == 2)
  const double* prev;    // conservative: previous level on the target grid
  double* out;
  int64_t nx, ny;
  int64_t trow0, ntrows, nty;
  int off, periodic;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;  // Dirichlet data for f0
  double g1scale;             // 1 for f1 Dirichlet data (unused: velocity reflects around 0)
};

template <int M, int NIN>
struct Taps2DParams {
  Taps2DArgs a;
  Taps2DTables<M, NIN> t;
};

template <int M>
struct Taps2DSmem {
  static constexpr int P = (M + 1) * (M + 1);
  static constexpr int PP = P | 1;
  static constexpr int NQ = kTileJ + 1;
};

template <int M, int NIN, int PA, int PB>
__device__ __forceinline__ void taps2d_class(const Taps2DTables<M, NIN>& T, const double* __restrict__ sraw,
                                             const double* __restrict__ prev_row, double* __restrict__ o,
                                             int lane, bool has_prev) {
  using S = Taps2DSmem<M>;
  constexpr int NK = (M - PA) / 2 + 1, NL = (M - PB) / 2 + 1;
  double acc[NK][NL];
#pragma unroll
  for (int x = 0; x < NK; ++x)
#pragma unroll
    for (int y = 0; y < NL; ++y) acc[x][y] = 0.0;

#pragma unroll
  for (int f = 0; f < NIN; ++f) {
    const double* base = sraw + f * 2 * S::NQ * S::PP;
    const double* u00 = base + (0 * S::NQ + lane) * S::PP;
    const double* u01 = base + (0 * S::NQ + lane + 1) * S::PP;
    const double* u10 = base + (1 * S::NQ + lane) * S::PP;
    const double* u11 = base + (1 * S::NQ + lane + 1) * S::PP;
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
#pragma unroll
    for (int b = PB; b < 2 * M + 2; b += 2) {
      double Y[M + 1];
#pragma unroll
      for (int k = 0; k <= M; ++k) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l <= M; ++l) s = fma(T.my[b][l], G[k][l], s);
        Y[k] = s;
      }
#pragma unroll
      for (int ia = 0; ia <= M; ++ia) {
        const int arow = PA + 2 * ia;
        if (arow > 2 * M + 1) continue;
        double c = 0.0;
#pragma unroll
        for (int k = 0; k <= M; ++k) c = fma(T.mx[arow][k], Y[k], c);
#pragma unroll
        for (int i = 0; i <= ia; ++i) {
          const int k = arow - 2 * i;
          if (k > M) continue;
#pragma unroll
          for (int j = 0; j <= M; ++j) {
            const int l = b - 2 * j;
            if (l < 0 || l > M) continue;
            acc[(k - PA) / 2][(l - PB) / 2] = fma(T.g[f][i][j], c, acc[(k - PA) / 2][(l - PB) / 2]);
          }
        }
      }
    }
  }
  constexpr int P = (M + 1) * (M + 1);
#pragma unroll
  for (int x = 0; x < NK; ++x)
#pragma unroll
    for (int y = 0; y < NL; ++y) {
      const int k = PA + 2 * x, l = PB + 2 * y;
      double r = T.inv[k][l] * acc[x][y];
      if (has_prev) r -= prev_row[lane * P + k * (M + 1) + l];
      o[lane * P + k * (M + 1) + l] = r;
    }
}

template <int M, int NIN>
__global__ void __launch_bounds__(128) taps2d_kernel(const __grid_constant__ Taps2DParams<M, NIN> Pm) {
  using S = Taps2DSmem<M>;
  constexpr int P = S::P;
  extern __shared__ __align__(16) double smem[];
  double* sraw = smem;
  double* so = smem + NIN * 2 * S::NQ * S::PP;
  const Taps2DArgs& a = Pm.a;
  const int64_t j0 = (int64_t)blockIdx.x * kTileJ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ncols = (a.nty - j0) < kTileJ ? (a.nty - j0) : kTileJ;
  Step2DArgs sa;  // reuse the staging helper's column/ghost logic
  sa.ny = a.ny;
  sa.periodic = a.periodic;
  sa.kyl = a.kyl;
  sa.kyh = a.kyh;
  sa.gyl = a.gyl;
  sa.gyh = a.gyh;

  for (int64_t tr = blockIdx.y; tr < a.ntrows; tr += gridDim.y) {
    const int64_t t = a.trow0 + tr;
    const int64_t s0 = t + a.off;
    __syncthreads();
#pragma unroll
    for (int f = 0; f < NIN; ++f) {
      const Rows& R = f ? a.f1 : a.f0;
      const double gl = f ? 0.0 : a.gxl, gh = f ? 0.0 : a.gxh;
      const RowRef r0 = resolve_row(R, s0, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, gl, gh);
      const RowRef r1 = resolve_row(R, s0 + 1, a.nx, a.ny * P, a.periodic, a.kxl, a.kxh, gl, gh);
      stage_rows<P, S::PP, M + 1>(sraw + f * 2 * S::NQ * S::PP, r0, r1, j0 + a.off, sa, f == 0);
    }
    __syncthreads();
    const bool has_prev = a.prev != nullptr;
    // `out` may alias `prev`: each CTA reads its own prev tile here and only
    // overwrites it after the barrier below.  Lanes past the last column skip
    // the prev read.
    const double* pv = has_prev ? a.prev + (tr * a.nty + j0) * P : nullptr;
    switch (warp) {
      case 0: taps2d_class<M, NIN, 0, 0>(Pm.t, sraw, pv, so, lane, has_prev && lane < ncols); break;
      case 1: taps2d_class<M, NIN, 0, 1>(Pm.t, sraw, pv, so, lane, has_prev && lane < ncols); break;
      case 2: taps2d_class<M, NIN, 1, 0>(Pm.t, sraw, pv, so, lane, has_prev && lane < ncols); break;
      default: taps2d_class<M, NIN, 1, 1>(Pm.t, sraw, pv, so, lane, has_prev && lane < ncols); break;
    }
    __syncthreads();
    double* go = a.out + (tr * a.nty + j0) * P;
    for (int idx = threadIdx.x; idx < ncols * P; idx += blockDim.x) go[idx] = so[idx];
  }
}

}  // namespace hw
