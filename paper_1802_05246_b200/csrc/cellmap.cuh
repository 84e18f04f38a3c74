// One fused sm_100a kernel for every 2D step of the hot path:
//   corner gather (periodic wrap / wall ghosts / slab halos, boundary.py:101-168)
//   + the per-class cell map out_c = W_c G^c (cellmap.h) on FP64 tensor cores.
//
// The class maps are dense, so the per-cell work is a GEMM over cells:
//   OUT[cells][n] = G[cells][e] . W_c[e][n]   (M = 8 cells, N = 8 outputs,
//   K = 4 inputs per mma.sync.m8n8k4.f64 — DMMA, the FP64 tensor-core path;
//   tcgen05.mma has no f64 kind on sm_100a).
// The A operand is formed in registers from the four staged corner values by
// a sign flip (integer XOR of the sign bit) and a 2x2 butterfly, which yields
// the four classes' G at once; the B operand (W, pre-arranged on the host in
// fragment order) is read conflict-free from shared memory.
//
// Data movement: persistent CTAs walk tiles of TR x TJ target cells.  Each
// tile is consumed in K-chunks of 16 inputs; a chunk stages the
// (TR+1) x (TJ+1) source nodes' 16 entries plus the matching 4 k-steps of W
// with cp.async into an NS-deep ring, so the loads of chunk g+2 overlap the
// tensor-core work of chunk g.  Accumulators live in registers for the whole
// tile; the epilogue stores them straight to the output records.
#pragma once

#include <stdint.h>

#include "cellmap_shape.h"
#include "common.cuh"

namespace hw {

struct CellMapArgs {
  Rows f0, f1;                 // source fields (f1 unused when the scheme has one input)
  const double* wfrag;         // [NK][NT][32] B fragments
  const int* ocode;            // [NT][8] field << 16 | offset, -1 = padding
  const int* icode;            // [NK*4] (kx & 1) | (ky & 1) << 1 of each input entry
  const double* prev;          // kCons: previous level (may alias out0)
  double* out0;
  double* out1;
  int64_t nx, ny;              // global source node counts
  int64_t trow0, ntrows, nty;  // target rows [trow0, trow0 + ntrows) x nty columns
  int off, periodic;           // source offset of a target (0 primal, -1 dual)
  int kxl, kxh, kyl, kyh;      // wall kinds (0 when periodic)
  double gxl, gxh, gyl, gyh;   // Dirichlet data, field 0 only
};

template <int M, int SCH>
struct CMCfg {
  static constexpr int W0 = cm_win(SCH, M, 0), W1 = cm_win(SCH, M, 1);
  static constexpr int P0 = W0 * W0, P1 = W1 * W1, DIN = P0 + P1;
  static constexpr int O0 = cm_wout(SCH, M, 0) * cm_wout(SCH, M, 0);
  static constexpr int O1 = cm_wout(SCH, M, 1) * cm_wout(SCH, M, 1);
  static constexpr int NK = cm_nk(SCH, M), NT = cm_nt(SCH, M);
  static constexpr int B1 = cm_ntbase(SCH, M, 1), B2 = cm_ntbase(SCH, M, 2), B3 = cm_ntbase(SCH, M, 3);
  static constexpr int KSC = 4;                    // k-steps per chunk
  static constexpr int KC = 4 * KSC;               // inputs per chunk
  static constexpr int NCH = (NK + KSC - 1) / KSC; // chunks per tile
  static constexpr int KCP = 20;                   // staged doubles per node (= 4 mod 16: conflict-free)
  // Tile and warp shape by accumulator footprint (MT x NT x 2 doubles per
  // thread): small maps give each warp two M-tiles (each W fragment feeds two
  // DMMAs) at two CTAs per SM; large maps one M-tile per warp at one CTA.
  static constexpr bool BIG = NT > 7;
  static constexpr int MT = BIG ? 1 : 2;           // 8-cell M-tiles per warp
  static constexpr int NW = 8;                     // warps per CTA
  static constexpr int TJ = 32;                    // target columns per tile
  static constexpr int TR = NW * MT / (TJ / 8);    // target rows per tile
  static constexpr int NODES = (TR + 1) * (TJ + 1);
  static constexpr int CBUF = NODES * KCP;
  static constexpr int WBUF = KSC * NT * 32;
  static constexpr int SBUF = CBUF + WBUF;         // doubles per pipeline stage
  static constexpr int NS = 3;                     // pipeline depth
  static constexpr int SMEM = NS * SBUF * 8 + (NK * 4 + NT * 8) * 4;
  static constexpr int MINB = 1;                   // CTAs per SM the register budget targets
  static constexpr bool UNROLL_KS = !BIG;          // software-pipeline the k-steps of a chunk
};

__device__ __forceinline__ void cm_cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cm_cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cm_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cm_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D += A B on the FP64 tensor cores (one 8x8x4 tile per warp).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ double flip_sign(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ mask);
}

// Source row s of a field: local rows, slab halos, periodic wrap, wall ghost
// (boundary.py:119-130).  kind = wall kind of a ghost row, else 0.
__device__ __forceinline__ const double* cm_row(const Rows& R, int64_t s, int64_t nx, int64_t rowlen, int periodic,
                                                int& ghost_side) {
  ghost_side = 0;
  if (s >= R.row0 && s < R.row0 + R.nrows) return R.base + (s - R.row0) * rowlen;
  if (s == R.row0 - 1 && R.lo) return R.lo;
  if (s == R.row0 + R.nrows && R.hi) return R.hi;
  if (periodic) {
    while (s < 0) s += nx;
    while (s >= nx) s -= nx;
    return R.base + (s - R.row0) * rowlen;
  }
  if (s < 0) {
    ghost_side = 1;
    return R.base + (0 - R.row0) * rowlen;
  }
  ghost_side = 2;
  return R.base + (nx - 1 - R.row0) * rowlen;
}

__device__ __forceinline__ int64_t cm_col(int64_t c, int64_t ny, int periodic, int& ghost_side) {
  ghost_side = 0;
  if (c >= 0 && c < ny) return c;
  if (periodic) {
    while (c < 0) c += ny;
    while (c >= ny) c -= ny;
    return c;
  }
  ghost_side = c < 0 ? 1 : 2;
  return c < 0 ? 0 : ny - 1;
}

template <int M, int SCH>
__global__ void __launch_bounds__(256, CMCfg<M, SCH>::MINB) cellmap_kernel(const __grid_constant__ CellMapArgs a) {
  using C = CMCfg<M, SCH>;
  constexpr int TR = C::TR, TJ = C::TJ, NT = C::NT, MT = C::MT, NS = C::NS, KSC = C::KSC, KC = C::KC,
                KCP = C::KCP, NCH = C::NCH;
  extern __shared__ __align__(16) double smem[];
  int* s_icode = reinterpret_cast<int*>(smem + NS * C::SBUF);
  int* s_ocode = s_icode + C::NK * 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < C::NK * 4; i += blockDim.x) s_icode[i] = a.icode[i];
  for (int i = tid; i < NT * 8; i += blockDim.x) s_ocode[i] = a.ocode[i];

  const int64_t tcols = (a.nty + TJ - 1) / TJ;
  const int64_t ntiles = tcols * ((a.ntrows + TR - 1) / TR);
  const int64_t my_tiles = ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nstages = my_tiles * NCH;
  const bool walls = !a.periodic;

  struct TileGeo {
    int64_t tr0, j0, s_first, c_first;
    int nvr, nvc;
  };
  auto geo = [&](int64_t g) {
    TileGeo t;
    const int64_t tile = blockIdx.x + (g / NCH) * (int64_t)gridDim.x;
    const int64_t ti = tile / tcols;
    t.tr0 = ti * TR;
    t.j0 = (tile - ti * tcols) * TJ;
    const int64_t vr = a.ntrows - t.tr0, vc = a.nty - t.j0;
    t.nvr = vr < TR ? (int)vr : TR;
    t.nvc = vc < TJ ? (int)vc : TJ;
    t.s_first = a.trow0 + t.tr0 + a.off;
    t.c_first = t.j0 + a.off;
    return t;
  };

  // Stage g = (tile, chunk): source entries [16 ch, 16 ch + 16) of the tile's
  // (TR+1) x (TJ+1) nodes, and k-steps [4 ch, 4 ch + 4) of W.
  auto issue = [&](int64_t g) {
    const TileGeo t = geo(g);
    const int ch = (int)(g % NCH);
    double* cb = smem + (g % NS) * C::SBUF;
#pragma unroll 1
    for (int idx = tid; idx < C::NODES * KC; idx += blockDim.x) {
      const int node = idx / KC, e = idx - (idx / KC) * KC;
      const int r = node / (TJ + 1), q = node - (node / (TJ + 1)) * (TJ + 1);
      const int ein = ch * KC + e;
      double* dst = cb + node * KCP + e;
      if (ein >= C::DIN || r > t.nvr || q > t.nvc) {
        *dst = 0.0;
        continue;
      }
      const bool f1 = ein >= C::P0;
      const int pf = f1 ? C::P1 : C::P0;
      int gs;
      const double* row = f1 ? cm_row(a.f1, t.s_first + r, a.nx, a.ny * pf, a.periodic, gs)
                             : cm_row(a.f0, t.s_first + r, a.nx, a.ny * pf, a.periodic, gs);
      const int64_t col = cm_col(t.c_first + q, a.ny, a.periodic, gs);
      cm_cp_async8(dst, row + col * pf + (f1 ? ein - C::P0 : ein));
    }
    const int nks = (C::NK - ch * KSC) < KSC ? (C::NK - ch * KSC) : KSC;
    const double* wsrc = a.wfrag + (size_t)ch * KSC * NT * 32;
    double* wb = cb + C::CBUF;
#pragma unroll 1
    for (int i = tid; i < nks * NT * 16; i += blockDim.x) cm_cp_async16(wb + 2 * i, wsrc + 2 * i);
  };

  // Wall ghosts: reflect the staged copies this thread issued (boundary.py:56-98;
  // the velocity / g1 reflects around zero, dissipative.py:229).
  auto fix_ghosts = [&](int64_t g) {
    const TileGeo t = geo(g);
    if (!(t.s_first < 0 || t.s_first + t.nvr >= a.nx || t.c_first < 0 || t.c_first + t.nvc >= a.ny)) return;
    const int ch = (int)(g % NCH);
    double* cb = smem + (g % NS) * C::SBUF;
#pragma unroll 1
    for (int idx = tid; idx < C::NODES * KC; idx += blockDim.x) {
      const int node = idx / KC, e = idx - (idx / KC) * KC;
      const int r = node / (TJ + 1), q = node - (node / (TJ + 1)) * (TJ + 1);
      const int ein = ch * KC + e;
      if (ein >= C::DIN || r > t.nvr || q > t.nvc) continue;
      const int64_t s = t.s_first + r, c = t.c_first + q;
      const int xk = s < 0 ? a.kxl : (s >= a.nx ? a.kxh : 0);
      const int yk = c < 0 ? a.kyl : (c >= a.ny ? a.kyh : 0);
      if (!(xk | yk)) continue;
      const bool f1 = ein >= C::P0;
      const int w = f1 ? C::W1 : C::W0;
      const int eo = f1 ? ein - C::P0 : ein;
      const double gx = f1 ? 0.0 : (s < 0 ? a.gxl : a.gxh);
      const double gy = f1 ? 0.0 : (c < 0 ? a.gyl : a.gyh);
      double* p = cb + node * KCP + e;
      *p = ghosted(*p, eo / w, eo % w, xk, gx, yk, gy);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

#pragma unroll
  for (int g = 0; g < NS - 1; ++g) {
    if (g < nstages) issue(g);
    cm_commit();
  }

  for (int64_t g = 0; g < nstages; ++g) {
    cm_wait<NS - 2>();
    if (walls) fix_ghosts(g);
    __syncthreads();
    if (g + NS - 1 < nstages) issue(g + NS - 1);
    cm_commit();

    const int ch = (int)(g % NCH);
    const double* cb = smem + (g % NS) * C::SBUF;
    const double* wb = cb + C::CBUF;
    const int nks = (C::NK - ch * KSC) < KSC ? (C::NK - ch * KSC) : KSC;
    auto kstep = [&](const int ks) {
      {
        const int code = s_icode[(ch * KSC + ks) * 4 + (lane & 3)];
        const unsigned long long mx = (unsigned long long)(code & 1) << 63;
        const unsigned long long my = (unsigned long long)((code >> 1) & 1) << 63;
        double A[MT][4];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int mt = warp * MT + t;
          const int trl = mt / (TJ / 8), tc = (mt % (TJ / 8)) * 8;
          const double* p = cb + (trl * (TJ + 1) + tc + (lane >> 2)) * KCP + ks * 4 + (lane & 3);
          const double c00 = p[0];
          const double c01 = flip_sign(p[KCP], my);
          const double c10 = flip_sign(p[(TJ + 1) * KCP], mx);
          const double c11 = flip_sign(p[(TJ + 2) * KCP], mx ^ my);
          const double ap = c00 + c10, am = c00 - c10, bp = c01 + c11, bm = c01 - c11;
          A[t][0] = ap + bp;  // class (0,0)
          A[t][1] = ap - bp;  // class (0,1)
          A[t][2] = am + bm;  // class (1,0)
          A[t][3] = am - bm;  // class (1,1)
        }
        const double* wk = wb + ks * NT * 32 + lane;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = nt < C::B1 ? 0 : (nt < C::B2 ? 1 : (nt < C::B3 ? 2 : 3));  // parity class of tile nt
          const double b = wk[nt * 32];
#pragma unroll
          for (int t = 0; t < MT; ++t) dmma(acc[t][nt], A[t][c], b);
        }
      }
    };
    if constexpr (C::UNROLL_KS) {
#pragma unroll
      for (int ks = 0; ks < KSC; ++ks)
        if (ks < nks) kstep(ks);
    } else {
#pragma unroll 1
      for (int ks = 0; ks < nks; ++ks) kstep(ks);
    }

    if (ch == NCH - 1) {  // epilogue: this tile's outputs straight to global
      const TileGeo tg = geo(g);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int mt = warp * MT + t;
        const int trl = mt / (TJ / 8), jl = (mt % (TJ / 8)) * 8 + (lane >> 2);
        if (trl < tg.nvr && jl < tg.nvc) {
          const int64_t cell = (tg.tr0 + trl) * a.nty + tg.j0 + jl;
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int code = s_ocode[n * 8 + (lane & 3) * 2 + i];
              if (code < 0) continue;
              const int o = code & 0xffff;
              if ((code >> 16) == 0) {
                const int64_t idx = cell * C::O0 + o;
                double v = acc[t][n][i];
                if (SCH == kCons) v -= a.prev[idx];
                a.out0[idx] = v;
              } else {
                a.out1[cell * C::O1 + o] = acc[t][n][i];
              }
            }
        }
#pragma unroll
        for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
      }
    }
  }
  cm_wait<0>();
}

}  // namespace hw
