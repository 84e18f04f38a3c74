// Streaming SIMT form of the 2D cell map (CUDA-core FP64).
//
// Used where it measured faster than the tensor-core cell map (cellmap.cuh):
// the conservative scheme at m <= 2 (2.1x at cons m = 2, 2048^2 walls), whose
// single-field maps are tiny (9 x 9 MACs per cell at m = 2) so the step is a
// stream: read each source node once, write each target record once.  (At
// the dissipative m = 1, 2 the DMMA kernel stays 10-25% faster; from m = 3 up
// this kernel is 2-8x slower: every weight is a uniform constant load
// (LDCU.64), and the constant cache sustains ~1 per 3 clocks per SM.
// tools/gpu_ab.sh, profiles/ab_r02_kernel_knobs.txt.)  The kernel
//   * stages a tile's (TR+1) x (TJ+1) source nodes in shared memory with
//     loads whose consecutive lanes read consecutive doubles of a node row
//     (periodic wrap, wall ghosts — boundary.py:56-132 — and slab halos
//     resolved per row / column on the way in),
//   * gives each thread one target cell: per input entry the four corner
//     values form the four parity classes' signed sums (the butterfly of
//     cellmap.h), which multiply the class maps read as warp-uniform
//     (broadcast) shared-memory operands — no DMMA padding, no fragments,
//   * writes the cell records into shared memory and copies the tile's rows
//     out as contiguous segments (consecutive lanes, consecutive doubles),
//     subtracting `previous` there for the conservative scheme
//     (conservative.py:136: out = 2 WT I(cur) - prev; prev may alias out).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <type_traits>

#include "cellmap_shape.h"
#include "common.cuh"

#ifndef HW_CM_PDL
#define HW_CM_PDL 1
#endif

namespace hw {

struct Simt2DArgs {
  Rows f0, f1;
  const double* wd;   // [DOUT][DIN] class-major dense maps (class 0 outputs, then 1, 2, 3)
  const int* code;    // [DOUT] output field << 16 | offset in the record
  const double* prev; // kCons
  double* out0;
  double* out1;
  int64_t nx, ny, trow0, ntrows, nty;
  int off, periodic;
  int kxl, kxh, kyl, kyh;
  double gxl, gxh, gyl, gyh;
};

template <int M, int SCH>
struct SimtCfg {
  static constexpr int W0 = cm_win(SCH, M, 0), W1 = cm_win(SCH, M, 1);
  static constexpr int P0 = W0 * W0, P1 = W1 * W1, DIN = P0 + P1;
  static constexpr int OW0 = cm_wout(SCH, M, 0), OW1 = cm_wout(SCH, M, 1);
  static constexpr int O0 = OW0 * OW0, O1 = OW1 * OW1, DOUT = O0 + O1;
  // tile: TR target rows x TJ columns, one thread per target cell
#ifdef HW_SIMT_TR
  static constexpr int TR = HW_SIMT_TR;
#else
  static constexpr int TR = 4;
#endif
#ifdef HW_SIMT_TJ
  static constexpr int TJ = HW_SIMT_TJ;
#else
  static constexpr int TJ = DIN > 30 ? 32 : 64;
#endif
  static constexpr int NTH = TR * TJ;
  static constexpr int NODES = (TR + 1) * (TJ + 1);
  static constexpr int SRC = NODES * DIN;  // doubles; reused for the output tile (TR TJ DOUT <= SRC)
  static_assert(TR * TJ * DOUT <= SRC, "output tile must fit the source tile's space");
  static constexpr int SMEM = SRC * 8;
  static constexpr int NC0 = cm_ncls(SCH, M, 0), NC1 = cm_ncls(SCH, M, 1), NC2 = cm_ncls(SCH, M, 2),
                       NC3 = cm_ncls(SCH, M, 3);
};

// The class maps ride in the kernel's parameter space (constant bank): every
// FMA takes its weight as a warp-uniform constant operand, no load at all.
// (Kernel parameters may hold up to 32764 bytes on sm_70+ with CUDA >= 12.1:
// the dense map fits up to m = 5, 61 x 61 doubles.)
template <int M, int SCH>
struct SimtParams {
  Simt2DArgs a;
  double w[SimtCfg<M, SCH>::DOUT * SimtCfg<M, SCH>::DIN];  // class-major [DOUT][DIN]
  int code[SimtCfg<M, SCH>::DOUT];
};

template <int M, int SCH>
__global__ void __launch_bounds__(SimtCfg<M, SCH>::NTH) simt2d_kernel(const __grid_constant__ SimtParams<M, SCH> prm) {
  using C = SimtCfg<M, SCH>;
  constexpr int TR = C::TR, TJ = C::TJ, DIN = C::DIN, DOUT = C::DOUT, P0 = C::P0, P1 = C::P1;
  const Simt2DArgs& a = prm.a;
  extern __shared__ __align__(16) double sm[];
  double* src = sm;  // [TR+1][TJ+1][DIN]
  const int tid = threadIdx.x;
#if HW_CM_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  const int64_t tcols = (a.nty + TJ - 1) / TJ;
  const int64_t tr0 = (int64_t)(blockIdx.x / tcols) * TR, j0 = (int64_t)(blockIdx.x % tcols) * TJ;
  const int nvr = (int)(a.ntrows - tr0 < TR ? a.ntrows - tr0 : TR);
  const int nvc = (int)(a.nty - j0 < TJ ? a.nty - j0 : TJ);
  const int64_t s_first = a.trow0 + tr0 + a.off, c_first = j0 + a.off;
  const bool col_interior = c_first >= 0 && c_first + nvc < a.ny;

  // ---- stage the source nodes: per row and field, a contiguous segment of
  // (nvc + 1) node records (consecutive lanes on consecutive doubles)
  auto stage = [&](auto f_c) {
    constexpr int F = decltype(f_c)::value;
    constexpr int PF = F ? P1 : P0, W = F ? C::W1 : C::W0, BASE = F ? P0 : 0;
    const int n = (nvc + 1) * PF;
    for (int r = 0; r <= nvr; ++r) {
      const RowRef rr = resolve_row(F ? a.f1 : a.f0, s_first + r, a.nx, a.ny * PF, a.periodic, a.kxl, a.kxh,
                                    F ? 0.0 : a.gxl, F ? 0.0 : a.gxh);
      double* dst = src + r * (TJ + 1) * DIN + BASE;
      if (col_interior && rr.kind == 0) {
        const double* seg = rr.p + c_first * PF;
        for (int i = tid; i < n; i += C::NTH) {
          const int q = i / PF, e = i - q * PF;
          dst[q * DIN + e] = seg[i];
        }
      } else {
        for (int i = tid; i < n; i += C::NTH) {
          const int q = i / PF, e = i - q * PF;
          const ColRef cc = resolve_col(c_first + q, a.ny, a.periodic, a.kyl, a.kyh, F ? 0.0 : a.gyl,
                                        F ? 0.0 : a.gyh);
          double v = rr.p[cc.c * PF + e];
          if (rr.kind | cc.kind) v = ghosted(v, e / W, e % W, rr.kind, rr.g, cc.kind, cc.g);
          dst[q * DIN + e] = v;
        }
      }
    }
  };
  stage(std::integral_constant<int, 0>{});
  if constexpr (P1 > 0) stage(std::integral_constant<int, 1>{});
  __syncthreads();

  // ---- one target cell per thread: out_c = W_c G^c
  const int tl = tid / TJ, tc = tid % TJ;
  double acc[DOUT];
#pragma unroll
  for (int o = 0; o < DOUT; ++o) acc[o] = 0.0;
  const bool valid = tl < nvr && tc < nvc;
  if (valid) {
    const double* n00 = src + (tl * (TJ + 1) + tc) * DIN;
    const double* n01 = n00 + DIN;
    const double* n10 = n00 + (TJ + 1) * DIN;
    const double* n11 = n10 + DIN;
#pragma unroll
    for (int e = 0; e < DIN; ++e) {
      // parity of input entry e (its field's k, l): sign flips of the x- / y-right corners
      const int ee = e < P0 ? e : e - P0, w = e < P0 ? C::W0 : C::W1;
      const bool kx = (ee / w) & 1, ky = (ee % w) & 1;
      const double c00 = n00[e];
      const double c01 = ky ? -n01[e] : n01[e];
      const double c10 = kx ? -n10[e] : n10[e];
      const double c11 = (kx != ky) ? -n11[e] : n11[e];
      const double ap = c00 + c10, am = c00 - c10, bp = c01 + c11, bm = c01 - c11;
      const double g[4] = {ap + bp, ap - bp, am + bm, am - bm};  // classes (0,0) (0,1) (1,0) (1,1)
      auto cls = [](int o) {
        return o < C::NC0 ? 0 : (o < C::NC0 + C::NC1 ? 1 : (o < C::NC0 + C::NC1 + C::NC2 ? 2 : 3));
      };
#pragma unroll
      for (int o = 0; o < DOUT; ++o) acc[o] = fma(prm.w[o * DIN + e], g[cls(o)], acc[o]);
    }
  }
  __syncthreads();  // the source tile is dead: reuse it for the output records
  double* outt = sm;  // [TR][TJ][O0] then [TR][TJ][O1]
  if (valid) {
#pragma unroll
    for (int o = 0; o < DOUT; ++o) {
      const int cd = prm.code[o], off = cd & 0xffff;
      if (cd >> 16)
        outt[TR * TJ * C::O0 + (tl * TJ + tc) * C::O1 + off] = acc[o];
      else
        outt[(tl * TJ + tc) * C::O0 + off] = acc[o];
    }
  }
  __syncthreads();

  // ---- copy out: each target row's records are one contiguous segment per field
  for (int r = 0; r < nvr; ++r) {
    const int64_t cell0 = (tr0 + r) * a.nty + j0;
    {
      double* d = a.out0 + cell0 * C::O0;
      const double* sv = outt + r * TJ * C::O0;
      const double* pv = SCH == kCons ? a.prev + cell0 * C::O0 : nullptr;
      for (int i = tid; i < nvc * C::O0; i += C::NTH) d[i] = SCH == kCons ? sv[i] - pv[i] : sv[i];
    }
    if (C::O1 > 0) {
      double* d = a.out1 + cell0 * C::O1;
      const double* sv = outt + TR * TJ * C::O0 + r * TJ * C::O1;
      for (int i = tid; i < nvc * C::O1; i += C::NTH) d[i] = sv[i];
    }
  }
}

// wd / code: HOST copies of the class maps (copied into the parameter block).
template <int M, int SCH>
cudaError_t launch_simt2d(const Simt2DArgs& a, const double* wd, const int* code, cudaStream_t st) {
  using C = SimtCfg<M, SCH>;
  static_assert(sizeof(SimtParams<M, SCH>) <= 32764, "class maps exceed the kernel parameter space");
  auto kern = simt2d_kernel<M, SCH>;
  constexpr int kDevs = 64;
  static std::atomic<bool> attr_set[kDevs];  // the shared-memory attribute, once per device
  cudaError_t e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if (dev >= kDevs || !attr_set[dev].load(std::memory_order_acquire)) {
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM)) != cudaSuccess)
      return e;
    if (dev < kDevs) attr_set[dev].store(true, std::memory_order_release);
  }
  const int64_t nblk = ((a.ntrows + C::TR - 1) / C::TR) * ((a.nty + C::TJ - 1) / C::TJ);
  if (nblk <= 0) return cudaSuccess;
  static thread_local SimtParams<M, SCH> prm;
  prm.a = a;
  for (int i = 0; i < C::DOUT * C::DIN; ++i) prm.w[i] = wd[i];
  for (int i = 0; i < C::DOUT; ++i) prm.code[i] = code[i];
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)nblk);
  lc.blockDim = dim3(C::NTH);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = HW_CM_PDL;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kern, prm);
}

// Generic (runtime-order) form for the orders above the templated fast paths
// (m = 9..12, interp.py:30 MAX_ORDER = 12): one thread per target cell reads
// its four corners straight from global memory (L1-cached; ghosts, wrap and
// halos as above), the class maps through the read-only cache, and
// accumulates GB outputs at a time.  Coverage for the reference's full order
// range, not a throughput path: these orders sit at the conditioning limit
// of the Hermite matrices (cond(M_12) ~ 1e10).
struct Gen2DArgs {
  Simt2DArgs s;
  int w0, w1, ow0, ow1, din, dout;
  int ncls[4];
};

static __global__ void __launch_bounds__(128) simt2d_generic_kernel(const __grid_constant__ Gen2DArgs g, int scheme) {
  constexpr int GB = 16;
  const Simt2DArgs& a = g.s;
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
#if HW_CM_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  if (cell >= a.ntrows * a.nty) return;
  const int64_t tl = cell / a.nty, tj = cell - tl * a.nty;
  const int64_t s0 = a.trow0 + tl + a.off, c0 = tj + a.off;
  const int p0 = g.w0 * g.w0, p1 = g.w1 * g.w1;
  RowRef rr[2][2];  // [field][sx]
  ColRef cc[2];
  for (int sx = 0; sx < 2; ++sx) {
    rr[0][sx] = resolve_row(a.f0, s0 + sx, a.nx, a.ny * p0, a.periodic, a.kxl, a.kxh, a.gxl, a.gxh);
    rr[1][sx] = p1 ? resolve_row(a.f1, s0 + sx, a.nx, a.ny * p1, a.periodic, a.kxl, a.kxh, 0.0, 0.0) : rr[0][sx];
    cc[sx] = resolve_col(c0 + sx, a.ny, a.periodic, a.kyl, a.kyh, a.gyl, a.gyh);
  }
  const int b1 = g.ncls[0], b2 = b1 + g.ncls[1], b3 = b2 + g.ncls[2];
  for (int ob = 0; ob < g.dout; ob += GB) {
    double acc[GB];
#pragma unroll
    for (int o = 0; o < GB; ++o) acc[o] = 0.0;
    for (int e = 0; e < g.din; ++e) {
      const int f = e < p0 ? 0 : 1, ee = f ? e - p0 : e, w = f ? g.w1 : g.w0, pf = f ? p1 : p0;
      const int k = ee / w, l = ee % w;
      double v[2][2];
      for (int sx = 0; sx < 2; ++sx)
        for (int sy = 0; sy < 2; ++sy) {
          const RowRef& r = rr[f][sx];
          const ColRef& c = cc[sy];
          double x = r.p[c.c * pf + ee];
          if (r.kind | c.kind) x = ghosted(x, k, l, r.kind, f ? 0.0 : r.g, c.kind, f ? 0.0 : c.g);
          v[sx][sy] = x;
        }
      const double c00 = v[0][0];
      const double c01 = (l & 1) ? -v[0][1] : v[0][1];
      const double c10 = (k & 1) ? -v[1][0] : v[1][0];
      const double c11 = ((k ^ l) & 1) ? -v[1][1] : v[1][1];
      const double ap = c00 + c10, am = c00 - c10, bp = c01 + c11, bm = c01 - c11;
      const double gc[4] = {ap + bp, ap - bp, am + bm, am - bm};
#pragma unroll
      for (int o = 0; o < GB; ++o) {
        const int row = ob + o;
        if (row < g.dout) {
          const int cl = row < b1 ? 0 : (row < b2 ? 1 : (row < b3 ? 2 : 3));
          acc[o] = fma(__ldg(a.wd + (int64_t)row * g.din + e), gc[cl], acc[o]);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < GB; ++o) {
      const int row = ob + o;
      if (row >= g.dout) continue;
      const int cd = __ldg(a.code + row), off = cd & 0xffff;
      if (cd >> 16) {
        a.out1[cell * (g.ow1 * g.ow1) + off] = acc[o];
      } else {
        const int64_t i = cell * (g.ow0 * g.ow0) + off;
        a.out0[i] = scheme == kCons ? acc[o] - a.prev[i] : acc[o];
      }
    }
  }
}

static inline cudaError_t launch_simt2d_generic(const Gen2DArgs& g, int scheme, cudaStream_t st) {
  const int64_t n = g.s.ntrows * g.s.nty;
  if (n <= 0) return cudaSuccess;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)((n + 127) / 128));
  lc.blockDim = dim3(128);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = HW_CM_PDL;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, simt2d_generic_kernel, g, scheme);
}

}  // namespace hw


#define HW_INSTANTIATE_SIMT2D(M)                                                                            \
  template cudaError_t launch_simt2d<M, kDiss>(const Simt2DArgs&, const double*, const int*, cudaStream_t); \
  template cudaError_t launch_simt2d<M, kCons>(const Simt2DArgs&, const double*, const int*, cudaStream_t); \
  template cudaError_t launch_simt2d<M, kBoot>(const Simt2DArgs&, const double*, const int*, cudaStream_t);
