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
// Warp specialisation.  Four producer warps stage, for every (tile, K-chunk)
// of the CTA's persistent tile sequence, the 16-entry slices of the tile's
// (TR+1) x (TJ+1) source nodes (plus the chunk's W fragments unless W is
// resident) into an NS-deep shared-memory ring with cp.async; completion is
// tracked by mbarriers (cp.async.mbarrier.arrive), never by a CTA-wide
// barrier.  Eight or twelve consumer warps wait on the ring's `full`
// barriers, run the DMMAs and release the slot on its `empty` barrier, so
// consumers drift freely relative to each other.  Each consumer dumps its
// accumulators into its own output slab and moves on; a producer warp drains
// the slab to HBM between staging steps (or, per order, the consumer stores
// directly / drains its own slab).
//
// Every per-order choice (consumer warps, M-tiles per warp, tile width, ring
// depth, resident W, epilogue kind, ...) lives in CMCfg / cellmap_shape.h with
// the measurement that picked it; profiles/ab_r01_kernel_knobs.txt has the
// A/B tables (tools/gpu_ab.sh, variant builds via -DHW_CM_* knobs).
#pragma once

#include <stdint.h>
#include <stdio.h>

#include <type_traits>

#include "cellmap_shape.h"
#include "common.cuh"

namespace hw {

struct CellMapArgs {
  Rows f0, f1;                 // source fields (f1 unused when the scheme has one input)
  const double* wfrag;         // [NK][NTB][32] B fragments of the DMMA tiles (cellmap_shape.h cm_ntb)
  const double* wleft;         // [NK][LC][4] weights of the SIMT columns (cellmap_shape.h hybrid tiles)
  const int* ocode;            // [NT][8] output field << 16 | offset in its record, -1 = padding
  const int* icode;            // [NK*4] (kx & 1) | (ky & 1) << 1 of each input slot
  const double* prev;          // kCons: previous level (may alias out0)
  double* out0;
  double* out1;
  int64_t nx, ny;              // global source node counts
  int64_t trow0, ntrows, nty;  // target rows [trow0, trow0 + ntrows) x nty columns
  int off, periodic;           // source offset of a target (0 primal, -1 dual)
  int kxl, kxh, kyl, kyh;      // wall kinds (0 when periodic)
  double gxl, gxh, gyl, gyh;   // Dirichlet data, field 0 only
  int* sched;                  // [2] dynamic tile counter + CTAs done (zero between launches); null = static schedule
};

// L2 prefetch size qualifier of the staging copies (A/B knob HW_CM_PFN = 64 / 128 / 256)
#if defined(HW_CM_PFN) && HW_CM_PFN == 64
#define HW_CM_PF ".L2::64B"
#elif defined(HW_CM_PFN) && HW_CM_PFN == 128
#define HW_CM_PF ".L2::128B"
#elif defined(HW_CM_PFN) && HW_CM_PFN == 256
#define HW_CM_PF ".L2::256B"
#else
#define HW_CM_PF ""
#endif
#ifndef HW_CM_PDL
#define HW_CM_PDL 1  // programmatic dependent launch between consecutive steps (A/B knob)
#endif
// HW_CM_DEBUG: race / bounds checking build (tools/race_stress.py; the pool
// has no compute-sanitizer).  Every ring slot is poisoned with NaN between
// its consumption and its refill, so a read of anything the producers did
// not stage reaches the outputs as NaN; producers and consumers sleep for
// random spans before each chunk, so orderings the barriers do not enforce
// show up as run-to-run differences; global reads and writes are bounds-
// checked against the field windows (trap on violation).
#ifndef HW_CM_DEBUG
#define HW_CM_DEBUG 0
#endif
#ifndef HW_CM_NOPADONCE
#define HW_CM_NOPADONCE 0  // A/B knob: zero the ring's padding slots at every stage
#endif
#if HW_CM_DEBUG
__device__ __forceinline__ unsigned cm_dbg_rand(unsigned a, unsigned b) {
  unsigned x = (unsigned)clock64() ^ (a * 2654435761u) ^ (b * 40503u) ^ (blockIdx.x * 2246822519u);
  x ^= x >> 13;
  x *= 0x5bd1e995u;
  x ^= x >> 15;
  return x;
}
#define CM_DBG_CHECK(cond, what)                                                                  \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("cellmap debug: %s violated (block %d thread %d)\n", what, blockIdx.x, threadIdx.x); \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define CM_DBG_CHECK(cond, what)
#endif
#ifndef HW_CM_DCODE
#define HW_CM_DCODE 1  // direct epilogue: per-lane output codes resolved once, branch-free stores (A/B knob)
#endif
#ifndef HW_CM_SLEEP
#define HW_CM_SLEEP 64  // producer back-off (ns) while its ring slot is busy and no slab is ready
#endif

template <int M, int SCH>
struct CMCfg {
  static constexpr int W0 = cm_win(SCH, M, 0), W1 = cm_win(SCH, M, 1);
  static constexpr int P0 = W0 * W0, P1 = W1 * W1;
  static constexpr int K0 = cm_k0(SCH, M);        // input slots of field 0 (P0 rounded up to 4)
  static constexpr int O0 = cm_wout(SCH, M, 0) * cm_wout(SCH, M, 0);
  static constexpr int O1 = cm_wout(SCH, M, 1) * cm_wout(SCH, M, 1);
  static constexpr int NK = cm_nk(SCH, M), NT = cm_nt(SCH, M);
  static constexpr int NTD = cm_ntd(SCH, M), LC = cm_lc(SCH, M);  // DMMA tiles; SIMT columns (hybrid tiles)
  static constexpr bool PXM = cm_pxm(SCH, M);      // merged x-classes (cellmap_shape.h)
  static constexpr int NTB = cm_ntb(SCH, M);       // B fragments per k-step
  static constexpr int TG1 = PXM ? cm_pxm_tiles(SCH, M, 0) : 0;  // PXM: first tile of the y-odd classes
  static constexpr int WLN = NK * LC * 4;                          // resident SIMT weights (doubles)
  static constexpr int B1 = cm_ntbase(SCH, M, 1), B2 = cm_ntbase(SCH, M, 2), B3 = cm_ntbase(SCH, M, 3);
  static constexpr int KSC = cm_ksc(SCH, M);       // k-steps per chunk
  static constexpr int KC = 4 * KSC;               // input slots per chunk
  static constexpr int NCH = (NK + KSC - 1) / KSC; // chunks per tile
  // staged doubles per node: = +-4 mod 16 keeps the fragment reads of 8 nodes x 4 slots conflict-free
  static constexpr int KCP = KC <= 12 ? 12 : 20;
  static_assert(KC <= KCP && (KCP % 16 == 4 || KCP % 16 == 12), "ring node stride");
  static constexpr int NW = cm_nw(SCH, M);         // consumer warps (a multiple of 4)
#ifdef HW_CM_NPW
  static constexpr int NPW = HW_CM_NPW;
#else
  static constexpr int NPW = 4;                    // producer warps (one per SM sub-partition)
#endif
  static constexpr int NTHREADS = 32 * (NW + NPW);
  static constexpr int TJ = cm_tj(SCH, M);         // target columns per tile
  static constexpr int NSMAX = 8;                  // ring slots the barrier arrays hold
  static constexpr int QT = 8;                     // tile-id ring (s_tile): tiles between fetch and last drain
  static constexpr int DO = O0 + O1;               // output record per cell
  // setmaxnreg split of the 512 registers per lane of each SM sub-partition
  // (NW / 4 consumer + NPW / 4 producer warps)
#ifdef HW_CM_PREGS
  static constexpr int PREGS = HW_CM_PREGS;
#else
  static constexpr int PREGS = NPW == 8 ? 56 : 72;
#endif
  static constexpr int LREGS = 65536 / NTHREADS / 8 * 8 * ((NW + NPW) / 4);  // per lane slot at launch
  static constexpr int CREGS0 = ((LREGS - (NPW / 4) * PREGS) / (NW / 4)) / 8 * 8;
  static constexpr int CREGS = CREGS0 > 232 ? 232 : CREGS0;
  static constexpr int SMEM_MAX = 227 * 1024;
  // Shared memory for MT M-tiles per consumer warp and an NS-slot ring:
  //   ring slot = the tile's (2 MT + 1) x 33 staged nodes x KCP + 4 k-steps of W
  //   per warp: one output slab in DMMA fragment order ([t][nt][lane][2],
  //   conflict-free 16-byte stores; drained by the producers through the
  //   inverse map s_inv) and, for kCons, one slab of `previous` records.
  // WRES: all NK k-steps of W stay resident in shared memory (loaded once per
  // CTA) instead of riding in every ring slot (cm_wres: where that measured
  // faster; W <= 40 KB).
  static constexpr bool WRES = cm_wres(SCH, M) && NK * NTB * 256 <= 40 * 1024;
  static constexpr int WRESN = WRES ? NK * NTB * 32 : 0;  // doubles
  static constexpr int sbuf(int mt) { return (NW * mt / (TJ / 8) + 1) * (TJ + 1) * KCP + (WRES ? 0 : KSC * NTB * 32); }
  // DIRECT: the consumers store their accumulators straight to HBM (no slab,
  // no producer drain).  SELF: each consumer warp drains its own slab
  // (fragment-order stores, record-order coalesced copy-out), no handoff.
  static constexpr bool DIRECT = cm_direct(SCH, M);
  static constexpr bool SELF = cm_self(SCH, M) && !DIRECT;
  static constexpr bool OWN = DIRECT || SELF;  // the consumers write HBM themselves
  // kCons `previous`: per-lane registers (loaded at the tile's first chunk, subtracted
  // in the epilogue) or a shared-memory slab (copied at the last chunk) — cm_prevreg
  static constexpr bool PREVREG = SCH == kCons && cm_prevreg(SCH, M);
  static constexpr bool PSMEM = SCH == kCons && !PREVREG;  // `previous` through a shared-memory slab
  static constexpr int tail(int mt) {
    return (WRESN + WLN) * 8 + NW * ((DIRECT ? 0 : mt * NT * 64) + (PSMEM ? mt * 8 * O0 : 0)) * 8 +
           (8 * DO + 8 * NT) * 4 +
           (2 * NSMAX + 2 * NW) * 8 + 64;
  }
  static constexpr bool fits(int mt, int ns) { return ns * sbuf(mt) * 8 + tail(mt) <= SMEM_MAX; }
  // Ring depth: 4 slots only where they leave >= 56 KB of the SM's 256 KB
  // L1/shared array to L1, else 3 where they fit at all.  A 4-slot ring that
  // eats into L1 measured slower than 3 slots (m = 5: 218 KB 0.44 ms vs 183 KB
  // 0.39 ms; m = 6 and conservative m = 8 likewise: the cp.async staging
  // needs the L1 lines), while 2 slots starve the consumers (m = 7: 3 slots at
  // 215 KB beat 2 at 178 KB by 8%).
  static constexpr int SMEM_SOFT = 200 * 1024;
  static constexpr bool fits_soft(int mt, int ns) { return ns * sbuf(mt) * 8 + tail(mt) <= SMEM_SOFT; }
  // 8-cell M-tiles per consumer warp.  Each staged W fragment feeds MT DMMAs
  // and each corner load feeds NT, so shared-memory traffic per DMMA falls as
  // (4 MT + NT) / (MT NT): take MT = 2 where its accumulators (2 MT NT
  // doubles) fit the consumer registers and its slabs fit beside a 2-slot ring.
  // (MT = 3 measured slower than 2 at m = 4: the ring shrinks to 3 slots.)
  // (conservative m = 3: three M-tiles with a 2-slot ring measured 6% faster)
  static constexpr int MT0 = (SCH == kCons && M == 3) ? 3 : ((2 * NT <= 32 && fits(2, 2)) ? 2 : 1);
#ifdef HW_CM_MT  // (A/B builds: where it fits)
  static constexpr int MT = cm_knob(SCH, M) && fits(HW_CM_MT, 2) ? HW_CM_MT : MT0;
#else
  static constexpr int MT = MT0;
#endif
  static constexpr int TR = NW * MT / (TJ / 8);    // target rows per tile
  static constexpr int NODES = (TR + 1) * (TJ + 1);
  static constexpr int CBUF = NODES * KCP;
  static constexpr int WBUF = WRES ? 0 : KSC * NTB * 32;
  static constexpr int SBUF = CBUF + WBUF;         // doubles per ring slot
  // bit ch: ring chunk ch lies inside one field whose record length is even
  // (so a multiple of 4: no padding slots) -> 16-byte staging copies
  static constexpr unsigned wide_mask() {
    unsigned mk = 0;
    for (int ch = 0; ch < NCH && ch < 32; ++ch) {
      const int s0 = ch * KC, s1 = (s0 + KC < 4 * NK) ? s0 + KC : 4 * NK;
      const bool in0 = s1 <= K0, in1 = s0 >= K0;
      if ((in0 && P0 % 2 == 0) || (in1 && P1 > 0 && P1 % 2 == 0)) mk |= 1u << ch;
    }
    return mk;
  }
#ifdef HW_CM_WIDE
  static constexpr unsigned WIDE = HW_CM_WIDE ? wide_mask() : 0u;
#else
  static constexpr unsigned WIDE = wide_mask();
#endif
  static constexpr int SLAB = DIRECT ? 0 : MT * NT * 64;
  // The fragment-order slab rotates n-tile nt's 32 lane slots by SWZ * nt:
  // the drain's record-order gather then spreads a cell's outputs of equal
  // column over more banks (the consumer's 16-byte stores stay conflict-free).
  // Measured 1.5-4% faster for every order (conservative m = 3: 4% slower with
  // its four class tiles in round 1, 2.5% faster with the merged ones).
  static constexpr int SWZ0 = 1;
#ifdef HW_CM_SWZ
  static constexpr int SWZ = cm_knob(SCH, M) ? HW_CM_SWZ : SWZ0;
#else
  static constexpr int SWZ = SWZ0;
#endif
  static constexpr int PSLAB = PSMEM ? MT * 8 * O0 : 0;
  static constexpr int TAIL = tail(MT);
#ifdef HW_CM_NS
  static constexpr int NS = cm_knob(SCH, M) && fits(MT, HW_CM_NS) ? HW_CM_NS :
      cm_ns(SCH, M) && fits(MT, cm_ns(SCH, M)) ? cm_ns(SCH, M) :
      (M == 4 ? 3 : (fits_soft(MT, 4) ? 4 : (fits(MT, 3) ? 3 : 2)));
#elif defined(HW_CM_NSDEEP)
  // deepest ring within the soft limit (at least 2)
  static constexpr int deepest(int ns) { return ns <= 2 ? 2 : (fits_soft(MT, ns) ? ns : deepest(ns - 1)); }
  static constexpr int NS = deepest(NSMAX);
#else
  // (m = 4: 3 slots measured faster than 4 — conservative 5%, dissipative 0.5-0.8%; tools/gpu_ab.sh)
  static constexpr int NS = cm_ns(SCH, M) && fits(MT, cm_ns(SCH, M)) ? cm_ns(SCH, M) :
      (M == 4 ? 3 : (fits_soft(MT, 4) ? 4 : (fits(MT, 3) ? 3 : 2)));
#endif
  static constexpr int WRES0 = NS * SBUF;          // double offset of the resident W
  static constexpr int WL0 = WRES0 + WRESN;        // double offset of the SIMT weights
  static constexpr int EPI0 = WL0 + WLN;           // double offset of the slabs
  static constexpr int SMEM = NS * SBUF * 8 + TAIL;
  // W fragments double-buffered in registers too where NT <= 8, except for the
  // dissipative m <= 4, where reading them at use measured 0.5-0.8% faster
  static constexpr bool PREFETCH_B0 = NTB <= 8 && !(SCH == kDiss && M <= 4);
#ifdef HW_CM_PREB
  static constexpr bool PREFETCH_B = cm_knob(SCH, M) ? HW_CM_PREB : PREFETCH_B0;
#else
  static constexpr bool PREFETCH_B = PREFETCH_B0;
#endif
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cm_cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global" HW_CM_PF " [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cm_cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global" HW_CM_PF " [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// mbarrier primitives (CTA scope).
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Arrive once all of this thread's prior cp.async copies have landed.
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// HW_CM_WAITHINT > 0: try_wait with a suspend-time hint (ns), so a waiting
// warp is parked by the hardware instead of spinning on issue slots (A/B knob).
#ifndef HW_CM_WAITHINT
#define HW_CM_WAITHINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#if HW_CM_WAITHINT > 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(HW_CM_WAITHINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

// Non-blocking probe of a phase (warp-uniform when called by one lane and
// broadcast).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Producer-side wait: back off between polls so a producer that runs ahead
// of the ring does not steal issue slots from the consumer warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(128);
  }
}

// D += A B on the FP64 tensor cores (one 8x8x4 tile per warp).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// D = A B (C = 0): the first k-step of a tile (no accumulator reset needed).
__device__ __forceinline__ void dmma_first(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%4};\n"
      : "=d"(d[0]), "=d"(d[1])
      : "d"(a), "d"(b), "d"(0.0));
}

__device__ __forceinline__ double flip_sign(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ mask);
}

// Source row s of a field: local rows, slab halos, periodic wrap, wall ghost
// (boundary.py:119-130).
__device__ __forceinline__ const double* cm_row(const Rows& R, int64_t s, int64_t nx, int64_t rowlen, int periodic) {
  if (s >= R.row0 && s < R.row0 + R.nrows) return R.base + (s - R.row0) * rowlen;
  if (s == R.row0 - 1 && R.lo) return R.lo;
  if (s == R.row0 + R.nrows && R.hi) return R.hi;
  if (periodic) {
    while (s < 0) s += nx;
    while (s >= nx) s -= nx;
    CM_DBG_CHECK(s >= R.row0 && s < R.row0 + R.nrows, "periodic source row inside the local window");
    return R.base + (s - R.row0) * rowlen;
  }
  const int64_t w = s < 0 ? 0 : nx - 1;  // wall: mirror node, reflected later
  CM_DBG_CHECK(w >= R.row0 && w < R.row0 + R.nrows, "wall mirror row inside the local window");
  return R.base + (w - R.row0) * rowlen;
}

// Tile geometry: target rows [tr0, tr0 + nvr) x columns [j0, j0 + nvc);
// source nodes s_first.., c_first.. (global indices).
struct CMTile {
  int64_t tr0, j0, s_first, c_first;
  int nvr, nvc;
};

// MODE is a profiling knob (tools/cellmap_probe.cu): 0 = the product kernel,
// 1 = skip the staging copies (compute on whatever the ring holds),
// 2 = skip the tensor-core work and stores (staging only), 3 = skip the
// output stores to HBM (staging + tensor cores + slab epilogue).
#ifdef HW_CM_CTA_TIMES
// profiling build only (tools/cta_times.cu): per-CTA start / end globaltimer
__device__ unsigned long long hw_cm_cta_t[2 * 1024];
__device__ __forceinline__ unsigned long long cm_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HW_CM_STAMP_END() \
  if ((threadIdx.x & 31) == 0) atomicMax(&hw_cm_cta_t[2 * blockIdx.x + 1], cm_gtimer())
#else
#define HW_CM_STAMP_END()
#endif

template <int M, int SCH, int MODE = 0>
__global__ void __launch_bounds__(CMCfg<M, SCH>::NTHREADS, 1) cellmap_kernel(const __grid_constant__ CellMapArgs a) {
  using C = CMCfg<M, SCH>;
  constexpr int TR = C::TR, TJ = C::TJ, NT = C::NT, MT = C::MT, NS = C::NS, KSC = C::KSC, KC = C::KC,
                KCP = C::KCP, NCH = C::NCH, NW = C::NW;
  extern __shared__ __align__(16) double smem[];
  double* slabs = smem + C::EPI0;                           // [NW][SLAB]
  double* pslabs = slabs + NW * C::SLAB;                    // [NW][PSLAB]   (kCons)
  int* s_inv = reinterpret_cast<int*>(pslabs + NW * C::PSLAB);  // [8 * DO]: output -> fragment slot
  int* s_ocode = s_inv + 8 * C::DO;                              // [NT * 8]: fragment column -> output
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_ocode + 8 * NT + (8 * C::DO + 8 * NT) % 2);
  uint64_t* full = bars;                  // [NS] producers -> consumers: ring slot staged
  uint64_t* empty = bars + C::NSMAX;      // [NS] consumers -> producers: ring slot consumed
  uint64_t* sfull = bars + 2 * C::NSMAX;  // [NW] consumer w -> producer: output slab written
  uint64_t* sempty = sfull + NW;          // [NW] producer -> consumer w: output slab drained
  int* s_tile = reinterpret_cast<int*>(sempty + NW);  // [QT] tile id of this CTA's k-th tile (in the tail's slack)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // Inverse fragment map: output q of an M-tile's records, laid out
  // [8 x O0 | 8 x O1], lives in fragment slot (nt * 32 + lane) * 2 + i, where
  // lane = 4 r + j holds columns 2j, 2j+1 of n-tile nt for cell r.
  for (int idx = tid; idx < NT * 8; idx += blockDim.x) {
    const int nt = idx / 8, col = idx % 8, code = a.ocode[idx];
    s_ocode[idx] = code;
    if (code < 0) continue;
    const int o = code & 0xffff;
    for (int r = 0; r < 8; ++r) {
      const int q = (code >> 16) ? 8 * C::O0 + r * C::O1 + o : r * C::O0 + o;
      s_inv[q] = (nt * 32 + ((r * 4 + col / 2 + C::SWZ * nt) & 31)) * 2 + col % 2;
    }
  }
  for (int i = tid; i < C::WLN; i += blockDim.x) smem[C::WL0 + i] = a.wleft[i];  // (not step data: before the PDL wait)
  if (tid == 0) {
    s_tile[0] = blockIdx.x;
    for (int b = 0; b < NS; ++b) {
      mbar_init(&full[b], 2 * 32 * C::NPW);  // each producer lane: one plain arrive + one cp.async arrive
      mbar_init(&empty[b], NW);               // one arrive per consumer warp
    }
    for (int w = 0; w < NW; ++w) {
      mbar_init(&sfull[w], 1);
      mbar_init(&sempty[w], 1);
    }
  }
  __syncthreads();
#if HW_CM_PDL
  // Programmatic dependent launch (cellmap_launch.cuh): the setup above ran
  // while the previous step's grid was still finishing; every read of step
  // data and every output store comes after this wait, which returns once
  // that grid has completed and its stores are visible.  Then let the next
  // step's grid be scheduled, so its CTAs take each SM as this grid's CTA
  // there exits and run their setup under this grid's tail.
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
#ifdef HW_CM_CTA_TIMES
  if (tid == 0) hw_cm_cta_t[2 * blockIdx.x] = cm_gtimer();
#endif

  const int tcols = (int)((a.nty + TJ - 1) / TJ);
  const int ntiles = tcols * (int)((a.ntrows + TR - 1) / TR);
  // Dynamic tile schedule: CTA b starts on tile b, then takes the next
  // unclaimed tile from the global counter a.sched[0] (one lead producer lane
  // claims tile k + 1 when the CTA starts tile k and publishes it in
  // s_tile[(k + 1) % QT]).  The persistent CTAs then finish within one tile
  // of each other instead of within the spread of their static shares
  // (tools/cta_times.cu: 11% at m = 4, 1024^2).  A claim past the last tile
  // ends the CTA's sequence; the last CTA to make that claim zeroes the
  // counters for the next launch.  Null a.sched: static round robin.
  static_assert(C::NS + 2 <= C::QT, "tile-id ring shorter than the tiles in flight");
  static_assert((2 * C::NSMAX + 2 * NW) * 8 + (8 * C::DO + 8 * NT) * 4 + 4 * C::QT + 4 <=
                    (2 * C::NSMAX + 2 * NW) * 8 + (8 * C::DO + 8 * NT) * 4 + 64,
                "s_tile must fit the tail's slack");

  // tile / tcols without an integer division (every warp decodes every tile
  // id it touches: at m = 2 that division was ~13% of the kernel's instructions):
  // float reciprocal (tile < 2^24, exact to within one) and one correction each way
  const float inv_tcols = 1.0f / (float)tcols;
  auto tile_geo = [&](int tile) {
    CMTile t;
    int ti = (int)((float)tile * inv_tcols);
    ti -= ti * tcols > tile;
    ti += (ti + 1) * tcols <= tile;
    t.tr0 = (int64_t)ti * TR;
    t.j0 = (int64_t)(tile - ti * tcols) * TJ;
    const int64_t vr = a.ntrows - t.tr0, vc = a.nty - t.j0;
    t.nvr = vr < TR ? (int)vr : TR;
    t.nvc = vc < TJ ? (int)vc : TJ;
    t.s_first = a.trow0 + t.tr0 + a.off;
    t.c_first = t.j0 + a.off;
    return t;
  };
  // M-tile t of consumer warp w in tile `tg`: first target cell and valid count
  // (the MT M-tiles of a warp are stacked in x: consecutive target rows, same
  // 8 columns, so neighbouring M-tiles share a row of staged corners)
  auto mtile = [&](const CMTile& tg, int w, int t, int64_t& cell0) {
    const int trl = (w / (TJ / 8)) * MT + t, jl0 = (w % (TJ / 8)) * 8;
    cell0 = (tg.tr0 + trl) * a.nty + tg.j0 + jl0;
    return trl < tg.nvr ? (tg.nvc - jl0 < 8 ? tg.nvc - jl0 : 8) : 0;
  };

  if (warp >= NW) {
    // ------------------------------------------------------------ producers
    // one warpgroup; hands registers to the consumer warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PREGS));
    constexpr int NPL = 32 * C::NPW;
    constexpr int QL = NPL / KC;
    constexpr int NQ = (TJ + QL) / QL;  // node columns per lane (ceil((TJ+1)/QL))
    const int pl = tid - 32 * NW, pw = warp - NW;
    const int e = pl % KC, q0 = pl / KC;
    const bool active = q0 < QL;  // (KC not dividing the producer lanes: the last few lanes stage nothing)
    // Padding slots (record lengths rounded up to 4 per field) are zero.  When
    // every ring slot always holds the same chunk (NS a multiple of NCH) they
    // are zeroed once here instead of at every stage: at m = 2 the per-stage
    // zero stores were 12% of the shared-memory wavefronts and a divergent
    // branch in every staging step (+8% at m = 2, +2% at m = 4).
    constexpr bool PADONCE = (NS % NCH == 0) && !HW_CM_NOPADONCE;
    auto pad_slot = [](int slot) {  // input slot past its field's record (and below the last k-step)
      const bool f1 = slot >= C::K0;
      return (f1 ? slot - C::K0 : slot) >= (f1 ? C::P1 : C::P0) && slot < 4 * C::NK;
    };
    if constexpr (PADONCE) {
      if (active) {
#pragma unroll 1
        for (int b = 0; b < NS; ++b) {
          if (!pad_slot((b % NCH) * KC + e)) continue;
          double* dst = smem + b * C::SBUF + q0 * KCP + e;
#pragma unroll 1
          for (int r = 0; r <= TR; ++r)
#pragma unroll
            for (int k = 0; k < NQ; ++k)
              if (q0 + k * QL <= TJ) dst[(r * (TJ + 1) + k * QL) * KCP] = 0.0;
        }
      }
    }

    // Output drain for consumer warps pw and pw + NPW: slab -> HBM, coalesced.
    int ktot = 0x7fffffff;  // this CTA's tile count, once its last claim has come back
    int dk[NW / C::NPW];  // tiles of consumer warp pw + NPW j drained so far
#pragma unroll
    for (int j = 0; j < NW / C::NPW; ++j) dk[j] = 0;
    // INVREG: this lane's inverse-map entries of a full M-tile held in
    // registers (record slot lane + 32 k of field 0, then of field 1) instead
    // of one extra shared load per drained value: 2% faster at m = 4 (both
    // schemes), slower where the producer's registers run out (m = 5: +5%)
    constexpr int K0N = (8 * C::O0 + 31) / 32, K1N = (8 * C::O1 + 31) / 32;
#ifdef HW_CM_INVREG
    constexpr bool INVREG = (cm_knob(SCH, M) ? HW_CM_INVREG : M == 4) && K0N + K1N <= 16;
#else
    constexpr bool INVREG = M == 4 && K0N + K1N <= 16;
#endif
    int inv[INVREG ? K0N + K1N : 1];
    if constexpr (INVREG) {
#pragma unroll
      for (int k = 0; k < K0N; ++k) inv[k] = lane + 32 * k < 8 * C::O0 ? s_inv[lane + 32 * k] : 0;
#pragma unroll
      for (int k = 0; k < K1N; ++k) inv[K0N + k] = lane + 32 * k < 8 * C::O1 ? s_inv[8 * C::O0 + lane + 32 * k] : 0;
    }
    auto try_drain = [&]() {
      bool any = false;
      if constexpr (!C::OWN) {  // (DIRECT / SELF: the consumers store their own outputs)
#pragma unroll
      for (int j = 0; j < NW / C::NPW; ++j) {
        const int w = pw + C::NPW * j;
        if (dk[j] >= ktot) continue;
        int ready = lane == 0 ? (int)mbar_test(&sfull[w], dk[j] & 1) : 0;
        ready = __shfl_sync(0xffffffffu, ready, 0);
        if (!ready) continue;
        const CMTile tg = tile_geo(s_tile[dk[j] % C::QT]);
        const double* sl = slabs + w * C::SLAB;
        const double* pl0 = pslabs + w * C::PSLAB;  // kCons: `previous`, record order
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          int64_t cell0;
          const int nv = mtile(tg, w, t, cell0);
          if (MODE == 2 || MODE == 3 || nv == 0) continue;
          double* o0 = a.out0 + cell0 * C::O0;
          const double* s0 = sl + t * NT * 64;
          CM_DBG_CHECK(cell0 >= 0 && cell0 + nv <= a.ntrows * a.nty, "drained cells inside the target window");
          if (nv == 8) {  // full M-tile: fixed trip counts, loads batched 4 ahead of the stores
#pragma unroll
            for (int k0 = 0; k0 < K0N; k0 += 4) {
              double v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int q = lane + 32 * (k0 + u);
                if (k0 + u < K0N && q < 8 * C::O0) {
                  v[u] = s0[INVREG ? inv[INVREG ? k0 + u : 0] : s_inv[q]];
                  if (C::PSMEM) v[u] -= pl0[t * 8 * C::O0 + q];  // conservative.py:136
                }
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int q = lane + 32 * (k0 + u);
                if (k0 + u < K0N && q < 8 * C::O0) o0[q] = v[u];
              }
            }
            if (C::O1 > 0) {
              double* o1 = a.out1 + cell0 * C::O1;
#pragma unroll
              for (int k0 = 0; k0 < K1N; k0 += 4) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int q = lane + 32 * (k0 + u);
                  if (k0 + u < K1N && q < 8 * C::O1)
                    v[u] = s0[INVREG ? inv[INVREG ? K0N + k0 + u : 0] : s_inv[8 * C::O0 + q]];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const int q = lane + 32 * (k0 + u);
                  if (k0 + u < K1N && q < 8 * C::O1) o1[q] = v[u];
                }
              }
            }
          } else {
            for (int q = lane; q < nv * C::O0; q += 32)
              o0[q] = C::PSMEM ? s0[s_inv[q]] - pl0[t * 8 * C::O0 + q] : s0[s_inv[q]];
            if (C::O1 > 0) {
              double* o1 = a.out1 + cell0 * C::O1;
              for (int q = lane; q < nv * C::O1; q += 32) o1[q] = s0[s_inv[8 * C::O0 + q]];
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[w]);
        ++dk[j];
        any = true;
      }
      }
      return any;
    };

    int tile = blockIdx.x, ch = 0, kp = 0;
    const bool lead = pl == 0;
    int nexttile = 0;
    // claim(): issue the claim of the tile after next; its result is first
    // read one tile later, so the atomic's round trip never stalls the
    // producers.  finish(): after this CTA's last (failed) claim.
    auto claim = [&]() {
      return a.sched == nullptr ? nexttile + (int)gridDim.x  // static: b, b + G, b + 2G, ...
                                : (int)gridDim.x + atomicAdd(a.sched, 1);
    };
    auto finish = [&]() {
      if (a.sched == nullptr) return;
      __threadfence();
      if (atomicAdd(a.sched + 1, 1) == (int)gridDim.x - 1) {  // the last CTA zeroes the counters
        __threadfence();
        atomicExch(a.sched, 0);
        atomicExch(a.sched + 1, 0);
      }
    };
    if (lead) {
      nexttile = tile;
      nexttile = claim();
    }
    CMTile t = tile_geo(tile);
    // 16-byte staging needs 16-byte aligned field bases (even-length records
    // keep every node and chunk offset even from there)
    const bool base_al16 = ((reinterpret_cast<uintptr_t>(a.f0.base) | reinterpret_cast<uintptr_t>(a.f1.base)) & 15) == 0;
    for (int g = 0;; ++g) {
      const int b = g % NS;
      if (g >= NS) {  // wait for the slot, draining finished output slabs meanwhile
        while (true) {
          int ok = lane == 0 ? (int)mbar_test(&empty[b], ((g / NS) - 1) & 1) : 0;
          if (__shfl_sync(0xffffffffu, ok, 0)) break;
          if (!try_drain()) __nanosleep(HW_CM_SLEEP);
        }
      } else {
        try_drain();
      }
      if (tile >= ntiles) {  // end of the sequence: wake the consumers on it (they read s_tile and exit)
        mbar_arrive(&full[b]);
        mbar_arrive(&full[b]);
        ktot = kp;
        break;
      }
      double* cb = smem + b * C::SBUF;
#if HW_CM_DEBUG
      {  // poison the slot (every consumer released it), then stage after a random delay
        const double nanv = __longlong_as_double(0x7ff8dead00000000ll);
        for (int i = pl; i < C::SBUF; i += NPL)  // (the once-zeroed padding slots stay)
          if (!(PADONCE && i < C::CBUF && i % KCP < KC && pad_slot(ch * KC + i % KCP))) cb[i] = nanv;
        asm volatile("bar.sync 2, %0;\n" ::"n"(NPL) : "memory");
        __nanosleep(cm_dbg_rand(g, tid) & 2047);
      }
#endif
      const int slot = ch * KC + e;  // input slot: field 0 in [0, K0), field 1 in [K0, 4 NK)
      const bool f1 = slot >= C::K0;
      const int eo = f1 ? slot - C::K0 : slot;
      const bool pad = eo >= (f1 ? C::P1 : C::P0);
      const bool edge = t.s_first < 0 || t.s_first + t.nvr >= a.nx || t.c_first < 0 || t.c_first + t.nvc >= a.ny;
      const bool manual = !a.periodic && edge;  // wall ghosts: reflect after the copies land
      double* dst = cb + q0 * KCP + e;
      const bool interior = t.nvr == TR && t.nvc == TJ && t.s_first >= a.f0.row0 &&
                            t.s_first + TR < a.f0.row0 + a.f0.nrows && t.c_first >= 0 && t.c_first + TJ < a.ny;
      if (MODE != 1 && interior && (C::WIDE >> ch & 1u) && base_al16) {
        // interior tile, chunk inside one field of even record length (no
        // padding slots): 16-byte L2-only copies of slot pairs, lane -> (pair
        // pl % (KC/2), node pl / (KC/2)); slots beyond the last k-step are never read
        constexpr int PAIRS = KC / 2, QW = NPL / PAIRS, NQW = (TJ + QW) / QW;
        const int e2 = 2 * (pl % PAIRS), qw = pl / PAIRS;
        if (qw < QW && ch * KC + e2 < 4 * C::NK) {
          const bool fw = ch * KC >= C::K0;
          const int pf = fw ? C::P1 : C::P0;
          const int64_t rowlen = a.ny * pf;
          const double* src = (fw ? a.f1.base : a.f0.base) + (t.s_first - a.f0.row0) * rowlen +
                              (t.c_first + qw) * pf + (fw ? ch * KC - C::K0 : ch * KC) + e2;
          double* dw = cb + qw * KCP + e2;
#pragma unroll
          for (int r = 0; r <= TR; ++r) {
#pragma unroll
            for (int k = 0; k < NQW; ++k)
              if (qw + k * QW <= TJ) cm_cp_async16(dw + (r * (TJ + 1) + k * QW) * KCP, src + k * QW * pf);
            src += rowlen;
          }
        }
      } else if (!active || (PADONCE && pad)) {
      } else if (pad) {
#pragma unroll 1
        for (int r = 0; r <= TR; ++r)
#pragma unroll
          for (int k = 0; k < NQ; ++k)
            if (q0 + k * QL <= TJ) dst[(r * (TJ + 1) + k * QL) * KCP] = 0.0;
      } else if (MODE != 1 && interior) {
        // interior tile: every staged row is a dense segment of the local slab
        const int pf = f1 ? C::P1 : C::P0;
        const int64_t rowlen = a.ny * pf;
        const double* src = (f1 ? a.f1.base : a.f0.base) + (t.s_first - a.f0.row0) * rowlen + (t.c_first + q0) * pf + eo;
        const int cstep = QL * pf;
        CM_DBG_CHECK(t.s_first >= a.f0.row0 && t.s_first + TR < a.f0.row0 + a.f0.nrows, "interior tile rows local");
#pragma unroll
        for (int r = 0; r <= TR; ++r) {
#pragma unroll
          for (int k = 0; k < NQ; ++k)
            if (k < NQ - 1 || q0 + k * QL <= TJ) cm_cp_async8(dst + (r * (TJ + 1) + k * QL) * KCP, src + k * cstep);
          src += rowlen;
        }
      } else if (MODE != 1) {
        const int pf = f1 ? C::P1 : C::P0;
        const int64_t rowlen = a.ny * pf;
        int col[NQ];  // offset of this lane's entry in each staged column (fits 32 bits: ny * P < 2^31)
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          int64_t c = t.c_first + q0 + k * QL;
          if (c < 0) c = a.periodic ? c + a.ny : 0;
          if (c >= a.ny) c = a.periodic ? c - a.ny : a.ny - 1;
          col[k] = (int)c * pf + eo;
        }
#pragma unroll 1
        for (int r = 0; r <= t.nvr; ++r) {
          const double* row = f1 ? cm_row(a.f1, t.s_first + r, a.nx, rowlen, a.periodic)
                                 : cm_row(a.f0, t.s_first + r, a.nx, rowlen, a.periodic);
#pragma unroll
          for (int k = 0; k < NQ; ++k)
            if (q0 + k * QL <= t.nvc) cm_cp_async8(dst + (r * (TJ + 1) + k * QL) * KCP, row + col[k]);
        }
        if (manual) {
          // wall ghosts: wait for this lane's copies, then reflect them in place
          // (boundary.py:56-98; field 1 reflects around zero, dissipative.py:229)
          asm volatile("cp.async.wait_all;\n" ::: "memory");
          const int w = f1 ? C::W1 : C::W0;
#pragma unroll 1
          for (int r = 0; r <= t.nvr; ++r) {
            const int64_t s = t.s_first + r;
            const int xk = s < 0 ? a.kxl : (s >= a.nx ? a.kxh : 0);
            const double gx = f1 ? 0.0 : (s < 0 ? a.gxl : a.gxh);
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
              const int q = q0 + k * QL;
              const int64_t c = t.c_first + q;
              const int yk = c < 0 ? a.kyl : (c >= a.ny ? a.kyh : 0);
              if (q > t.nvc || !(xk | yk)) continue;
              const double gy = f1 ? 0.0 : (c < 0 ? a.gyl : a.gyh);
              double* pv = dst + (r * (TJ + 1) + k * QL) * KCP;
              *pv = ghosted(*pv, eo / w, eo % w, xk, gx, yk, gy);
            }
          }
        }
      }
      // W fragments of the chunk (contiguous, 16-byte aligned)
      const int nks = (C::NK - ch * KSC) < KSC ? (C::NK - ch * KSC) : KSC;
      if (!C::WRES) {
        const double* wsrc = a.wfrag + ch * KSC * C::NTB * 32;
        double* wb = cb + C::CBUF;
#pragma unroll 1
        for (int i = pl; i < nks * C::NTB * 16; i += NPL) cm_cp_async16(wb + 2 * i, wsrc + 2 * i);
      } else if (g == 0) {  // the whole W once; stage 0's cp.async arrive covers it
#pragma unroll 1
        for (int i = pl; i < C::NK * C::NTB * 16; i += NPL) cm_cp_async16(smem + C::WRES0 + 2 * i, a.wfrag + 2 * i);
      }
      mbar_arrive(&full[b]);           // orders this lane's plain shared stores
      mbar_arrive_cp_async(&full[b]);  // fires when this lane's copies have landed
      if (++ch == NCH) {
        ch = 0;
        ++kp;
        if (lead) {
          s_tile[kp % C::QT] = nexttile;
          if (nexttile < ntiles)
            nexttile = claim();
          else
            finish();
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(NPL) : "memory");  // producers: s_tile[kp] published
        tile = s_tile[kp % C::QT];
        if (tile < ntiles) t = tile_geo(tile);
      }
    }
    // drain the remaining output slabs
    while (!C::OWN) {
      bool left = false;
#pragma unroll
      for (int j = 0; j < NW / C::NPW; ++j) left |= dk[j] < ktot;
      if (!left) break;
      if (!try_drain()) __nanosleep(HW_CM_SLEEP);
    }
    HW_CM_STAMP_END();
    return;
  }

  // -------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CREGS));
  // Parity bits (kx & 1, ky & 1) of this lane's input slot 4 s + (lane & 3)
  // at every k-step s (sign flips of the x- / y-right corners).
  unsigned long long kxbits = 0, kybits = 0;
#pragma unroll 1
  for (int st = 0; st < C::NK; ++st) {
    const int code = a.icode[st * 4 + (lane & 3)];
    kxbits |= (unsigned long long)(code & 1) << st;
    kybits |= (unsigned long long)((code >> 1) & 1) << st;
  }
#if HW_CM_DCODE
  int dcode[C::DIRECT ? NT : 1][2];  // DIRECT epilogue: this lane's output codes (field << 16 | offset, -1 pad)
  if constexpr (C::DIRECT) {
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int i = 0; i < 2; ++i) dcode[n][i] = s_ocode[n * 8 + 2 * (lane & 3) + i];
  }
#endif
  double acc[MT][NT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
  constexpr int LC = C::LC, NTD = C::NTD, NTB = C::NTB;
  double part[MT][LC > 0 ? LC : 1];  // SIMT columns: this lane's partial sums over its input slots
  double pvr[C::PREVREG ? MT : 1][C::PREVREG ? NT : 1][2];  // PREVREG: `previous` at this lane's accumulator slots

  int ch = 0, k = 0;  // k = this warp's tile count
  CMTile cg;
  double* slab = slabs + warp * C::SLAB;
  for (int g = 0;; ++g) {
    const int b = g % NS;
    if (ch == 0) {  // a new tile: its id is published with its first chunk
      mbar_wait(&full[b], (g / NS) & 1);
      const int tile = s_tile[k % C::QT];
      if (tile >= ntiles) break;
      cg = tile_geo(tile);
      if constexpr (C::PREVREG) {
        // `previous` of this lane's accumulator slots (cell r = lane / 4 of each
        // M-tile, columns 2 (lane & 3), +1 of each n-tile): plain loads issued
        // now land while the tile's DMMAs run; used in the epilogue.  In place
        // is safe: only this tile's epilogue writes these records, later.
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          int64_t cell0;
          const int nv = mtile(cg, warp, t, cell0);
          const double* pc = a.prev + (cell0 + (lane >> 2)) * C::O0;
#pragma unroll
          for (int n = 0; n < NT; ++n)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int code = s_ocode[n * 8 + 2 * (lane & 3) + i];
              pvr[t][n][i] = (code >= 0 && (lane >> 2) < nv) ? pc[code & 0xffff] : 0.0;
            }
        }
      }
    }
    if (ch == NCH - 1) {
      // The tile's last chunk: the previous tile's slab must be drained before
      // this tile's epilogue reuses it (and, for kCons, before its `previous`
      // records are staged — contiguous, with cp.async, landing under the
      // last chunk's DMMAs).
      if (!C::OWN && k >= 1) mbar_wait(&sempty[warp], (k - 1) & 1);
      if (C::PSMEM) {
        double* pv = pslabs + warp * C::PSLAB;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          int64_t cell0;
          const int nv = mtile(cg, warp, t, cell0);
          const double* p = a.prev + cell0 * C::O0;
          for (int q = lane; q < nv * C::O0; q += 32) cm_cp_async8(pv + t * 8 * C::O0 + q, p + q);
        }
      }
    }
#if HW_CM_DEBUG
    __nanosleep(cm_dbg_rand(g, tid) & 1023);
#endif
    if (ch != 0) mbar_wait(&full[b], (g / NS) & 1);
    const double* cb = smem + b * C::SBUF;
    const double* wb = C::WRES ? smem + C::WRES0 + ch * KSC * NTB * 32 : cb + C::CBUF;
    // One chunk of NKS k-steps, software-pipelined: the shared-memory
    // operands of k-step ks+1 (corner values; W fragments when registers
    // allow) are loaded before the DMMAs of k-step ks issue.  FIRST: the
    // tile's first chunk, whose first k-step starts the accumulators (C = 0).
    auto run_chunk = [&](auto nks_c, auto first_c) {
      constexpr int NKS = decltype(nks_c)::value;
      constexpr bool FIRST = decltype(first_c)::value;
      constexpr bool PREB = C::PREFETCH_B;
      // raw[.][r] = the two y-corners of staged row trl0 + r (row r + 1 of
      // M-tile r is row 0 of M-tile r + 1: MT + 1 rows feed MT M-tiles)
      double raw[2][MT + 1][2];
      double bb[PREB ? 2 : 1][NTB];
      const int trl0 = (warp / (TJ / 8)) * MT, tc = (warp % (TJ / 8)) * 8;
      const double* pbase = cb + (trl0 * (TJ + 1) + tc + (lane >> 2)) * KCP + (lane & 3);
      auto load = [&](const int ks, const int slot) {
#pragma unroll
        for (int r = 0; r <= MT; ++r) {
          const double* p = pbase + r * (TJ + 1) * KCP + ks * 4;
          raw[slot][r][0] = p[0];
          raw[slot][r][1] = p[KCP];
        }
        if (PREB) {
          const double* wk = wb + ks * NTB * 32 + lane;
#pragma unroll
          for (int nt = 0; nt < NTB; ++nt) bb[PREB ? slot : 0][nt] = wk[nt * 32];
        }
      };
      load(0, 0);
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int cur = ks & 1;
        if (ks + 1 < NKS) load(ks + 1, cur ^ 1);
        const int step = ch * KSC + ks;
        const unsigned long long mx = ((kxbits >> step) & 1ull) << 63;
        const unsigned long long my = ((kybits >> step) & 1ull) << 63;
        double A[MT][4];
        const double* wk = wb + ks * NTB * 32 + lane;
        if constexpr (C::PXM) {
          // y-pair sums per staged row; the tensor cores combine the rows
          double P[MT + 1], Q[MT + 1];
#pragma unroll
          for (int r = 0; r <= MT; ++r) {
            const double yl = raw[cur][r][0], yr = flip_sign(raw[cur][r][1], my);
            P[r] = yl + yr;  // y-even classes
            Q[r] = yl - yr;  // y-odd classes
          }
#pragma unroll
          for (int nt = 0; nt < NTD; ++nt) {
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
              const double bf = PREB ? bb[PREB ? cur : 0][2 * nt + dx] : wk[(2 * nt + dx) * 32];
#pragma unroll
              for (int t = 0; t < MT; ++t) {
                const double av = nt < C::TG1 ? P[t + dx] : Q[t + dx];
                if (FIRST && ks == 0 && dx == 0)
                  dmma_first(acc[t][nt], av, bf);
                else
                  dmma(acc[t][nt], av, bf);
              }
            }
          }
          continue;
        }
        if constexpr (cm_yfirst(SCH, M)) {
          // y-pairs first, per staged row (row t + 1 is shared by M-tiles t and
          // t + 1): 2 (MT + 1) + 4 MT additions instead of 8 MT
          double P[MT + 1], Q[MT + 1];
#pragma unroll
          for (int r = 0; r <= MT; ++r) {
            const double yl = raw[cur][r][0], yr = flip_sign(raw[cur][r][1], my);
            P[r] = yl + yr;  // y-even classes
            Q[r] = yl - yr;  // y-odd classes
          }
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const double p1 = flip_sign(P[t + 1], mx), q1 = flip_sign(Q[t + 1], mx);
            A[t][0] = P[t] + p1;  // class (0,0)
            A[t][1] = Q[t] + q1;  // class (0,1)
            A[t][2] = P[t] - p1;  // class (1,0)
            A[t][3] = Q[t] - q1;  // class (1,1)
          }
        } else {
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            const double c00 = raw[cur][t][0];
            const double c01 = flip_sign(raw[cur][t][1], my);
            const double c10 = flip_sign(raw[cur][t + 1][0], mx);
            const double c11 = flip_sign(raw[cur][t + 1][1], mx ^ my);
            const double ap = c00 + c10, am = c00 - c10, bp = c01 + c11, bm = c01 - c11;
            A[t][0] = ap + bp;  // class (0,0)
            A[t][1] = ap - bp;  // class (0,1)
            A[t][2] = am + bm;  // class (1,0)
            A[t][3] = am - bm;  // class (1,1)
          }
        }
        if constexpr (LC > 0) {
          // SIMT columns: W_c[o][slot] for this lane's slot (4 distinct per warp: one wavefront)
          const double* wl = smem + C::WL0 + step * LC * 4 + (lane & 3);
#pragma unroll
          for (int j = 0; j < LC; ++j) {
            const double w = wl[j * 4];
#pragma unroll
            for (int t = 0; t < MT; ++t) {
              const double av = A[t][cm_lclass(SCH, M, j)];
              part[t][j] = (FIRST && ks == 0) ? w * av : fma(w, av, part[t][j]);
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < NTD; ++nt) {
          const int c = nt < C::B1 ? 0 : (nt < C::B2 ? 1 : (nt < C::B3 ? 2 : 3));  // parity class of tile nt
          const double bf = PREB ? bb[PREB ? cur : 0][nt] : wk[nt * 32];
#pragma unroll
          for (int t = 0; t < MT; ++t) {
            if (FIRST && ks == 0)
              dmma_first(acc[t][nt], A[t][c], bf);
            else
              dmma(acc[t][nt], A[t][c], bf);
          }
        }
      }
    };
    if constexpr (MODE != 2) {
      using KF = std::integral_constant<int, KSC>;
      using KL = std::integral_constant<int, C::NK - (NCH - 1) * KSC>;
      if constexpr (NCH == 1) {
        run_chunk(KL{}, std::true_type{});
      } else {
        if (ch == 0)
          run_chunk(KF{}, std::true_type{});
        else if (ch == NCH - 1)
          run_chunk(KL{}, std::false_type{});
        else
          run_chunk(KF{}, std::false_type{});
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);  // ring slot b may be refilled
    if constexpr (LC > 0) {
      if (ch == NCH - 1) {
        // the four lanes of a cell (lane & 3 = its input slots) sum their partials;
        // lane 4 r + q then holds SIMT columns 2 q, 2 q + 1 of each SIMT tile (fragment layout)
#pragma unroll
        for (int t = 0; t < MT; ++t) {
#pragma unroll
          for (int j = 0; j < LC; ++j) {
            double v = part[t][j];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            part[t][j] = v;
          }
#pragma unroll
          for (int s2 = 0; s2 < C::NT - NTD; ++s2)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              double v = 0.0;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int j = 8 * s2 + 2 * q + i;
                if (j < LC && (lane & 3) == q) v = part[t][j < LC ? j : 0];
              }
              acc[t][NTD + s2][i] = v;
            }
        }
      }
    }

    if (C::PREVREG && ch == NCH - 1) {  // conservative.py:136: new = 2 WT I(cur) - previous
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          acc[t][n][0] -= pvr[t][n][0];
          acc[t][n][1] -= pvr[t][n][1];
        }
    }
    if (ch == NCH - 1 && C::DIRECT) {
      // Epilogue straight to HBM: lane 4 r + j stores outputs 2 j, 2 j + 1 of
      // every n-tile for cell r of each M-tile.
      if (C::PSMEM) asm volatile("cp.async.wait_all;\n" ::: "memory");  // `previous` landed
      const double* pv = pslabs + warp * C::PSLAB;
      const int r = lane >> 2;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        int64_t cell0;
        const int nv = mtile(cg, warp, t, cell0);
        if (MODE == 3 || r >= nv) continue;
        double* d0 = a.out0 + (cell0 + r) * C::O0;
        double* d1 = C::O1 > 0 ? a.out1 + (cell0 + r) * C::O1 : nullptr;
#if HW_CM_DCODE
        // branch-free: this lane's destinations were resolved once (dcode)
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int code = dcode[n][i];
            double* base = (C::O1 > 0 && (code >> 16) > 0) ? d1 : d0;
            double v = acc[t][n][i];
            if (C::PSMEM) v -= (code >= 0 && (code >> 16) == 0) ? pv[t * 8 * C::O0 + r * C::O0 + (code & 0xffff)] : 0.0;
            if (code >= 0) base[code & 0xffff] = v;
          }
#else
#pragma unroll
        for (int n = 0; n < NT; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int code = s_ocode[n * 8 + 2 * (lane & 3) + i];  // (held in registers: 13% slower at m=2)
            if (code < 0) continue;
            const int o = code & 0xffff;
            if (code >> 16)
              d1[o] = acc[t][n][i];
            else
              d0[o] = C::PSMEM ? acc[t][n][i] - pv[t * 8 * C::O0 + r * C::O0 + o] : acc[t][n][i];
          }
#endif
      }
      __syncwarp();
    } else if (ch == NCH - 1) {
      // Epilogue: accumulators -> this warp's output slab in fragment order; a
      // producer warp drains the slab to HBM while this warp moves on.
#pragma unroll
      for (int t = 0; t < MT; ++t)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          *reinterpret_cast<double2*>(slab + t * NT * 64 + (n * 32 + ((lane + C::SWZ * n) & 31)) * 2) =
              make_double2(acc[t][n][0], acc[t][n][1]);
      if (C::PSMEM) asm volatile("cp.async.wait_all;\n" ::: "memory");  // `previous` landed
      __syncwarp();
      if constexpr (C::SELF) {
        // drain it ourselves: record order, consecutive lanes on consecutive doubles
        const double* pv = pslabs + warp * C::PSLAB;
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          int64_t cell0;
          const int nv = mtile(cg, warp, t, cell0);
          if (MODE == 3 || nv == 0) continue;
          const double* s0 = slab + t * NT * 64;
          double* o0 = a.out0 + cell0 * C::O0;
          for (int q = lane; q < nv * C::O0; q += 32)
            o0[q] = C::PSMEM ? s0[s_inv[q]] - pv[t * 8 * C::O0 + q] : s0[s_inv[q]];
          if (C::O1 > 0) {
            double* o1 = a.out1 + cell0 * C::O1;
            for (int q = lane; q < nv * C::O1; q += 32) o1[q] = s0[s_inv[8 * C::O0 + q]];
          }
        }
        __syncwarp();
      } else {
        if (lane == 0) mbar_arrive(&sfull[warp]);
      }
    }
    if (ch == NCH - 1) {
      ++k;
      ch = 0;
    } else {
      ++ch;
    }
  }
  HW_CM_STAMP_END();
}

}  // namespace hw
