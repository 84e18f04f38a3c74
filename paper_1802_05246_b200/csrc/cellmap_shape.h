// Compile-time shape of the per-class cell maps (shared by the host builder
// and the sm_100a kernel so both agree on the class/tile layout).
#pragma once

namespace hw {

enum Scheme : int { kDiss = 0, kCons = 1, kBoot = 2 };

// field widths (orders + 1) of the inputs / outputs of each scheme
constexpr int cm_win(int sch, int m, int f) { return f == 0 ? m + 1 : (sch == 0 ? m : (sch == 2 ? m + 1 : 0)); }
constexpr int cm_wout(int sch, int m, int f) { return f == 0 ? m + 1 : (sch == 0 ? m : 0); }

// (A/B knob filter, as cm_knob below)
constexpr bool cm_knob_h(int sch, int m) {
#ifdef HW_CM_KNOB_M
  if (m != HW_CM_KNOB_M) return false;
#endif
#ifdef HW_CM_KNOB_SCH
  if (sch != HW_CM_KNOB_SCH) return false;
#endif
  return sch >= 0 && m >= 0;
}

// number of k in [0, w) with k % 2 == p
constexpr int cm_cnt_par(int w, int p) { return w > p ? (w - 1 - p) / 2 + 1 : 0; }

constexpr int cm_din(int sch, int m) { return cm_win(sch, m, 0) * cm_win(sch, m, 0) + cm_win(sch, m, 1) * cm_win(sch, m, 1); }
constexpr int cm_dout(int sch, int m) {
  return cm_wout(sch, m, 0) * cm_wout(sch, m, 0) + cm_wout(sch, m, 1) * cm_wout(sch, m, 1);
}

// outputs of parity class c = (PA, PB) = (c >> 1, c & 1)
constexpr int cm_ncls(int sch, int m, int c) {
  return cm_cnt_par(cm_wout(sch, m, 0), c >> 1) * cm_cnt_par(cm_wout(sch, m, 0), c & 1) +
         cm_cnt_par(cm_wout(sch, m, 1), c >> 1) * cm_cnt_par(cm_wout(sch, m, 1), c & 1);
}

// Merged x-classes (PXM; the dissipative m <= 2, conservative / bootstrap
// m = 3, bootstrap m <= 2 — where the merged tiles need no more DMMAs): the outputs of classes
// (0, PB) and (1, PB) share n-tiles, and the x-combination of the corners
// runs on the tensor cores instead of the butterfly: each tile takes two DMMAs
// per k-step, one on the upper and one on the lower corner row's y-pair sums
// (P = U(r,0) + s U(r,1), Q = U(r,0) - s U(r,1); s = (-1)^ky), with the
// x-signs (-1)^((PA + kx) dx) folded into the W fragments of the lower row.
// At m = 2 the classes hold 5 / 3 / 3 / 2 outputs, so 4 class tiles become
// 2 merged tiles x 2 rows (the same DMMA count) while the additions per
// k-step fall from 8 MT to 2 (MT + 1) — the FP64 datapath DMMA and DADD share.
constexpr bool cm_pxm(int sch, int m) {
#ifdef HW_CM_PXM
  if (cm_knob_h(sch, m)) return HW_CM_PXM && (sch == 0 ? m <= 2 : (m == 3 || (sch == 2 && m <= 2)));
#endif
  // (the conservative m <= 2 runs on the SIMT kernel; the bootstrap m <= 2 on this one)
  return sch == 0 ? m <= 2 : (m == 3 || (sch == 2 && m <= 2));
}
// Hybrid tiles.  A class's outputs fill 8-wide DMMA n-tiles (m8n8k4: N = 8);
// where class c's remainder r_c = n_c mod 8 is in the class mask cm_lmask,
// those r_c outputs are computed on the CUDA cores instead of padding a
// whole n-tile: each lane accumulates W_c[o][e] G^c[e] over its own input
// slots (the A fragment it already holds) and the four lanes of a cell sum
// by shuffles.  The left-over outputs of all masked classes form the columns
// of extra "SIMT" tiles laid out like DMMA fragments, so the epilogue is
// unchanged.  (Pipe cost per M-tile and k-step: a padded DMMA tile 4 clocks
// of the SM's FP64 datapath, r_c SIMT columns r_c / 2 clocks.)
constexpr int cm_lmask(int sch, int m) {
#ifdef HW_CM_LMASK
  if (cm_knob_h(sch, m)) return HW_CM_LMASK;
#endif
  // measured (profiles/ab_r02_kernel_knobs.txt): cons m = 5 (+7%); one left-over output of class (0,0) on
  // the CUDA cores in place of a whole n-tile at diss m = 6, 8 (+2.6%, +2.7%) and cons m = 8 (+1%);
  // off elsewhere (diss m = 4 -2% (0x6) / -7% (0xf), m = 2 20-39% slower, cons m = 4 0x1 -8%)
  if (sch == 1 && m == 5) return 0xf;
  return ((sch == 0 && (m == 6 || m == 8)) || (sch == 1 && m == 8)) ? 0x1 : 0;
}
constexpr int cm_rem(int sch, int m, int c) { return cm_ncls(sch, m, c) % 8; }
constexpr int cm_left(int sch, int m, int c) {
  return (cm_lmask(sch, m) >> c & 1) && !cm_pxm(sch, m) ? cm_rem(sch, m, c) : 0;  // (none under PXM)
}
// DMMA n-tiles of class c and their prefix sums
constexpr int cm_ntc(int sch, int m, int c) {
  return cm_left(sch, m, c) ? cm_ncls(sch, m, c) / 8 : (cm_ncls(sch, m, c) + 7) / 8;
}
constexpr int cm_ntbase(int sch, int m, int c) {  // non-recursive: folds inside unrolled device loops
  return (c > 0 ? cm_ntc(sch, m, 0) : 0) + (c > 1 ? cm_ntc(sch, m, 1) : 0) + (c > 2 ? cm_ntc(sch, m, 2) : 0) +
         (c > 3 ? cm_ntc(sch, m, 3) : 0);
}
constexpr int cm_pxm_n(int sch, int m, int pb) { return cm_ncls(sch, m, pb) + cm_ncls(sch, m, 2 + pb); }
constexpr int cm_pxm_tiles(int sch, int m, int pb) { return (cm_pxm_n(sch, m, pb) + 7) / 8; }
constexpr int cm_ntd(int sch, int m) {  // DMMA tiles
  return cm_pxm(sch, m) ? cm_pxm_tiles(sch, m, 0) + cm_pxm_tiles(sch, m, 1) : cm_ntbase(sch, m, 4);
}
// B fragments per k-step: one per DMMA tile, two (upper / lower corner row) under PXM
constexpr int cm_ntb(int sch, int m) { return cm_pxm(sch, m) ? 2 * cm_ntd(sch, m) : cm_ntd(sch, m); }
// SIMT columns (left-over outputs, class 0's first) and SIMT tiles
constexpr int cm_lbase(int sch, int m, int c) {
  return (c > 0 ? cm_left(sch, m, 0) : 0) + (c > 1 ? cm_left(sch, m, 1) : 0) + (c > 2 ? cm_left(sch, m, 2) : 0) +
         (c > 3 ? cm_left(sch, m, 3) : 0);
}
constexpr int cm_lc(int sch, int m) { return cm_lbase(sch, m, 4); }
constexpr int cm_lclass(int sch, int m, int j) {  // class of SIMT column j
  return j < cm_lbase(sch, m, 1) ? 0 : (j < cm_lbase(sch, m, 2) ? 1 : (j < cm_lbase(sch, m, 3) ? 2 : 3));
}
constexpr int cm_nts(int sch, int m) { return (cm_lc(sch, m) + 7) / 8; }
// all fragment-layout tiles (accumulators, epilogue): DMMA, then SIMT
constexpr int cm_nt(int sch, int m) { return cm_ntd(sch, m) + cm_nts(sch, m); }

// parity class that DMMA output tile nt belongs to
constexpr int cm_class_of_tile(int sch, int m, int nt) {
  return nt < cm_ntbase(sch, m, 1) ? 0 : (nt < cm_ntbase(sch, m, 2) ? 1 : (nt < cm_ntbase(sch, m, 3) ? 2 : 3));
}

// Conservative scheme: `previous` loaded into registers at the tile's first
// chunk and subtracted from the accumulators (1), or copied into a
// shared-memory slab at the last chunk (0): registers measured +2% at m = 5,
// +12% at m = 6; the slab stays where the registers run out (m = 3: -27%,
// m = 8: -55%) (profiles/ab_r02_kernel_knobs.txt).
constexpr bool cm_prevreg(int sch, int m) {
#ifdef HW_CM_PREVREG
  if (cm_knob_h(sch, m)) return HW_CM_PREVREG;
#endif
  return sch == 1 && (m == 5 || m == 6);
}

// Corner butterfly order: y-pairs per staged row first (shared by the stacked
// M-tiles: 2 (MT + 1) + 4 MT additions instead of 8 MT) where it measured
// faster — dissipative m = 3..5 (+0.6% m = 4, +1.3% m = 5); x-pairs first
// elsewhere (m = 2: 4.5% slower y-first; m = 6..8 ~1%)
// (profiles/ab_r02_kernel_knobs.txt).
constexpr bool cm_yfirst(int sch, int m) {
#ifdef HW_CM_YFIRST
  if (cm_knob_h(sch, m)) return HW_CM_YFIRST;
#endif
  return sch == 0 && m >= 3 && m <= 5;
}

// Input slots: each field's entries padded to a multiple of 4 (a 4-deep
// DMMA k-step never straddles the two fields): field 0 in [0, K0), field 1
// from K0.  k-steps of 4 slots: NK.
constexpr int cm_k0(int sch, int m) { return (cm_win(sch, m, 0) * cm_win(sch, m, 0) + 3) / 4 * 4; }
constexpr int cm_nk(int sch, int m) {
  return (cm_k0(sch, m) + (cm_win(sch, m, 1) * cm_win(sch, m, 1) + 3) / 4 * 4) / 4;
}

// A/B builds (tools/build_variant.sh): -DHW_CM_<KNOB>=v overrides one of the
// per-order choices below, for every order or, with -DHW_CM_KNOB_M=m (and
// -DHW_CM_KNOB_SCH=s), for one.
constexpr bool cm_knob(int sch, int m) {
#ifdef HW_CM_KNOB_M
  if (m != HW_CM_KNOB_M) return false;
#endif
#ifdef HW_CM_KNOB_SCH
  if (sch != HW_CM_KNOB_SCH) return false;
#endif
  return sch >= 0 && m >= 0;
}

// The kernel's staging unit: k-steps per ring chunk.
constexpr int cm_ksc(int sch, int m) {
#ifdef HW_CM_KSC
  if (cm_knob_h(sch, m)) return HW_CM_KSC;
#endif
  // conservative m = 5 (NK = 9): three 3-k-step chunks instead of 4 + 4 + 1, with the smaller ring
  // slots (node stride 12) allowing a 5-deep ring: 1.23x; conservative m = 6 likewise 1.06x
  // (profiles/ab_r02_kernel_knobs.txt: 2-k-step chunks and 3-k-step chunks elsewhere measured slower)
  return (sch == 1 && (m == 5 || m == 6)) ? 3 : 4;
}

// Ring depth override (0 = the shared-memory rule in CMCfg).
constexpr int cm_ns(int sch, int m) { return (sch == 1 && (m == 5 || m == 6)) ? 5 : 0; }

// Consumer warps per CTA: 12 (three per SM sub-partition, more warps to hide
// the LDS -> butterfly -> DMMA latency) where that measured faster — the low
// orders, whose k-steps carry the most non-tensor work per DMMA, and the
// conservative m = 5 map; 8 elsewhere, where the larger ring and accumulator
// budget of two warps per sub-partition win (tools/gpu_perf.sh, round 1).
constexpr int cm_nw(int sch, int m) {
#ifdef HW_CM_NW
  if (cm_knob(sch, m)) return HW_CM_NW;
#endif
  return (m <= 3 || (sch != 0 && m == 5) || (sch == 0 && (m == 6 || m == 7))) ? 12 : 8;
}

// W resident in shared memory for the whole kernel instead of staged per
// ring chunk: measured 2-6% faster for diss m = 3, 4 and cons m = 3..5,
// neutral at diss m = 5 (tools/cellmap_probe, round 1); at diss m = 2 5%
// slower with the four-class tiles, 1.3% faster with the merged ones (round 2).
constexpr bool cm_wres(int sch, int m) {
#ifdef HW_CM_WRES
  if (cm_knob(sch, m)) return HW_CM_WRES;
#endif
  return sch == 0 ? (m >= 2 && m <= 4) : (m >= 3 && m <= 5);
}

// Target columns per tile (tile = TR rows x TJ columns; the staged halo is
// (TR + 1)(TJ + 1) nodes).  32 by default; 16 (taller tiles, less halo)
// where that measured faster (profiles/ab_r01_kernel_knobs.txt).  TJ / 8
// must divide the consumer warp count (cellmap_launch.cuh asserts it).
constexpr int cm_tj(int sch, int m) {
#ifdef HW_CM_TJ
  if (cm_knob(sch, m)) return HW_CM_TJ;
#endif
  // (diss m = 3, round 2: 16 columns, whose smaller ring slots give a 4-deep ring, 6-9% faster)
  return (sch == 0 && (m == 3 || m == 4)) || (sch != 0 && (m == 4 || m == 8)) ? 16 : 32;
}

// Epilogue straight from the accumulators to HBM (no slab, no producer
// drain): 20% faster at diss m = 2, whose map is so small that the step is
// HBM-bound, 4-40% slower everywhere else (profiles/ab_r01_kernel_knobs.txt).
constexpr bool cm_direct(int sch, int m) {
#ifdef HW_CM_DIRECT
  if (cm_knob(sch, m)) return HW_CM_DIRECT;
#endif
  return sch == 0 && m <= 2;
}

// Each consumer warp drains its own output slab (no producer handoff):
// measured 7% faster at diss m = 3 and 3% at cons m = 3, slower from m = 4 up
// where the producers' otherwise idle issue slots are worth more.
constexpr bool cm_self(int sch, int m) {
#ifdef HW_CM_SELF
  if (cm_knob(sch, m)) return HW_CM_SELF;
#endif
  return sch != 2 && m == 3;
}

// Dynamic tile schedule (a global tile counter, cellmap_kernel) instead of
// static round robin.  The persistent CTAs of a static schedule finish up to
// 11% apart (tools/cta_times.cu, m = 4, 1024^2); claiming tiles evens that
// out: +4% at diss m = 4 (1024^2), +3% at m = 3, 5, +0.4-0.8% at m = 6..8,
// +5% cons m = 3, +0.5% cons m = 8.  Static stays where the claimed order
// measured slower per tile: diss m = 2 (HBM-bound, -7%) and cons m = 5 (-2%)
// (profiles/ab_r01_kernel_knobs.txt).
constexpr bool cm_dyn(int sch, int m) {
#ifdef HW_CM_DYN
  if (cm_knob(sch, m)) return HW_CM_DYN;
#endif
  return !(sch == 0 && m <= 2) && !(sch == 1 && m == 5);
}

}  // namespace hw
