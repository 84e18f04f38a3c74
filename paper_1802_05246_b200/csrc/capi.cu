// extern "C" boundary (include/hermb200.h): argument checking, constant-table
// construction and kernel dispatch.  Never throws across the ABI.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "cellmap.cuh"
#include "cellmap.h"
#include "common.cuh"
#include "diag.cuh"
#include "line1d.cuh"
#include "lowlevel.cuh"
#include "simt2d.cuh"
#include "tables.h"

// Which 2D steps run the SIMT cell map (simt2d.cuh: CUDA-core FP64, class
// maps as constant operands) instead of the tensor-core cell map
// (cellmap.cuh): the conservative scheme at m <= 2, where it measured 2.1x
// faster (profiles/ab_r02_kernel_knobs.txt).  A/B knob HW_SIMT_M: every
// scheme at m <= HW_SIMT_M (0..5).
static constexpr bool use_simt(int sch, int m) {
#ifdef HW_SIMT_M
  static_assert(HW_SIMT_M <= 5, "the SIMT kernel's class maps fit the parameter space up to m = 5");
  return m <= HW_SIMT_M;
#else
  return sch == hw::kCons && m <= 2;
#endif
}

namespace hw {

template <int M, int SCH>
cudaError_t launch_cellmap(const CellMapArgs& a, cudaStream_t st);  // kern_m*.cu
template <int M, int SCH>
cudaError_t launch_simt2d(const Simt2DArgs& a, const double* wd, const int* code, cudaStream_t st);  // kern_m1..5.cu

static thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& s) : std::runtime_error(s), code(c) {}
};

#define HW_CHECK(cond, msg) \
  do {                      \
    if (!(cond)) throw Error(HW_EINVAL, msg); \
  } while (0)

static void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(HW_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
static int guard(F&& f) {
  try {
    f();
    return HW_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HW_EINVAL;
  }
}

static Rows to_rows(const hw_rows2d* r) {
  Rows o;
  o.base = r->base;
  o.lo = r->halo_lo;
  o.hi = r->halo_hi;
  o.row0 = r->row0;
  o.nrows = r->nrows;
  return o;
}

static void check_bc_axis(const hw_axis_bc& b, int periodic) {
  auto ok = [](int k) { return k == HW_PERIODIC || k == HW_DIRICHLET0 || k == HW_NEUMANN0; };
  HW_CHECK(ok(b.left_kind) && ok(b.right_kind), "unknown boundary kind");
  HW_CHECK((b.left_kind == HW_PERIODIC) == (b.right_kind == HW_PERIODIC),
           "periodic must be specified on both opposing sides");
  HW_CHECK((b.left_kind == HW_PERIODIC) == (periodic != 0),
           "boundary spec and grid disagree about periodicity");
}

// ------------------------------------------------------------------ cell maps
// Device copies of the class maps in DMMA fragment order, cached per
// (device, scheme, m, dt, hx, hy, speed, stages).
struct DevMap {
  double* wfrag = nullptr;
  double* wleft = nullptr;
  int* ocode = nullptr;
  int* icode = nullptr;
  double* wdense = nullptr;  // [dout][din] class-major (simt2d.cuh)
  int* dcode = nullptr;      // [dout]
  std::shared_ptr<const std::vector<double>> hwd;  // host copies (the SIMT kernel's parameter block)
  std::shared_ptr<const std::vector<int>> hdc;
};

struct MapKey {
  int dev, scheme, m, stages;
  double dt, hx, hy, speed;
  bool operator==(const MapKey& o) const {
    return dev == o.dev && scheme == o.scheme && m == o.m && stages == o.stages &&
           std::memcmp(&dt, &o.dt, 8) == 0 && std::memcmp(&hx, &o.hx, 8) == 0 &&
           std::memcmp(&hy, &o.hy, 8) == 0 && std::memcmp(&speed, &o.speed, 8) == 0;
  }
};

static std::mutex g_map_mu;
static std::list<std::pair<MapKey, DevMap>> g_maps;  // most recent first
constexpr size_t kMaxMaps = 48;

static void free_map(DevMap& d) {
  cudaFree(d.wfrag);
  cudaFree(d.wleft);
  cudaFree(d.ocode);
  cudaFree(d.icode);
  cudaFree(d.wdense);
  cudaFree(d.dcode);
}

static DevMap device_map(int scheme, int m, double dt, double hx, double hy, double speed, int stages) {
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  cuda_check(cudaGetDevice(&key.dev), "cudaGetDevice");
  key.scheme = scheme;
  key.m = m;
  key.stages = stages;
  key.dt = dt;
  key.hx = hx;
  key.hy = hy;
  key.speed = speed;
  std::lock_guard<std::mutex> lk(g_map_mu);
  for (auto it = g_maps.begin(); it != g_maps.end(); ++it)
    if (it->first == key) {
      g_maps.splice(g_maps.begin(), g_maps, it);
      return g_maps.front().second;
    }
  const CellMap cm = build_cell_map(scheme, m, dt, hx, hy, speed, stages);
  // fragment tiles: DMMA tiles (ntd) then SIMT tiles, whose columns are the
  // left-over outputs of the hybrid classes (cellmap_shape.h)
  const int nk = cm_nk(scheme, m), nt = cm_nt(scheme, m), ntd = cm_ntd(scheme, m), lc = cm_lc(scheme, m);
  const int ntb = cm_ntb(scheme, m);  // B fragments per k-step
  std::vector<double> wf((size_t)nk * ntb * 32, 0.0), wl((size_t)nk * lc * 4, 0.0);
  std::vector<int> oc((size_t)nt * 8, -1), ic((size_t)nk * 4, 0);
  // input slot -> map input e (field 0 entries, then field 1); -1 = pad slot
  const int p0 = cm.w_in[0] * cm.w_in[0], p1 = cm.w_in[1] * cm.w_in[1], k0 = cm_k0(scheme, m);
  std::vector<int> slot_e((size_t)nk * 4, -1);
  for (int sl = 0; sl < nk * 4; ++sl) {
    const bool f1 = sl >= k0;
    const int ee = f1 ? sl - k0 : sl;
    if (ee >= (f1 ? p1 : p0)) continue;
    const int w = cm.w_in[f1 ? 1 : 0];
    slot_e[sl] = f1 ? p0 + ee : ee;
    ic[sl] = ((ee / w) & 1) | (((ee % w) & 1) << 1);
  }
  for (int c = 0; c < 4; ++c)
    if (cm.ncls[c] != cm_ncls(scheme, m, c)) throw Error(HW_EINVAL, "internal: class size mismatch");
  if (cm_pxm(scheme, m)) {
    // merged x-classes (cellmap_shape.h): tile group PB holds the outputs of
    // classes (0, PB) then (1, PB); fragment 2 j + dx of k-step ks multiplies
    // corner row dx's y-pair sums, the lower row's x-sign (-1)^(PA + kx) folded in
    for (int pb = 0; pb < 2; ++pb) {
      const int base = pb ? cm_pxm_tiles(scheme, m, 0) : 0, ntile = cm_pxm_tiles(scheme, m, pb);
      std::vector<std::pair<int, int>> cols;  // (class, output)
      for (int pa = 0; pa < 2; ++pa)
        for (int o = 0; o < cm.ncls[2 * pa + pb]; ++o) cols.emplace_back(2 * pa + pb, o);
      for (size_t j = 0; j < cols.size(); ++j) oc[(size_t)(base + j / 8) * 8 + j % 8] = cm.code[cols[j].first][cols[j].second];
      for (int ks = 0; ks < nk; ++ks)
        for (int jt = 0; jt < ntile; ++jt)
          for (int dx = 0; dx < 2; ++dx)
            for (int lane = 0; lane < 32; ++lane) {
              const int col = 8 * jt + lane / 4, sl = 4 * ks + lane % 4, e = slot_e[sl];
              if (col >= (int)cols.size() || e < 0) continue;
              const int c = cols[col].first, o = cols[col].second, pa = c >> 1, kx = ic[sl] & 1;
              const double sg = (dx && ((pa + kx) & 1)) ? -1.0 : 1.0;
              wf[((size_t)ks * ntb + 2 * (base + jt) + dx) * 32 + lane] = sg * cm.w[c][(size_t)o * cm.din + e];
            }
    }
  }
  for (int c = 0; c < 4 && !cm_pxm(scheme, m); ++c) {
    const int base = cm_ntbase(scheme, m, c), ntc = cm_ntc(scheme, m, c);
    const int ndm = std::min(cm.ncls[c], 8 * ntc);  // outputs in DMMA tiles; the rest are SIMT columns
    for (int o = 0; o < ndm; ++o) oc[(size_t)(base + o / 8) * 8 + o % 8] = cm.code[c][o];
    for (int ks = 0; ks < nk; ++ks)
      for (int j = 0; j < ntc; ++j)
        for (int lane = 0; lane < 32; ++lane) {
          const int o = 8 * j + lane / 4, e = slot_e[4 * ks + lane % 4];
          if (o < ndm && e >= 0) wf[((size_t)ks * ntb + base + j) * 32 + lane] = cm.w[c][(size_t)o * cm.din + e];
        }
    for (int q = 0; q < cm_left(scheme, m, c); ++q) {
      const int jcol = cm_lbase(scheme, m, c) + q, o = ndm + q;
      oc[(size_t)(ntd + jcol / 8) * 8 + jcol % 8] = cm.code[c][o];
      for (int ks = 0; ks < nk; ++ks)
        for (int kk = 0; kk < 4; ++kk) {
          const int e = slot_e[4 * ks + kk];
          if (e >= 0) wl[((size_t)ks * lc + jcol) * 4 + kk] = cm.w[c][(size_t)o * cm.din + e];
        }
    }
  }
  // class-major dense maps for the SIMT kernel
  std::vector<double> wd((size_t)cm.dout * cm.din);
  std::vector<int> dc((size_t)cm.dout);
  for (int c = 0, row = 0; c < 4; ++c)
    for (int o = 0; o < cm.ncls[c]; ++o, ++row) {
      dc[row] = cm.code[c][o];
      for (int e = 0; e < cm.din; ++e) wd[(size_t)row * cm.din + e] = cm.w[c][(size_t)o * cm.din + e];
    }
  DevMap d;
  d.hwd = std::make_shared<const std::vector<double>>(wd);
  d.hdc = std::make_shared<const std::vector<int>>(dc);
  try {
    cuda_check(cudaMalloc(&d.wdense, wd.size() * sizeof(double)), "cudaMalloc(wdense)");
    cuda_check(cudaMalloc(&d.dcode, dc.size() * sizeof(int)), "cudaMalloc(dcode)");
    cuda_check(cudaMemcpy(d.wdense, wd.data(), wd.size() * sizeof(double), cudaMemcpyHostToDevice), "upload wd");
    cuda_check(cudaMemcpy(d.dcode, dc.data(), dc.size() * sizeof(int), cudaMemcpyHostToDevice), "upload dcode");
    cuda_check(cudaMalloc(&d.wfrag, wf.size() * sizeof(double)), "cudaMalloc(wfrag)");
    cuda_check(cudaMalloc(&d.wleft, std::max<size_t>(wl.size(), 1) * sizeof(double)), "cudaMalloc(wleft)");
    if (!wl.empty())
      cuda_check(cudaMemcpy(d.wleft, wl.data(), wl.size() * sizeof(double), cudaMemcpyHostToDevice), "upload wl");
    cuda_check(cudaMalloc(&d.ocode, oc.size() * sizeof(int)), "cudaMalloc(ocode)");
    cuda_check(cudaMalloc(&d.icode, ic.size() * sizeof(int)), "cudaMalloc(icode)");
    cuda_check(cudaMemcpy(d.wfrag, wf.data(), wf.size() * sizeof(double), cudaMemcpyHostToDevice), "upload wfrag");
    cuda_check(cudaMemcpy(d.ocode, oc.data(), oc.size() * sizeof(int), cudaMemcpyHostToDevice), "upload ocode");
    cuda_check(cudaMemcpy(d.icode, ic.data(), ic.size() * sizeof(int), cudaMemcpyHostToDevice), "upload icode");
    // a pageable H2D cudaMemcpy may return before its DMA lands, and the kernel
    // runs on the caller's (possibly non-blocking) stream: wait once per new map
    cuda_check(cudaDeviceSynchronize(), "upload map");
  } catch (...) {
    free_map(d);
    throw;
  }
  if (g_maps.size() >= kMaxMaps) {
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    free_map(g_maps.back().second);
    g_maps.pop_back();
  }
  g_maps.emplace_front(key, d);
  return d;
}

template <int SCH>
static void dispatch_cellmap(int m, const CellMapArgs& a, const DevMap& dm, cudaStream_t st) {
  cudaError_t e;
  if (use_simt(SCH, m) || m > kMaxFast) {
    Simt2DArgs s;
    std::memset(&s, 0, sizeof(s));
    s.f0 = a.f0;
    s.f1 = a.f1;
    s.wd = dm.wdense;
    s.code = dm.dcode;
    s.prev = a.prev;
    s.out0 = a.out0;
    s.out1 = a.out1;
    s.nx = a.nx;
    s.ny = a.ny;
    s.trow0 = a.trow0;
    s.ntrows = a.ntrows;
    s.nty = a.nty;
    s.off = a.off;
    s.periodic = a.periodic;
    s.kxl = a.kxl;
    s.kxh = a.kxh;
    s.kyl = a.kyl;
    s.kyh = a.kyh;
    s.gxl = a.gxl;
    s.gxh = a.gxh;
    s.gyl = a.gyl;
    s.gyh = a.gyh;
    if (m > kMaxFast) {  // m = 9..12: the generic runtime-order path
      Gen2DArgs g;
      std::memset(&g, 0, sizeof(g));
      g.s = s;
      g.w0 = cm_win(SCH, m, 0);
      g.w1 = cm_win(SCH, m, 1);
      g.ow0 = cm_wout(SCH, m, 0);
      g.ow1 = cm_wout(SCH, m, 1);
      g.din = cm_din(SCH, m);
      g.dout = cm_dout(SCH, m);
      for (int c = 0; c < 4; ++c) g.ncls[c] = cm_ncls(SCH, m, c);
      e = launch_simt2d_generic(g, SCH, st);
    } else {
      const double* hw = dm.hwd->data();
      const int* hc = dm.hdc->data();
      switch (m) {
        case 1: e = launch_simt2d<1, SCH>(s, hw, hc, st); break;
        case 2: e = launch_simt2d<2, SCH>(s, hw, hc, st); break;
        case 3: e = launch_simt2d<3, SCH>(s, hw, hc, st); break;
        case 4: e = launch_simt2d<4, SCH>(s, hw, hc, st); break;
        default: e = launch_simt2d<5, SCH>(s, hw, hc, st); break;
      }
    }
    cuda_check(e, "simt2d launch");
    return;
  }
  switch (m) {
    case 1: e = launch_cellmap<1, SCH>(a, st); break;
    case 2: e = launch_cellmap<2, SCH>(a, st); break;
    case 3: e = launch_cellmap<3, SCH>(a, st); break;
    case 4: e = launch_cellmap<4, SCH>(a, st); break;
    case 5: e = launch_cellmap<5, SCH>(a, st); break;
    case 6: e = launch_cellmap<6, SCH>(a, st); break;
    case 7: e = launch_cellmap<7, SCH>(a, st); break;
    case 8: e = launch_cellmap<8, SCH>(a, st); break;
    default: throw Error(HW_EUNSUPPORTED, "method order m=" + std::to_string(m) + " has no 2D path (1..12)");
  }
  cuda_check(e, "cellmap launch");
}

struct Geo {
  int64_t nx, ny, ntx, nty, trow0, ntrows;
  int off, periodic;
};

static Geo check_geom(const hw_geom2d* g) {
  HW_CHECK(g, "null geometry");
  HW_CHECK(g->nx >= 1 && g->ny >= 1, "need at least one source node per axis");
  HW_CHECK(g->parity_src == HW_PRIMAL || g->parity_src == HW_DUAL, "unknown parity");
  check_bc_axis(g->bcx, g->periodic);
  check_bc_axis(g->bcy, g->periodic);
  Geo o;
  o.nx = g->nx;
  o.ny = g->ny;
  o.periodic = g->periodic != 0;
  o.off = src_offset(g->parity_src);
  o.ntx = target_count(g->nx, g->parity_src, o.periodic);
  o.nty = target_count(g->ny, g->parity_src, o.periodic);
  HW_CHECK(o.ntx >= 1 && o.nty >= 1, "grid too small for a half step");
  o.trow0 = g->trow0;
  o.ntrows = g->ntrows < 0 ? o.ntx - g->trow0 : g->ntrows;
  HW_CHECK(o.trow0 >= 0 && o.trow0 + o.ntrows <= o.ntx, "target row range out of bounds");
  return o;
}

static CellMapArgs cellmap_args(const Geo& g, const hw_geom2d* geom, const hw_rows2d* f0, const hw_rows2d* f1,
                                const DevMap& dm, int m) {
  // the kernel stages with 32-bit offsets within a source row
  HW_CHECK(g.ny * (int64_t)(m + 1) * (m + 1) < ((int64_t)1 << 31), "grid row too long for the 2D kernels");
  CellMapArgs a;
  std::memset(&a, 0, sizeof(a));
  a.f0 = to_rows(f0);
  a.f1 = f1 ? to_rows(f1) : a.f0;
  a.wfrag = dm.wfrag;
  a.wleft = dm.wleft;
  a.ocode = dm.ocode;
  a.icode = dm.icode;
  a.nx = g.nx;
  a.ny = g.ny;
  a.trow0 = g.trow0;
  a.ntrows = g.ntrows;
  a.nty = g.nty;
  a.off = g.off;
  a.periodic = g.periodic;
  a.kxl = g.periodic ? 0 : geom->bcx.left_kind;
  a.kxh = g.periodic ? 0 : geom->bcx.right_kind;
  a.kyl = g.periodic ? 0 : geom->bcy.left_kind;
  a.kyh = g.periodic ? 0 : geom->bcy.right_kind;
  a.gxl = geom->bcx.left_value;
  a.gxh = geom->bcx.right_value;
  a.gyl = geom->bcy.left_value;
  a.gyh = geom->bcy.right_value;
  return a;
}

static void check_rows(const hw_rows2d* r, const Geo& g, const hw_rows2d* first = nullptr) {
  HW_CHECK(r->nrows >= 0 && r->row0 >= 0 && r->row0 + r->nrows <= g.nx, "source row window out of bounds");
  HW_CHECK(!first || (first->row0 == r->row0 && first->nrows == r->nrows),
           "both source fields must cover the same row window");
}

}  // namespace hw

using namespace hw;

extern "C" {

const char* hw_last_error(void) { return g_err.c_str(); }
int hw_version(void) { return 4; }
int hw_max_order(void) { return kMaxFast; }

int hw_interp_matrix(int mu, double* out) {
  return guard([&] {
    HW_CHECK(out, "null output");
    HW_CHECK(mu >= 0 && mu <= kMaxOrder, "interpolation order must be in [0, 12]");
    const std::vector<double> m = hermite_matrix(mu);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

int64_t hw_target_count(int64_t n_src, int parity_src, int periodic) {
  return target_count(n_src, parity_src, periodic);
}

int hw_cell_map_dims(int scheme, int m, int* din, int* dout) {
  return guard([&] {
    HW_CHECK(din && dout, "null output");
    HW_CHECK(scheme >= kDiss && scheme <= kBoot, "unknown scheme");
    HW_CHECK(m >= 1 && m <= kMaxOrder, "method order out of range");
    *din = cm_din(scheme, m);
    *dout = cm_dout(scheme, m);
  });
}

int hw_cell_map_2d(int scheme, int m, double dt, double hx, double hy, double speed, int stages, double* out) {
  return guard([&] {
    HW_CHECK(out, "null output");
    HW_CHECK(scheme >= kDiss && scheme <= kBoot, "unknown scheme");
    HW_CHECK(m >= 1 && m <= kMaxOrder, "method order out of range");
    HW_CHECK(stages >= 1 || scheme == kCons, "stage count must be >= 1");
    const CellMap cm = build_cell_map(scheme, m, dt, hx, hy, speed, stages);
    const std::vector<double> d = dense_cell_map(cm);
    std::memcpy(out, d.data(), d.size() * sizeof(double));
  });
}

int hw_diss2d_half_step(const hw_rows2d* u_src, const hw_rows2d* v_src, double* u_dst, double* v_dst, int m,
                        const hw_geom2d* geom, double dt, double hx, double hy, double speed, int stage_cap,
                        void* stream) {
  return guard([&] {
    HW_CHECK(u_src && v_src && u_src->base && v_src->base && u_dst && v_dst, "null field pointer");
    HW_CHECK(m >= 1, "method order must be >= 1");
    const Geo g = check_geom(geom);
    check_rows(u_src, g);
    check_rows(v_src, g, u_src);
    if (g.ntrows == 0) return;
    const int S = stage_cap > 0 ? stage_cap : 4 * m + 4;  // dissipative.py:73-74
    HW_CHECK(m <= kMaxOrder, "method order m=" + std::to_string(m) + " out of range (interp.py:62-63: 1..12)");
    const DevMap dm = device_map(kDiss, m, dt, hx, hy, speed, S);
    CellMapArgs a = cellmap_args(g, geom, u_src, v_src, dm, m);
    a.out0 = u_dst;
    a.out1 = v_dst;
    dispatch_cellmap<kDiss>(m, a, dm, (cudaStream_t)stream);
  });
}

int hw_cons2d_step(const hw_rows2d* cur_src, const double* prev, double* out, int m, const hw_geom2d* geom,
                   double dt, double hx, double hy, double speed, void* stream) {
  return guard([&] {
    HW_CHECK(cur_src && cur_src->base && prev && out, "null field pointer");
    HW_CHECK(m >= 1, "method order must be >= 1");
    const Geo g = check_geom(geom);
    check_rows(cur_src, g);
    if (g.ntrows == 0) return;
    HW_CHECK(m <= kMaxOrder, "method order m=" + std::to_string(m) + " out of range (interp.py:62-63: 1..12)");
    const DevMap dm = device_map(kCons, m, dt, hx, hy, speed, 0);
    CellMapArgs a = cellmap_args(g, geom, cur_src, nullptr, dm, m);
    a.prev = prev;
    a.out0 = out;
    dispatch_cellmap<kCons>(m, a, dm, (cudaStream_t)stream);
  });
}

int hw_boot2d(const hw_rows2d* g0_src, const hw_rows2d* g1_src, double* out, int m, const hw_geom2d* geom,
              double dt, double hx, double hy, double speed, void* stream) {
  return guard([&] {
    HW_CHECK(g0_src && g1_src && g0_src->base && g1_src->base && out, "null field pointer");
    HW_CHECK(m >= 1, "method order must be >= 1");
    const Geo g = check_geom(geom);
    check_rows(g0_src, g);
    check_rows(g1_src, g, g0_src);
    if (g.ntrows == 0) return;
    HW_CHECK(m <= kMaxOrder, "method order m=" + std::to_string(m) + " out of range (interp.py:62-63: 1..12)");
    const DevMap dm = device_map(kBoot, m, dt, hx, hy, speed, 4 * m + 4);  // conservative.py:192
    CellMapArgs a = cellmap_args(g, geom, g0_src, g1_src, dm, m);
    a.out0 = out;
    dispatch_cellmap<kBoot>(m, a, dm, (cudaStream_t)stream);
  });
}

// ------------------------------------------------------------------ 1D
static std::unordered_map<int, double*>& hl_cache() {
  static std::unordered_map<int, double*> c;
  return c;
}
static std::mutex g_hl_mu;

static const double* device_hl(int mu) {
  std::lock_guard<std::mutex> lk(g_hl_mu);
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const int key = dev * 64 + mu;
  auto it = hl_cache().find(key);
  if (it != hl_cache().end()) return it->second;
  const std::vector<double> h = hermite_left_block(mu);
  double* d = nullptr;
  cuda_check(cudaMalloc(&d, h.size() * sizeof(double)), "cudaMalloc(hl)");
  cuda_check(cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(hl)");
  cuda_check(cudaDeviceSynchronize(), "upload hl");  // see device_map
  hl_cache()[key] = d;
  return d;
}

static Line1DArgs line_args(int m, int64_t n_src, int parity_src, const hw_axis_bc* bc) {
  HW_CHECK(bc, "null boundary spec");
  HW_CHECK(m >= 1 && m <= kMax1D, "1D method order must be in [1, 12]");
  const int periodic = bc->left_kind == HW_PERIODIC;
  check_bc_axis(*bc, periodic);
  HW_CHECK(parity_src == HW_PRIMAL || parity_src == HW_DUAL, "unknown parity");
  Line1DArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = n_src;
  a.nt = target_count(n_src, parity_src, periodic);
  HW_CHECK(n_src >= 1 && a.nt >= 1, "grid too small for a half step");
  a.off = src_offset(parity_src);
  a.periodic = periodic;
  a.kl = periodic ? 0 : bc->left_kind;
  a.kh = periodic ? 0 : bc->right_kind;
  a.gl = bc->left_value;
  a.gh = bc->right_value;
  a.m = m;
  return a;
}

int hw_diss1d_half_step(const double* u_src, const double* v_src, double* u_dst, double* v_dst, int m,
                        int64_t n_src, int parity_src, const hw_axis_bc* bc, double dt, double h, double speed,
                        int stages, const double* forcing, void* stream) {
  return guard([&] {
    HW_CHECK(u_src && v_src && u_dst && v_dst, "null field pointer");
    Line1DArgs a = line_args(m, n_src, parity_src, bc);
    HW_CHECK(stages >= 1 && stages <= 4 * kMax1D, "stage count out of range");
    a.u = u_src;
    a.v = v_src;
    a.ou = u_dst;
    a.ov = v_dst;
    a.forcing = forcing;
    a.stages = stages;
    a.dt = dt;
    a.h = h;
    a.speed = speed;
    a.hl_u = device_hl(m);
    a.hl_v = device_hl(m - 1);
    const int thr = 128;
    diss1d_kernel<<<(unsigned)((a.nt + thr - 1) / thr), thr, 0, (cudaStream_t)stream>>>(a);
    cuda_check(cudaGetLastError(), "diss1d launch");
  });
}

int hw_cons1d_step(const double* cur, const double* prev, double* out, int m, int64_t n_src, int parity_src,
                   const hw_axis_bc* bc, double lam, void* stream) {
  return guard([&] {
    HW_CHECK(cur && prev && out, "null field pointer");
    Line1DArgs a = line_args(m, n_src, parity_src, bc);
    a.u = cur;
    a.prev = prev;
    a.ou = out;
    a.rho = 0.5 * lam;  // conservative.py:125
    a.hl_u = device_hl(m);
    const int thr = 128;
    cons1d_kernel<<<(unsigned)((a.nt + thr - 1) / thr), thr, 0, (cudaStream_t)stream>>>(a);
    cuda_check(cudaGetLastError(), "cons1d launch");
  });
}

int hw_boot1d(const double* g0, const double* g1, double* out, int m, int64_t n_src, int parity_src,
              const hw_axis_bc* bc, double dt, double h, double speed, void* stream) {
  return guard([&] {
    HW_CHECK(g0 && g1 && out, "null field pointer");
    Line1DArgs a = line_args(m, n_src, parity_src, bc);
    a.u = g0;
    a.v = g1;
    a.ou = out;
    a.stages = 2 * m + 3;  // conservative.py:183-184
    a.dt = dt;
    a.h = h;
    a.speed = speed;
    a.hl_u = device_hl(m);
    const int thr = 128;
    boot1d_kernel<<<(unsigned)((a.nt + thr - 1) / thr), thr, 0, (cudaStream_t)stream>>>(a);
    cuda_check(cudaGetLastError(), "boot1d launch");
  });
}

// ------------------------------------------------------------------ diagnostics
struct DevBuf {
  double* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

static double reduce_partials(double* part, int64_t n, cudaStream_t st) {
  DevBuf out;
  cuda_check(cudaMallocAsync(&out.p, sizeof(double), st), "cudaMallocAsync");
  sum_partials_kernel<<<1, kRedThreads, 0, st>>>(part, n, out.p);
  cuda_check(cudaGetLastError(), "sum_partials launch");
  double h = 0.0;
  cuda_check(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  cudaFreeAsync(out.p, st);
  out.p = nullptr;
  return h;
}

// Ex[p][c] = sum_a d^d/dxi^d (xi_p)^a M[a][c] / h^d at xi_p = xg_p / 2
// (diagnostics.py:128-130 at d = 0): the tensor interpolant's d-th derivative
// at the Gauss points, as a map of the cell's stacked corner data.
static std::vector<double> deriv_eval_matrix(int mu, int d, double h, const std::vector<double>& gx) {
  const std::vector<double> M = hermite_matrix(mu);
  const int n = 2 * mu + 2, npts = (int)gx.size();
  std::vector<double> e((size_t)npts * n, 0.0);
  for (int p = 0; p < npts; ++p) {
    const double xi = 0.5 * gx[p];
    for (int c = 0; c < n; ++c) {
      double s = 0.0, pw = 1.0;
      for (int a2 = d; a2 < n; ++a2) {
        double fall = 1.0;  // a2! / (a2 - d)!
        for (int k = 0; k < d; ++k) fall *= (double)(a2 - k);
        s += fall * pw * M[(size_t)a2 * n + c];
        pw *= xi;
      }
      e[(size_t)p * n + c] = d ? s * std::pow(h, -(double)d) : s;
    }
  }
  return e;
}

// Shared by hw_l2err2d and hw_seminorm2d: the tensor interpolant of every
// target cell evaluated at the npts^2 Gauss points, d-th derivative along each
// axis (d = 0: the values), reduced to sum_cells sum_pq w_p w_q (val - exact)^2.
static double cell_quadrature_2d(const hw_rows2d* src, int mx, int my, const hw_geom2d* geom, double x_left,
                                 double y_left, double hx, double hy, int dx, int dy, int npts,
                                 const double* gauss_x, const double* gauss_w, int exact_kind, const double* exact,
                                 const double* params, cudaStream_t st) {
  const Geo g = check_geom(geom);
  // Ex[p][e] = sum_a d^dx/dx^dx (xg_p/2)^a M[a][e]   (diagnostics.py:128-130 at dx = 0);
  // the interpolant is a polynomial in xi = (x - xc) / h, so each derivative brings 1/h
  std::vector<double> gx(npts), gw(npts);
  cuda_check(cudaMemcpy(gx.data(), gauss_x, npts * sizeof(double), cudaMemcpyDefault), "copy gauss x");
  cuda_check(cudaMemcpy(gw.data(), gauss_w, npts * sizeof(double), cudaMemcpyDefault), "copy gauss w");
  const std::vector<double> ex = deriv_eval_matrix(mx, dx, hx, gx), ey = deriv_eval_matrix(my, dy, hy, gx);
  const int64_t ncell = g.ntrows * g.nty;
  if (ncell == 0) return 0.0;
  const int64_t nblk = (ncell + kRedThreads - 1) / kRedThreads;
  DevBuf dex, dey, dgx, dgw, dpart;
  cuda_check(cudaMalloc(&dex.p, ex.size() * 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dey.p, ey.size() * 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dgx.p, npts * 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dgw.p, npts * 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dpart.p, nblk * 8), "cudaMalloc");
  cuda_check(cudaMemcpyAsync(dex.p, ex.data(), ex.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  cuda_check(cudaMemcpyAsync(dey.p, ey.data(), ey.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  cuda_check(cudaMemcpyAsync(dgx.p, gx.data(), npts * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  cuda_check(cudaMemcpyAsync(dgw.p, gw.data(), npts * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  L2Err2DArgs a;
  std::memset(&a, 0, sizeof(a));
  a.f = to_rows(src);
  a.nx = g.nx;
  a.ny = g.ny;
  a.ntx = g.ntx;
  a.nty = g.nty;
  a.trow0 = g.trow0;
  a.ntrows = g.ntrows;
  a.off = g.off;
  a.periodic = g.periodic;
  a.kxl = g.periodic ? 0 : geom->bcx.left_kind;
  a.kxh = g.periodic ? 0 : geom->bcx.right_kind;
  a.kyl = g.periodic ? 0 : geom->bcy.left_kind;
  a.kyh = g.periodic ? 0 : geom->bcy.right_kind;
  a.gxl = geom->bcx.left_value;
  a.gxh = geom->bcx.right_value;
  a.gyl = geom->bcy.left_value;
  a.gyh = geom->bcy.right_value;
  a.mx = mx;
  a.my = my;
  a.npts = npts;
  a.ex = dex.p;
  a.ey = dey.p;
  a.gw = dgw.p;
  a.gx = dgx.p;
  a.exact_kind = exact_kind;
  a.exact = exact;
  for (int q = 0; q < 4; ++q) a.prm[q] = params ? params[q] : 0.0;
  a.x0 = x_left;
  a.y0 = y_left;
  a.hx = hx;
  a.hy = hy;
  a.coff = geom->parity_src == HW_PRIMAL ? 0.5 : 0.0;  // targets live on the flipped parity
  a.part = dpart.p;
  l2err2d_kernel<<<(unsigned)nblk, kRedThreads, 0, st>>>(a);
  cuda_check(cudaGetLastError(), "l2err2d launch");
  return reduce_partials(dpart.p, nblk, st);
}

int hw_l2err2d(const hw_rows2d* src, int mx, int my, const hw_geom2d* geom, double x_left, double y_left,
               double hx, double hy, int npts, const double* gauss_x, const double* gauss_w, int exact_kind,
               const double* exact, const double* params, double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(src && src->base && gauss_x && gauss_w && out_host, "null pointer");
    HW_CHECK(mx >= 0 && my >= 0 && mx <= kMaxOrder && my <= kMaxOrder, "orders out of range");
    HW_CHECK(npts >= 1 && npts <= 64, "npts out of range");
    HW_CHECK(exact_kind >= 0 && exact_kind <= 2, "unknown exact kind");
    HW_CHECK(exact_kind != 0 || exact, "null exact array");
    const double s = cell_quadrature_2d(src, mx, my, geom, x_left, y_left, hx, hy, 0, 0, npts, gauss_x, gauss_w,
                                        exact_kind, exact, params, (cudaStream_t)stream);
    *out_host = s * (0.25 * hx * hy);
  });
}

int hw_seminorm2d(const hw_rows2d* src, int mx, int my, const hw_geom2d* geom, double hx, double hy, int dx, int dy,
                  int npts, const double* gauss_x, const double* gauss_w, double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(src && src->base && gauss_x && gauss_w && out_host, "null pointer");
    HW_CHECK(mx >= 0 && my >= 0 && mx <= kMaxOrder && my <= kMaxOrder, "orders out of range");
    HW_CHECK(dx >= 0 && dy >= 0 && dx <= 2 * mx + 1 && dy <= 2 * my + 1, "derivative orders out of range");
    HW_CHECK(npts >= 1 && npts <= 64, "npts out of range");
    const double s = cell_quadrature_2d(src, mx, my, geom, 0.0, 0.0, hx, hy, dx, dy, npts, gauss_x, gauss_w, 3,
                                        nullptr, nullptr, (cudaStream_t)stream);
    *out_host = s * (0.25 * hx * hy);
  });
}

int hw_inner2d(const hw_rows2d* f, const hw_rows2d* g, int mx, int my, const hw_geom2d* geom, double hx, double hy,
               int dx, int dy, int npts, const double* gauss_x, const double* gauss_w, int wall_half,
               double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(f && f->base && gauss_x && gauss_w && out_host, "null pointer");
    HW_CHECK(!g || g->base, "null field pointer");
    HW_CHECK(mx >= 0 && my >= 0 && mx <= kMaxOrder && my <= kMaxOrder, "orders out of range");
    HW_CHECK(dx >= 0 && dy >= 0 && dx <= 2 * mx + 1 && dy <= 2 * my + 1, "derivative orders out of range");
    HW_CHECK(npts >= 1 && npts <= 64, "npts out of range");
    const Geo gg = check_geom(geom);
    check_rows(f, gg);
    if (g) check_rows(g, gg, f);
    cudaStream_t st = (cudaStream_t)stream;
    *out_host = 0.0;
    const int64_t ncell = gg.ntrows * gg.nty;
    if (ncell == 0) return;
    std::vector<double> gx(gauss_x, gauss_x + npts), gw(gauss_w, gauss_w + npts);
    const std::vector<double> ex = deriv_eval_matrix(mx, dx, hx, gx), ey = deriv_eval_matrix(my, dy, hy, gx);
    const int64_t nblk = (ncell + kRedThreads - 1) / kRedThreads;
    DevBuf dex, dey, dgw, dpart, dout;
    cuda_check(cudaMalloc(&dex.p, ex.size() * 8), "cudaMalloc");
    cuda_check(cudaMalloc(&dey.p, ey.size() * 8), "cudaMalloc");
    cuda_check(cudaMalloc(&dgw.p, npts * 8), "cudaMalloc");
    cuda_check(cudaMalloc(&dpart.p, nblk * 16), "cudaMalloc");
    cuda_check(cudaMalloc(&dout.p, 8), "cudaMalloc");
    cuda_check(cudaMemcpyAsync(dex.p, ex.data(), ex.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(dey.p, ey.data(), ey.size() * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(dgw.p, gw.data(), npts * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
    Inner2DArgs a;
    std::memset(&a, 0, sizeof(a));
    a.f = to_rows(f);
    a.g = g ? to_rows(g) : a.f;
    a.same = g == nullptr || (g->base == f->base && g->halo_lo == f->halo_lo && g->halo_hi == f->halo_hi);
    a.nx = gg.nx;
    a.ny = gg.ny;
    a.nty = gg.nty;
    a.trow0 = gg.trow0;
    a.ntrows = gg.ntrows;
    a.off = gg.off;
    a.periodic = gg.periodic;
    a.kxl = gg.periodic ? 0 : geom->bcx.left_kind;
    a.kxh = gg.periodic ? 0 : geom->bcx.right_kind;
    a.kyl = gg.periodic ? 0 : geom->bcy.left_kind;
    a.kyh = gg.periodic ? 0 : geom->bcy.right_kind;
    a.gxl = geom->bcx.left_value;
    a.gxh = geom->bcx.right_value;
    a.gyl = geom->bcy.left_value;
    a.gyh = geom->bcy.right_value;
    a.mx = mx;
    a.my = my;
    a.npts = npts;
    a.wall_half = wall_half != 0;
    a.ex = dex.p;
    a.ey = dey.p;
    a.gw = dgw.p;
    a.part = dpart.p;
    inner2d_kernel<<<(unsigned)nblk, kRedThreads, 0, st>>>(a);
    cuda_check(cudaGetLastError(), "inner2d launch");
    sum_partials_dd_kernel<<<1, kRedThreads, 0, st>>>(dpart.p, nblk, dout.p);
    cuda_check(cudaGetLastError(), "sum_partials_dd launch");
    double h = 0.0;
    cuda_check(cudaMemcpyAsync(&h, dout.p, sizeof(double), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    *out_host = h * (0.25 * hx * hy);  // Gauss rule on [-1, 1]^2 -> the hx x hy cell
  });
}

int hw_l2err1d(const double* src, int mu, int64_t n_src, int parity_src, const hw_axis_bc* bc, double h, int deriv,
               int npts, const double* xi, const double* w, const double* ex, double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(src && xi && w && ex && out_host, "null pointer");
    HW_CHECK(mu >= 0 && mu <= kMaxOrder, "order out of range");
    HW_CHECK(bc, "null boundary spec");
    const int periodic = bc->left_kind == HW_PERIODIC;
    check_bc_axis(*bc, periodic);
    cudaStream_t st = (cudaStream_t)stream;
    L2Err1DArgs a;
    std::memset(&a, 0, sizeof(a));
    a.f = src;
    a.n = n_src;
    a.nt = target_count(n_src, parity_src, periodic);
    a.off = src_offset(parity_src);
    a.periodic = periodic;
    a.kl = periodic ? 0 : bc->left_kind;
    a.kh = periodic ? 0 : bc->right_kind;
    a.gl = bc->left_value;
    a.gh = bc->right_value;
    a.mu = mu;
    a.deriv = deriv;
    a.npts = npts;
    a.h = h;
    a.hl = device_hl(mu);
    a.xi = xi;
    a.w = w;
    a.ex = ex;
    const int64_t nblk = (a.nt + kRedThreads - 1) / kRedThreads;
    DevBuf part;
    cuda_check(cudaMalloc(&part.p, nblk * 8), "cudaMalloc");
    a.part = part.p;
    l2err1d_kernel<<<(unsigned)nblk, kRedThreads, 0, st>>>(a);
    cuda_check(cudaGetLastError(), "l2err1d launch");
    *out_host = reduce_partials(part.p, nblk, st);
  });
}

static Energy1DArgs energy_args(int mu, int64_t n_src, int parity, const hw_axis_bc* bc, double h, int npts,
                                const double* gx, const double* gw) {
  HW_CHECK(bc, "null boundary spec");
  HW_CHECK(mu >= 0 && mu <= kMax1D, "order out of range");
  HW_CHECK(npts >= 1 && npts <= 64 && gx && gw, "bad Gauss rule");
  const int periodic = bc->left_kind == HW_PERIODIC;
  check_bc_axis(*bc, periodic);
  HW_CHECK(parity == HW_PRIMAL || parity == HW_DUAL, "unknown parity");
  Energy1DArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = n_src;
  a.nt = target_count(n_src, parity, periodic);
  HW_CHECK(n_src >= 1 && a.nt >= 1, "grid too small");
  a.off = src_offset(parity);
  a.periodic = periodic;
  a.kl = periodic ? 0 : bc->left_kind;
  a.kh = periodic ? 0 : bc->right_kind;
  a.gl = bc->left_value;
  a.gh = bc->right_value;
  a.mu = mu;
  a.h = h;
  a.npts = npts;
  a.hl = device_hl(mu);
  return a;
}

// Gauss rule (host arrays) -> device copies owned by the caller's DevBufs.
static void upload_rule(Energy1DArgs& a, const double* gx, const double* gw, DevBuf& dx, DevBuf& dw,
                        cudaStream_t st) {
  cuda_check(cudaMalloc(&dx.p, a.npts * 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dw.p, a.npts * 8), "cudaMalloc");
  // stream-ordered before the kernel that reads them (pageable sources are staged before return)
  cuda_check(cudaMemcpyAsync(dx.p, gx, a.npts * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  cuda_check(cudaMemcpyAsync(dw.p, gw, a.npts * 8, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync");
  a.gx = dx.p;
  a.gw = dw.p;
}

int hw_seminorm1d(const double* f, int mu, int64_t n_src, int parity, const hw_axis_bc* bc, double h, int order,
                  double scale, int npts, const double* gx, const double* gw, double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(f && out_host, "null pointer");
    HW_CHECK(order >= 0, "derivative order must be nonnegative");
    Energy1DArgs a = energy_args(mu, n_src, parity, bc, h, npts, gx, gw);
    a.f = f;
    a.order = order;
    a.scale = scale;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf dx, dw;
    upload_rule(a, gx, gw, dx, dw, st);
    const int64_t nblk = (a.nt + kRedThreads - 1) / kRedThreads;
    DevBuf part;
    cuda_check(cudaMalloc(&part.p, nblk * 8), "cudaMalloc");
    a.part = part.p;
    seminorm1d_kernel<<<(unsigned)nblk, kRedThreads, 0, st>>>(a);
    cuda_check(cudaGetLastError(), "seminorm1d launch");
    *out_host = reduce_partials(part.p, nblk, st);
  });
}

int hw_cons_energy1d(const double* cur, const double* prev, int m, int64_t n_src, int parity_cur, double h,
                     double delta, int npts, const double* gx, const double* gw, double* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(cur && prev && out_host, "null pointer");
    hw_axis_bc per = {HW_PERIODIC, HW_PERIODIC, 0.0, 0.0};
    Energy1DArgs a = energy_args(m, n_src, parity_cur, &per, h, npts, gx, gw);
    HW_CHECK(delta >= 0.0 && delta < h, "shift distance must be smaller than the smallest cell");
    a.f = cur;
    a.g = prev;
    a.offg = src_offset(parity_cur == HW_PRIMAL ? HW_DUAL : HW_PRIMAL);
    a.order = m + 1;
    a.delta = delta;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf dx, dw;
    upload_rule(a, gx, gw, dx, dw, st);
    const int64_t nblk = (a.nt + kRedThreads - 1) / kRedThreads;
    DevBuf part;
    cuda_check(cudaMalloc(&part.p, nblk * 8), "cudaMalloc");
    a.part = part.p;
    cons_energy1d_kernel<<<(unsigned)nblk, kRedThreads, 0, st>>>(a);
    cuda_check(cudaGetLastError(), "cons_energy1d launch");
    *out_host = reduce_partials(part.p, nblk, st);
  });
}

// ------------------------------------------------------------------ lower-level API (lowlevel.cuh)
// A host table uploaded for one call (stream-ordered; freed after the launch).
struct CallTable {
  double* p = nullptr;
  cudaStream_t st;
  CallTable(const std::vector<double>& h, cudaStream_t s) : st(s) {
    cuda_check(cudaMallocAsync((void**)&p, h.size() * sizeof(double), st), "cudaMallocAsync");
    cuda_check(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, st),
               "cudaMemcpyAsync");
  }
  ~CallTable() {
    if (p) cudaFreeAsync(p, st);
  }
};

static unsigned ll_blocks(int64_t n) { return (unsigned)((n + 127) / 128); }

int hw_apply_interp(const double* data, double* out, int64_t batch, int mu, void* stream) {
  return guard([&] {
    HW_CHECK(mu >= 0 && mu <= kMaxOrder, "interpolation order out of range");
    HW_CHECK(batch >= 0 && (batch == 0 || (data && out)), "null pointer");
    if (batch == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    const CallTable M(hermite_matrix(mu), st);
    const int n = 2 * mu + 2;
    apply_interp_kernel<<<ll_blocks(batch * n), 128, 0, st>>>(data, out, batch, n, M.p);
    cuda_check(cudaGetLastError(), "apply_interp launch");
  });
}

int hw_apply_interp_2d(const double* data, double* out, int64_t batch, int mux, int muy, void* stream) {
  return guard([&] {
    HW_CHECK(mux >= 0 && muy >= 0 && mux <= kMaxOrder && muy <= kMaxOrder, "interpolation order out of range");
    HW_CHECK(batch >= 0 && (batch == 0 || (data && out)), "null pointer");
    if (batch == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    const CallTable Mx(hermite_matrix(mux), st), My(hermite_matrix(muy), st);
    apply_interp2d_kernel<<<ll_blocks(batch * (2 * mux + 2)), 128, 0, st>>>(data, out, batch, mux, muy, Mx.p, My.p);
    cuda_check(cudaGetLastError(), "apply_interp_2d launch");
  });
}

int hw_expand_taylor(const double* cu, const double* cv, double* cu_tab, double* cv_tab, int64_t batch, int lu,
                     int lv, double dt, double r, int smax, const double* fterm, void* stream) {
  return guard([&] {
    HW_CHECK(lu >= 1 && lv >= 0 && lv <= lu && smax >= 0, "table sizes out of range");
    HW_CHECK(batch >= 0 && (batch == 0 || (cu && cu_tab && (lv == 0 || (cv && cv_tab)))), "null pointer");
    if (batch == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    expand_taylor_kernel<<<ll_blocks(batch), 128, 0, st>>>(cu, cv, cu_tab, cv_tab, batch, lu, lv, dt, r, smax, fterm);
    cuda_check(cudaGetLastError(), "expand_taylor launch");
  });
}

int hw_expand_taylor_2d(const double* c0, const double* d0, const double* d1, double* c_tab, double* d_tab,
                        int64_t batch, int K, int lv, double dt, double rx, double ry, int smax, void* stream) {
  return guard([&] {
    HW_CHECK(K >= 2 && lv >= 0 && lv <= K && smax >= 0, "table sizes out of range");
    HW_CHECK(batch >= 0 && (batch == 0 || (c0 && d0 && c_tab && d_tab)), "null pointer");
    if (batch == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    expand_taylor2d_kernel<<<ll_blocks(batch), 128, 0, st>>>(c0, d0, d1, c_tab, d_tab, batch, K, lv, dt, rx, ry, smax);
    cuda_check(cudaGetLastError(), "expand_taylor_2d launch");
  });
}

int hw_eval_series(const double* table, double* out, int64_t batch, int nstages, double theta, void* stream) {
  return guard([&] {
    HW_CHECK(nstages >= 1, "empty series");
    HW_CHECK(batch >= 0 && (batch == 0 || (table && out)), "null pointer");
    if (batch == 0) return;
    cudaStream_t st = (cudaStream_t)stream;
    eval_series_kernel<<<ll_blocks(batch), 128, 0, st>>>(table, out, batch, nstages, theta);
    cuda_check(cudaGetLastError(), "eval_series launch");
  });
}

// conservative.py:77-84 _update_matrix_1d: W[k][j] = C(j, k) rho^(j-k), j = k, k+2, ...
int hw_cons_update_1d(const double* coeffs, const double* prev, double* out, int64_t batch, int m, double rho,
                      void* stream) {
  return guard([&] {
    HW_CHECK(m >= 1 && m < kMaxOrder, "method order out of range");
    HW_CHECK(batch >= 0 && (batch == 0 || (coeffs && prev && out)), "null pointer");
    if (batch == 0) return;
    const int nj = 2 * m + 2;
    std::vector<double> w((size_t)(m + 1) * nj, 0.0);
    for (int k = 0; k <= m; ++k)
      for (int j = k; j < nj; j += 2) w[(size_t)k * nj + j] = binom(j, k) * std::pow(rho, (double)(j - k));
    cudaStream_t st = (cudaStream_t)stream;
    const CallTable W(w, st);
    cons_update_kernel<<<ll_blocks(batch * (m + 1)), 128, 0, st>>>(coeffs, prev, out, batch, m + 1, nj, W.p);
    cuda_check(cudaGetLastError(), "conservative_update_1d launch");
  });
}

// conservative.py:87-112 _update_tensor_2d: WT[k][l][a][b] at a = k + 2i, b = l + 2j is
// float(C(a,k) C(b,l) C(i+j,i) / C(2i+2j,2i)) rho_x^(2i) rho_y^(2j)
int hw_cons_update_2d(const double* coeffs, const double* prev, double* out, int64_t batch, int m, double rho_x,
                      double rho_y, void* stream) {
  return guard([&] {
    // (the exact-integer numerator below stays under 2^53 up to m = 9)
    HW_CHECK(m >= 1 && m <= 9, "2D conservative update order must be in [1, 9]");
    HW_CHECK(batch >= 0 && (batch == 0 || (coeffs && prev && out)), "null pointer");
    if (batch == 0) return;
    const int kk = 2 * m + 2, nq = (m + 1) * (m + 1), nj = kk * kk;
    std::vector<double> w((size_t)nq * nj, 0.0);
    for (int k = 0; k <= m; ++k)
      for (int l = 0; l <= m; ++l)
        for (int i = 0; k + 2 * i <= 2 * m + 1; ++i)
          for (int j = 0; l + 2 * j <= 2 * m + 1; ++j) {
            const int a = k + 2 * i, b = l + 2 * j;
            // the numerator (< 2^53) and denominator are exact doubles: one correctly rounded division
            const double num = binom(a, k) * binom(b, l) * binom(i + j, i);
            const double frac = num / binom(2 * i + 2 * j, 2 * i);
            w[(size_t)(k * (m + 1) + l) * nj + a * kk + b] =
                frac * std::pow(rho_x, (double)(2 * i)) * std::pow(rho_y, (double)(2 * j));
          }
    cudaStream_t st = (cudaStream_t)stream;
    const CallTable W(w, st);
    cons_update_kernel<<<ll_blocks(batch * nq), 128, 0, st>>>(coeffs, prev, out, batch, nq, nj, W.p);
    cuda_check(cudaGetLastError(), "conservative_update_2d launch");
  });
}

int hw_gather(const double* src, double* out, int dims, int64_t nx, int64_t ny, int w0, int w1, int parity_src,
              const hw_axis_bc* bcx, const hw_axis_bc* bcy, void* stream) {
  return guard([&] {
    HW_CHECK(dims == 1 || dims == 2, "dims must be 1 or 2");
    HW_CHECK(bcx && (dims == 1 || bcy), "null boundary spec");
    HW_CHECK(w0 >= 1 && w1 >= 1 && (dims == 2 || w1 == 1), "block widths out of range");
    HW_CHECK(parity_src == HW_PRIMAL || parity_src == HW_DUAL, "unknown parity");
    const int periodic = bcx->left_kind == HW_PERIODIC;
    check_bc_axis(*bcx, periodic);
    if (dims == 2) check_bc_axis(*bcy, periodic);
    HW_CHECK(nx >= 1 && (dims == 1 ? ny == 1 : ny >= 1), "node counts out of range");
    GatherArgs a;
    std::memset(&a, 0, sizeof(a));
    a.src = src;
    a.out = out;
    a.nx = nx;
    a.ny = ny;
    a.ntx = target_count(nx, parity_src, periodic);
    a.nty = dims == 2 ? target_count(ny, parity_src, periodic) : 1;
    a.w0 = w0;
    a.w1 = w1;
    a.off = src_offset(parity_src);
    a.periodic = periodic;
    a.dims = dims;
    if (!periodic) {
      a.kxl = bcx->left_kind;
      a.kxh = bcx->right_kind;
      a.gxl = bcx->left_value;
      a.gxh = bcx->right_value;
      if (dims == 2) {
        a.kyl = bcy->left_kind;
        a.kyh = bcy->right_kind;
        a.gyl = bcy->left_value;
        a.gyh = bcy->right_value;
      }
    }
    const int64_t n = a.ntx * a.nty * (dims == 2 ? 4 : 2) * w0 * w1;
    if (n == 0) return;
    HW_CHECK(src && out, "null pointer");
    gather_kernel<<<ll_blocks(n), 128, 0, (cudaStream_t)stream>>>(a);
    cuda_check(cudaGetLastError(), "gather launch");
  });
}

int hw_ghost(const double* in, double* out, int64_t batch, int n0, int n1, int axis, int kind, double value,
             void* stream) {
  return guard([&] {
    HW_CHECK(kind == HW_DIRICHLET0 || kind == HW_NEUMANN0, "ghosts reflect across dirichlet0 or neumann0 walls");
    HW_CHECK(axis == 0 || axis == 1, "axis must be 0 or 1");
    HW_CHECK(n0 >= 1 && n1 >= 1 && batch >= 0, "sizes out of range");
    const int64_t n = batch * n0 * n1;
    if (n == 0) return;
    HW_CHECK(in && out, "null pointer");
    ghost_kernel<<<ll_blocks(n), 128, 0, (cudaStream_t)stream>>>(in, out, batch, n0, n1, axis, kind, value);
    cuda_check(cudaGetLastError(), "ghost launch");
  });
}

int hw_scale_cols(const double* in, double* out, int64_t rows, int cols, double h, void* stream) {
  return guard([&] {
    HW_CHECK(rows >= 0 && cols >= 1, "sizes out of range");
    if (rows == 0) return;
    HW_CHECK(in && out, "null pointer");
    scale_cols_kernel<<<ll_blocks(rows * cols), 128, 0, (cudaStream_t)stream>>>(in, out, rows, cols, h);
    cuda_check(cudaGetLastError(), "scale_cols launch");
  });
}

int hw_count_nonfinite(const double* x, int64_t n, int64_t* out_host, void* stream) {
  return guard([&] {
    HW_CHECK(out_host, "null output");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
      *out_host = 0;
      return;
    }
    HW_CHECK(x, "null pointer");
    unsigned long long* d = nullptr;
    cuda_check(cudaMallocAsync((void**)&d, 8, st), "cudaMallocAsync");
    cuda_check(cudaMemsetAsync(d, 0, 8, st), "cudaMemsetAsync");
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    nonfinite_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, n, d);
    cuda_check(cudaGetLastError(), "nonfinite launch");
    unsigned long long h = 0;
    cuda_check(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    cudaFreeAsync(d, st);
    *out_host = (int64_t)h;
  });
}

static void launch_init(const Init2DArgs& a, cudaStream_t st) {
  const int64_t n = a.nx * a.ny;
  if (n == 0) return;
  init2d_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(a);
  cuda_check(cudaGetLastError(), "init2d launch");
}

int hw_init_planewave2d(double* out, int64_t nx, int64_t ny, int64_t row0, int kx, int ky, double x0, double y0,
                        double off,
                        double t, double kappa, double hx, double hy, int tder, void* stream) {
  return guard([&] {
    HW_CHECK(out, "null output");
    Init2DArgs a;
    std::memset(&a, 0, sizeof(a));
    a.out = out;
    HW_CHECK(row0 >= 0, "row offset must be nonnegative");
    a.nx = nx;
    a.ny = ny;
    a.row0 = row0;
    a.kx = kx;
    a.ky = ky;
    a.x0 = x0;
    a.y0 = y0;
    a.off = off;
    a.t = t;
    a.hx = hx;
    a.hy = hy;
    a.kind = 1;
    a.w = 2.0 * 3.141592653589793 * kappa;
    a.tder = tder;
    launch_init(a, (cudaStream_t)stream);
  });
}

int hw_init_standing2d(double* out, int64_t nx, int64_t ny, int64_t row0, int kx, int ky, double x0, double y0,
                       double off,
                       double t, double ax, double ay, double px, double py, double om, double hx, double hy,
                       int tder, void* stream) {
  return guard([&] {
    HW_CHECK(out, "null output");
    Init2DArgs a;
    std::memset(&a, 0, sizeof(a));
    a.out = out;
    HW_CHECK(row0 >= 0, "row offset must be nonnegative");
    a.nx = nx;
    a.ny = ny;
    a.row0 = row0;
    a.kx = kx;
    a.ky = ky;
    a.x0 = x0;
    a.y0 = y0;
    a.off = off;
    a.t = t;
    a.hx = hx;
    a.hy = hy;
    a.kind = 2;
    a.ax = ax;
    a.ay = ay;
    a.px = px;
    a.py = py;
    a.om = om;
    a.tder = tder;
    launch_init(a, (cudaStream_t)stream);
  });
}

int hw_init_1d(double* out, const double* x, int64_t n, int kmax, int kind, double x0, double h, double off,
               int scaled, double t, double a, int tder, void* stream) {
  return guard([&] {
    HW_CHECK(out, "null output");
    HW_CHECK(n >= 0, "node count must be nonnegative");
    HW_CHECK(kmax >= 0 && kmax <= kMax1D, "derivative count out of range (0..12)");
    HW_CHECK(kind >= 0 && kind <= 2, "unknown 1D data kind");
    HW_CHECK(tder == 0 || (tder == 1 && kind == 1), "only the gaussian box has a time derivative");
    if (n == 0) return;
    Init1DArgs g;
    std::memset(&g, 0, sizeof(g));
    g.out = out;
    g.xs = x;
    g.n = n;
    g.kmax = kmax;
    g.kind = kind;
    g.tder = tder;
    g.scaled = scaled != 0;
    g.x0 = x0;
    g.h = h;
    g.off = off;
    g.t = t;
    g.a = a;
    init1d_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(g);
    cuda_check(cudaGetLastError(), "init1d launch");
  });
}

}  // extern "C"
