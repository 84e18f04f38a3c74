// Host construction of the per-class cell maps (see cellmap.h).
#include "cellmap.h"

#include <map>
#include <mutex>
#include <stdexcept>

#include "cellmap_shape.h"
#include "tables.h"

namespace hw {

using LD = long double;

void cellmap_widths(int scheme, int m, int w_in[2], int w_out[2]) {
  for (int f = 0; f < 2; ++f) {
    w_in[f] = cm_win(scheme, m, f);
    w_out[f] = cm_wout(scheme, m, f);
  }
}

static const std::vector<LD>& hermite_ld(int mu) {
  static std::mutex mu_lock;
  static std::map<int, std::vector<LD>> cache;
  std::lock_guard<std::mutex> lk(mu_lock);
  auto it = cache.find(mu);
  if (it != cache.end()) return it->second;
  const std::vector<double> h = hermite_matrix(mu);  // exact dyadic rationals
  return cache.emplace(mu, std::vector<LD>(h.begin(), h.end())).first->second;
}

// interp.py:93-111 apply_interp_2d for one cell: C = M_x St M_y^T with the
// stacked corner block St[sx*(mux+1)+k][sy*(muy+1)+l] = U[sx][sy][k][l].
template <class Get>
static std::vector<LD> interp2(Get get, int mux, int muy) {
  const int nx = 2 * mux + 2, ny = 2 * muy + 2;
  const std::vector<LD>& Mx = hermite_ld(mux);
  const std::vector<LD>& My = hermite_ld(muy);
  std::vector<LD> st((size_t)nx * ny, 0.0L), t((size_t)nx * ny, 0.0L), c((size_t)nx * ny, 0.0L);
  for (int sx = 0; sx < 2; ++sx)
    for (int sy = 0; sy < 2; ++sy)
      for (int k = 0; k <= mux; ++k)
        for (int l = 0; l <= muy; ++l) st[(size_t)(sx * (mux + 1) + k) * ny + sy * (muy + 1) + l] = get(sx, sy, k, l);
  for (int a = 0; a < nx; ++a)
    for (int j = 0; j < ny; ++j) {
      LD s = 0.0L;
      for (int i = 0; i < nx; ++i) s += Mx[(size_t)a * nx + i] * st[(size_t)i * ny + j];
      t[(size_t)a * ny + j] = s;
    }
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < ny; ++b) {
      LD s = 0.0L;
      for (int j = 0; j < ny; ++j) s += t[(size_t)a * ny + j] * My[(size_t)b * ny + j];
      c[(size_t)a * ny + b] = s;
    }
  return c;
}

static LD binom_ld(int n, int k) { return (LD)binom(n, k); }

// dissipative.py:184-212 expand_taylor_2d (+ eval_series at theta = 1/2,
// dissipative.py:116-121) on K x K tables.  d1 (may be empty) replaces
// stage 1 of the v table.  Returns the two theta-sums.
static void taylor_sum(int K, const std::vector<LD>& c0, const std::vector<LD>& d0pad, const std::vector<LD>* d1,
                       int n1, double dt, double rx, double ry, int smax, std::vector<LD>& su, std::vector<LD>& sv) {
  std::vector<LD> uc = c0, vc = d0pad, un(K * K), vn(K * K);
  su = uc;
  sv = vc;
  LD th = 1.0L;
  for (int s = 1; s <= smax; ++s) {
    th *= 0.5L;
    const LD fdt = (LD)dt / s, frx = (LD)rx / s, fry = (LD)ry / s;
    for (int i = 0; i < K * K; ++i) un[i] = fdt * vc[i];
    std::fill(vn.begin(), vn.end(), 0.0L);
    if (s == 1 && d1) {
      for (int a = 0; a < n1; ++a)
        for (int b = 0; b < n1; ++b) vn[a * K + b] = (*d1)[a * n1 + b];
    } else {
      for (int a = 0; a < K - 2; ++a)
        for (int b = 0; b < K; ++b) vn[a * K + b] = frx * (LD)((a + 2) * (a + 1)) * uc[(a + 2) * K + b];
      for (int a = 0; a < K; ++a)
        for (int b = 0; b < K - 2; ++b) vn[a * K + b] += fry * (LD)((b + 2) * (b + 1)) * uc[a * K + b + 2];
    }
    uc.swap(un);
    vc.swap(vn);
    for (int i = 0; i < K * K; ++i) {
      su[i] += th * uc[i];
      sv[i] += th * vc[i];
    }
  }
}

void eval_cell_reference(int scheme, int m, double dt, double hx, double hy, double speed, int stages,
                         const long double* in, long double* out) {
  int wi[2], wo[2];
  cellmap_widths(scheme, m, wi, wo);
  const int p0 = wi[0] * wi[0], din = p0 + wi[1] * wi[1];
  const int K = 2 * m + 2;
  auto field = [&](int f) {
    const int base = f ? p0 : 0, w = wi[f];
    return [=](int sx, int sy, int k, int l) { return in[(sx * 2 + sy) * din + base + k * w + l]; };
  };
  // rx, ry exactly as the reference forms them (dissipative.py:234-235,204-205)
  const double rx = speed * speed * dt / (hx * hx);
  const double ry = speed * speed * dt / (hy * hy);
  if (scheme == kDiss) {
    auto u = field(0);
    auto v = field(1);
    const std::vector<LD> cmm = interp2(u, m, m);
    const std::vector<LD> cx = interp2(u, m, m - 1);  // du[..., :, :m]
    const std::vector<LD> cy = interp2(u, m - 1, m);  // du[..., :m, :]
    const std::vector<LD> d0 = interp2(v, m - 1, m - 1);
    const int n1 = 2 * m;
    std::vector<LD> d1((size_t)n1 * n1), d0p((size_t)K * K, 0.0L);
    for (int a = 0; a < n1; ++a)
      for (int b = 0; b < n1; ++b) {
        d1[a * n1 + b] = (LD)rx * (LD)((a + 2) * (a + 1)) * cx[(a + 2) * n1 + b] +
                         (LD)ry * (LD)((b + 2) * (b + 1)) * cy[a * K + b + 2];
        d0p[a * K + b] = d0[a * n1 + b];
      }
    std::vector<LD> su, sv;
    taylor_sum(K, cmm, d0p, &d1, n1, dt, rx, ry, stages, su, sv);
    for (int k = 0; k <= m; ++k)
      for (int l = 0; l <= m; ++l) out[k * (m + 1) + l] = su[k * K + l];
    const int q0 = (m + 1) * (m + 1);
    for (int k = 0; k < m; ++k)
      for (int l = 0; l < m; ++l) out[q0 + k * m + l] = sv[k * K + l];
  } else if (scheme == kCons) {
    // conservative.py:87-112,130-136: new = 2 WT . I_{m,m}(cur)
    const std::vector<LD> c = interp2(field(0), m, m);
    const LD rhx = (LD)(0.5 * speed * dt / hx), rhy = (LD)(0.5 * speed * dt / hy);
    for (int k = 0; k <= m; ++k)
      for (int l = 0; l <= m; ++l) {
        LD s = 0.0L;
        for (int i = 0; k + 2 * i <= 2 * m + 1; ++i)
          for (int j = 0; l + 2 * j <= 2 * m + 1; ++j) {
            const int a = k + 2 * i, b = l + 2 * j;
            LD wt = binom_ld(a, k) * binom_ld(b, l) * binom_ld(i + j, i) / binom_ld(2 * i + 2 * j, 2 * i);
            for (int q = 0; q < 2 * i; ++q) wt *= rhx;
            for (int q = 0; q < 2 * j; ++q) wt *= rhy;
            s += wt * c[a * K + b];
          }
        out[k * (m + 1) + l] = 2.0L * s;
      }
  } else if (scheme == kBoot) {
    // conservative.py:185-195: plain recursion on I_m g0, I_m g1
    const std::vector<LD> c0 = interp2(field(0), m, m);
    const std::vector<LD> d0 = interp2(field(1), m, m);
    std::vector<LD> su, sv;
    taylor_sum(K, c0, d0, nullptr, 0, dt, rx, ry, stages, su, sv);
    for (int k = 0; k <= m; ++k)
      for (int l = 0; l <= m; ++l) out[k * (m + 1) + l] = su[k * K + l];
  } else {
    throw std::invalid_argument("unknown scheme");
  }
}

CellMap build_cell_map(int scheme, int m, double dt, double hx, double hy, double speed, int stages) {
  if (scheme < kDiss || scheme > kBoot) throw std::invalid_argument("unknown scheme");
  if (m < 1 || m > kMaxOrder) throw std::invalid_argument("method order out of range");
  CellMap cm;
  cm.scheme = scheme;
  cm.m = m;
  cellmap_widths(scheme, m, cm.w_in, cm.w_out);
  cm.din = cm.w_in[0] * cm.w_in[0] + cm.w_in[1] * cm.w_in[1];
  cm.dout = cm.w_out[0] * cm.w_out[0] + cm.w_out[1] * cm.w_out[1];
  // output enumeration: field 0 (k, l) row-major, then field 1; class = (k&1, l&1)
  std::vector<int> cls_of, pos_of;
  for (int f = 0; f < 2; ++f) {
    const int w = cm.w_out[f];
    for (int k = 0; k < w; ++k)
      for (int l = 0; l < w; ++l) {
        const int c = (k & 1) * 2 + (l & 1);
        cls_of.push_back(c);
        pos_of.push_back(cm.ncls[c]++);
        cm.code[c].push_back((f << 16) | (k * w + l));
      }
  }
  for (int c = 0; c < 4; ++c) cm.w[c].assign((size_t)cm.ncls[c] * cm.din, 0.0);
  std::vector<LD> in((size_t)4 * cm.din, 0.0L), out((size_t)cm.dout, 0.0L);
  for (int e = 0; e < cm.din; ++e) {
    in[e] = 1.0L;  // unit entry of corner (0, 0): G^c[e] = 1 for every class
    eval_cell_reference(scheme, m, dt, hx, hy, speed, stages, in.data(), out.data());
    in[e] = 0.0L;
    for (int o = 0; o < cm.dout; ++o) cm.w[cls_of[o]][(size_t)pos_of[o] * cm.din + e] = (double)out[o];
  }
  return cm;
}

std::vector<double> dense_cell_map(const CellMap& cm) {
  const int din = cm.din, p0 = cm.w_in[0] * cm.w_in[0];
  std::vector<double> d((size_t)cm.dout * 4 * din, 0.0);
  int o = 0;
  for (int f = 0; f < 2; ++f) {
    const int w = cm.w_out[f];
    for (int k = 0; k < w; ++k)
      for (int l = 0; l < w; ++l, ++o) {
        const int PA = k & 1, PB = l & 1, c = PA * 2 + PB;
        int pos = 0;
        while (cm.code[c][pos] != ((f << 16) | (k * w + l))) ++pos;
        for (int e = 0; e < din; ++e) {
          const int wi = e < p0 ? cm.w_in[0] : cm.w_in[1];
          const int ee = e < p0 ? e : e - p0;
          const int kx = ee / wi, ky = ee % wi;
          const double wv = cm.w[c][(size_t)pos * din + e];
          for (int sx = 0; sx < 2; ++sx)
            for (int sy = 0; sy < 2; ++sy) {
              const bool neg = ((sx * (PA + kx)) + (sy * (PB + ky))) & 1;
              d[(size_t)(k * w + l + (f ? cm.w_out[0] * cm.w_out[0] : 0)) * 4 * din + (sx * 2 + sy) * din + e] =
                  neg ? -wv : wv;
            }
        }
      }
  }
  return d;
}

}  // namespace hw
