#include "tables.h"

#include <stdexcept>

namespace hw {

using i128 = __int128;

static i128 ibinom(int n, int k) {
  if (k < 0 || k > n) return 0;
  i128 r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

double factorial(int n) {
  double r = 1.0;
  for (int i = 2; i <= n; ++i) r *= i;
  return r;
}

double binom(int n, int k) { return (double)ibinom(n, k); }

std::vector<double> hermite_left_block(int mu) {
  if (mu < 0 || mu > kMaxOrder) throw std::invalid_argument("interpolation order out of range");
  const int n = 2 * mu + 2;
  const int deg = 2 * mu + 1;
  std::vector<double> hl((size_t)n * (mu + 1), 0.0);
  for (int k = 0; k <= mu; ++k) {
    // integer coefficients of B_k(t) in powers of t
    std::vector<i128> b(deg + 1, 0);
    for (int r = 0; r <= mu + 1; ++r) {          // (1-t)^(mu+1)
      const i128 cr = ((r & 1) ? -1 : 1) * ibinom(mu + 1, r);
      for (int i = 0; i <= mu - k; ++i) {        // sum C(mu+i,i) t^i
        const int p = k + r + i;
        b[p] += cr * ibinom(mu + i, i);
      }
    }
    // B_k(xi + 1/2): coefficient of xi^j = sum_r b_r C(r,j) 2^(j-r)
    //              = 2^-deg * sum_r b_r C(r,j) 2^(deg-r+j)
    for (int j = 0; j <= deg; ++j) {
      i128 acc = 0;
      for (int r = j; r <= deg; ++r) {
        if (b[r] == 0) continue;
        acc += b[r] * ibinom(r, j) * ((i128)1 << (deg - r + j));
      }
      // acc = num * 2^e with a short num: the conversion is exact
      const bool neg = acc < 0;
      i128 mag = neg ? -acc : acc;
      int e = 0;
      while (mag != 0 && (mag & 1) == 0) {
        mag >>= 1;
        ++e;
      }
      if (mag >= ((i128)1 << 53)) throw std::runtime_error("hermite entry not exactly representable");
      double v = std::ldexp((double)(int64_t)mag, e - deg);
      hl[(size_t)j * (mu + 1) + k] = neg ? -v : v;
    }
  }
  return hl;
}

std::vector<double> hermite_matrix(int mu) {
  const int n = 2 * mu + 2, w = mu + 1;
  std::vector<double> hl = hermite_left_block(mu);
  std::vector<double> m((size_t)n * n, 0.0);
  for (int a = 0; a < n; ++a)
    for (int k = 0; k < w; ++k) {
      const double v = hl[(size_t)a * w + k];
      m[(size_t)a * n + k] = v;
      m[(size_t)a * n + w + k] = ((a + k) & 1) ? -v : v;
    }
  return m;
}

}  // namespace hw
