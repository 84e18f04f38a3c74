// Host-side constant tables: exact two-point Hermite matrices and the
// per-launch scaled tap weights that the kernels read as constant-bank operands.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

namespace hw {

constexpr int kMaxOrder = 12;  // interp.py:30 MAX_ORDER

// Left block HL_mu[a][k] of interp.py:51-75 interp_matrix(mu), shape
// (2mu+2) x (mu+1).  The right block is (-1)^(a+k) * HL (exact symmetry of
// the centred two-point problem), so HL determines the whole matrix.
//
// Computed in exact integer arithmetic from the closed-form two-point Hermite
// basis B_k(t) = t^k (1-t)^(mu+1) sum_{i<=mu-k} C(mu+i,i) t^i on t in [0,1]
// (B_k^(l)(0)/l! = delta_kl, B_k^(l)(1) = 0), re-expanded about the cell
// centre t = xi + 1/2.  Every entry is a dyadic rational with a short
// numerator, so the double result is exact and equals the reference's
// Fraction-based inverse bit for bit (pinned in tests/test_tables.py).
std::vector<double> hermite_left_block(int mu);

// Full (2mu+2)^2 matrix in the reference's column order (left 0..mu, right).
std::vector<double> hermite_matrix(int mu);

double factorial(int n);
double binom(int n, int k);

}  // namespace hw
