// Per-cell linear maps of the 2D half step (host side).
//
// Every 2D step the path performs is, per target cell, a LINEAR map of the
// four flanking source nodes (plus the affine Dirichlet ghost datum, which the
// kernel folds into its staged loads):
//   kDiss  half_step_2d          (dissipative.py:215-247)  u,v -> u,v
//   kCons  full_step_conservative (conservative.py:139-157) cur -> 2 WT I(cur)
//                                 (the kernel subtracts `previous`)
//   kBoot  bootstrap_first_half   (conservative.py:185-195) g0,g1 -> u
//
// Parity split.  The right block of every Hermite matrix is (-1)^(a+k) times
// the left block (interp.py:51-75, exact), so output coefficient (k, l) of
// parity class c = (k&1, l&1) depends on the corners only through the signed
// sum  G^c[e] = U00 + (-1)^(PA+kx) U10 + (-1)^(PB+ky) U01 + (-1)^(..) U11
// of input entry e = (kx, ky).  Hence  out_c = W_c G^c  with a dense
// n_c x D_in matrix W_c per class and sum_c n_c = D_out.
//
// W_c is obtained by evaluating the reference algorithm for ONE cell in
// extended precision (long double) on unit inputs of corner (0,0) — the
// same interpolation, stage recursion (with the stage cap) and Horner sum at
// theta = 1/2, so W is the reference's own operator rounded once to double.
#pragma once

#include <cstdint>
#include <vector>

#include "cellmap_shape.h"

namespace hw {

struct CellMap {
  int scheme = 0, m = 0;
  int w_in[2] = {0, 0};    // input field widths (orders + 1); 0 = absent
  int w_out[2] = {0, 0};   // output field widths
  int din = 0, dout = 0;   // inputs per corner node, outputs per target node
  int ncls[4] = {0, 0, 0, 0};
  std::vector<int> code[4];     // per class: field << 16 | offset in the node record
  std::vector<double> w[4];     // per class: w[c][o * din + e]
};

// Field widths of a scheme at order m.
void cellmap_widths(int scheme, int m, int w_in[2], int w_out[2]);

// Build the class maps.  dt, hx, hy, speed are exactly the doubles the
// reference uses; stages = Taylor stage count (kDiss: stage cap or 4m+4;
// kBoot: 4m+4; ignored for kCons).
CellMap build_cell_map(int scheme, int m, double dt, double hx, double hy, double speed, int stages);

// Dense single-cell map (dout x 4*din; column = corner*din + e with
// corner = sx*2 + sy) assembled from the class maps and the parity signs.
std::vector<double> dense_cell_map(const CellMap& cm);

// Reference evaluation of one cell in long double (for tests): corners
// in[corner][din] -> out[dout].
void eval_cell_reference(int scheme, int m, double dt, double hx, double hy, double speed, int stages,
                         const long double* in, long double* out);

}  // namespace hw
