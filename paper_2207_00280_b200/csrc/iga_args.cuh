// Argument blocks passed by value to the kernels (shared between the
// launchers and the C-ABI entry points).
#pragma once

#include <stdint.h>

namespace iga {

struct ElemArgs {
  int dim, K, q, op, method;
  double jac, coef_scalar;
  const double* knots;         // general knot vector [K + 2p + 1], or null (open uniform)
  const double* wt;            // [K][q] per-element weights of a general knot vector, or null
  const double* coef;
  const double* weights;
  const double* ref_nodes;
  const int32_t* elem_ids;
  const double* elem_nodes;
  const double* elem_weights;  // [count][dim][q] per-axis weights, or null (weights on every axis)
  const double* elem_coef;     // [count][q^dim] per-element coefficients, or null (coef / scalar)
  int64_t count;
  double* out;
  double* scratch;             // per-CTA sum-factorization stage buffers in global memory
                               // (high degrees), or null (shared memory)
};

struct ScatterArgs {
  int dim, K, op;
  const double* wt;               // [K][Q] per-element weights (general knots), or null
  int el_begin, el_end;           // slab along the slowest axis
  int64_t row_first, row_last;    // global rows [row_first, row_last) written
  int64_t base;                   // rowptr(row_first)
  double jac, coef_scalar;
  const double* coef;
  const double* weights;
  const double* V;  // [K][m][Q]
  const double* D;  // [K][m][Q] or null (mass)
  double* values;
  // element colour of this launch: the elements e with e_d = c_d (mod p+1) -- a colour's
  // elements share no dof, so each value receives at most one contribution per launch and
  // the colours, launched in a fixed order, fix the summation order (no atomics)
  int first0;                     // smallest e0 in [el_begin, el_end) of the colour
  int c1, c2;                     // colour along axes 1, 2 (2D: c1 only)
  int n0, n1, n2;                 // colour elements per axis (2D: n2 = 1)
  int split;                      // CTAs per element (classical DMMA kernel: tile ranges)
  double* scratch;                // element-local sum factorization, high degrees: per-CTA
                                  // stage buffers in global memory (else shared memory)
};

struct GsfArgs {
  int K, op;
  const double* wt;              // [K][Q] per-element weights (general knots), or null
  int el_begin, el_end;          // element slab along axis 0
  int plane_begin, plane_end;    // row planes I0 computed
  int segs;                      // segments of the element column e2 per tile (>= 1)
  int seg_len;                   // elements per segment
  int tiles1;                    // tiles along axis 1
  int64_t base;                  // rowptr of (plane_begin, 0, 0)
  double jac, coef_scalar;
  const double* coef;            // [K^3][Q^3] or null
  const double* weights;         // [Q]
  const double* V;               // [K][P+1][Q]
  const double* D;               // [K][P+1][Q] (null for mass)
  double* values;
};

struct KronArgs {
  int K, op;
  const double* wt;              // [K][Q] per-element weights (general knots), or null
  int el_begin, el_end;          // element slab along axis 0
  int plane_begin, plane_end;    // row planes I0 written
  int64_t base;                  // rowptr of (plane_begin, 0, 0)
  double jc;                     // jac * scalar coefficient
  const double* weights;         // [Q]
  const double* V;               // [K][P+1][Q]
  const double* D;               // [K][P+1][Q] (null for mass)
  const double2* band;           // [N][2P+1] (m, k) from iga_band_tables, or null
  double* values;
};

}  // namespace iga
