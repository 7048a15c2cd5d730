/*
 * oracle/iga_oracle.c -- CPU restatement of the reference `igabench` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_2207_00280_b200/) never links or calls
 * it and fails loudly if its CUDA library is missing.
 *
 * It restates, function by function, the reference files under
 * /root/reference/pkg/src/igabench (cited as file:line):
 *   - knots / Cox-de Boor / nonzero values and derivatives  splines.py:59-178
 *   - per-1D-element node mapping and tables                 runtime.py:142-149
 *   - classical quadrature loop                               integrators.py:77-109
 *   - three-stage sum factorization                           integrators.py:112-151
 *   - lexicographic dof map and scatter-assembly to CSR       assembly.py:19-25, 46-83
 *   - symbolic CSR pattern (sorted columns, both triangles)   assembly.py:99-115
 * and extends them the way SURVEY.md §8(c) prescribes for what the reference
 * lacks: stiffness = the reference kernels called once per axis with the
 * derivative table substituted on that axis, summed in axis order (then the
 * mass term for stiffness+mass); a per-quadrature-point coefficient appended
 * as the last factor of the classical product and of the stage-1 product;
 * 2D = the same loops with the third axis dropped.
 *
 * Must be compiled with -ffp-contract=off (no FMA contraction) so the loops
 * are strict IEEE left-to-right like the numba kernels (bitwise pinned against
 * the reference by tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OP_MASS 0
#define ORC_OP_STIFFNESS 1
#define ORC_OP_STIFFNESS_MASS 2

/* Absolute mode: tables and coefficient replaced by their absolute values, so
 * every quadrature term becomes |term| and an assembled entry becomes
 * A[I,J] = sum |terms|, the scale of any fp64 summation's rounding error
 * (used by tests/parity.py for entries that cancel).  Off by default. */
static int g_absolute = 0;
void orc_set_absolute(int on) { g_absolute = on; }

static void abs_inplace(double* a, size_t n) {
  if (!g_absolute) return;
  for (size_t i = 0; i < n; ++i) a[i] = fabs(a[i]);
}

/* General open knot vector mode (off by default): the tables are
 * evaluated from these knots at x = lo + (ref+1)*(h/2) in each span [t_{p+e}, t_{p+e+1}],
 * and element e's Jacobian is folded into per-axis weights wt[e][k] = w_k * (h_e / 2)
 * with jac = 1 -- the definition tools/gen_golden.py (section 12) feeds the reference's own
 * kernels with. */
static double* g_knots = NULL;
static int g_nknots = 0;
static double* g_wt = NULL;
void orc_set_knots(const double* t, int nt, const double* wt, int K, int q) {
  free(g_knots);
  free(g_wt);
  g_knots = NULL;
  g_wt = NULL;
  g_nknots = 0;
  if (t == NULL) return;
  g_knots = (double*)malloc(sizeof(double) * nt);
  memcpy(g_knots, t, sizeof(double) * nt);
  g_nknots = nt;
  g_wt = (double*)malloc(sizeof(double) * K * q);
  memcpy(g_wt, wt, sizeof(double) * K * q);
}

/* per-axis weights of element alpha[d] (general knots) or the reference weights */
static inline const double* axis_w(const double* w, const int* alpha, int d, int q) {
  return g_wt ? g_wt + (size_t)alpha[d] * q : w;
}

/* ---------------------------------------------------------------- splines */

/* splines.py:59-75 make_knot_vector: p+1 zeros, arange(1,K)/K, p+1 ones. */
void orc_knots(int K, int p, double* t) {
  int n = 0;
  for (int i = 0; i <= p; ++i) t[n++] = 0.0;
  for (int i = 1; i < K; ++i) t[n++] = (double)i / (double)K;
  for (int i = 0; i <= p; ++i) t[n++] = 1.0;
}

/* splines.py:78-91 eval_basis_order0 (closed last non-empty span). */
static double orc_order0(const double* t, int nt, int i, double x) {
  if (t[i] <= x && x < t[i + 1]) return 1.0;
  if (x == t[nt - 1] && t[i] < t[i + 1] && t[i + 1] == t[nt - 1]) return 1.0;
  return 0.0;
}

/* splines.py:108-118 _cox: zero-denominator terms contribute nothing. */
double orc_cox(const double* t, int nt, int i, int q, double x) {
  if (q == 0) return orc_order0(t, nt, i, x);
  double out = 0.0;
  double d_left = t[i + q] - t[i];
  if (d_left > 0.0) out += (x - t[i]) / d_left * orc_cox(t, nt, i, q - 1, x);
  double d_right = t[i + q + 1] - t[i + 1];
  if (d_right > 0.0) out += (t[i + q + 1] - x) / d_right * orc_cox(t, nt, i + 1, q - 1, x);
  return out;
}

/* splines.py:127-136 values and :139-161 derivatives of the p+1 functions
 * supported on element e at x.  ders may be NULL (p == 0 has none). */
void orc_nonzero_basis(const double* t, int nt, int p, int e, double x, double* vals,
                       double* ders) {
  for (int r = 0; r <= p; ++r) vals[r] = orc_cox(t, nt, e + r, p, x);
  if (ders == NULL || p < 1) return;
  for (int r = 0; r <= p; ++r) {
    int i = e + r;
    double d = 0.0;
    double d_left = t[i + p] - t[i];
    if (d_left > 0.0) d += orc_cox(t, nt, i, p - 1, x) / d_left;
    double d_right = t[i + p + 1] - t[i + 1];
    if (d_right > 0.0) d -= orc_cox(t, nt, i + 1, p - 1, x) / d_right;
    ders[r] = (double)p * d;
  }
}

/* runtime.py:142-149 build_tables (+ heat.py:94-98 for derivatives):
 * nodes e*h + (ref+1)*(h/2), h = 1/K; tables V[e][r][k], D[e][r][k]. */
void orc_tables(int K, int p, int q, const double* ref_nodes, double* V, double* D) {
  int nt = K + 2 * p + 1;
  double* t = (double*)malloc(sizeof(double) * nt);
  if (g_knots && g_nknots == nt)
    memcpy(t, g_knots, sizeof(double) * nt);
  else
    orc_knots(K, p, t);
  int m = p + 1;
  double h = 1.0 / (double)K;
  double vals[32], ders[32];
  for (int e = 0; e < K; ++e) {
    for (int k = 0; k < q; ++k) {
      double x = (double)e * h + (ref_nodes[k] + 1.0) * (h / 2.0);
      if (g_knots) {
        double lo = t[p + e], he = t[p + e + 1] - t[p + e];
        x = lo + (ref_nodes[k] + 1.0) * (he / 2.0);
      }
      orc_nonzero_basis(t, nt, p, e, x, vals, D ? ders : NULL);
      for (int r = 0; r < m; ++r) {
        V[((size_t)e * m + r) * q + k] = vals[r];
        if (D) D[((size_t)e * m + r) * q + k] = p >= 1 ? ders[r] : 0.0;
      }
    }
  }
  free(t);
}

/* ----------------------------------------------------------- element kernels */

/* Select per-axis table for term `term` (0..dim-1: derivative on that axis;
 * dim: the mass term). */
static inline const double* pick(const double* V, const double* D, int axis, int term) {
  return axis == term ? D : V;
}

/* integrators.py:77-109 classical_kernel, all n*n entries (canonical pairs
 * computed, mirrored).  tabs: per-axis value tables tv[d] and derivative
 * tables td[d] ([m][q] each); coef: q^dim factors (k1 slowest) or NULL. */
static void classical_term(int dim, int m, int q, const double* b0, const double* b1,
                           const double* b2, const double* w0, const double* w1,
                           const double* w2, double jac, const double* coef, double* out) {
  int n = dim == 3 ? m * m * m : m * m;
  int m2 = m * m;
  for (int row = 0; row < n; ++row) {
    for (int col = 0; col <= row; ++col) {
      double acc = 0.0;
      if (dim == 3) {
        int i1 = row / m2, i2 = (row / m) % m, i3 = row % m;
        int j1 = col / m2, j2 = (col / m) % m, j3 = col % m;
        for (int k1 = 0; k1 < q; ++k1)
          for (int k2 = 0; k2 < q; ++k2)
            for (int k3 = 0; k3 < q; ++k3) {
              double v = b0[i1 * q + k1] * b0[j1 * q + k1] * b1[i2 * q + k2] * b1[j2 * q + k2] *
                         b2[i3 * q + k3] * b2[j3 * q + k3] * w0[k1] * w1[k2] * w2[k3] * jac;
              if (coef) v = v * coef[(k1 * q + k2) * q + k3];
              acc += v;
            }
      } else {
        int i1 = row / m, i2 = row % m;
        int j1 = col / m, j2 = col % m;
        for (int k1 = 0; k1 < q; ++k1)
          for (int k2 = 0; k2 < q; ++k2) {
            double v = b0[i1 * q + k1] * b0[j1 * q + k1] * b1[i2 * q + k2] * b1[j2 * q + k2] *
                       w0[k1] * w1[k2] * jac;
            if (coef) v = v * coef[k1 * q + k2];
            acc += v;
          }
      }
      out[row * n + col] = acc;
      out[col * n + row] = acc;
    }
  }
}

/* integrators.py:112-151 sumfact_kernel (3D) with the coefficient appended to
 * the stage-1 product; 2D = stage 1 then the last stage over axis 2. */
static void sumfact_term(int dim, int m, int q, const double* b0, const double* b1,
                         const double* b2, const double* w0, const double* w1, const double* w2,
                         double jac, const double* coef, double* Dbuf, double* Cbuf,
                         double* out) {
  int m2 = m * m;
  if (dim == 3) {
    int n = m2 * m;
    memset(Dbuf, 0, sizeof(double) * m * m * q * q);
    memset(Cbuf, 0, sizeof(double) * m * m * m * m * q);
    for (int i1 = 0; i1 < m; ++i1)
      for (int j1 = 0; j1 < m; ++j1)
        for (int k2 = 0; k2 < q; ++k2)
          for (int k3 = 0; k3 < q; ++k3)
            for (int k1 = 0; k1 < q; ++k1) {
              double v = b0[i1 * q + k1] * b0[j1 * q + k1] * w0[k1] * jac;
              if (coef) v = v * coef[(k1 * q + k2) * q + k3];
              Dbuf[((i1 * m + j1) * q + k2) * q + k3] += v;
            }
    for (int i2 = 0; i2 < m; ++i2)
      for (int j2 = 0; j2 < m; ++j2)
        for (int i1 = 0; i1 < m; ++i1)
          for (int j1 = 0; j1 < m; ++j1)
            for (int k3 = 0; k3 < q; ++k3)
              for (int k2 = 0; k2 < q; ++k2)
                Cbuf[(((i2 * m + i1) * m + j2) * m + j1) * q + k3] +=
                    b1[i2 * q + k2] * b1[j2 * q + k2] * Dbuf[((i1 * m + j1) * q + k2) * q + k3] *
                    w1[k2];
    for (int row = 0; row < n; ++row)
      for (int col = 0; col <= row; ++col) {
        int i1 = row / m2, i2 = (row / m) % m, i3 = row % m;
        int j1 = col / m2, j2 = (col / m) % m, j3 = col % m;
        double acc = 0.0;
        for (int k3 = 0; k3 < q; ++k3)
          acc += b2[i3 * q + k3] * b2[j3 * q + k3] *
                 Cbuf[(((i2 * m + i1) * m + j2) * m + j1) * q + k3] * w2[k3];
        out[row * n + col] = acc;
        out[col * n + row] = acc;
      }
  } else {
    int n = m2;
    memset(Dbuf, 0, sizeof(double) * m * m * q);
    for (int i1 = 0; i1 < m; ++i1)
      for (int j1 = 0; j1 < m; ++j1)
        for (int k2 = 0; k2 < q; ++k2)
          for (int k1 = 0; k1 < q; ++k1) {
            double v = b0[i1 * q + k1] * b0[j1 * q + k1] * w0[k1] * jac;
            if (coef) v = v * coef[k1 * q + k2];
            Dbuf[(i1 * m + j1) * q + k2] += v;
          }
    for (int row = 0; row < n; ++row)
      for (int col = 0; col <= row; ++col) {
        int i1 = row / m, i2 = row % m, j1 = col / m, j2 = col % m;
        double acc = 0.0;
        for (int k2 = 0; k2 < q; ++k2)
          acc += b1[i2 * q + k2] * b1[j2 * q + k2] * Dbuf[(i1 * m + j1) * q + k2] * w1[k2];
        out[row * n + col] = acc;
        out[col * n + row] = acc;
      }
  }
}

/* One element matrix (n x n) for operator op.  V, D: mesh tables [K][m][q];
 * alpha: 1D element indices; method 0 = classical, 1 = sumfact.  Terms are
 * summed in the fixed order: derivative on axis 0, 1, (2), then mass. */
static void element_scratch(int dim, int p, int q, int op, int method, const double* V,
                            const double* D, const double* w, double jac, const double* coef,
                            const int* alpha, double* out, double* scratch);

void orc_element(int dim, int K, int p, int q, int op, int method, const double* V,
                 const double* D, const double* w, double jac, const double* coef,
                 const int* alpha, double* out) {
  (void)K;
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  double* scratch = (double*)malloc(sizeof(double) * (n * n + m * m * q * q + m * m * m * m * q));
  element_scratch(dim, p, q, op, method, V, D, w, jac, coef, alpha, out, scratch);
  free(scratch);
}

/* scratch: n*n + m*m*q*q + m^4*q doubles. */
static void element_scratch(int dim, int p, int q, int op, int method, const double* V,
                            const double* D, const double* w, double jac, const double* coef,
                            const int* alpha, double* out, double* scratch) {
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  const double* tv[3];
  const double* td[3];
  for (int d = 0; d < dim; ++d) {
    tv[d] = V + (size_t)alpha[d] * m * q;
    td[d] = D ? D + (size_t)alpha[d] * m * q : NULL;
  }
  if (dim == 2) { tv[2] = tv[1]; td[2] = td[1]; }
  int terms[4], nterm = 0;
  if (op == ORC_OP_MASS) {
    terms[nterm++] = dim;
  } else {
    for (int d = 0; d < dim; ++d) terms[nterm++] = d;
    if (op == ORC_OP_STIFFNESS_MASS) terms[nterm++] = dim;
  }
  double* tmp = scratch;
  double* Dbuf = scratch + n * n;
  double* Cbuf = Dbuf + m * m * q * q;
  for (int t = 0; t < nterm; ++t) {
    int term = terms[t];
    const double* b0 = pick(tv[0], td[0], 0, term);
    const double* b1 = pick(tv[1], td[1], 1, term);
    const double* b2 = pick(tv[2], td[2], 2, term);
    double* dst = t == 0 ? out : tmp;
    const double* w0 = axis_w(w, alpha, 0, q);
    const double* w1 = axis_w(w, alpha, 1, q);
    const double* w2 = axis_w(w, alpha, dim == 3 ? 2 : 1, q);
    const double jj = g_wt ? 1.0 : jac;
    if (method == 0)
      classical_term(dim, m, q, b0, b1, b2, w0, w1, w2, jj, coef, dst);
    else
      sumfact_term(dim, m, q, b0, b1, b2, w0, w1, w2, jj, coef, Dbuf, Cbuf, dst);
    if (t > 0)
      for (int i = 0; i < n * n; ++i) out[i] = out[i] + tmp[i];
  }
}

/* Row il of the classical element matrix only (same per-entry operation order
 * as classical_term / orc_element: canonical (row >= col) factor order, terms
 * summed in the same order), for the sampled-row oracle at full mesh sizes. */
static void classical_row(int dim, int p, int q, int op, const double* V, const double* D,
                          const double* w, double jac, const double* coef, const int* alpha,
                          int il, double* out) {
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  int m2 = m * m;
  const double* tv[3];
  const double* td[3];
  for (int d = 0; d < dim; ++d) {
    tv[d] = V + (size_t)alpha[d] * m * q;
    td[d] = D ? D + (size_t)alpha[d] * m * q : NULL;
  }
  if (dim == 2) { tv[2] = tv[1]; td[2] = td[1]; }
  int terms[4], nterm = 0;
  if (op == ORC_OP_MASS) {
    terms[nterm++] = dim;
  } else {
    for (int d = 0; d < dim; ++d) terms[nterm++] = d;
    if (op == ORC_OP_STIFFNESS_MASS) terms[nterm++] = dim;
  }
  const double* w0 = axis_w(w, alpha, 0, q);
  const double* w1 = axis_w(w, alpha, 1, q);
  const double* w2 = axis_w(w, alpha, dim == 3 ? 2 : 1, q);
  if (g_wt) jac = 1.0;
  for (int j = 0; j < n; ++j) {
    int row = il > j ? il : j, col = il > j ? j : il;
    double total = 0.0;
    for (int t = 0; t < nterm; ++t) {
      const double* b0 = pick(tv[0], td[0], 0, terms[t]);
      const double* b1 = pick(tv[1], td[1], 1, terms[t]);
      const double* b2 = pick(tv[2], td[2], 2, terms[t]);
      double acc = 0.0;
      if (dim == 3) {
        int i1 = row / m2, i2 = (row / m) % m, i3 = row % m;
        int j1 = col / m2, j2 = (col / m) % m, j3 = col % m;
        for (int k1 = 0; k1 < q; ++k1)
          for (int k2 = 0; k2 < q; ++k2)
            for (int k3 = 0; k3 < q; ++k3) {
              double v = b0[i1 * q + k1] * b0[j1 * q + k1] * b1[i2 * q + k2] * b1[j2 * q + k2] *
                         b2[i3 * q + k3] * b2[j3 * q + k3] * w0[k1] * w1[k2] * w2[k3] * jac;
              if (coef) v = v * coef[(k1 * q + k2) * q + k3];
              acc += v;
            }
      } else {
        int i1 = row / m, i2 = row % m, j1 = col / m, j2 = col % m;
        for (int k1 = 0; k1 < q; ++k1)
          for (int k2 = 0; k2 < q; ++k2) {
            double v = b0[i1 * q + k1] * b0[j1 * q + k1] * b1[i2 * q + k2] * b1[j2 * q + k2] *
                       w0[k1] * w1[k2] * jac;
            if (coef) v = v * coef[k1 * q + k2];
            acc += v;
          }
      }
      total = t == 0 ? acc : total + acc;
    }
    out[j] = total;
  }
}

/* --------------------------------------------------------------- CSR pattern */

/* Columns coupled to 1D dof I: [max(I-p,0), min(I+p,n1d-1)]. */
static inline int64_t band_lo(int64_t I, int p) { return I - p > 0 ? I - p : 0; }
static inline int64_t band_cnt(int64_t I, int p, int64_t n1d) {
  int64_t hi = I + p < n1d - 1 ? I + p : n1d - 1;
  return hi - band_lo(I, p) + 1;
}

/* assembly.py:99-115 symbolic_pattern (sorted columns, both triangles), for
 * rows [row_begin, row_end); indptr is relative (indptr[0] = 0). */
int64_t orc_pattern(int dim, int K, int p, int64_t row_begin, int64_t row_end, int64_t* indptr,
                    int64_t* indices) {
  int64_t n1d = K + p;
  int64_t nnz = 0;
  for (int64_t row = row_begin; row < row_end; ++row) {
    if (indptr) indptr[row - row_begin] = nnz;
    int64_t I[3];
    if (dim == 3) {
      I[0] = row / (n1d * n1d); I[1] = (row / n1d) % n1d; I[2] = row % n1d;
    } else {
      I[0] = row / n1d; I[1] = row % n1d; I[2] = 0;
    }
    int64_t lo[3], c[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = d < dim ? band_lo(I[d], p) : 0;
      c[d] = d < dim ? band_cnt(I[d], p, n1d) : 1;
    }
    for (int64_t a = 0; a < c[0]; ++a)
      for (int64_t b = 0; b < c[1]; ++b)
        for (int64_t cc = 0; cc < c[2]; ++cc) {
          if (indices) {
            int64_t col = dim == 3 ? ((lo[0] + a) * n1d + lo[1] + b) * n1d + lo[2] + cc
                                   : (lo[0] + a) * n1d + lo[1] + b;
            indices[nnz] = col;
          }
          nnz++;
        }
  }
  if (indptr) indptr[row_end - row_begin] = nnz;
  return nnz;
}

/* Offset of (row, col) in the structured CSR, relative to row_base's first entry. */
static inline int64_t csr_pos(int dim, int64_t n1d, int p, const int64_t* indptr,
                              int64_t row_base, int64_t row, int64_t col) {
  int64_t I[3], J[3];
  if (dim == 3) {
    I[0] = row / (n1d * n1d); I[1] = (row / n1d) % n1d; I[2] = row % n1d;
    J[0] = col / (n1d * n1d); J[1] = (col / n1d) % n1d; J[2] = col % n1d;
  } else {
    I[0] = row / n1d; I[1] = row % n1d; J[0] = col / n1d; J[1] = col % n1d;
  }
  int64_t off = 0;
  for (int d = 0; d < dim; ++d) off = off * band_cnt(I[d], p, n1d) + (J[d] - band_lo(I[d], p));
  return indptr[row - row_base] + off;
}

/* assembly.py:46-83 assemble, restated as a scatter in lexicographic element
 * order into the structured CSR (rows [row_begin,row_end) only; entries whose
 * row falls outside are skipped).  Elements [el_begin, el_end) along the
 * slowest axis are integrated on the fly (runtime.py:187-219 without the
 * N_el x n x n staging array).  coef: [N_el][q^dim] or NULL; coef_scalar
 * multiplies every quadrature point when coef == NULL and coef_scalar != 1. */
void orc_integrate_assemble(int dim, int K, int p, int q, int op, int method,
                            const double* ref_nodes, const double* w, double jac,
                            const double* coef, int el_begin, int el_end, int64_t row_begin,
                            int64_t row_end, const int64_t* indptr, double* values) {
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  int nq = dim == 3 ? q * q * q : q * q;
  int64_t n1d = K + p;
  double* V = (double*)malloc(sizeof(double) * K * m * q);
  double* D = (double*)malloc(sizeof(double) * K * m * q);
  orc_tables(K, p, q, ref_nodes, V, p >= 1 ? D : NULL);
  abs_inplace(V, (size_t)K * m * q);
  abs_inplace(D, (size_t)K * m * q);
  double* cabs = NULL;
  if (coef && g_absolute) {
    int64_t nel = dim == 3 ? (int64_t)K * K * K : (int64_t)K * K;
    cabs = (double*)malloc(sizeof(double) * nel * nq);
    for (int64_t i = 0; i < nel * nq; ++i) cabs[i] = fabs(coef[i]);
    coef = cabs;
  }
  double* E = (double*)malloc(sizeof(double) * n * n);
  int64_t nvals = indptr[row_end - row_begin];
  memset(values, 0, sizeof(double) * nvals);
  int K2 = dim == 3 ? K : 1;
  int64_t dofs[512];
  for (int e0 = el_begin; e0 < el_end; ++e0)
    for (int e1 = 0; e1 < K; ++e1)
      for (int e2 = 0; e2 < K2; ++e2) {
        int alpha[3] = {e0, e1, e2};
        int64_t eid = dim == 3 ? ((int64_t)e0 * K + e1) * K + e2 : (int64_t)e0 * K + e1;
        orc_element(dim, K, p, q, op, method, V, D, w, jac, coef ? coef + eid * nq : NULL,
                    alpha, E);
        for (int i = 0; i < n; ++i) {
          int64_t g;
          if (dim == 3)
            g = ((int64_t)(e0 + i / (m * m)) * n1d + e1 + (i / m) % m) * n1d + e2 + i % m;
          else
            g = (int64_t)(e0 + i / m) * n1d + e1 + i % m;
          dofs[i] = g;
        }
        for (int i = 0; i < n; ++i) {
          if (dofs[i] < row_begin || dofs[i] >= row_end) continue;
          for (int j = 0; j < n; ++j) {
            int64_t pos = csr_pos(dim, n1d, p, indptr, row_begin, dofs[i], dofs[j]);
            values[pos] += E[i * n + j];
          }
        }
      }
  free(V);
  free(D);
  free(E);
  free(cabs);
}

/* Sampled-row oracle: full CSR rows for the listed
 * global rows, summing element contributions in lexicographic element
 * order.  out_offsets[r] is where row r's values start in out. */
void orc_rows(int dim, int K, int p, int q, int op, int method, const double* ref_nodes,
              const double* w, double jac, const double* coef, const int64_t* rows, int nrows,
              const int64_t* out_offsets, double* out) {
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  int nq = dim == 3 ? q * q * q : q * q;
  int64_t n1d = K + p;
  double* V = (double*)malloc(sizeof(double) * K * m * q);
  double* D = (double*)malloc(sizeof(double) * K * m * q);
  orc_tables(K, p, q, ref_nodes, V, p >= 1 ? D : NULL);
  abs_inplace(V, (size_t)K * m * q);
  abs_inplace(D, (size_t)K * m * q);
  double* cabs = NULL;
  if (coef && g_absolute) {
    int64_t nel = dim == 3 ? (int64_t)K * K * K : (int64_t)K * K;
    cabs = (double*)malloc(sizeof(double) * nel * nq);
    for (int64_t i = 0; i < nel * nq; ++i) cabs[i] = fabs(coef[i]);
    coef = cabs;
  }
  double* E = (double*)malloc(sizeof(double) * n * n);
  for (int r = 0; r < nrows; ++r) {
    int64_t row = rows[r];
    int64_t I[3] = {0, 0, 0};
    if (dim == 3) {
      I[0] = row / (n1d * n1d); I[1] = (row / n1d) % n1d; I[2] = row % n1d;
    } else {
      I[0] = row / n1d; I[1] = row % n1d;
    }
    int64_t c[3], lo[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = d < dim ? band_lo(I[d], p) : 0;
      c[d] = d < dim ? band_cnt(I[d], p, n1d) : 1;
    }
    int64_t cnt = c[0] * c[1] * c[2];
    double* o = out + out_offsets[r];
    for (int64_t j = 0; j < cnt; ++j) o[j] = 0.0;
    int elo[3], ehi[3];
    for (int d = 0; d < 3; ++d) {
      if (d < dim) {
        elo[d] = (int)(I[d] - p > 0 ? I[d] - p : 0);
        ehi[d] = (int)(I[d] < K - 1 ? I[d] : K - 1);
      } else {
        elo[d] = 0; ehi[d] = 0;
      }
    }
    for (int a0 = elo[0]; a0 <= ehi[0]; ++a0)
      for (int a1 = elo[1]; a1 <= ehi[1]; ++a1)
        for (int a2 = elo[2]; a2 <= ehi[2]; ++a2) {
          int alpha[3] = {a0, a1, a2};
          int64_t eid = dim == 3 ? ((int64_t)a0 * K + a1) * K + a2 : (int64_t)a0 * K + a1;
          int il = dim == 3 ? (int)(((I[0] - a0) * m + (I[1] - a1)) * m + (I[2] - a2))
                            : (int)((I[0] - a0) * m + (I[1] - a1));
          const double* ce = coef ? coef + eid * nq : NULL;
          double* Erow = E + (size_t)il * n;
          if (method == 0)
            classical_row(dim, p, q, op, V, D, w, jac, ce, alpha, il, Erow);
          else
            orc_element(dim, K, p, q, op, method, V, D, w, jac, ce, alpha, E);
          for (int j = 0; j < n; ++j) {
            int64_t J[3];
            if (dim == 3) {
              J[0] = a0 + j / (m * m); J[1] = a1 + (j / m) % m; J[2] = a2 + j % m;
            } else {
              J[0] = a0 + j / m; J[1] = a1 + j % m; J[2] = 0;
            }
            int64_t off = 0;
            for (int d = 0; d < dim; ++d) off = off * c[d] + (J[d] - lo[d]);
            o[off] += E[il * n + j];
          }
        }
  }
  free(V);
  free(D);
  free(E);
  free(cabs);
}

/* ------------------------------------------------------ CPU baseline (timed) */

/* The reference's mesh-wide CPU path (runtime.py:258-267 over_elements +
 * assembly.py:46-83), restated for timing on the host cores: element matrices
 * by the chosen method on `nthreads` OpenMP threads (planes e0 of the slowest
 * axis coloured mod p+1 so concurrent planes never touch the same rows), each
 * scattered straight into the structured CSR.  Not bitwise-ordered like
 * orc_integrate_assemble; used only for the reported CPU baseline. */
void orc_cpu_baseline(int dim, int K, int p, int q, int op, int method, const double* ref_nodes,
                      const double* w, double jac, const double* coef, int el_begin, int el_end,
                      const int64_t* indptr, double* values, int nthreads) {
  int m = p + 1;
  int n = dim == 3 ? m * m * m : m * m;
  int nq = dim == 3 ? q * q * q : q * q;
  int64_t n1d = K + p;
  double* V = (double*)malloc(sizeof(double) * K * m * q);
  double* D = (double*)malloc(sizeof(double) * K * m * q);
  orc_tables(K, p, q, ref_nodes, V, p >= 1 ? D : NULL);
  /* zero the rows the slab touches: planes [el_begin, el_end + p) */
  int64_t plane = dim == 3 ? n1d * n1d : n1d;
  int64_t r0 = (int64_t)el_begin * plane;
  int64_t r1 = ((int64_t)el_end + p < n1d ? (int64_t)el_end + p : n1d) * plane;
  memset(values + indptr[r0], 0, sizeof(double) * (indptr[r1] - indptr[r0]));
  int K2 = dim == 3 ? K : 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  /* colour (e0 mod p+1, e1 mod p+1): concurrent (e0, e1) pencils of one colour
   * touch disjoint rows, each pencil runs its e2 elements in order. */
  int nc1 = dim == 3 ? p + 1 : 1;
  for (int color = 0; color < (p + 1) * nc1; ++color) {
    int c0 = color / nc1, c1 = color % nc1;
    int n0 = (el_end - el_begin - c0 + p) / (p + 1);
    int n1 = dim == 3 ? (K - c1 + p) / (p + 1) : 1;
    if (n0 <= 0 || n1 <= 0) continue;
#pragma omp parallel
    {
      double* E = (double*)malloc(sizeof(double) * n * n);
      double* scratch = (double*)malloc(sizeof(double) * (n * n + m * m * q * q + m * m * m * m * q));
      int64_t dofs[512];
#pragma omp for schedule(dynamic, 1)
      for (int task = 0; task < n0 * n1; ++task) {
        int e0 = el_begin + c0 + (task / n1) * (p + 1);
        int e1_lo = dim == 3 ? c1 + (task % n1) * (p + 1) : 0;
        int e1_hi = dim == 3 ? e1_lo + 1 : K;
        for (int e1 = e1_lo; e1 < e1_hi; ++e1)
          for (int e2 = 0; e2 < K2; ++e2) {
            int alpha[3] = {e0, e1, e2};
            int64_t eid = dim == 3 ? ((int64_t)e0 * K + e1) * K + e2 : (int64_t)e0 * K + e1;
            element_scratch(dim, p, q, op, method, V, D, w, jac, coef ? coef + eid * nq : NULL,
                            alpha, E, scratch);
            for (int i = 0; i < n; ++i)
              dofs[i] = dim == 3 ? ((int64_t)(e0 + i / (m * m)) * n1d + e1 + (i / m) % m) * n1d +
                                       e2 + i % m
                                 : (int64_t)(e0 + i / m) * n1d + e1 + i % m;
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j)
                values[csr_pos(dim, n1d, p, indptr, 0, dofs[i], dofs[j])] += E[i * n + j];
          }
      }
      free(E);
      free(scratch);
    }
  }
  free(V);
  free(D);
}
