/*
 * iga_b200.h -- C-ABI of the B200-native IGA integration + assembly path.
 *
 * Plain C types only (no torch, no C++): every pointer is a device pointer
 * owned by the caller unless stated otherwise, every call takes the CUDA
 * stream it is enqueued on as `void* stream` (NULL = legacy default stream),
 * nothing is allocated or synchronised inside, and calls on different streams
 * are reentrant.  Return value: IGA_OK, or an IGA_E* code with a message in
 * iga_last_error() (thread-local).  The Python shims map IGA_EINVAL and
 * IGA_EUNSUPPORTED to ValueError (the reference's convention for bad sizes
 * and shapes, integrators.py:180-190, assembly.py:22-24) and IGA_ECUDA to
 * RuntimeError.
 *
 * Reference interfaces each entry point replaces are cited as
 * /root/reference/pkg/src/igabench/<file>:<line>.
 */
#ifndef IGA_B200_H
#define IGA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGA_ABI_VERSION 5

#define IGA_OK 0
#define IGA_EINVAL 1       /* invalid argument -> ValueError            */
#define IGA_ECUDA 2        /* CUDA launch/runtime failure -> RuntimeError */
#define IGA_EUNSUPPORTED 3 /* (p, q, dim) outside the device grid -> ValueError */
#define IGA_ENOCONV 4      /* iterative solve did not converge -> RuntimeError  */

/* Operators (SURVEY.md §8(b) superset of the reference's mass-only Gram). */
#define IGA_OP_MASS 0           /* int c B_i B_j                              */
#define IGA_OP_STIFFNESS 1      /* int c grad B_i . grad B_j                  */
#define IGA_OP_STIFFNESS_MASS 2 /* int c (grad B_i . grad B_j + B_i B_j)      */

/* Integration methods. */
#define IGA_METHOD_CLASSICAL 0        /* Algorithm 1, integrators.py:77-109              */
#define IGA_METHOD_SUMFACT 1          /* Algorithm 2, element-local, integrators.py:112-151 */
#define IGA_METHOD_SUMFACT_ASSEMBLED 2 /* sum factorization with the inter-element sum
                                          folded into each axis contraction (row owner) */
#define IGA_METHOD_SEPARABLE 3         /* scalar coefficient only: the 3D quadrature factorised
                                          into assembled 1D band matrices (Kronecker form),
                                          HBM-bound CSR fill; dim = 3 */

/* One mesh-wide problem: open uniform knots on [0,1]^dim, K elements per
 * axis, degree p, q Gauss points per axis (mesh.py:73-93). */
typedef struct iga_problem {
  int32_t dim;          /* 2 or 3 */
  int32_t K;            /* elements per axis */
  int32_t p;            /* degree */
  int32_t q;            /* quadrature points per axis */
  int32_t op;           /* IGA_OP_* */
  int32_t reserved;     /* must be 0 */
  double jac;           /* constant Jacobian, host-computed as (1/(2K))**dim (mesh.py:90) */
  double coef_scalar;   /* coefficient when coef == NULL (1.0 = the reference Gram) */
  const double* coef;   /* device [K^dim][q^dim] per-quadrature-point coefficient, element
                           lexicographic (slowest axis first), then k1 slowest; or NULL */
  const double* weights; /* device [q] reference Gauss weights (leggauss, mesh.py:82) */
  const double* tables_v; /* device [K][p+1][q] basis values from iga_mesh_tables */
  const double* tables_d; /* device [K][p+1][q] basis derivatives (NULL for IGA_OP_MASS) */
  const double* band;     /* device [K+p][2p+1][2] assembled 1D band matrices from
                             iga_band_tables, or NULL.  Used by the separable method only:
                             with it the integration kernel reads the 1D integrals instead of
                             forming them in every CTA (a shorter prologue).  Read-only: the
                             same buffer may feed concurrent launches on several streams. */
  /* General open knot vector, the same on every axis like the
   * reference's single KnotVector: knots [K + 2p + 1] non-decreasing, p + 1 equal at each
   * end, K non-empty spans (element e = [t_{p+e}, t_{p+e+1}]), or NULL for the open uniform
   * vector of make_knot_vector (splines.py:59-75).  With knots, element e's Jacobian is
   * folded into the per-axis weights elem_weights [K][q] = w_k h_e / 2 (h_e the span
   * length; iga_mesh_tables_general writes them) and jac must be 1.0; the CSR pattern is
   * unchanged. */
  const double* knots;
  const double* elem_weights;
} iga_problem;

const char* iga_last_error(void);
int32_t iga_abi_version(void);

/* K1 -- per-1D-element basis tables at the mapped Gauss nodes.
 * vals/ders: [K][p+1][q]; ders may be NULL.  Bitwise equal to
 * runtime._MeshContext.build_tables (runtime.py:142-149) ->
 * splines.basis_value_table / basis_derivative_table (splines.py:164-178). */
int32_t iga_mesh_tables(int32_t K, int32_t p, int32_t q, const double* ref_nodes, double* vals,
                        double* ders, void* stream);

/* K1 on a general open knot vector knots [K + 2p + 1]: tables at the Gauss points mapped
 * into each span (x = lo + (ref + 1) h / 2, h = hi - lo) and the per-element weights
 * elem_weights [K][q] = weights[k] * (h_e / 2) (either output may be NULL: not written). */
int32_t iga_mesh_tables_general(int32_t K, int32_t p, int32_t q, const double* knots,
                                const double* ref_nodes, const double* weights, double* vals,
                                double* ders, double* elem_weights, void* stream);

/* K1' -- nonzero basis values/derivatives at arbitrary points:
 * vals/ders [n][p+1] for point x[i] in element elem[i]
 * (splines.eval_nonzero_basis / eval_nonzero_basis_derivatives, splines.py:127-161);
 * knots: device general knot vector [K + 2p + 1], or NULL for the open uniform one. */
int32_t iga_basis_eval(int32_t K, int32_t p, const double* knots, int64_t n,
                       const int32_t* elem, const double* x, double* vals, double* ders,
                       void* stream);

/* eval_basis / eval_basis_order0 (splines.py:78-118) on any non-decreasing knot vector
 * knots[n_knots]: out[i] = B_{index[i], order}(x[i]) by the reference's two-term
 * recursion (0/0 := 0, last non-empty span closed at the last knot), bitwise equal.
 * An index outside [0, n_knots - order - 2] yields NaN (the Python shim raises
 * IndexError before the call, as splines.py:85-86 / :103-104 do). */
int32_t iga_eval_basis(const double* knots, int32_t n_knots, int32_t order, int64_t n,
                       const int32_t* index, const double* x, double* out, void* stream);

/* K1 + the assembled 1D band matrices of the separable method in one launch:
 * vals/ders [K][p+1][q] as iga_mesh_tables (either may be NULL: not stored), and
 * band[I][d] = (m, k), I < K+p, d = J-I+p in [0, 2p] ((K+p)(2p+1)*2 doubles):
 *   m(I,J) = sum_e sum_k w_k V_e(I-e,k) V_e(J-e,k)   (k(I,J): the same with derivatives)
 * over all elements, elements ascending -- the 1D factors of the Kronecker form of the
 * reference's element quadrature summed by assemble (integrators.py:77-151,
 * assembly.py:80-82).  Uses prob->K, p, q, op, weights and, for a general knot vector
 * (prob->knots), writes the per-element weights into elem_weights [K][q] (the same values
 * as iga_mesh_tables_general; NULL for the uniform mesh). */
int32_t iga_band_tables(const iga_problem* prob, const double* ref_nodes, double* vals,
                        double* ders, double* band, double* elem_weights, void* stream);

/* Host arithmetic: number of CSR entries in global rows [row_begin, row_end). */
int64_t iga_csr_nnz(int32_t dim, int32_t K, int32_t p, int64_t row_begin, int64_t row_end);

/* K5 -- structured CSR pattern for rows [row_begin, row_end): indptr[rows+1]
 * (relative, indptr[0] = 0) and sorted column indices, both triangles.
 * Replaces assembly.symbolic_pattern (assembly.py:99-115) and the
 * COO->CSR index build of assembly.assemble (assembly.py:68-82). */
int32_t iga_csr_pattern(int32_t dim, int32_t K, int32_t p, int64_t row_begin, int64_t row_end,
                        int64_t* indptr, int32_t* indices, void* stream);

/* K2/K3 per-element matrices: out[count][n][n], n = (p+1)^dim, for the
 * elements elem_ids[count][dim].  Strict IEEE, same operation order as the
 * reference kernels, so mass matrices are bitwise equal to
 * integrate_element_classical / integrate_element_sumfact (integrators.py:193-230).
 * elem_nodes: optional device [count][dim][q] physical nodes (the caller's
 * QuadratureRule.nodes); NULL maps prob->weights' reference nodes as gauss_rule
 * does.  ref_nodes [q] must be given when elem_nodes is NULL.
 * elem_weights: optional device [count][dim][q] per-axis weights (the reference
 * passes rule.weights[0], [1], [2] separately, integrators.py:200-203); NULL uses
 * prob->weights on every axis.  elem_coef: optional device [count][q^dim]
 * coefficients at each listed element's points (k1 slowest); NULL uses prob->coef
 * indexed by element id, or prob->coef_scalar.
 * prob->tables_* are ignored (tables are evaluated from the nodes). */
int32_t iga_element_matrices(const iga_problem* prob, int32_t method, const double* ref_nodes,
                             const int32_t* elem_ids, const double* elem_nodes,
                             const double* elem_weights, const double* elem_coef, int64_t count,
                             double* out, void* stream);

/* Fused mesh-wide integration + assembly (runtime.run_integration,
 * runtime.py:187-219 + assembly.assemble, assembly.py:46-83, without the
 * N_el x n x n staging array).  Integrates the elements whose slowest index is in
 * [el_begin, el_end) and writes CSR values of the global rows
 * [row_plane_begin, row_plane_end) x (K+p)^(dim-1) into `values`, which starts at
 * the first entry of row_plane_begin.  Rows touched by elements outside the slab
 * receive partial sums (the multi-GPU interface rows).  The call overwrites
 * every value of its rows. */
int32_t iga_integrate_assemble(const iga_problem* prob, int32_t method, int32_t el_begin,
                               int32_t el_end, int32_t row_plane_begin, int32_t row_plane_end,
                               double* values, void* stream);

/* assembly.assemble (assembly.py:46-83) from precomputed element matrices
 * mats[K^dim][n][n] (element lexicographic): every CSR value of the rows
 * [row_plane_begin, row_plane_end) planes is the sum of its element
 * contributions in lexicographic element order (deterministic, no atomics). */
int32_t iga_assemble_elements(int32_t dim, int32_t K, int32_t p, const double* mats,
                              int32_t row_plane_begin, int32_t row_plane_end, double* values,
                              void* stream);

/* Matrix-free operator application y = alpha M x + beta S x over the whole mesh
 * (x, y: [(K+p)^dim] dof vectors, lexicographic like dof_index), by sum
 * factorization per element with the problem's coefficient; y is overwritten.
 * Device version of heat.HeatProblem.assemble_rhs (heat.py:131-158), which is
 * apply(alpha = 1, beta = -dt).  dim = 3. */
int32_t iga_apply(const iga_problem* prob, double alpha, double beta, const double* x, double* y,
                  void* stream);

/* y[i] += x[i], i < n  (interface-row accumulation after the NCCL receive). */
int32_t iga_axpy(int64_t n, const double* x, double* y, void* stream);

/* Matrix Market export (assembly.write_matrix_market, assembly.py:118-120 =
 * scipy.io.mmwrite(path, coo, symmetry="symmetric")): the lower triangle of the
 * structured CSR whose values are given, byte-identical to scipy 1.18's output.
 * The device version streams row blocks to the host (two pinned staging buffers
 * it allocates and frees, one cudaMemcpyAsync per block on `stream`) and formats
 * them with `threads` host threads while the next block is in flight; it returns
 * after the file is closed.  The _host version takes host values and needs no GPU. */
int32_t iga_write_matrix_market(int32_t dim, int32_t K, int32_t p, const double* values,
                                const char* path, int32_t threads, void* stream);
int32_t iga_write_matrix_market_host(int32_t dim, int32_t K, int32_t p, const double* values,
                                     const char* path, int32_t threads);

/* CSR SpMV y = A x over the structured pattern (assembly.spmv, assembly.py:86-91). */
int32_t iga_spmv(int32_t dim, int32_t K, int32_t p, const double* values, const double* x,
                 double* y, void* stream);

/* Conjugate gradients for G x = b on the device: the solve of the heat demo's implicit
 * step (heat.HeatProblem._solve, heat.py:168-175, scipy cg with rtol 1e-10 and maxiter
 * 10 n).  G is the assembled structured CSR (values != NULL: iga_spmv(dim, K, p, values))
 * or, with values == NULL, the matrix-free alpha M + beta S of prob (iga_apply, dim 3).
 * x holds x0 on entry and the solution on return; work holds iga_cg_work_size(n) doubles.
 * Stops when ||b - G x|| <= rtol ||b||.  The iterations run stream-ordered on the device
 * (four launches each, deterministic fixed-order reductions); the host reads a 32-byte
 * state every check_every iterations.  *iters: iterations done.  IGA_ENOCONV if maxiter
 * iterations did not converge. */
int64_t iga_cg_work_size(int64_t n);
int32_t iga_cg(int32_t dim, int32_t K, int32_t p, const double* values, const iga_problem* prob,
               double alpha, double beta, int64_t n, const double* b, double* x, double* work,
               double rtol, int64_t maxiter, int32_t check_every, int64_t* iters, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* IGA_B200_H */
