// Element-local kernels.
//
//  * k_element_strict  -- per-element matrices with the reference's exact
//    operation order (strict IEEE via __dmul_rn/__dadd_rn): classical =
//    integrators.py:77-109, sum factorization = integrators.py:112-151.
//    Bitwise equal to the numba kernels for the mass operator; stiffness =
//    the same kernels once per axis with derivative tables, summed in axis
//    order (oracle/iga_oracle.c orc_element defines the same order).
//  * k_classical_scatter -- Algorithm 1 mesh-wide: grid over elements, warps
//    over canonical pairs, lanes over quadrature points, warp-shuffle
//    reduction, fused scatter into the structured CSR (by element colour).
//  * k_sumfact_scatter -- Algorithm 2 element-local, stages in shared memory
//    (Foata classes p+1..p+6 of taskgraph.py:204-223 -> barrier phases),
//    fused scatter (by element colour).
#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

// ---------------------------------------------------------------- strict
// Shared layout: tabs[dim][2][m][Q] (values, derivatives), w[dim][Q] (per-axis weights:
// integrators.py:200-203 passes rule.weights[0..2] separately), then sumfact buffers
// D [m][m][Q][Q] and C [m][m][m][m][Q] (3D).
template <int DIM, int P, int Q>
__global__ void __launch_bounds__(256) k_element_strict(ElemArgs a) {
  constexpr int m = P + 1;
  constexpr int n = DIM == 3 ? m * m * m : m * m;
  constexpr int nq = DIM == 3 ? Q * Q * Q : Q * Q;
  extern __shared__ double smem[];
  double* tabs = smem;                       // DIM*2*m*Q
  double* w = tabs + DIM * 2 * m * Q;        // DIM*Q
  // sum-factorization stage buffers: shared memory, or (high degrees: m^4 Q doubles do not
  // fit) this CTA's slice of the global scratch
  double* Dbuf = a.scratch ? a.scratch + (int64_t)blockIdx.x * (m * m * Q * Q + m * m * m * m * Q)
                           : w + DIM * Q;    // m*m*Q*Q (3D) or m*m*Q (2D)
  double* Cbuf = Dbuf + m * m * Q * Q;       // m^4*Q (3D)
  const int64_t el = blockIdx.x;
  if (el >= a.count) return;
  int alpha[3] = {0, 0, 0};
  for (int d = 0; d < DIM; ++d) alpha[d] = a.elem_ids[el * DIM + d];
  // tables: thread per (axis, point)
  for (int t = threadIdx.x; t < DIM * Q; t += blockDim.x) {
    const int d = t / Q, k = t % Q;
    const double x = a.elem_nodes ? a.elem_nodes[(el * DIM + d) * Q + k]
                                  : map_node(alpha[d], a.ref_nodes[k], a.K, P, a.knots);
    double vals[m], ders[m];
    cox_de_boor_ool<P>(alpha[d], x, a.K, vals, ders, a.knots);
    for (int r = 0; r < m; ++r) {
      tabs[((d * 2 + 0) * m + r) * Q + k] = vals[r];
      tabs[((d * 2 + 1) * m + r) * Q + k] = ders[r];
    }
  }
  for (int u = threadIdx.x; u < DIM * Q; u += blockDim.x)
    w[u] = a.elem_weights ? a.elem_weights[el * DIM * Q + u]
                          : axis_w(a.weights, a.wt, alpha[u / Q], u % Q, Q);
  __syncthreads();
  const double* w0 = w;
  const double* w1 = w + Q;
  const double* w2 = w + (DIM - 1) * Q;
  const double* coef = nullptr;
  if (a.elem_coef) {
    coef = a.elem_coef + el * nq;
  } else if (a.coef) {
    int64_t eid = DIM == 3 ? ((int64_t)alpha[0] * a.K + alpha[1]) * a.K + alpha[2]
                           : (int64_t)alpha[0] * a.K + alpha[1];
    coef = a.coef + eid * nq;
  }
  const bool scal = a.coef == nullptr && a.coef_scalar != 1.0;
  int terms[4], nterm = 0;
  if (a.op == IGA_OP_MASS) {
    terms[nterm++] = DIM;
  } else {
    for (int d = 0; d < DIM; ++d) terms[nterm++] = d;
    if (a.op == IGA_OP_STIFFNESS_MASS) terms[nterm++] = DIM;
  }
  double* out = a.out + el * n * n;
  constexpr int npairs = n * (n + 1) / 2;
  for (int ti = 0; ti < nterm; ++ti) {
    const int term = terms[ti];
    const double* b0 = tabs + ((0 * 2 + (term == 0)) * m) * Q;
    const double* b1 = tabs + ((1 * 2 + (term == 1)) * m) * Q;
    const double* b2 = DIM == 3 ? tabs + ((2 * 2 + (term == 2)) * m) * Q : b1;
    if (a.method == IGA_METHOD_CLASSICAL) {
      for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
        // canonical pair t -> (row >= col), row-major lower triangle (integrators.py:69-74)
        int row = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
        while (row * (row + 1) / 2 > t) --row;
        while ((row + 1) * (row + 2) / 2 <= t) ++row;
        const int col = t - row * (row + 1) / 2;
        double acc = 0.0;
        if (DIM == 3) {
          const int i1 = row / (m * m), i2 = (row / m) % m, i3 = row % m;
          const int j1 = col / (m * m), j2 = (col / m) % m, j3 = col % m;
#pragma unroll 1
          for (int k1 = 0; k1 < Q; ++k1)
#pragma unroll 1
            for (int k2 = 0; k2 < Q; ++k2)
              for (int k3 = 0; k3 < Q; ++k3) {
                double v = mul(b0[i1 * Q + k1], b0[j1 * Q + k1]);
                v = mul(v, b1[i2 * Q + k2]);
                v = mul(v, b1[j2 * Q + k2]);
                v = mul(v, b2[i3 * Q + k3]);
                v = mul(v, b2[j3 * Q + k3]);
                v = mul(v, w0[k1]);
                v = mul(v, w1[k2]);
                v = mul(v, w2[k3]);
                v = mul(v, a.jac);
                if (coef) v = mul(v, coef[(k1 * Q + k2) * Q + k3]);
                else if (scal) v = mul(v, a.coef_scalar);
                acc = add(acc, v);
              }
        } else {
          const int i1 = row / m, i2 = row % m, j1 = col / m, j2 = col % m;
#pragma unroll 1
          for (int k1 = 0; k1 < Q; ++k1)
            for (int k2 = 0; k2 < Q; ++k2) {
              double v = mul(b0[i1 * Q + k1], b0[j1 * Q + k1]);
              v = mul(v, b1[i2 * Q + k2]);
              v = mul(v, b1[j2 * Q + k2]);
              v = mul(v, w0[k1]);
              v = mul(v, w1[k2]);
              v = mul(v, a.jac);
              if (coef) v = mul(v, coef[k1 * Q + k2]);
              else if (scal) v = mul(v, a.coef_scalar);
              acc = add(acc, v);
            }
        }
        if (ti == 0) {
          out[row * n + col] = acc;
          out[col * n + row] = acc;
        } else {
          const double s = add(out[row * n + col], acc);
          out[row * n + col] = s;
          out[col * n + row] = s;
        }
      }
    } else {
      // stage 1: D[i1][j1][k2][k3] = sum_k1 b0 b0 w jac [c]   (integrators.py:120-126)
      constexpr int nD = DIM == 3 ? m * m * Q * Q : m * m * Q;
      for (int t = threadIdx.x; t < nD; t += blockDim.x) {
        int i1, j1, k2, k3 = 0;
        if (DIM == 3) {
          k3 = t % Q; k2 = (t / Q) % Q; j1 = (t / (Q * Q)) % m; i1 = t / (Q * Q * m);
        } else {
          k2 = t % Q; j1 = (t / Q) % m; i1 = t / (Q * m);
        }
        double acc = 0.0;
        for (int k1 = 0; k1 < Q; ++k1) {
          double v = mul(mul(mul(b0[i1 * Q + k1], b0[j1 * Q + k1]), w0[k1]), a.jac);
          if (coef) v = mul(v, DIM == 3 ? coef[(k1 * Q + k2) * Q + k3] : coef[k1 * Q + k2]);
          else if (scal) v = mul(v, a.coef_scalar);
          acc = add(acc, v);
        }
        Dbuf[t] = acc;
      }
      __syncthreads();
      if (DIM == 3) {
        // stage 2: C[i2][i1][j2][j1][k3] = sum_k2 b1 b1 D w   (integrators.py:128-136)
        constexpr int nC = m * m * m * m * Q;
        for (int t = threadIdx.x; t < nC; t += blockDim.x) {
          const int k3 = t % Q, j1 = (t / Q) % m, j2 = (t / (Q * m)) % m;
          const int i1 = (t / (Q * m * m)) % m, i2 = t / (Q * m * m * m);
          double acc = 0.0;
          for (int k2 = 0; k2 < Q; ++k2)
            acc = add(acc, mul(mul(mul(b1[i2 * Q + k2], b1[j2 * Q + k2]),
                                   Dbuf[((i1 * m + j1) * Q + k2) * Q + k3]),
                               w1[k2]));
          Cbuf[t] = acc;
        }
        __syncthreads();
      }
      // stage 3 (2D: stage 2) for canonical pairs, mirrored (integrators.py:138-151)
      for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
        int row = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
        while (row * (row + 1) / 2 > t) --row;
        while ((row + 1) * (row + 2) / 2 <= t) ++row;
        const int col = t - row * (row + 1) / 2;
        double acc = 0.0;
        if (DIM == 3) {
          const int i1 = row / (m * m), i2 = (row / m) % m, i3 = row % m;
          const int j1 = col / (m * m), j2 = (col / m) % m, j3 = col % m;
          const double* Cp = Cbuf + (((i2 * m + i1) * m + j2) * m + j1) * Q;
          for (int k3 = 0; k3 < Q; ++k3)
            acc = add(acc, mul(mul(mul(b2[i3 * Q + k3], b2[j3 * Q + k3]), Cp[k3]), w2[k3]));
        } else {
          const int i1 = row / m, i2 = row % m, j1 = col / m, j2 = col % m;
          const double* Dp = Dbuf + (i1 * m + j1) * Q;
          for (int k2 = 0; k2 < Q; ++k2)
            acc = add(acc, mul(mul(mul(b1[i2 * Q + k2], b1[j2 * Q + k2]), Dp[k2]), w1[k2]));
        }
        if (ti == 0) {
          out[row * n + col] = acc;
          out[col * n + row] = acc;
        } else {
          const double s = add(out[row * n + col], acc);
          out[row * n + col] = s;
          out[col * n + row] = s;
        }
      }
    }
    __syncthreads();
  }
}

template <int P, int Q>
struct ElementStrictLaunch {
  static int run(const ElemArgs& a0, cudaStream_t s) {
    constexpr int m = P + 1;
    if (a0.count == 0) return IGA_OK;
    if (a0.count > 0x7fffffff) return fail_einval("too many elements");
    if (a0.dim == 2) {
      const size_t shm = sizeof(double) * (2 * 2 * m * Q + 2 * Q + m * m * Q * Q);
      if (shm > 48 * 1024) {
        cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(k_element_strict<2, P, Q>), shm);
        if (e != cudaSuccess) return check_cuda(e, "element smem attr");
      }
      k_element_strict<2, P, Q><<<(unsigned)a0.count, 256, shm, s>>>(a0);
      return check_cuda(cudaGetLastError(), "iga_element_matrices launch");
    }
    constexpr size_t stage = (size_t)m * m * Q * Q + (size_t)m * m * m * m * Q;  // D + C doubles
    constexpr size_t base = 3 * 2 * m * Q + 3 * Q;
    const bool global = a0.method == IGA_METHOD_SUMFACT && sizeof(double) * (base + stage) > 200 * 1024;
    const size_t shm = sizeof(double) * (global || a0.method != IGA_METHOD_SUMFACT ? base : base + stage);
    if (shm > 48 * 1024) {
      cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(k_element_strict<3, P, Q>), shm);
      if (e != cudaSuccess) return check_cuda(e, "element smem attr");
    }
    if (!global) {
      k_element_strict<3, P, Q><<<(unsigned)a0.count, 256, shm, s>>>(a0);
      return check_cuda(cudaGetLastError(), "iga_element_matrices launch");
    }
    // high degrees: the m^4 Q stage buffer of every CTA in stream-ordered global scratch
    // (cudaMallocAsync: graph-capturable, freed in stream order), chunks of <= 256 elements
    constexpr int64_t kChunk = 256;
    const int64_t chunk = a0.count < kChunk ? a0.count : kChunk;
    double* scratch = nullptr;
    int rc = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                                        sizeof(double) * stage * chunk, s), "element scratch");
    if (rc) return rc;
    constexpr int n = m * m * m, nq = Q * Q * Q;
    for (int64_t off = 0; off < a0.count && !rc; off += chunk) {
      ElemArgs a = a0;
      a.count = a0.count - off < chunk ? a0.count - off : chunk;
      a.elem_ids = a0.elem_ids + off * 3;
      if (a0.elem_nodes) a.elem_nodes = a0.elem_nodes + off * 3 * Q;
      if (a0.elem_weights) a.elem_weights = a0.elem_weights + off * 3 * Q;
      if (a0.elem_coef) a.elem_coef = a0.elem_coef + off * nq;
      a.out = a0.out + off * (int64_t)n * n;
      a.scratch = scratch;
      k_element_strict<3, P, Q><<<(unsigned)a.count, 256, shm, s>>>(a);
      rc = check_cuda(cudaGetLastError(), "iga_element_matrices launch");
    }
    const int rf = check_cuda(cudaFreeAsync(scratch, s), "element scratch free");
    return rc ? rc : rf;
  }
};

int launch_element_strict(const ElemArgs& a, int p, int q, cudaStream_t s) {
  return dispatch_pq_all<ElementStrictLaunch>(p, q, a, s);
}

}  // namespace iga

using namespace iga;

extern "C" int32_t iga_element_matrices(const iga_problem* prob, int32_t method,
                                        const double* ref_nodes, const int32_t* elem_ids,
                                        const double* elem_nodes, const double* elem_weights,
                                        const double* elem_coef, int64_t count, double* out,
                                        void* stream) {
  if (!prob) return fail_einval("null problem");
  if (prob->dim != 2 && prob->dim != 3) return fail_einval("dim must be 2 or 3");
  if (prob->K < 1 || prob->p < 0) return fail_einval("mesh must be >= 1 and degree >= 0");
  if (prob->op < 0 || prob->op > 2) return fail_einval("unknown operator %d", prob->op);
  if (prob->op != IGA_OP_MASS && prob->p < 1) return fail_einval("derivatives require degree >= 1");
  if (method != IGA_METHOD_CLASSICAL && method != IGA_METHOD_SUMFACT)
    return fail_einval("element matrices: method must be classical or sumfact");
  if (count < 0) return fail_einval("negative count");
  if (count > 0 && (!elem_ids || !out || !prob->weights || (!elem_nodes && !ref_nodes)))
    return fail_einval("null pointer");
  ElemArgs a;
  a.dim = prob->dim; a.K = prob->K; a.q = prob->q; a.op = prob->op; a.method = method;
  a.jac = prob->jac; a.coef_scalar = prob->coef_scalar; a.coef = prob->coef;
  a.knots = prob->knots; a.wt = prob->knots ? prob->elem_weights : nullptr;
  if (prob->knots && !elem_weights && !prob->elem_weights)
    return fail_einval("a general knot vector needs elem_weights (iga_mesh_tables_general)");
  a.weights = prob->weights; a.ref_nodes = ref_nodes; a.elem_ids = elem_ids;
  a.elem_nodes = elem_nodes; a.elem_weights = elem_weights; a.elem_coef = elem_coef;
  a.count = count; a.out = out; a.scratch = nullptr;
  return launch_element_strict(a, prob->p, prob->q, as_stream(stream));
}
