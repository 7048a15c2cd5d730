// Matrix-free operator application y = alpha M x + beta S x:
// the element quadrature of the assembled operators applied to a coefficient
// vector without forming the matrix, by sum factorization -- the device version of
// heat.HeatProblem.assemble_rhs (heat.py:131-158: field values and gradients at
// the Gauss points by per-axis contractions, weighted, then the transposed
// contractions, scattered into the result).
//
// Per element: forward x_e (m^3) -> u, du/dx0, du/dx1, du/dx2 at the q^3 points
// (three axis contractions, value and derivative tables); pointwise f = W (alpha u,
// beta grad u), W = w w w jac c; backward: the transposed contractions, then
// atomicAdd of the element result into y.  A CTA runs a batch of E elements.
#include "iga_args.cuh"
#include "iga_band.cuh"
#include "iga_dispatch.cuh"

namespace iga {

struct ApplyArgs {
  int K;
  double alpha, beta, jac, coef_scalar;
  const double* wt;  // [K][Q] per-element weights (general knots), or null
  const double* coef;
  const double* weights;
  const double* V;
  const double* D;
  const double* x;
  double* y;
};

// E consecutive elements along the fastest axis per CTA (they share the axis-0/1
// tables and overlap in their dof windows): every stage runs over the E elements at
// once (fewer barriers per element), and the backward axis-2 contraction sums the
// batch's contributions per dof in shared memory, so only (E+P) m^2 atomics leave
// the CTA instead of E m^3.
template <int P, int Q, int E>
__global__ void __launch_bounds__(256, 4) k_apply3(ApplyArgs a) {
  constexpr int m = P + 1, W2 = E + P;  // dof window of the batch along axis 2
  __shared__ double sx[m][m][W2];
  __shared__ double t0[E][m][m][Q], t1[E][m][m][Q];               // axis-2 contractions
  __shared__ double u0[E][m][Q][Q], u1[E][m][Q][Q], u2[E][m][Q][Q];  // axis-1
  __shared__ double f[4][E][Q][Q][Q];                              // point values
  __shared__ double h0[E][m][Q][Q], h1[E][m][Q][Q], h2[E][m][Q][Q];  // backward axis 0
  __shared__ double j0[E][m][m][Q], j1[E][m][m][Q];               // backward axis 1
  __shared__ double tv01[2][m][Q], td01[2][m][Q], tv2[E][m][Q], td2[E][m][Q], w[Q];
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int nb = (K + E - 1) / E;  // batches along axis 2
  const int64_t n_batch = (int64_t)K * K * nb;
  const bool stiff = a.beta != 0.0;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t bt = blockIdx.x; bt < n_batch; bt += gridDim.x) {
    const int eb = (int)(bt % nb) * E, e1 = (int)((bt / nb) % K), e0 = (int)(bt / ((int64_t)nb * K));
    const int ne = min(E, K - eb);  // elements in this batch
    __syncthreads();
    for (int u = tid; u < 2 * m * Q; u += nt) {
      const int d = u / (m * Q), rk = u % (m * Q);
      const int64_t e = d == 0 ? e0 : e1;
      tv01[d][rk / Q][rk % Q] = a.V[e * m * Q + rk];
      td01[d][rk / Q][rk % Q] = stiff ? a.D[e * m * Q + rk] : 0.0;
    }
    for (int u = tid; u < E * m * Q; u += nt) {
      const int b = u / (m * Q), rk = u % (m * Q);
      const bool ok = b < ne;
      tv2[b][rk / Q][rk % Q] = ok ? a.V[(int64_t)(eb + b) * m * Q + rk] : 0.0;
      td2[b][rk / Q][rk % Q] = ok && stiff ? a.D[(int64_t)(eb + b) * m * Q + rk] : 0.0;
    }
    if (tid < Q) w[tid] = a.weights[tid];
    for (int u = tid; u < m * m * W2; u += nt) {
      const int i0 = u / (m * W2), i1 = (u / W2) % m, z = u % W2;
      sx[i0][i1][z] = eb + z < N ? a.x[((int64_t)(e0 + i0) * N + e1 + i1) * N + eb + z] : 0.0;
    }
    __syncthreads();
    // forward axis 2: t0 = sum x V2, t1 = sum x D2
    for (int u = tid; u < E * m * m * Q; u += nt) {
      const int b = u / (m * m * Q), i0 = (u / (m * Q)) % m, i1 = (u / Q) % m, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i2 = 0; i2 < m; ++i2) {
        const double xv = sx[i0][i1][b + i2];
        s0 += xv * tv2[b][i2][k2];
        s1 += xv * td2[b][i2][k2];
      }
      t0[b][i0][i1][k2] = s0;
      t1[b][i0][i1][k2] = s1;
    }
    __syncthreads();
    // forward axis 1: u0 = t0 V1, u1 = t0 D1, u2 = t1 V1
    for (int u = tid; u < E * m * Q * Q; u += nt) {
      const int b = u / (m * Q * Q), i0 = (u / (Q * Q)) % m, k1 = (u / Q) % Q, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < m; ++i1) {
        s0 += t0[b][i0][i1][k2] * tv01[1][i1][k1];
        s1 += t0[b][i0][i1][k2] * td01[1][i1][k1];
        s2 += t1[b][i0][i1][k2] * tv01[1][i1][k1];
      }
      u0[b][i0][k1][k2] = s0;
      u1[b][i0][k1][k2] = s1;
      u2[b][i0][k1][k2] = s2;
    }
    __syncthreads();
    // forward axis 0 + pointwise weights: f0 = W a u, f1..3 = W b du/dx_d
    for (int u = tid; u < E * Q * Q * Q; u += nt) {
      const int b = u / (Q * Q * Q), k = u % (Q * Q * Q);
      const int k0 = k / (Q * Q), k1 = (k / Q) % Q, k2 = k % Q;
      double val = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < m; ++i0) {
        val += u0[b][i0][k1][k2] * tv01[0][i0][k0];
        g0 += u0[b][i0][k1][k2] * td01[0][i0][k0];
        g1 += u1[b][i0][k1][k2] * tv01[0][i0][k0];
        g2 += u2[b][i0][k1][k2] * tv01[0][i0][k0];
      }
      double Wt = 0.0;
      if (b < ne) {
        Wt = axis_w(w, a.wt, e0, k0, Q) * axis_w(w, a.wt, e1, k1, Q) * axis_w(w, a.wt, eb + b, k2, Q) *
             a.jac;
        const int64_t el = ((int64_t)e0 * K + e1) * K + eb + b;
        Wt *= a.coef ? a.coef[el * (Q * Q * Q) + k] : a.coef_scalar;
      }
      f[0][b][k0][k1][k2] = Wt * a.alpha * val;
      f[1][b][k0][k1][k2] = Wt * a.beta * g0;
      f[2][b][k0][k1][k2] = Wt * a.beta * g1;
      f[3][b][k0][k1][k2] = Wt * a.beta * g2;
    }
    __syncthreads();
    // backward axis 0: h0 = V0 f0 + D0 f1 (pairs with V1 V2), h1 = V0 f2 (D1 V2), h2 = V0 f3 (V1 D2)
    for (int u = tid; u < E * m * Q * Q; u += nt) {
      const int b = u / (m * Q * Q), i0 = (u / (Q * Q)) % m, k1 = (u / Q) % Q, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < Q; ++k0) {
        s0 += tv01[0][i0][k0] * f[0][b][k0][k1][k2] + td01[0][i0][k0] * f[1][b][k0][k1][k2];
        s1 += tv01[0][i0][k0] * f[2][b][k0][k1][k2];
        s2 += tv01[0][i0][k0] * f[3][b][k0][k1][k2];
      }
      h0[b][i0][k1][k2] = s0;
      h1[b][i0][k1][k2] = s1;
      h2[b][i0][k1][k2] = s2;
    }
    __syncthreads();
    // backward axis 1: j0 = V1 h0 + D1 h1 (pairs with V2), j1 = V1 h2 (D2)
    for (int u = tid; u < E * m * m * Q; u += nt) {
      const int b = u / (m * m * Q), i0 = (u / (m * Q)) % m, i1 = (u / Q) % m, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) {
        s0 += tv01[1][i1][k1] * h0[b][i0][k1][k2] + td01[1][i1][k1] * h1[b][i0][k1][k2];
        s1 += tv01[1][i1][k1] * h2[b][i0][k1][k2];
      }
      j0[b][i0][i1][k2] = s0;
      j1[b][i0][i1][k2] = s1;
    }
    __syncthreads();
    // backward axis 2, summed over the batch's elements per dof, then one atomic per dof
    for (int u = tid; u < m * m * W2; u += nt) {
      const int i0 = u / (m * W2), i1 = (u / W2) % m, z = u % W2;
      if (eb + z >= N) continue;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < E; ++b) {
        const int i2 = z - b;
        if (b < ne && i2 >= 0 && i2 < m) {
#pragma unroll
          for (int k2 = 0; k2 < Q; ++k2) s += tv2[b][i2][k2] * j0[b][i0][i1][k2] + td2[b][i2][k2] * j1[b][i0][i1][k2];
        }
      }
      atomicAdd(a.y + ((int64_t)(e0 + i0) * N + e1 + i1) * N + eb + z, s);
    }
  }
}

// static shared memory of k_apply3<P,Q,E> in doubles (must stay under 48 KB)
constexpr int apply_smem(int P, int Q, int E) {
  return (P + 1) * (P + 1) * (E + P) + 4 * E * (P + 1) * (P + 1) * Q + 6 * E * (P + 1) * Q * Q +
         4 * E * Q * Q * Q + 4 * (P + 1) * Q + 2 * E * (P + 1) * Q + Q;
}
constexpr int apply_batch(int P, int Q) {
  return apply_smem(P, Q, 4) * 8 <= 48 * 1024 ? 4 : (apply_smem(P, Q, 2) * 8 <= 48 * 1024 ? 2 : 1);
}

template <int P, int Q>
struct ApplyLaunch {
  static int run(const ApplyArgs& a, cudaStream_t s) {
    constexpr int E = apply_batch(P, Q);
    const int64_t n_batch = (int64_t)a.K * a.K * ((a.K + E - 1) / E);
    const int64_t cap = (int64_t)sm_count() * 8;
    const int64_t grid = n_batch < cap ? n_batch : cap;
    k_apply3<P, Q, E><<<(unsigned)grid, 256, 0, s>>>(a);
    return check_cuda(cudaGetLastError(), "iga_apply launch");
  }
};

// Scalar coefficient: the operator is a sum of Kronecker products of 1D band matrices
// (iga_kron.cu header),  y = cj [ (alpha m0 + beta k0) c + beta m0 (k1 a + m1 b) ]
// with a = m2 x, b = k2 x, c = m1 a (each a 2P+1-point stencil along one axis), so
// y costs ~7 (2P+1) flops per dof instead of an element-by-element quadrature.
// One CTA per T0 x T1 block of (I0, I1) dof lines, the lines swept in z-chunks of
// ZC dofs; the x window (with a P halo on every side) and the intermediates live in
// shared memory, and every y value is written once by its owner (no atomics).
constexpr int AK_T = 4, AK_ZC = 32;

template <int P>
__host__ __device__ constexpr int apply_kron_work(int) {
  return (AK_T + 2 * P) * (AK_T + 2 * P) * (AK_ZC + 2 * P) +      // X
         2 * (AK_T + 2 * P) * (AK_T + 2 * P) * AK_ZC +           // (a, b)
         2 * (AK_T + 2 * P) * AK_T * AK_ZC;                      // (c, de)
}

template <int P, int Q>
__global__ void __launch_bounds__(256) k_apply_kron(ApplyArgs a) {
  constexpr int NB = 2 * P + 1, T = AK_T, W = T + 2 * P, ZC = AK_ZC, ZH = ZC + 2 * P;
  extern __shared__ __align__(16) double2 tb[];  // [N][NB] (m, k), then the work area
  __shared__ double w_s[Q];
  const int K = a.K, tid = threadIdx.x, nt = blockDim.x;
  const int N = K + P;
  const bool stiff = a.beta != 0.0;
  double* work = reinterpret_cast<double*>(tb + N * NB);
  double* X = work;                                        // [W][W][ZH]
  double2* AB = reinterpret_cast<double2*>(X + W * W * ZH);  // [W][W][ZC]
  double2* CD = AB + W * W * ZC;                           // [W][T][ZC]
  build_band_tables<P, Q>(a.V, a.D, a.weights, K, stiff, 0, K, false, tb, work,
                          apply_kron_work<P>(0), w_s, tid, nt, a.wt);
  const double cj = a.jac * a.coef_scalar;
  const int nblk = (N + T - 1) / T;
  for (int blk = blockIdx.x; blk < nblk * nblk; blk += gridDim.x) {
    const int i0 = (blk / nblk) * T, j0 = (blk % nblk) * T;
    for (int z0 = 0; z0 < N; z0 += ZC) {
      __syncthreads();  // previous chunk's CD / X consumed
      for (int u = tid; u < W * W * ZH; u += nt) {
        const int w0 = u / (W * ZH), w1 = (u / ZH) % W, zz = u % ZH;
        const int I0 = i0 - P + w0, I1 = j0 - P + w1, I2 = z0 - P + zz;
        X[u] = (I0 >= 0 && I0 < N && I1 >= 0 && I1 < N && I2 >= 0 && I2 < N)
                   ? a.x[((int64_t)I0 * N + I1) * N + I2]
                   : 0.0;
      }
      __syncthreads();
      // axis 2: a = m2 x, b = k2 x
      for (int u = tid; u < W * W * ZC; u += nt) {
        const int wl = u / ZC, z = u % ZC;
        const double2* t = tb + min(z0 + z, N - 1) * NB;
        const double* xl = X + wl * ZH + z;
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int d = 0; d < NB; ++d) {
          sa += t[d].x * xl[d];
          sb += t[d].y * xl[d];
        }
        AB[u] = make_double2(sa, sb);
      }
      __syncthreads();
      // axis 1: c = m1 a, de = k1 a + m1 b
      for (int u = tid; u < W * T * ZC; u += nt) {
        const int w0 = u / (T * ZC), o1 = (u / ZC) % T, z = u % ZC;
        const double2* t = tb + min(j0 + o1, N - 1) * NB;
        const double2* ab = AB + (w0 * W + o1) * ZC + z;
        double sc = 0.0, sd = 0.0;
#pragma unroll
        for (int d = 0; d < NB; ++d) {
          const double2 v = ab[d * ZC];
          sc += t[d].x * v.x;
          sd += t[d].y * v.x + t[d].x * v.y;
        }
        CD[u] = make_double2(sc, sd);
      }
      __syncthreads();
      // axis 0 and the output
      for (int u = tid; u < T * T * ZC; u += nt) {
        const int o0 = u / (T * ZC), o1 = (u / ZC) % T, z = u % ZC;
        const int I0 = i0 + o0, I1 = j0 + o1, I2 = z0 + z;
        if (I0 >= N || I1 >= N || I2 >= N) continue;
        const double2* t = tb + I0 * NB;
        const double2* cd = CD + (o0 * T + o1) * ZC + z;
        double sy = 0.0;
#pragma unroll
        for (int d = 0; d < NB; ++d) {
          const double2 v = cd[d * T * ZC];
          sy += (a.alpha * t[d].x + a.beta * t[d].y) * v.x + a.beta * t[d].x * v.y;
        }
        a.y[((int64_t)I0 * N + I1) * N + I2] = cj * sy;
      }
    }
  }
}

template <int P, int Q>
struct ApplyKronLaunch {
  static int run(const ApplyArgs& a, cudaStream_t s) {
    const int N = a.K + P;
    const size_t smem = sizeof(double2) * (size_t)N * (2 * P + 1) + sizeof(double) * apply_kron_work<P>(0);
    if (smem > 220 * 1024) {
      set_error("separable apply: 1D band tables of K=%d do not fit shared memory", a.K);
      return IGA_EUNSUPPORTED;
    }
    const void* fn = reinterpret_cast<const void*>(k_apply_kron<P, Q>);
    cudaError_t e = smem_attr_once(fn, smem, true);
    if (e != cudaSuccess) return check_cuda(e, "apply smem attr");
    const int nblk = (N + AK_T - 1) / AK_T;
    const int64_t slots = (int64_t)sm_count() * blocks_per_sm_once(fn, 256, smem);
    const int64_t grid = (int64_t)nblk * nblk < slots ? (int64_t)nblk * nblk : slots;
    k_apply_kron<P, Q><<<(unsigned)grid, 256, smem, s>>>(a);
    return check_cuda(cudaGetLastError(), "iga_apply (separable) launch");
  }
};

}  // namespace iga

using namespace iga;

extern "C" int32_t iga_apply(const iga_problem* prob, double alpha, double beta, const double* x,
                             double* y, void* stream) {
  if (!prob) return fail_einval("null problem");
  if (prob->dim != 3) return fail_einval("matrix-free application is implemented for dim=3");
  if (prob->K < 1 || prob->p < 0 || prob->q < 1) return fail_einval("bad mesh/degree/points");
  if (beta != 0.0 && (prob->p < 1 || !prob->tables_d)) return fail_einval("stiffness needs p >= 1 and tables_d");
  if (!prob->weights || !prob->tables_v || !x || !y) return fail_einval("null pointer");
  const int64_t N = (int64_t)prob->K + prob->p;
  cudaStream_t s = as_stream(stream);
  ApplyArgs a;
  if (prob->knots && !prob->elem_weights)
    return fail_einval("a general knot vector needs elem_weights (iga_mesh_tables_general)");
  a.K = prob->K; a.alpha = alpha; a.beta = beta; a.jac = prob->jac;
  a.wt = prob->knots ? prob->elem_weights : nullptr;
  a.coef_scalar = prob->coef_scalar; a.coef = prob->coef; a.weights = prob->weights;
  a.V = prob->tables_v; a.D = prob->tables_d; a.x = x; a.y = y;
  if (!prob->coef) {  // scalar coefficient: separable operator, y written once per dof
    const int rc = dispatch_pq<ApplyKronLaunch>(prob->p, prob->q, a, s);
    if (rc != IGA_EUNSUPPORTED) return rc;  // (too large for the shared-memory tables)
  }
  int rc = check_cuda(cudaMemsetAsync(y, 0, sizeof(double) * N * N * N, s), "zero y");
  if (rc) return rc;
  return dispatch_pq<ApplyLaunch>(prob->p, prob->q, a, s);
}
