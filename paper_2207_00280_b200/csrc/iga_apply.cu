// Matrix-free operator application y = alpha M x + beta S x:
// the element quadrature of the assembled operators applied to a coefficient
// vector without forming the matrix, by sum factorization -- the device version of
// heat.HeatProblem.assemble_rhs (heat.py:131-158: field values and gradients at
// the Gauss points by per-axis contractions, weighted, then the transposed
// contractions, scattered into the result).
//
// One CTA per element (grid-stride).  Forward: x_e (m^3) -> u, du/dx0, du/dx1,
// du/dx2 at the q^3 points (three axis contractions, value and derivative tables).
// Pointwise: f = W (alpha u, beta grad u), W = w w w jac c.  Backward: the
// transposed contractions, then an atomicAdd of the m^3 element result into y.
#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

struct ApplyArgs {
  int K;
  double alpha, beta, jac, coef_scalar;
  const double* coef;
  const double* weights;
  const double* V;
  const double* D;
  const double* x;
  double* y;
};

template <int P, int Q>
__global__ void __launch_bounds__(128) k_apply3(ApplyArgs a) {
  constexpr int m = P + 1;
  __shared__ double sx[m * m * m];
  __shared__ double t0[m][m][Q], t1[m][m][Q];                  // axis-2 contractions
  __shared__ double u0[m][Q][Q], u1[m][Q][Q], u2[m][Q][Q];     // axis-1
  __shared__ double f[4][Q][Q][Q];                             // point values
  __shared__ double h0[m][Q][Q], h1[m][Q][Q], h2[m][Q][Q];     // backward axis 0
  __shared__ double j0[m][m][Q], j1[m][m][Q];                  // backward axis 1
  __shared__ double tv[3][m][Q], td[3][m][Q], w[Q];
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int64_t n_el = (int64_t)K * K * K;
  const bool stiff = a.beta != 0.0;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t el = blockIdx.x; el < n_el; el += gridDim.x) {
    const int e2 = (int)(el % K), e1 = (int)((el / K) % K), e0 = (int)(el / ((int64_t)K * K));
    const int ev[3] = {e0, e1, e2};
    __syncthreads();
    for (int u = tid; u < 3 * m * Q; u += nt) {
      const int d = u / (m * Q), rk = u % (m * Q);
      tv[d][rk / Q][rk % Q] = a.V[(int64_t)ev[d] * m * Q + rk];
      td[d][rk / Q][rk % Q] = stiff ? a.D[(int64_t)ev[d] * m * Q + rk] : 0.0;
    }
    if (tid < Q) w[tid] = a.weights[tid];
    for (int u = tid; u < m * m * m; u += nt) {
      const int i0 = u / (m * m), i1 = (u / m) % m, i2 = u % m;
      sx[u] = a.x[((int64_t)(e0 + i0) * N + e1 + i1) * N + e2 + i2];
    }
    __syncthreads();
    // forward axis 2: t0 = sum x V2, t1 = sum x D2
    for (int u = tid; u < m * m * Q; u += nt) {
      const int i0 = u / (m * Q), i1 = (u / Q) % m, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i2 = 0; i2 < m; ++i2) {
        const double xv = sx[(i0 * m + i1) * m + i2];
        s0 += xv * tv[2][i2][k2];
        s1 += xv * td[2][i2][k2];
      }
      t0[i0][i1][k2] = s0;
      t1[i0][i1][k2] = s1;
    }
    __syncthreads();
    // forward axis 1: u0 = t0 V1, u1 = t0 D1, u2 = t1 V1
    for (int u = tid; u < m * Q * Q; u += nt) {
      const int i0 = u / (Q * Q), k1 = (u / Q) % Q, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < m; ++i1) {
        s0 += t0[i0][i1][k2] * tv[1][i1][k1];
        s1 += t0[i0][i1][k2] * td[1][i1][k1];
        s2 += t1[i0][i1][k2] * tv[1][i1][k1];
      }
      u0[i0][k1][k2] = s0;
      u1[i0][k1][k2] = s1;
      u2[i0][k1][k2] = s2;
    }
    __syncthreads();
    // forward axis 0 + pointwise weights: f0 = W a u, f1..3 = W b du/dx_d
    for (int u = tid; u < Q * Q * Q; u += nt) {
      const int k0 = u / (Q * Q), k1 = (u / Q) % Q, k2 = u % Q;
      double val = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < m; ++i0) {
        val += u0[i0][k1][k2] * tv[0][i0][k0];
        g0 += u0[i0][k1][k2] * td[0][i0][k0];
        g1 += u1[i0][k1][k2] * tv[0][i0][k0];
        g2 += u2[i0][k1][k2] * tv[0][i0][k0];
      }
      double W = w[k0] * w[k1] * w[k2] * a.jac;
      W *= a.coef ? a.coef[el * (Q * Q * Q) + u] : a.coef_scalar;
      f[0][k0][k1][k2] = W * a.alpha * val;
      f[1][k0][k1][k2] = W * a.beta * g0;
      f[2][k0][k1][k2] = W * a.beta * g1;
      f[3][k0][k1][k2] = W * a.beta * g2;
    }
    __syncthreads();
    // backward axis 0: h0 = V0 f0 + D0 f1 (pairs with V1 V2), h1 = V0 f2 (D1 V2), h2 = V0 f3 (V1 D2)
    for (int u = tid; u < m * Q * Q; u += nt) {
      const int i0 = u / (Q * Q), k1 = (u / Q) % Q, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < Q; ++k0) {
        s0 += tv[0][i0][k0] * f[0][k0][k1][k2] + td[0][i0][k0] * f[1][k0][k1][k2];
        s1 += tv[0][i0][k0] * f[2][k0][k1][k2];
        s2 += tv[0][i0][k0] * f[3][k0][k1][k2];
      }
      h0[i0][k1][k2] = s0;
      h1[i0][k1][k2] = s1;
      h2[i0][k1][k2] = s2;
    }
    __syncthreads();
    // backward axis 1: j0 = V1 h0 + D1 h1 (pairs with V2), j1 = V1 h2 (D2)
    for (int u = tid; u < m * m * Q; u += nt) {
      const int i0 = u / (m * Q), i1 = (u / Q) % m, k2 = u % Q;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) {
        s0 += tv[1][i1][k1] * h0[i0][k1][k2] + td[1][i1][k1] * h1[i0][k1][k2];
        s1 += tv[1][i1][k1] * h2[i0][k1][k2];
      }
      j0[i0][i1][k2] = s0;
      j1[i0][i1][k2] = s1;
    }
    __syncthreads();
    // backward axis 2 and scatter
    for (int u = tid; u < m * m * m; u += nt) {
      const int i0 = u / (m * m), i1 = (u / m) % m, i2 = u % m;
      double s = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) s += tv[2][i2][k2] * j0[i0][i1][k2] + td[2][i2][k2] * j1[i0][i1][k2];
      atomicAdd(a.y + ((int64_t)(e0 + i0) * N + e1 + i1) * N + e2 + i2, s);
    }
  }
}

template <int P, int Q>
struct ApplyLaunch {
  static int run(const ApplyArgs& a, cudaStream_t s) {
    const int64_t n_el = (int64_t)a.K * a.K * a.K;
    const int64_t grid = n_el < 148 * 16 ? n_el : 148 * 16;
    k_apply3<P, Q><<<(unsigned)grid, 128, 0, s>>>(a);
    return check_cuda(cudaGetLastError(), "iga_apply launch");
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
  int rc = check_cuda(cudaMemsetAsync(y, 0, sizeof(double) * N * N * N, s), "zero y");
  if (rc) return rc;
  ApplyArgs a;
  a.K = prob->K; a.alpha = alpha; a.beta = beta; a.jac = prob->jac;
  a.coef_scalar = prob->coef_scalar; a.coef = prob->coef; a.weights = prob->weights;
  a.V = prob->tables_v; a.D = prob->tables_d; a.x = x; a.y = y;
  return dispatch_pq<ApplyLaunch>(prob->p, prob->q, a, s);
}
