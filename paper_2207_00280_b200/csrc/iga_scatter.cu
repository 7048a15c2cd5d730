// Element-local mesh-wide kernels with fused atomic scatter (see iga_element.cu header).
//
//  * k_element_strict  -- per-element matrices with the reference's exact
//    operation order (strict IEEE via __dmul_rn/__dadd_rn): classical =
//    integrators.py:77-109, sum factorization = integrators.py:112-151.
//    Bitwise equal to the numba kernels for the mass operator; stiffness =
//    the same kernels once per axis with derivative tables, summed in axis
//    order (oracle/iga_oracle.c orc_element defines the same order).
//  * k_classical_scatter -- Algorithm 1 mesh-wide: grid over elements, warps
//    over canonical pairs, lanes over quadrature points, warp-shuffle
//    reduction, fused atomic scatter into the structured CSR.
//  * k_sumfact_scatter -- Algorithm 2 element-local, stages in shared memory
//    (Foata classes p+1..p+6 of taskgraph.py:204-223 -> barrier phases),
//    fused atomic scatter.
#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

// --------------------------------------------------------- fused scatter
__device__ __forceinline__ void scatter_add(const ScatterArgs& a, int P, int64_t N,
                                            const int64_t* I, const int64_t* J, double v) {
  int64_t row;
  if (a.dim == 3) row = (I[0] * N + I[1]) * N + I[2];
  else row = I[0] * N + I[1];
  if (row < a.row_first || row >= a.row_last) return;
  int64_t off;
  if (a.dim == 3) {
    off = rowptr3(I[0], I[1], I[2], P, N) + col_slot3(I, J, P, N);
  } else {
    off = rowptr2(I[0], I[1], P, N) + (J[0] - band_lo(I[0], P)) * band_cnt(I[1], P, N) +
          (J[1] - band_lo(I[1], P));
  }
  atomicAdd(a.values + (off - a.base), v);
}

// Algorithm 1 over the mesh.  One CTA per element (grid-stride), 8 warps over
// canonical pairs, lanes over the q^dim quadrature points, shuffle reduction.
// Per quadrature point the shared factor W = w w w jac c is formed once and
// the per-axis pair products are read from shared memory.
template <int DIM, int P, int Q>
__global__ void __launch_bounds__(256) k_classical_scatter(ScatterArgs a) {
  constexpr int m = P + 1;
  constexpr int n = DIM == 3 ? m * m * m : m * m;
  constexpr int nq = DIM == 3 ? Q * Q * Q : Q * Q;
  constexpr int npairs = n * (n + 1) / 2;
  __shared__ double sV[3][m][Q], sD[3][m][Q], sW[nq];
  const int64_t N = (int64_t)a.K + P;
  const int Kb = DIM == 3 ? a.K : 1;
  const int64_t n_el = (int64_t)(a.el_end - a.el_begin) * a.K * Kb;
  const bool stiff = a.op != IGA_OP_MASS;
  const bool with_mass = a.op != IGA_OP_STIFFNESS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t el = blockIdx.x; el < n_el; el += gridDim.x) {
    int alpha[3];
    if (DIM == 3) {
      alpha[2] = (int)(el % a.K);
      alpha[1] = (int)((el / a.K) % a.K);
      alpha[0] = a.el_begin + (int)(el / ((int64_t)a.K * a.K));
    } else {
      alpha[2] = 0;
      alpha[1] = (int)(el % a.K);
      alpha[0] = a.el_begin + (int)(el / a.K);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < DIM * m * Q; t += blockDim.x) {
      const int d = t / (m * Q), rk = t % (m * Q);
      sV[d][rk / Q][rk % Q] = a.V[(int64_t)alpha[d] * m * Q + rk];
      sD[d][rk / Q][rk % Q] = stiff ? a.D[(int64_t)alpha[d] * m * Q + rk] : 0.0;
    }
    const int64_t eid = DIM == 3 ? ((int64_t)alpha[0] * a.K + alpha[1]) * a.K + alpha[2]
                                 : (int64_t)alpha[0] * a.K + alpha[1];
    for (int t = threadIdx.x; t < nq; t += blockDim.x) {
      const int k1 = DIM == 3 ? t / (Q * Q) : t / Q;
      const int k2 = DIM == 3 ? (t / Q) % Q : t % Q;
      const int k3 = DIM == 3 ? t % Q : 0;
      double W = a.weights[k1] * a.weights[k2] * a.jac;
      if (DIM == 3) W *= a.weights[k3];
      W *= a.coef ? a.coef[eid * nq + t] : a.coef_scalar;
      sW[t] = W;
    }
    __syncthreads();
    for (int t = warp; t < npairs; t += blockDim.x >> 5) {
      int row = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
      while (row * (row + 1) / 2 > t) --row;
      while ((row + 1) * (row + 2) / 2 <= t) ++row;
      const int col = t - row * (row + 1) / 2;
      int ri[3], ci[3];
      if (DIM == 3) {
        ri[0] = row / (m * m); ri[1] = (row / m) % m; ri[2] = row % m;
        ci[0] = col / (m * m); ci[1] = (col / m) % m; ci[2] = col % m;
      } else {
        ri[0] = row / m; ri[1] = row % m; ri[2] = 0;
        ci[0] = col / m; ci[1] = col % m; ci[2] = 0;
      }
      double acc = 0.0;
#pragma unroll 1
      for (int k = lane; k < nq; k += 32) {
        const int k1 = DIM == 3 ? k / (Q * Q) : k / Q;
        const int k2 = DIM == 3 ? (k / Q) % Q : k % Q;
        const int k3 = DIM == 3 ? k % Q : 0;
        const double v0 = sV[0][ri[0]][k1] * sV[0][ci[0]][k1];
        const double v1 = sV[1][ri[1]][k2] * sV[1][ci[1]][k2];
        const double v2 = DIM == 3 ? sV[2][ri[2]][k3] * sV[2][ci[2]][k3] : 1.0;
        double f = 0.0;
        if (stiff) {
          const double d0 = sD[0][ri[0]][k1] * sD[0][ci[0]][k1];
          const double d1 = sD[1][ri[1]][k2] * sD[1][ci[1]][k2];
          f = d0 * v1 * v2 + v0 * d1 * v2;
          if (DIM == 3) f += v0 * v1 * (sD[2][ri[2]][k3] * sD[2][ci[2]][k3]);
        }
        if (with_mass) f += v0 * v1 * v2;
        acc += f * sW[k];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        int64_t I[3], J[3];
        for (int d = 0; d < 3; ++d) {
          I[d] = alpha[d] + ri[d];
          J[d] = alpha[d] + ci[d];
        }
        scatter_add(a, P, N, I, J, acc);
        if (row != col) scatter_add(a, P, N, J, I, acc);
      }
    }
  }
}

// Algorithm 2 element-local, merged stiffness form, fused atomic scatter.
//   X_T[i1][j1][k2][k3] = sum_k1 T_i1 T_j1 W             (T in {V, D})
//   Y_A[i2 i1 j2 j1][k3] = sum_k2 X_D VV + X_V DD,  Y_B = sum_k2 X_V VV
//   S[pair] = sum_k3 Y_A VV3 + Y_B Z3  (Z3 = DD3, + VV3 for stiffness+mass)
template <int P, int Q>
__global__ void __launch_bounds__(256) k_sumfact_scatter(ScatterArgs a) {
  constexpr int m = P + 1;
  constexpr int n = m * m * m;
  constexpr int npairs = n * (n + 1) / 2;
  constexpr int nX = m * m * Q * Q;
  constexpr int nY = m * m * m * m * Q;
  extern __shared__ double smem[];
  double* sV = smem;                 // [3][m][Q]
  double* sD = sV + 3 * m * Q;       // [3][m][Q]
  double* sW = sD + 3 * m * Q;       // [Q^3]
  double* XV = sW + Q * Q * Q;
  double* XD = XV + nX;
  double* YA = XD + nX;
  double* YB = YA + nY;
  const int64_t N = (int64_t)a.K + P;
  const int64_t n_el = (int64_t)(a.el_end - a.el_begin) * a.K * a.K;
  const int op = a.op;
  for (int64_t el = blockIdx.x; el < n_el; el += gridDim.x) {
    int alpha[3];
    alpha[2] = (int)(el % a.K);
    alpha[1] = (int)((el / a.K) % a.K);
    alpha[0] = a.el_begin + (int)(el / ((int64_t)a.K * a.K));
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * m * Q; t += blockDim.x) {
      const int d = t / (m * Q), rk = t % (m * Q);
      sV[t] = a.V[(int64_t)alpha[d] * m * Q + rk];
      sD[t] = op != IGA_OP_MASS ? a.D[(int64_t)alpha[d] * m * Q + rk] : 0.0;
    }
    const int64_t eid = ((int64_t)alpha[0] * a.K + alpha[1]) * a.K + alpha[2];
    for (int t = threadIdx.x; t < Q * Q * Q; t += blockDim.x) {
      const int k1 = t / (Q * Q), k2 = (t / Q) % Q, k3 = t % Q;
      double W = a.weights[k1] * a.weights[k2] * a.weights[k3] * a.jac;
      W *= a.coef ? a.coef[eid * Q * Q * Q + t] : a.coef_scalar;
      sW[t] = W;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nX; t += blockDim.x) {
      const int k3 = t % Q, k2 = (t / Q) % Q, j1 = (t / (Q * Q)) % m, i1 = t / (Q * Q * m);
      double xv = 0.0, xd = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) {
        const double W = sW[(k1 * Q + k2) * Q + k3];
        xv += sV[i1 * Q + k1] * sV[j1 * Q + k1] * W;
        xd += sD[i1 * Q + k1] * sD[j1 * Q + k1] * W;
      }
      XV[t] = xv;
      XD[t] = xd;
    }
    __syncthreads();
    const double* V1 = sV + m * Q;
    const double* D1 = sD + m * Q;
    for (int t = threadIdx.x; t < nY; t += blockDim.x) {
      const int k3 = t % Q, j1 = (t / Q) % m, j2 = (t / (Q * m)) % m;
      const int i1 = (t / (Q * m * m)) % m, i2 = t / (Q * m * m * m);
      double ya = 0.0, yb = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) {
        const double vv = V1[i2 * Q + k2] * V1[j2 * Q + k2];
        const int xi = ((i1 * m + j1) * Q + k2) * Q + k3;
        if (op == IGA_OP_MASS) {
          ya += XV[xi] * vv;
        } else {
          const double dd = D1[i2 * Q + k2] * D1[j2 * Q + k2];
          ya += XD[xi] * vv + XV[xi] * dd;
          yb += XV[xi] * vv;
        }
      }
      YA[t] = ya;
      YB[t] = yb;
    }
    __syncthreads();
    const double* V2 = sV + 2 * m * Q;
    const double* D2 = sD + 2 * m * Q;
    for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
      int row = (int)((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
      while (row * (row + 1) / 2 > t) --row;
      while ((row + 1) * (row + 2) / 2 <= t) ++row;
      const int col = t - row * (row + 1) / 2;
      const int i1 = row / (m * m), i2 = (row / m) % m, i3 = row % m;
      const int j1 = col / (m * m), j2 = (col / m) % m, j3 = col % m;
      const int yi = (((i2 * m + i1) * m + j2) * m + j1) * Q;
      double acc = 0.0;
#pragma unroll
      for (int k3 = 0; k3 < Q; ++k3) {
        const double vv = V2[i3 * Q + k3] * V2[j3 * Q + k3];
        if (op == IGA_OP_MASS) {
          acc += YA[yi + k3] * vv;
        } else {
          double z = D2[i3 * Q + k3] * D2[j3 * Q + k3];
          if (op == IGA_OP_STIFFNESS_MASS) z += vv;
          acc += YA[yi + k3] * vv + YB[yi + k3] * z;
        }
      }
      int64_t I[3] = {alpha[0] + i1, alpha[1] + i2, alpha[2] + i3};
      int64_t J[3] = {alpha[0] + j1, alpha[1] + j2, alpha[2] + j3};
      scatter_add(a, P, N, I, J, acc);
      if (row != col) scatter_add(a, P, N, J, I, acc);
    }
  }
}

template <int P, int Q>
struct ScatterLaunch {
  static int run(const ScatterArgs& a, int method, cudaStream_t s) {
    const int64_t Kb = a.dim == 3 ? a.K : 1;
    const int64_t n_el = (int64_t)(a.el_end - a.el_begin) * a.K * Kb;
    if (n_el <= 0) return IGA_OK;
    int64_t grid = n_el < 148 * 64 ? n_el : 148 * 64;
    if (method == IGA_METHOD_CLASSICAL) {
      if (a.dim == 3)
        k_classical_scatter<3, P, Q><<<(unsigned)grid, 256, 0, s>>>(a);
      else
        k_classical_scatter<2, P, Q><<<(unsigned)grid, 256, 0, s>>>(a);
    } else {
      if (a.dim != 3) return fail_einval("element-local sum factorization scatter is 3D only");
      constexpr int m = P + 1;
      const size_t shm = sizeof(double) * (6 * m * Q + Q * Q * Q + 2 * m * m * Q * Q +
                                           2 * m * m * m * m * Q);
      if (shm > 48 * 1024) {
        cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(k_sumfact_scatter<P, Q>), shm);
        if (e != cudaSuccess) return check_cuda(e, "sumfact smem attr");
      }
      k_sumfact_scatter<P, Q><<<(unsigned)grid, 256, shm, s>>>(a);
    }
    return check_cuda(cudaGetLastError(), "scatter launch");
  }
};

int launch_scatter(const ScatterArgs& a, int method, int p, int q, cudaStream_t s) {
  return dispatch_pq<ScatterLaunch>(p, q, a, method, s);
}

}  // namespace iga
