// Element-local mesh-wide kernels with a fused, deterministic scatter (see iga_element.cu
// header).  The elements are launched by colour (e_d mod (p+1), (p+1)^dim launches in a fixed
// order): elements of one colour share no dof, so every CSR value receives at most one
// contribution per launch, added with a plain read-modify-write -- the summation order is
// the colour order whatever the schedule, and two runs give the same bits (the reference
// promises bitwise-identical matrices for every schedule, runtime.py:16-20).
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
#include <cstdlib>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

// --------------------------------------------------------- fused scatter
// Element `el` of the launch's colour (elements lexicographic within the colour).
__device__ __forceinline__ void colour_element(const ScatterArgs& a, int64_t el, int m, int dim,
                                               int* alpha) {
  if (dim == 3) {
    const int i2 = (int)(el % a.n2), i1 = (int)((el / a.n2) % a.n1);
    const int i0 = (int)(el / ((int64_t)a.n1 * a.n2));
    alpha[0] = a.first0 + m * i0;
    alpha[1] = a.c1 + m * i1;
    alpha[2] = a.c2 + m * i2;
  } else {
    const int i1 = (int)(el % a.n1), i0 = (int)(el / a.n1);
    alpha[0] = a.first0 + m * i0;
    alpha[1] = a.c1 + m * i1;
    alpha[2] = 0;
  }
}

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
  a.values[off - a.base] += v;  // one contribution per value per colour launch
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
  const int64_t n_el = (int64_t)a.n0 * a.n1 * a.n2;
  const bool stiff = a.op != IGA_OP_MASS;
  const bool with_mass = a.op != IGA_OP_STIFFNESS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t el = blockIdx.x; el < n_el; el += gridDim.x) {
    int alpha[3];
    colour_element(a, el, m, DIM, alpha);
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
      double W = axis_w(a.weights, a.wt, alpha[0], k1, Q) * axis_w(a.weights, a.wt, alpha[1], k2, Q) *
                 a.jac;
      if (DIM == 3) W *= axis_w(a.weights, a.wt, alpha[2], k3, Q);
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

// Algorithm 1 in 3D on the FP64 tensor cores (mma.sync m8n8k4 f64, "DMMA").
// Per element the local matrix is a sum of Gram products over the quadrature
// points,  M_e = sum_t  A_t^T diag(W) B_t,  A_t(q, i) = prod_d T_{t,d}(i_d, q_d),
// with t over the terms of the operator (mass: V V V; stiffness: D V V, V D V,
// V V D), so each 8x8 output tile of the n x n matrix is KS = ceil(q^3 / 4)
// DMMA steps per term with operands formed on the fly from the per-axis tables.
// Only the upper triangle of tiles is computed; each warp owns a balanced
// contiguous range of the row-major tile list, walked in segments of <= CH
// tiles of one row tile, so an A fragment is built once per k-step and reused
// over the segment.  The scatter mirrors every strictly-upper value to the
// lower triangle, so each element matrix is exactly symmetric like the
// reference's (integrators.py:5 fills the mirror of each canonical pair, and
// assembly.py:71-79 adds all n^2 entries of the symmetric element matrix); the
// inter-element (colour) order makes the assembled matrix symmetric to rounding.
// Column slots come from per-element tables (row offset into the CSR window,
// per-axis band shifts and counts) instead of per-entry int64 index math.
__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int P, int Q>
struct ClassicalMma {
  static constexpr int m = P + 1, n = m * m * m, nq = Q * Q * Q;
  static constexpr int MT = (n + 7) / 8, KS = (nq + 3) / 4, CH = 4;
  static constexpr int NTILES = MT * (MT + 1) / 2;  // upper 8x8 tiles (nt >= mt)
};

template <int P, int Q>
__global__ void __launch_bounds__(256) k_classical_mma(ScatterArgs a) {
  using C = ClassicalMma<P, Q>;
  constexpr int m = C::m, n = C::n, nq = C::nq, MT = C::MT, KS = C::KS, CH = C::CH;
  constexpr int NTILES = C::NTILES;
  __shared__ double sV[3][m][Q], sD[3][m][Q], sW[nq];
  __shared__ int64_t s_rowoff[n];  // CSR offset of local row i (relative to a.base), -1: not owned
  __shared__ int s_shift[3][m], s_cnt[3][m];
  const int64_t N = (int64_t)a.K + P;
  const int64_t n_el = (int64_t)a.n0 * a.n1 * a.n2;
  const bool stiff = a.op != IGA_OP_MASS;
  const bool with_mass = a.op != IGA_OP_STIFFNESS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  // high degrees: `split` CTAs share an element, each taking a contiguous part of its
  // tile list (the parts write disjoint values, so the scatter stays one contribution per
  // value and element)
  const int split = a.split > 1 ? a.split : 1;
  for (int64_t item = blockIdx.x; item < n_el * split; item += gridDim.x) {
    const int64_t el = item / split;
    const int part = (int)(item % split);
    int alpha[3];
    colour_element(a, el, m, 3, alpha);
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * m * Q; t += blockDim.x) {
      const int d = t / (m * Q), rk = t % (m * Q);
      sV[d][rk / Q][rk % Q] = a.V[(int64_t)alpha[d] * m * Q + rk];
      sD[d][rk / Q][rk % Q] = stiff ? a.D[(int64_t)alpha[d] * m * Q + rk] : 0.0;
    }
    const int64_t eid = ((int64_t)alpha[0] * a.K + alpha[1]) * a.K + alpha[2];
    for (int t = threadIdx.x; t < nq; t += blockDim.x) {
      const int k1 = t / (Q * Q), k2 = (t / Q) % Q, k3 = t % Q;
      double W = axis_w(a.weights, a.wt, alpha[0], k1, Q) * axis_w(a.weights, a.wt, alpha[1], k2, Q) *
                 a.jac * axis_w(a.weights, a.wt, alpha[2], k3, Q);
      W *= a.coef ? a.coef[eid * nq + t] : a.coef_scalar;
      sW[t] = W;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int64_t I0 = alpha[0] + t / (m * m), I1 = alpha[1] + (t / m) % m, I2 = alpha[2] + t % m;
      const int64_t row = (I0 * N + I1) * N + I2;
      s_rowoff[t] = row >= a.row_first && row < a.row_last ? rowptr3(I0, I1, I2, P, N) - a.base : -1;
    }
    for (int t = threadIdx.x; t < 3 * m; t += blockDim.x) {
      const int d = t / m, k = t % m;
      const int64_t I = alpha[d] + k;
      s_shift[d][k] = (int)(alpha[d] - band_lo(I, P));  // slot of column alpha_d + c: c + shift
      s_cnt[d][k] = (int)band_cnt(I, P, N);
    }
    __syncthreads();
    // contiguous, balanced ranges of the row-major upper-tile list per warp, cut into
    // segments of <= CH tiles sharing the row tile mt
    const int nwarps = blockDim.x >> 5;
    const int p_lo = (int)((int64_t)part * NTILES / split), p_n = (int)((int64_t)(part + 1) * NTILES / split) - p_lo;
    const int t_hi = p_lo + (warp + 1) * p_n / nwarps;
    for (int t = p_lo + warp * p_n / nwarps; t < t_hi;) {
      int mt = 0, nt0 = t;
      while (nt0 >= MT - mt) nt0 -= MT - mt++;
      nt0 += mt;
      const int len = min(min(CH, t_hi - t), MT - nt0);
      t += len;
      // A row of this lane, B columns of this lane per segment tile (clamped; zeroed below)
      const int ia = min(8 * mt + g, n - 1);
      const int a0 = ia / (m * m), a1 = (ia / m) % m, a2 = ia % m;
      const bool a_ok = 8 * mt + g < n;
      int b0[CH], b1[CH], b2[CH];
      bool b_ok[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int jb = 8 * (nt0 + c) + g;
        b_ok[c] = jb < n;
        const int j = min(jb, n - 1);
        b0[c] = j / (m * m); b1[c] = (j / m) % m; b2[c] = j % m;
      }
      double acc[CH][2];
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll 2
      for (int ks = 0; ks < KS; ++ks) {
        const int qr = 4 * ks + tq;
        const int q = min(qr, nq - 1);
        const int q0 = q / (Q * Q), q1 = (q / Q) % Q, q2 = q % Q;
        const double w = a_ok && qr < nq ? sW[q] : 0.0;
        const double va0 = sV[0][a0][q0], va1 = sV[1][a1][q1], va2 = sV[2][a2][q2];
        const double wv12 = w * va1 * va2;
        const double am = wv12 * va0;
        double ad0 = 0.0, ad1 = 0.0, ad2 = 0.0;
        if (stiff) {
          const double wv0 = w * va0;
          ad0 = wv12 * sD[0][a0][q0];
          ad1 = wv0 * sD[1][a1][q1] * va2;
          ad2 = wv0 * va1 * sD[2][a2][q2];
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          if (c >= len) break;  // warp-uniform
          const double z = b_ok[c] ? 1.0 : 0.0;
          const double vb0 = sV[0][b0[c]][q0] * z, vb1 = sV[1][b1[c]][q1], vb2 = sV[2][b2[c]][q2];
          if (stiff) {
            const double v12 = vb1 * vb2;
            dmma_acc(acc[c][0], acc[c][1], ad0, sD[0][b0[c]][q0] * z * v12);
            dmma_acc(acc[c][0], acc[c][1], ad1, vb0 * sD[1][b1[c]][q1] * vb2);
            dmma_acc(acc[c][0], acc[c][1], ad2, vb0 * vb1 * sD[2][b2[c]][q2]);
            if (with_mass) dmma_acc(acc[c][0], acc[c][1], am, vb0 * v12);
          } else {
            dmma_acc(acc[c][0], acc[c][1], am, vb0 * vb1 * vb2);
          }
        }
      }
      // C fragment: lane holds (i = 8 mt + g, j = 8 nt + 2 tq + e), e = 0, 1
      const int i = 8 * mt + g;
      if (i < n) {
        const int i0 = i / (m * m), i1 = (i / m) % m, i2 = i % m;
        const int64_t off_i = s_rowoff[i];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int nt = nt0 + c;
          if (c >= len) break;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 8 * nt + 2 * tq + e;
            if (j >= n || (nt == mt && j < i)) continue;
            const int j0 = j / (m * m), j1 = (j / m) % m, j2 = j % m;
            const double v = acc[c][e];
            if (off_i >= 0) {
              const int slot = ((j0 + s_shift[0][i0]) * s_cnt[1][i1] + j1 + s_shift[1][i1]) * s_cnt[2][i2] +
                               j2 + s_shift[2][i2];
              a.values[off_i + slot] += v;
            }
            const int64_t off_j = s_rowoff[j];
            if (j != i && off_j >= 0) {
              const int slot = ((i0 + s_shift[0][j0]) * s_cnt[1][j1] + i1 + s_shift[1][j1]) * s_cnt[2][j2] +
                               i2 + s_shift[2][j2];
              a.values[off_j + slot] += v;
            }
          }
        }
      }
    }
  }
}

// Algorithm 2 element-local, merged stiffness form, fused scatter (by element colour).
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
  // stage buffers: shared memory, or (high degrees) this CTA's slice of the global scratch
  double* XV = a.scratch ? a.scratch + (int64_t)blockIdx.x * (2 * nX + 2 * nY) : sW + Q * Q * Q;
  double* XD = XV + nX;
  double* YA = XD + nX;
  double* YB = YA + nY;
  const int64_t N = (int64_t)a.K + P;
  const int64_t n_el = (int64_t)a.n0 * a.n1 * a.n2;
  const int op = a.op;
  for (int64_t el = blockIdx.x; el < n_el; el += gridDim.x) {
    int alpha[3];
    colour_element(a, el, m, 3, alpha);
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * m * Q; t += blockDim.x) {
      const int d = t / (m * Q), rk = t % (m * Q);
      sV[t] = a.V[(int64_t)alpha[d] * m * Q + rk];
      sD[t] = op != IGA_OP_MASS ? a.D[(int64_t)alpha[d] * m * Q + rk] : 0.0;
    }
    const int64_t eid = ((int64_t)alpha[0] * a.K + alpha[1]) * a.K + alpha[2];
    for (int t = threadIdx.x; t < Q * Q * Q; t += blockDim.x) {
      const int k1 = t / (Q * Q), k2 = (t / Q) % Q, k3 = t % Q;
      double W = axis_w(a.weights, a.wt, alpha[0], k1, Q) * axis_w(a.weights, a.wt, alpha[1], k2, Q) *
                 axis_w(a.weights, a.wt, alpha[2], k3, Q) * a.jac;
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
  static constexpr int m = P + 1;
  static constexpr size_t kStage = 2 * (size_t)m * m * Q * Q + 2 * (size_t)m * m * m * m * Q;
  static constexpr size_t kBase = 6 * m * Q + Q * Q * Q;
  static constexpr bool kGlobalStage = sizeof(double) * (kBase + kStage) > 200 * 1024;

  static int launch_colour(const ScatterArgs& a, int method, size_t shm, int64_t slots,
                           cudaStream_t s) {
    const int64_t n_el = (int64_t)a.n0 * a.n1 * a.n2;
    if (n_el <= 0) return IGA_OK;
    int64_t grid = n_el < 148 * 64 ? n_el : 148 * 64;
    if (method == IGA_METHOD_CLASSICAL) {
      static const bool scalar = [] {
        const char* e = getenv("IGA_CLASSICAL_SCALAR");
        return e && e[0] == '1' && e[1] == 0;
      }();
      if (a.dim == 3 && !scalar) {
        ScatterArgs b = a;
        // few, large elements per colour (high degrees): several CTAs per element
        constexpr int NT = ClassicalMma<P, Q>::NTILES;
        b.split = 1;
        if (P > kMaxPLow && n_el < 2 * 148) {
          const int64_t want = (2 * 148 + n_el - 1) / n_el;
          b.split = (int)(want < NT / 64 ? want : (NT / 64 > 1 ? NT / 64 : 1));
        }
        const int64_t items = n_el * b.split;
        grid = items < 148 * 64 ? items : 148 * 64;
        k_classical_mma<P, Q><<<(unsigned)grid, 256, 0, s>>>(b);
      } else if (a.dim == 3) {
        k_classical_scatter<3, P, Q><<<(unsigned)grid, 256, 0, s>>>(a);
      } else {
        k_classical_scatter<2, P, Q><<<(unsigned)grid, 256, 0, s>>>(a);
      }
    } else {
      if (slots > 0 && grid > slots) grid = slots;  // one scratch slice per CTA
      k_sumfact_scatter<P, Q><<<(unsigned)grid, 256, shm, s>>>(a);
    }
    return check_cuda(cudaGetLastError(), "scatter launch");
  }

  static int run(const ScatterArgs& a0, int method, cudaStream_t s) {
    if (a0.el_end <= a0.el_begin) return IGA_OK;
    size_t shm = 0;
    int64_t slots = 0;
    double* scratch = nullptr;
    if (method != IGA_METHOD_CLASSICAL) {
      if (a0.dim != 3) return fail_einval("element-local sum factorization scatter is 3D only");
      shm = sizeof(double) * (kGlobalStage ? kBase : kBase + kStage);
      if (shm > 48 * 1024) {
        cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(k_sumfact_scatter<P, Q>), shm);
        if (e != cudaSuccess) return check_cuda(e, "sumfact smem attr");
      }
      if (kGlobalStage) {
        // high degrees: the stage buffers (m^4 Q doubles each) of one resident wave of CTAs
        // in stream-ordered global scratch (cudaMallocAsync; graph-capturable), freed after
        // the last colour
        slots = (int64_t)sm_count() *
                blocks_per_sm_once(reinterpret_cast<const void*>(k_sumfact_scatter<P, Q>), 256, shm);
        const int rc = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&scratch),
                                                  sizeof(double) * kStage * slots, s),
                                  "sumfact scratch");
        if (rc) return rc;
      }
    }
    auto count = [](int lo, int hi, int c) {  // e in [lo, hi) with e = c (mod m)
      const int first = lo + ((c - lo % m) % m + m) % m;
      return first >= hi ? 0 : (hi - 1 - first) / m + 1;
    };
    const int colours = a0.dim == 3 ? m * m * m : m * m;
    int rc = IGA_OK;
    for (int col = 0; col < colours && !rc; ++col) {  // fixed colour order = fixed summation order
      ScatterArgs a = a0;
      const int c0 = a0.dim == 3 ? col / (m * m) : col / m;
      a.c1 = a0.dim == 3 ? (col / m) % m : col % m;
      a.c2 = a0.dim == 3 ? col % m : 0;
      a.first0 = a0.el_begin + ((c0 - a0.el_begin % m) % m + m) % m;
      a.n0 = count(a0.el_begin, a0.el_end, c0);
      a.n1 = count(0, a0.K, a.c1);
      a.n2 = a0.dim == 3 ? count(0, a0.K, a.c2) : 1;
      a.split = 1;
      a.scratch = scratch;
      rc = launch_colour(a, method, shm, slots, s);
    }
    if (scratch) {
      const int rf = check_cuda(cudaFreeAsync(scratch, s), "sumfact scratch free");
      if (!rc) rc = rf;
    }
    return rc;
  }
};

int launch_scatter(const ScatterArgs& a, int method, int p, int q, cudaStream_t s) {
  return dispatch_pq_all<ScatterLaunch>(p, q, a, method, s);
}

}  // namespace iga
