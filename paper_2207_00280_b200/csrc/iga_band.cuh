// 1D band matrices of the separable (scalar-coefficient) paths (iga_kron.cu, iga_apply.cu):
//   m(I,J) = sum_e sum_q w_q V_e(I-e,q) V_e(J-e,q),  k: the same with derivatives D,
// for band offsets d = J - I + P in [0, 2P], elements e in a range (a slab restricts
// the axis-0 factor only).  Element order ascending, points ascending.
#pragma once

#include "iga_common.cuh"

namespace iga {

// 1D band entry (I, J = I + d - P) over the elements e in [e_lo, e_hi): value and
// derivative products, elements ascending, quadrature points ascending.
template <int P, int Q>
__device__ __forceinline__ double2 band1d(const double* V, const double* D, int K, const double* w,
                                          int I, int d, int e_lo, int e_hi, bool stiff,
                                          const double* wt = nullptr) {
  constexpr int M = P + 1;
  const int J = I + d - P;
  double m = 0.0, k = 0.0;
  const int lo = max(max(I, J) - P, max(e_lo, 0)), hi = min(min(I, J) + 1, min(e_hi, K));
  // at most P+1 elements
#pragma unroll
  for (int t = 0; t <= P; ++t) {
    const int e = lo + t;
    if (e < hi) {
      const double* Ve = V + e * M * Q;
      const int i = I - e, j = J - e;
#pragma unroll
      for (int q = 0; q < Q; ++q) m += (axis_w(w, wt, e, q, Q) * Ve[i * Q + q]) * Ve[j * Q + q];
      if (stiff) {
        const double* De = D + e * M * Q;
#pragma unroll
        for (int q = 0; q < Q; ++q) k += (axis_w(w, wt, e, q, Q) * De[i * Q + q]) * De[j * Q + q];
      }
    }
  }
  return make_double2(m, k);
}


// band1d summed as build_band_tables' shared-memory path does (each element's integral
// over its points first, then the elements ascending), so it reproduces those bits
template <int P, int Q>
__device__ __forceinline__ double2 band1d_el(const double* V, const double* D, int K, const double* w,
                                             int I, int d, int e_lo, int e_hi, bool stiff,
                                             const double* wt = nullptr) {
  constexpr int M = P + 1;
  const int J = I + d - P;
  double m = 0.0, k = 0.0;
  const int lo = max(max(I, J) - P, max(e_lo, 0)), hi = min(min(I, J) + 1, min(e_hi, K));
  for (int e = lo; e < hi; ++e) {
    const double* Ve = V + e * M * Q;
    const int i = I - e, j = J - e;
    double me = 0.0, ke = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) me += (axis_w(w, wt, e, q, Q) * Ve[i * Q + q]) * Ve[j * Q + q];
    if (stiff) {
      const double* De = D + e * M * Q;
#pragma unroll
      for (int q = 0; q < Q; ++q) ke += (axis_w(w, wt, e, q, Q) * De[i * Q + q]) * De[j * Q + q];
    }
    m += me;
    k += ke;
  }
  return make_double2(m, k);
}

// Fill tb[0][N][NB] (all elements) and, if with_slab, tb[1][N][NB] (elements in
// [slab_lo, slab_hi)) in shared memory, (m, k) per entry.  When the basis tables and
// the element integrals fit in `scratch` (small K, where this prologue is not
// amortised) the element integrals m_e(r,s), k_e(r,s) are formed first -- one short
// dot product per thread -- and summed per band entry over the <= P+1 elements of
// the pair; otherwise each entry is integrated from the global tables.  w_s: [Q]
// shared.  Ends with a barrier.
template <int P, int Q>
__device__ void build_band_tables(const double* V, const double* D, const double* weights, int K,
                                  bool stiff, int slab_lo, int slab_hi, bool with_slab,
                                  double2* tb, double* scratch, int scratch_doubles, double* w_s,
                                  int tid, int nt, const double* wt = nullptr) {
  constexpr int M = P + 1, NB = 2 * P + 1;
  const int N = K + P;
  const int nvd = K * M * Q, nem = K * M * M;
  const int ntab = (with_slab ? 2 : 1) * N * NB;
  if (tid < Q) w_s[tid] = weights[tid];
  if (2 * nvd + 2 * nem <= scratch_doubles) {
    double* Vs = scratch;
    double* Ds = scratch + nvd;
    double2* em = reinterpret_cast<double2*>(scratch + 2 * nvd);  // [K][M][M] (m, k)
    for (int u = tid; u < nvd; u += nt) {
      Vs[u] = __ldg(V + u);
      if (stiff) Ds[u] = __ldg(D + u);
    }
    __syncthreads();
    for (int u = tid; u < nem; u += nt) {
      const int e = u / (M * M), r = (u / M) % M, c = u % M;
      const double* vr = Vs + (e * M + r) * Q;
      const double* vc = Vs + (e * M + c) * Q;
      double m = 0.0, k = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) m += (axis_w(w_s, wt, e, q, Q) * vr[q]) * vc[q];
      if (stiff) {
        const double* dr = Ds + (e * M + r) * Q;
        const double* dc = Ds + (e * M + c) * Q;
#pragma unroll
        for (int q = 0; q < Q; ++q) k += (axis_w(w_s, wt, e, q, Q) * dr[q]) * dc[q];
      }
      em[u] = make_double2(m, k);
    }
    __syncthreads();
    for (int u = tid; u < ntab; u += nt) {
      const int v = u < N * NB ? u : u - N * NB;
      const bool slab = u >= N * NB;
      const int I = v / NB, J = I + v % NB - P;
      const int lo = max(max(I, J) - P, slab ? max(slab_lo, 0) : 0);
      const int hi = min(min(I, J) + 1, slab ? min(slab_hi, K) : K);
      double m = 0.0, k = 0.0;
      for (int e = lo; e < hi; ++e) {
        const double2 x = em[(e * M + I - e) * M + J - e];
        m += x.x;
        k += x.y;
      }
      tb[u] = make_double2(m, k);
    }
  } else {
    __syncthreads();
    for (int u = tid; u < ntab; u += nt) {
      const int v = u < N * NB ? u : u - N * NB;
      const bool slab = u >= N * NB;
      tb[u] = band1d<P, Q>(V, D, K, w_s, v / NB, v % NB, slab ? slab_lo : 0, slab ? slab_hi : K,
                           stiff, wt);
    }
  }
  __syncthreads();
}

}  // namespace iga
