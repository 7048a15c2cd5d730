// Shared device helpers for the B200 IGA integration + assembly kernels.
//
//  * strict-IEEE Cox-de Boor evaluation (bitwise equal to splines.py:78-161)
//  * structured CSR arithmetic: row pointers and column slots of the global
//    pattern computed in closed form (the pattern assembly.py:99-115 builds is
//    a tensor product of 1D bands, so no indptr/indices reads are needed)
//  * error reporting for the C-ABI
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/iga_b200.h"

namespace iga {

constexpr int kMaxP = 9;    // highest degree with device kernels (iga_dispatch.cuh: p <= 5 on
                            // every path, 6..9 on the paths that opt in)
constexpr int kMaxQ = 10;   // highest quadrature-point count per axis
constexpr int kMaxKnots = 1 << 16;

// ------------------------------------------------------------ error state
void set_error(const char* fmt, ...);
int fail_einval(const char* fmt, ...);
int check_cuda(cudaError_t err, const char* what);

// ------------------------------------------------ cached launch set-up (host)
// Function attributes and occupancy are per (kernel, device) and cost host
// microseconds per call -- time the GPU would otherwise idle between
// back-to-back launches -- so they are set / queried once (iga_abi.cu).
cudaError_t smem_attr_once(const void* fn, size_t bytes, bool max_carveout = false);
int sm_count();
int blocks_per_sm_once(const void* fn, int threads, size_t smem);

// ----------------------------------------------------- strict IEEE helpers
// __dmul_rn / __dadd_rn are never contracted into DFMA, so expressions built
// from them round exactly like the numba kernels (strict left-to-right).
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// Knot t_i of the open uniform vector (splines.py:59-75): p+1 zeros,
// i/K for the interior (np.arange(1,K)/K is a correctly rounded division),
// p+1 ones.  Computed, never stored -- unless a general knot vector `t`
// (K + 2p + 1 non-decreasing knots) is given.
__device__ __forceinline__ double knot(int i, int K, int p, const double* t = nullptr) {
  if (t != nullptr) return __ldg(t + i);
  if (i <= p) return 0.0;
  if (i >= K + p) return 1.0;
  return dvd((double)(i - p), (double)K);
}

// Bottom-up Cox-de Boor: N[j] holds B_{lo+j, level}(x).  The value of
// B_{i,r}(x) does not depend on the recursion path, so evaluating the
// triangle level by level with the same two-term expression as _cox
// (splines.py:108-118) reproduces the reference bits.
// Fills vals[r] = B_{e+r,p}(x), r = 0..p, and (if ders) the derivatives of
// splines.py:139-161.
template <int P>
__device__ __forceinline__ void cox_de_boor(int e, double x, int K, double* vals, double* ders,
                                            const double* t = nullptr) {
  // the 2P+2 knots t_e .. t_{e+2P+1} this point touches, each divided once
  double kn[2 * P + 2];
#pragma unroll
  for (int j = 0; j <= 2 * P + 1; ++j) kn[j] = knot(e + j, K, P, t);
  // level-0 indices e .. e+2P  (2P+1 values); level r needs e .. e+2P-r.
  // order0 (splines.py:78-91) with the closed last span: the last knot (1.0 for the
  // uniform vector)
  const double tl = t != nullptr ? __ldg(t + K + 2 * P) : 1.0;
  double N[2 * P + 1];
#pragma unroll
  for (int j = 0; j <= 2 * P; ++j) {
    const double ti = kn[j], ti1 = kn[j + 1];
    N[j] = (ti <= x && x < ti1) || (x == tl && ti < ti1 && ti1 == tl) ? 1.0 : 0.0;
  }
  double Nprev[2 * P + 1];  // level P-1 values, for derivatives
#pragma unroll
  for (int j = 0; j <= 2 * P; ++j) Nprev[j] = N[j];
  // the triangle's divisions depend only on x and the knots: all of them are issued
  // before the level recursion (independent, so their latencies overlap)
  double cl[P + 1][2 * P + 1], cr[P + 1][2 * P + 1];
#pragma unroll
  for (int q = 1; q <= P; ++q)
#pragma unroll
    for (int j = 0; j <= 2 * P - q; ++j) {
      const double d_left = sub(kn[j + q], kn[j]), d_right = sub(kn[j + q + 1], kn[j + 1]);
      cl[q][j] = d_left > 0.0 ? dvd(sub(x, kn[j]), d_left) : 0.0;
      cr[q][j] = d_right > 0.0 ? dvd(sub(kn[j + q + 1], x), d_right) : 0.0;
    }
#pragma unroll
  for (int q = 1; q <= P; ++q) {
#pragma unroll
    for (int j = 0; j <= 2 * P - q; ++j) {
      double out = 0.0;
      if (sub(kn[j + q], kn[j]) > 0.0) out = add(out, mul(cl[q][j], N[j]));
      if (sub(kn[j + q + 1], kn[j + 1]) > 0.0) out = add(out, mul(cr[q][j], N[j + 1]));
      N[j] = out;
    }
    if (q == P - 1) {
#pragma unroll
      for (int j = 0; j <= 2 * P; ++j) Nprev[j] = N[j];
    }
  }
#pragma unroll
  for (int r = 0; r <= P; ++r) vals[r] = N[r];
  if (ders != nullptr) {
    if (P == 0) {
      ders[0] = 0.0;
    } else {
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        double d = 0.0;
        const double d_left = sub(kn[r + P], kn[r]);
        if (d_left > 0.0) d = add(d, dvd(Nprev[r], d_left));
        const double d_right = sub(kn[r + P + 1], kn[r + 1]);
        if (d_right > 0.0) d = sub(d, dvd(Nprev[r + 1], d_right));
        ders[r] = mul((double)P, d);
      }
    }
  }
}

// Out-of-line copy (one per P per translation unit) for kernels templated on
// more than P, to keep their code size and compile time bounded.
template <int P>
__device__ __noinline__ void cox_de_boor_ool(int e, double x, int K, double* vals, double* ders,
                                             const double* t) {
  cox_de_boor<P>(e, x, K, vals, ders, t);
}

// Node mapping of runtime.py:147 / mesh.py:88: e*h + (ref+1)*(h/2), h = 1/K.  For a
// general knot vector t the element is the span [t_{p+e}, t_{p+e+1}]:
// lo + (ref+1)*(h/2), h = hi - lo (tools/gen_golden.py nonuniform_tables).
__device__ __forceinline__ double map_node(int e, double ref, int K, int p = 0,
                                           const double* t = nullptr) {
  if (t != nullptr) {
    const double lo = __ldg(t + p + e), hi = __ldg(t + p + e + 1);
    return add(lo, mul(add(ref, 1.0), dvd(sub(hi, lo), 2.0)));
  }
  const double h = dvd(1.0, (double)K);
  return add(mul((double)e, h), mul(add(ref, 1.0), dvd(h, 2.0)));
}

// Weight of quadrature point k of element e along an axis: the reference weight (uniform
// mesh: the Jacobian is the scalar jac) or, for a general knot vector, the per-element
// table wt[e][k] = w_k h_e / 2 that K1 writes (the element's Jacobian folded per axis).
__device__ __forceinline__ double axis_w(const double* w, const double* wt, int e, int k, int q) {
  return wt != nullptr ? __ldg(wt + e * q + k) : w[k];
}

// ------------------------------------------------- structured CSR helpers
// 1D band of dof I: columns [max(I-p,0), min(I+p,N-1)], N = K+p.
__host__ __device__ __forceinline__ int64_t band_lo(int64_t I, int p) { return I - p > 0 ? I - p : 0; }
__host__ __device__ __forceinline__ int64_t band_cnt(int64_t I, int p, int64_t N) {
  const int64_t hi = I + p < N - 1 ? I + p : N - 1;
  return hi - band_lo(I, p) + 1;
}
// Prefix sum of band_cnt over I' < I (closed form).
__host__ __device__ __forceinline__ int64_t band_prefix(int64_t I, int p, int64_t N) {
  int64_t L = N - p;
  if (L < 0) L = 0;
  if (L > I) L = I;
  int64_t s = L * (L - 1) / 2 + (int64_t)p * L + (I - L) * (N - 1);
  if (I > p) s -= (I - p) * (I - p - 1) / 2;
  return s + I;
}
// Row pointer of global row (I0,I1,I2) (I0 slowest) in the full CSR.
__host__ __device__ __forceinline__ int64_t rowptr3(int64_t I0, int64_t I1, int64_t I2, int p, int64_t N) {
  const int64_t T = band_prefix(N, p, N);
  return T * T * band_prefix(I0, p, N) +
         band_cnt(I0, p, N) * (T * band_prefix(I1, p, N) + band_cnt(I1, p, N) * band_prefix(I2, p, N));
}
__host__ __device__ __forceinline__ int64_t rowptr2(int64_t I0, int64_t I1, int p, int64_t N) {
  const int64_t T = band_prefix(N, p, N);
  return T * band_prefix(I0, p, N) + band_cnt(I0, p, N) * band_prefix(I1, p, N);
}
__host__ __device__ __forceinline__ int64_t rowptr(int dim, int64_t row, int p, int64_t N) {
  if (dim == 3) return rowptr3(row / (N * N), (row / N) % N, row % N, p, N);
  return rowptr2(row / N, row % N, p, N);
}
// Offset of column J inside row I (both as per-axis indices).
__host__ __device__ __forceinline__ int64_t col_slot3(const int64_t* I, const int64_t* J, int p, int64_t N) {
  return ((J[0] - band_lo(I[0], p)) * band_cnt(I[1], p, N) + (J[1] - band_lo(I[1], p))) *
             band_cnt(I[2], p, N) +
         (J[2] - band_lo(I[2], p));
}

}  // namespace iga

