// C-ABI entry points of the mesh-wide path: fused integrate+assemble,
// assembly from element matrices, and SpMV over the structured CSR.
#include <cstdlib>

#include "iga_dispatch.cuh"

#include "iga_args.cuh"

namespace iga {

int launch_scatter(const ScatterArgs& a, int method, int p, int q, cudaStream_t s);
int launch_gsf(const GsfArgs& a, int p, int q, cudaStream_t s);
int launch_kron(const KronArgs& a, int p, int q, cudaStream_t s);
int launch_band_tables(int K, int p, int q, const double* ref, const double* weights, int stiff,
                       double* V, double* D, double* band, const double* knots, double* wt,
                       cudaStream_t s);

// assembly.assemble from element matrices: one warp per CSR row, lanes over
// its columns; every value sums its element contributions in lexicographic
// element order (deterministic; SPEC's "lexicographic element order").
__global__ void k_assemble_elements(int dim, int K, int p, const double* __restrict__ mats,
                                    int64_t row_first, int64_t nrows, int64_t base,
                                    double* __restrict__ values) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nrows) return;
  const int64_t N = (int64_t)K + p;
  const int m = p + 1;
  const int64_t n = dim == 3 ? (int64_t)m * m * m : (int64_t)m * m;
  const int64_t row = row_first + warp;
  int64_t I[3] = {0, 0, 0};
  if (dim == 3) {
    I[0] = row / (N * N); I[1] = (row / N) % N; I[2] = row % N;
  } else {
    I[0] = row / N; I[1] = row % N;
  }
  int64_t lo[3], c[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = d < dim ? band_lo(I[d], p) : 0;
    c[d] = d < dim ? band_cnt(I[d], p, N) : 1;
  }
  const int64_t cnt = c[0] * c[1] * c[2];
  const int64_t off = rowptr(dim, row, p, N) - base;
  for (int64_t j = lane; j < cnt; j += 32) {
    int64_t J[3] = {lo[0] + j / (c[1] * c[2]), lo[1] + (j / c[2]) % c[1], lo[2] + j % c[2]};
    int64_t elo[3], ehi[3];
    for (int d = 0; d < 3; ++d) {
      if (d < dim) {
        const int64_t mx = I[d] > J[d] ? I[d] : J[d], mn = I[d] < J[d] ? I[d] : J[d];
        elo[d] = mx - p > 0 ? mx - p : 0;
        ehi[d] = mn < K - 1 ? mn : K - 1;
      } else {
        elo[d] = 0; ehi[d] = 0;
      }
    }
    double acc = 0.0;
    for (int64_t a0 = elo[0]; a0 <= ehi[0]; ++a0)
      for (int64_t a1 = elo[1]; a1 <= ehi[1]; ++a1)
        for (int64_t a2 = elo[2]; a2 <= ehi[2]; ++a2) {
          int64_t eid, il, jl;
          if (dim == 3) {
            eid = (a0 * K + a1) * K + a2;
            il = ((I[0] - a0) * m + (I[1] - a1)) * m + (I[2] - a2);
            jl = ((J[0] - a0) * m + (J[1] - a1)) * m + (J[2] - a2);
          } else {
            eid = a0 * K + a1;
            il = (I[0] - a0) * m + (I[1] - a1);
            jl = (J[0] - a0) * m + (J[1] - a1);
          }
          acc += mats[(eid * n + il) * n + jl];
        }
    values[off + j] = acc;
  }
}

// y = A x over the structured CSR: one warp per row, lanes over the row's values
// (contiguous, so each warp load is one coalesced 256-byte segment); the column of
// value j is (lo0 + a, lo1 + b, lo2 + c) with j = (a c1 + b) c2 + c, decomposed with
// compile-time divisors for the full-band rows.  HBM-bound on the values.
template <int P>
__global__ void __launch_bounds__(256, 5) k_spmv3(int K, const double* __restrict__ values,
                                               const double* __restrict__ x,
                                               double* __restrict__ y, int nseg) {
  constexpr int NB = 2 * P + 1;
  const int lane = threadIdx.x & 31;
  const int64_t N = (int64_t)K + P;
  // work unit: a run of rows I2 in [h0, h1) of one (I0, I1) pencil; the row offset and
  // the x window advance incrementally along the run (no per-row 64-bit arithmetic)
  const int64_t nunits = N * N * nseg;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nunits;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t pen = u / nseg;
    const int sg = (int)(u - pen * nseg);
    const int I0 = (int)(pen / N), I1 = (int)(pen - (int64_t)I0 * N);
    const int h0 = (int)(N * sg / nseg), h1 = (int)(N * (sg + 1) / nseg);
    const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N), c01 = c0 * c1;
    const double* v = values + rowptr3(I0, I1, h0, P, N);
    const double* xp = x + ((int64_t)band_lo(I0, P) * N + band_lo(I1, P)) * N;
    double* yp = y + ((int64_t)I0 * N + I1) * N;
    // x offsets of this lane's values in a full-band row (the same for every such row)
    constexpr int NE = (NB * NB * NB + 31) / 32;
    int xo[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) {
      const int j = lane + 32 * k, a = j / (NB * NB), b = (j / NB) % NB, c = j % NB;
      xo[k] = (int)(((int64_t)a * N + b) * N + c);
    }
    for (int I2 = h0; I2 < h1; ++I2) {
      const int lo2 = I2 - P < 0 ? 0 : I2 - P;
      const int c2 = (int)band_cnt(I2, P, N);
      const double* xb = xp + lo2;
      const int cnt = c01 * c2;
      double acc = 0.0;
      if (cnt == NB * NB * NB) {
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int j = lane + 32 * k;
          if (j < NB * NB * NB) acc += v[j] * xb[xo[k]];
        }
      } else {
        for (int j = lane; j < cnt; j += 32) {
          const int a = j / (c1 * c2), b = (j / c2) % c1, c = j % c2;
          acc += v[j] * xb[((int64_t)a * N + b) * N + c];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) yp[I2] = acc;
      v += cnt;
    }
  }
}

// Same product with the x window in shared memory: a CTA takes one dof plane I0, a block
// of SB1 pencils I1 (one warp each) and a segment of SEG rows I2; the x values its rows
// touch (<= 2P+1 planes x SB1+2P pencils x SEG+2P rows) are staged once, so the per-value
// gathers hit shared memory instead of L1/L2 (the values stream from HBM as before).
constexpr int kSpmvSB1 = 8, kSpmvSeg = 64;
template <int P>
__global__ void __launch_bounds__(32 * kSpmvSB1) k_spmv3s(int K, const double* __restrict__ values,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ y) {
  constexpr int NB = 2 * P + 1, WB = kSpmvSB1 + 2 * P, WC = kSpmvSeg + 2 * P;
  extern __shared__ double xs[];  // [NB][WB][WC]
  const int N = K + P;
  const int nb1 = (N + kSpmvSB1 - 1) / kSpmvSB1, nsg = (N + kSpmvSeg - 1) / kSpmvSeg;
  const int seg = (N + nsg - 1) / nsg;  // balanced segments of <= kSpmvSeg rows
  const int blk = blockIdx.x;
  const int I0 = blk / (nb1 * nsg), r = blk - I0 * nb1 * nsg, i1b = (r / nsg) * kSpmvSB1,
            h0 = (r % nsg) * seg, h1 = min(N, h0 + seg);
  const int lo0 = max(0, I0 - P), c0 = (int)band_cnt(I0, P, N);
  const int b_lo = max(0, i1b - P), b_hi = min(N, i1b + kSpmvSB1 + P);
  const int c_lo = max(0, h0 - P), c_hi = min(N, h1 + P);
  const int nbw = b_hi - b_lo, ncw = c_hi - c_lo;
  for (int u = threadIdx.x; u < c0 * nbw * ncw; u += blockDim.x) {
    const int a = u / (nbw * ncw), rr = u - a * nbw * ncw, b = rr / ncw, c = rr - b * ncw;
    xs[(a * WB + b) * WC + c] = __ldg(x + ((int64_t)(lo0 + a) * N + b_lo + b) * N + c_lo + c);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, I1 = i1b + (threadIdx.x >> 5);
  if (I1 >= N) return;
  const int c1 = (int)band_cnt(I1, P, N), c01 = c0 * c1;
  const double* v = values + rowptr3(I0, I1, h0, P, N);
  const double* xw = xs + (band_lo(I1, P) - b_lo) * WC - c_lo;  // + (a WB + b) WC + column
  constexpr int NE = (NB * NB * NB + 31) / 32;
  int xo[NE];
#pragma unroll
  for (int k = 0; k < NE; ++k) {
    const int j = lane + 32 * k, a = j / (NB * NB), b = (j / NB) % NB, c = j % NB;
    xo[k] = (a * WB + b) * WC + c;
  }
  double* yp = y + ((int64_t)I0 * N + I1) * N;
  for (int I2 = h0; I2 < h1; ++I2) {
    const int lo2 = I2 - P < 0 ? 0 : I2 - P;
    const int c2 = (int)band_cnt(I2, P, N);
    const double* xb = xw + lo2;
    const int cnt = c01 * c2;
    double acc = 0.0;
    if (cnt == NB * NB * NB) {
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const int j = lane + 32 * k;
        if (j < NB * NB * NB) acc += v[j] * xb[xo[k]];
      }
    } else {
      for (int j = lane; j < cnt; j += 32) {
        const int a = j / (c1 * c2), b = (j / c2) % c1, c = j % c2;
        acc += v[j] * xb[(a * WB + b) * WC + c];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) yp[I2] = acc;
    v += cnt;
  }
}

template <int P>
struct Spmv3Launch {
  static int run(int K, const double* values, const double* x, double* y, cudaStream_t s) {
    const int64_t N = (int64_t)K + P;
    // ~4 row runs per resident warp (balance), runs of >= 8 rows
    const int64_t want_units = (int64_t)sm_count() * 64 * 4;
    int nseg = (int)((want_units + N * N - 1) / (N * N));
    if (nseg > (int)(N / 8)) nseg = (int)(N / 8);
    if (nseg < 1) nseg = 1;
    const int64_t units = N * N * nseg;
    const int64_t want = (units * 32 + 255) / 256;
    const int64_t grid = want < (int64_t)sm_count() * 5 ? want : (int64_t)sm_count() * 5;
    // the staged-window kernel wins on large meshes only (measured: K = 256 9.8 vs 11.5 ms,
    // K = 192 4.3 vs 4.8; K <= 128 the L1 version is faster); IGA_SPMV_L1=1 forces L1
    // (an A/B knob read per call so a test can compare both kernels in one process; only
    // the value "1" enables it)
    const char* force_l1 = getenv("IGA_SPMV_L1");
    constexpr size_t staged_sm = sizeof(double) * (2 * P + 1) * (kSpmvSB1 + 2 * P) * (kSpmvSeg + 2 * P);
    if (staged_sm <= 200 * 1024 && N >= 160 &&
        !(force_l1 != nullptr && force_l1[0] == '1' && force_l1[1] == 0)) {
      const int64_t nb1 = (N + kSpmvSB1 - 1) / kSpmvSB1, nsg = (N + kSpmvSeg - 1) / kSpmvSeg;
      const size_t sm = sizeof(double) * (2 * P + 1) * (kSpmvSB1 + 2 * P) * (kSpmvSeg + 2 * P);
      const void* fn = reinterpret_cast<const void*>(k_spmv3s<P>);
      cudaError_t e = smem_attr_once(fn, sm, false);
      if (e != cudaSuccess) return check_cuda(e, "spmv smem attr");
      k_spmv3s<P><<<(unsigned)(N * nb1 * nsg), 32 * kSpmvSB1, sm, s>>>(K, values, x, y);
      return check_cuda(cudaGetLastError(), "iga_spmv");
    }
    k_spmv3<P><<<(unsigned)grid, 256, 0, s>>>(K, values, x, y, nseg);
    return check_cuda(cudaGetLastError(), "iga_spmv");
  }
};

// 2D: one warp per row (general path).
__global__ void k_spmv(int dim, int K, int p, const double* __restrict__ values,
                       const double* __restrict__ x, double* __restrict__ y, int64_t nrows) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nrows) return;
  const int64_t N = (int64_t)K + p;
  const int64_t row = warp;
  int64_t I[3] = {0, 0, 0};
  if (dim == 3) {
    I[0] = row / (N * N); I[1] = (row / N) % N; I[2] = row % N;
  } else {
    I[0] = row / N; I[1] = row % N;
  }
  int64_t lo[3], c[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = d < dim ? band_lo(I[d], p) : 0;
    c[d] = d < dim ? band_cnt(I[d], p, N) : 1;
  }
  const int64_t cnt = c[0] * c[1] * c[2];
  const int64_t off = rowptr(dim, row, p, N);
  double acc = 0.0;
  for (int64_t j = lane; j < cnt; j += 32) {
    const int64_t a = j / (c[1] * c[2]), b = (j / c[2]) % c[1], cc = j % c[2];
    const int64_t col = dim == 3 ? ((lo[0] + a) * N + lo[1] + b) * N + lo[2] + cc
                                 : (lo[0] + a) * N + lo[1] + b;
    acc += values[off + j] * x[col];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[row] = acc;
}

static int validate_problem(const iga_problem* prob) {
  if (!prob) return fail_einval("null problem");
  if (prob->dim != 2 && prob->dim != 3) return fail_einval("dim must be 2 or 3, got %d", prob->dim);
  if (prob->K < 1) return fail_einval("mesh must be >= 1, got %d", prob->K);
  if (prob->p < 0) return fail_einval("degree must be >= 0, got %d", prob->p);
  if (prob->q < 1) return fail_einval("quadrature points must be >= 1, got %d", prob->q);
  if (prob->op < 0 || prob->op > 2) return fail_einval("unknown operator %d", prob->op);
  if (prob->op != IGA_OP_MASS && prob->p < 1)
    return fail_einval("derivatives require degree >= 1");
  if (!prob->weights || !prob->tables_v) return fail_einval("null weights/tables");
  if (prob->op != IGA_OP_MASS && !prob->tables_d) return fail_einval("stiffness needs tables_d");
  if (prob->reserved != 0) return fail_einval("reserved field must be 0");
  if (prob->knots && !prob->elem_weights)
    return fail_einval("a general knot vector needs elem_weights (iga_mesh_tables_general)");
  return IGA_OK;
}

}  // namespace iga

using namespace iga;

extern "C" {

int32_t iga_band_tables(const iga_problem* prob, const double* ref_nodes, double* vals,
                        double* ders, double* band, double* elem_weights, void* stream) {
  if (!prob) return fail_einval("null problem");
  if (prob->knots && !elem_weights) return fail_einval("a general knot vector needs elem_weights");
  iga_problem pr = *prob;  // the weights are this call's output
  if (pr.knots) pr.elem_weights = elem_weights;
  int rc = validate_problem(&pr);
  if (rc) return rc;
  if (!ref_nodes || !band) return fail_einval("null ref_nodes/band");
  return launch_band_tables(prob->K, prob->p, prob->q, ref_nodes, prob->weights,
                            prob->op != IGA_OP_MASS, vals, ders, band, prob->knots,
                            prob->knots ? elem_weights : nullptr, as_stream(stream));
}

int32_t iga_integrate_assemble(const iga_problem* prob, int32_t method, int32_t el_begin,
                               int32_t el_end, int32_t row_plane_begin, int32_t row_plane_end,
                               double* values, void* stream) {
  int rc = validate_problem(prob);
  if (rc) return rc;
  const int K = prob->K, p = prob->p, dim = prob->dim;
  const int64_t N = (int64_t)K + p;
  if (el_begin < 0 || el_end > K || el_end < el_begin)
    return fail_einval("element slab [%d, %d) outside [0, %d)", el_begin, el_end, K);
  if (row_plane_begin < 0 || row_plane_end > N || row_plane_end < row_plane_begin)
    return fail_einval("row planes [%d, %d) outside [0, %lld)", row_plane_begin, row_plane_end,
                       (long long)N);
  if (!values) return fail_einval("null values");
  cudaStream_t s = as_stream(stream);
  const int64_t plane_rows = dim == 3 ? N * N : N;
  const int64_t row_first = row_plane_begin * plane_rows, row_last = row_plane_end * plane_rows;
  const int64_t base = rowptr(dim, row_first, p, N);
  const int64_t nvals = rowptr(dim, row_last, p, N) - base;
  if (nvals == 0) return IGA_OK;
  if (method == IGA_METHOD_SEPARABLE) {
    if (dim != 3) {
      set_error("the separable method is implemented for dim=3 only");
      return IGA_EUNSUPPORTED;
    }
    if (prob->coef) return fail_einval("the separable method needs a scalar coefficient (coef == NULL)");
    KronArgs a;
    a.K = K; a.op = prob->op; a.el_begin = el_begin; a.el_end = el_end;
    a.wt = prob->knots ? prob->elem_weights : nullptr;
    a.plane_begin = row_plane_begin; a.plane_end = row_plane_end; a.base = base;
    a.jc = prob->jac * prob->coef_scalar; a.weights = prob->weights;
    a.V = prob->tables_v; a.D = prob->tables_d; a.values = values;
    a.band = reinterpret_cast<const double2*>(prob->band);
    return launch_kron(a, p, prob->q, s);
  }
  if (method == IGA_METHOD_SUMFACT_ASSEMBLED) {
    if (dim != 3) {
      set_error("assembled sum factorization is implemented for dim=3 only");
      return IGA_EUNSUPPORTED;
    }
    GsfArgs a;
    a.K = K; a.op = prob->op; a.el_begin = el_begin; a.el_end = el_end;
    a.wt = prob->knots ? prob->elem_weights : nullptr;
    a.plane_begin = row_plane_begin; a.plane_end = row_plane_end; a.tiles1 = 0;
    a.segs = 1; a.seg_len = K;
    a.base = base; a.jac = prob->jac; a.coef_scalar = prob->coef_scalar; a.coef = prob->coef;
    a.weights = prob->weights; a.V = prob->tables_v; a.D = prob->tables_d; a.values = values;
    return launch_gsf(a, p, prob->q, s);
  }
  if (method != IGA_METHOD_CLASSICAL && method != IGA_METHOD_SUMFACT)
    return fail_einval("unknown method %d", method);
  rc = check_cuda(cudaMemsetAsync(values, 0, sizeof(double) * nvals, s), "zero values");
  if (rc) return rc;
  ScatterArgs a;
  a.dim = dim; a.K = K; a.op = prob->op; a.el_begin = el_begin; a.el_end = el_end;
  a.wt = prob->knots ? prob->elem_weights : nullptr;
  a.row_first = row_first; a.row_last = row_last; a.base = base; a.jac = prob->jac;
  a.coef_scalar = prob->coef_scalar; a.coef = prob->coef; a.weights = prob->weights;
  a.V = prob->tables_v; a.D = prob->tables_d; a.values = values;
  return launch_scatter(a, method, p, prob->q, s);
}

int32_t iga_assemble_elements(int32_t dim, int32_t K, int32_t p, const double* mats,
                              int32_t row_plane_begin, int32_t row_plane_end, double* values,
                              void* stream) {
  if (dim != 2 && dim != 3) return fail_einval("dim must be 2 or 3");
  if (K < 1 || p < 0) return fail_einval("mesh must be >= 1 and degree >= 0");
  const int64_t N = (int64_t)K + p;
  if (row_plane_begin < 0 || row_plane_end > N || row_plane_end < row_plane_begin)
    return fail_einval("row planes outside [0, %lld)", (long long)N);
  if (!mats || !values) return fail_einval("null pointer");
  const int64_t plane_rows = dim == 3 ? N * N : N;
  const int64_t row_first = row_plane_begin * plane_rows;
  const int64_t nrows = (row_plane_end - row_plane_begin) * plane_rows;
  if (nrows == 0) return IGA_OK;
  const int64_t base = rowptr(dim, row_first, p, N);
  const int64_t threads = nrows * 32;
  k_assemble_elements<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
      dim, K, p, mats, row_first, nrows, base, values);
  return check_cuda(cudaGetLastError(), "iga_assemble_elements");
}

int32_t iga_spmv(int32_t dim, int32_t K, int32_t p, const double* values, const double* x,
                 double* y, void* stream) {
  if (dim != 2 && dim != 3) return fail_einval("dim must be 2 or 3");
  if (K < 1 || p < 0) return fail_einval("mesh must be >= 1 and degree >= 0");
  if (!values || !x || !y) return fail_einval("null pointer");
  const int64_t N = (int64_t)K + p;
  if (dim == 3) return dispatch_p_all<Spmv3Launch>(p, K, values, x, y, as_stream(stream));
  const int64_t nrows = N * N;
  const int64_t threads = nrows * 32;
  k_spmv<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(dim, K, p, values, x,
                                                                          y, nrows);
  return check_cuda(cudaGetLastError(), "iga_spmv");
}

}  // extern "C"
