// C-ABI plumbing: error state, version, host-side CSR arithmetic, small
// vector kernels, and the K1 (basis tables) and K5 (CSR pattern) kernels.
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>

#include "iga_dispatch.cuh"

namespace iga {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail_einval(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return IGA_EINVAL;
}

int check_cuda(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return IGA_OK;
  set_error("%s: %s", what, cudaGetErrorString(err));
  return IGA_ECUDA;
}

static std::mutex g_launch_mu;

cudaError_t smem_attr_once(const void* fn, size_t bytes, bool max_carveout) {
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_launch_mu);
  auto it = done.find({fn, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && max_carveout)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done[{fn, dev}] = bytes;
  return e;
}

int sm_count() {
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> g(g_launch_mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n;
  return n;
}

int blocks_per_sm_once(const void* fn, int threads, size_t smem) {
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  std::lock_guard<std::mutex> g(g_launch_mu);
  auto key = std::make_tuple(fn, dev, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess || n < 1)
    n = 1;
  cache[key] = n;
  return n;
}

// ------------------------------------------------------------------ K1
// One thread per (element e, point k): x = e*h + (ref_k + 1)*(h/2), then the
// bottom-up Cox-de Boor triangle (bitwise equal to splines.py:108-161).
template <int P>
__global__ void k_mesh_tables(int K, int q, const double* __restrict__ ref, double* __restrict__ V,
                              double* __restrict__ D, const double* __restrict__ knots,
                              const double* __restrict__ w, double* __restrict__ wt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * q) return;
  const int e = t / q, k = t % q;
  const double x = map_node(e, ref[k], K, P, knots);
  double vals[P + 1], ders[P + 1];
  cox_de_boor<P>(e, x, K, vals, D ? ders : nullptr, knots);
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    if (V) V[((size_t)e * (P + 1) + r) * q + k] = vals[r];
    if (D) D[((size_t)e * (P + 1) + r) * q + k] = ders[r];
  }
  if (wt) {  // w_k * (h_e / 2): the element's Jacobian folded into this axis' weights
    const double h = sub(__ldg(knots + P + e + 1), __ldg(knots + P + e));
    wt[e * q + k] = mul(w[k], dvd(h, 2.0));
  }
}

template <int P>
struct MeshTablesLaunch {
  static int run(int K, int q, const double* ref, double* V, double* D, const double* knots,
                 const double* w, double* wt, cudaStream_t s) {
    const int n = K * q;
    k_mesh_tables<P><<<(n + 127) / 128, 128, 0, s>>>(K, q, ref, V, D, knots, w, wt);
    return check_cuda(cudaGetLastError(), "iga_mesh_tables launch");
  }
};

template <int P>
__global__ void k_basis_eval(int K, const double* __restrict__ knots, int64_t n,
                             const int32_t* __restrict__ elem, const double* __restrict__ x,
                             double* __restrict__ V, double* __restrict__ D) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double vals[P + 1], ders[P + 1];
  cox_de_boor<P>(elem[t], x[t], K, vals, D ? ders : nullptr, knots);
#pragma unroll
  for (int r = 0; r <= P; ++r) {
    V[t * (P + 1) + r] = vals[r];
    if (D) D[t * (P + 1) + r] = ders[r];
  }
}

template <int P>
struct BasisEvalLaunch {
  static int run(int K, const double* knots, int64_t n, const int32_t* elem, const double* x,
                 double* V, double* D, cudaStream_t s) {
    if (n == 0) return IGA_OK;
    k_basis_eval<P><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(K, knots, n, elem, x, V, D);
    return check_cuda(cudaGetLastError(), "iga_basis_eval launch");
  }
};

// eval_basis / eval_basis_order0 (splines.py:78-118) on any non-decreasing knot
// vector: B_{i,order}(x) by the same two-term triangle as cox_de_boor, bottom-up over
// the order+1 level-0 spans i .. i+order (the value of B_{i,r}(x) does not depend on the
// recursion path, and every level uses _cox's expression and 0/0 := 0 branches).
constexpr int kMaxEvalOrder = 31;
__global__ void k_eval_basis(const double* __restrict__ t, int nt, int order, int64_t n,
                             const int32_t* __restrict__ index, const double* __restrict__ xs,
                             double* __restrict__ out) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int i = index[u];
  const double x = xs[u];
  if (i < 0 || i > nt - order - 2) {  // the host raises IndexError first; never read outside t
    out[u] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  const double tl = t[nt - 1];
  double N[kMaxEvalOrder + 1];
  for (int j = 0; j <= order; ++j) {  // order 0 with the closed last non-empty span
    const double a = t[i + j], b = t[i + j + 1];
    N[j] = (a <= x && x < b) || (x == tl && a < b && b == tl) ? 1.0 : 0.0;
  }
  for (int q = 1; q <= order; ++q)
    for (int j = 0; j <= order - q; ++j) {
      const int ii = i + j;
      double v = 0.0;
      const double d_left = sub(t[ii + q], t[ii]);
      if (d_left > 0.0) v = add(v, mul(dvd(sub(x, t[ii]), d_left), N[j]));
      const double d_right = sub(t[ii + q + 1], t[ii + 1]);
      if (d_right > 0.0) v = add(v, mul(dvd(sub(t[ii + q + 1], x), d_right), N[j + 1]));
      N[j] = v;
    }
  out[u] = N[0];
}

// ------------------------------------------------------------------ K5
// indptr: one thread per row (closed-form row pointer); indices: one warp per
// row writes its <= (2p+1)^dim sorted columns, coalesced.
__global__ void k_csr_indptr(int dim, int p, int64_t N, int64_t row_begin, int64_t nrows,
                             int64_t base, int64_t* __restrict__ indptr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nrows) return;
  indptr[t] = rowptr(dim, row_begin + t, p, N) - base;
}

__global__ void k_csr_indices(int dim, int p, int64_t N, int64_t row_begin, int64_t nrows,
                              int64_t base, int32_t* __restrict__ indices) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nrows) return;
  const int64_t row = row_begin + warp;
  int64_t I[3];
  if (dim == 3) {
    I[0] = row / (N * N); I[1] = (row / N) % N; I[2] = row % N;
  } else {
    I[0] = row / N; I[1] = row % N; I[2] = 0;
  }
  int64_t lo[3], c[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = d < dim ? band_lo(I[d], p) : 0;
    c[d] = d < dim ? band_cnt(I[d], p, N) : 1;
  }
  const int64_t cnt = c[0] * c[1] * c[2];
  const int64_t off = rowptr(dim, row, p, N) - base;
  for (int64_t j = lane; j < cnt; j += 32) {
    const int64_t a = j / (c[1] * c[2]), b = (j / c[2]) % c[1], cc = j % c[2];
    int64_t col;
    if (dim == 3)
      col = ((lo[0] + a) * N + lo[1] + b) * N + lo[2] + cc;
    else
      col = (lo[0] + a) * N + lo[1] + b;
    indices[off + j] = (int32_t)col;
  }
}

__global__ void k_axpy(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (; i + 1 < n; i += stride) {
    y[i] += x[i];
    y[i + 1] += x[i + 1];
  }
  if (i < n) y[i] += x[i];
}

int64_t n_rows(int dim, int K, int p) {
  const int64_t N = (int64_t)K + p;
  return dim == 3 ? N * N * N : N * N;
}

}  // namespace iga

using namespace iga;

extern "C" {

const char* iga_last_error(void) { return g_err; }

int32_t iga_eval_basis(const double* knots, int32_t n_knots, int32_t order, int64_t n,
                       const int32_t* index, const double* x, double* out, void* stream) {
  if (n < 0) return fail_einval("negative point count");
  if (order < 0 || order > kMaxEvalOrder)
    return fail_einval("order %d outside [0, %d]", order, kMaxEvalOrder);
  if (n_knots < order + 2) return fail_einval("%d knots cannot carry order %d", n_knots, order);
  if (n == 0) return IGA_OK;
  if (!knots || !index || !x || !out) return fail_einval("null pointer");
  k_eval_basis<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(knots, n_knots, order,
                                                                          n, index, x, out);
  return check_cuda(cudaGetLastError(), "iga_eval_basis launch");
}

int32_t iga_abi_version(void) { return IGA_ABI_VERSION; }

int32_t iga_mesh_tables(int32_t K, int32_t p, int32_t q, const double* ref_nodes, double* vals,
                        double* ders, void* stream) {
  if (K < 1) return fail_einval("element count must be >= 1, got %d", K);
  if (p < 0) return fail_einval("degree must be >= 0, got %d", p);
  if (q < 1 || q > kMaxQ) return fail_einval("quadrature points q=%d outside 1..%d", q, kMaxQ);
  if (!ref_nodes || !vals) return fail_einval("null pointer");
  return dispatch_p_all<MeshTablesLaunch>(p, K, q, ref_nodes, vals, ders, nullptr, nullptr,
                                          nullptr, as_stream(stream));
}

int32_t iga_mesh_tables_general(int32_t K, int32_t p, int32_t q, const double* knots,
                                const double* ref_nodes, const double* weights, double* vals,
                                double* ders, double* elem_weights, void* stream) {
  if (K < 1) return fail_einval("element count must be >= 1, got %d", K);
  if (p < 0) return fail_einval("degree must be >= 0, got %d", p);
  if (q < 1 || q > kMaxQ) return fail_einval("quadrature points q=%d outside 1..%d", q, kMaxQ);
  if (!knots || !ref_nodes) return fail_einval("null pointer");
  if (elem_weights && !weights) return fail_einval("elem_weights need the reference weights");
  return dispatch_p_all<MeshTablesLaunch>(p, K, q, ref_nodes, vals, ders, knots, weights,
                                          elem_weights, as_stream(stream));
}

int32_t iga_basis_eval(int32_t K, int32_t p, const double* knots, int64_t n,
                       const int32_t* elem, const double* x, double* vals, double* ders,
                       void* stream) {
  if (K < 1) return fail_einval("element count must be >= 1, got %d", K);
  if (p < 0) return fail_einval("degree must be >= 0, got %d", p);
  if (n < 0) return fail_einval("negative point count");
  if (n > 0 && (!elem || !x || !vals)) return fail_einval("null pointer");
  return dispatch_p_all<BasisEvalLaunch>(p, K, knots, n, elem, x, vals, ders, as_stream(stream));
}

int64_t iga_csr_nnz(int32_t dim, int32_t K, int32_t p, int64_t row_begin, int64_t row_end) {
  if ((dim != 2 && dim != 3) || K < 1 || p < 0) return -1;
  const int64_t N = (int64_t)K + p;
  const int64_t nr = n_rows(dim, K, p);
  if (row_begin < 0 || row_end < row_begin || row_end > nr) return -1;
  return rowptr(dim, row_end, p, N) - rowptr(dim, row_begin, p, N);
}

int32_t iga_csr_pattern(int32_t dim, int32_t K, int32_t p, int64_t row_begin, int64_t row_end,
                        int64_t* indptr, int32_t* indices, void* stream) {
  if (dim != 2 && dim != 3) return fail_einval("dim must be 2 or 3, got %d", dim);
  if (K < 1 || p < 0) return fail_einval("mesh must be >= 1 and degree >= 0");
  const int64_t N = (int64_t)K + p;
  const int64_t nr = n_rows(dim, K, p);
  if (row_begin < 0 || row_end < row_begin || row_end > nr)
    return fail_einval("row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                       (long long)row_end, (long long)nr);
  if (N > INT32_MAX / N / (dim == 3 ? N : 1))
    return fail_einval("column ids exceed int32");
  const int64_t nrows = row_end - row_begin;
  const int64_t base = rowptr(dim, row_begin, p, N);
  cudaStream_t s = as_stream(stream);
  if (indptr) {
    k_csr_indptr<<<(unsigned)((nrows + 1 + 255) / 256), 256, 0, s>>>(dim, p, N, row_begin, nrows,
                                                                     base, indptr);
    int rc = check_cuda(cudaGetLastError(), "iga_csr_pattern indptr");
    if (rc) return rc;
  }
  if (indices && nrows > 0) {
    const int64_t threads = nrows * 32;
    k_csr_indices<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(dim, p, N, row_begin, nrows,
                                                                    base, indices);
    return check_cuda(cudaGetLastError(), "iga_csr_pattern indices");
  }
  return IGA_OK;
}

int32_t iga_axpy(int64_t n, const double* x, double* y, void* stream) {
  if (n < 0) return fail_einval("negative length");
  if (n == 0) return IGA_OK;
  if (!x || !y) return fail_einval("null pointer");
  int64_t blocks = (n / 2 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_axpy<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(n, x, y);
  return check_cuda(cudaGetLastError(), "iga_axpy");
}

}  // extern "C"
