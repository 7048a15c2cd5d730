// Conjugate gradients on the device: the solve of the heat demo's implicit step
// (heat.HeatProblem._solve, heat.py:168-175: scipy cg, rtol 1e-10, maxiter 10 n), with the
// operator applied by iga_spmv (assembled structured CSR) or iga_apply (matrix-free
// alpha M + beta S).  SURVEY.md 8(f) row 2.
//
// Each iteration is four stream-ordered launches and no host synchronisation:
//   apply(p) -> Ap;  k_cg_dot: per-block partial sums of p.Ap;
//   k_cg_step: every block sums the partials (fixed order), alpha = rr / pAp,
//              x += alpha p, r -= alpha Ap, per-block partial sums of r.r;
//   k_cg_dir:  rr' = sum of partials, p = r + (rr' / rr) p, block 0 stores rr' and the
//              convergence flag ||r|| <= rtol ||b|| for the next iteration.
// The scalars live in a small device state with parity-indexed slots (iteration i reads slot
// i & 1 and writes slot (i + 1) & 1), so no launch reads a value another block of the same
// launch writes.  Once converged, every kernel returns at entry: the iterations launched
// between two host checks leave x unchanged.  The host reads the 32-byte state every
// `check_every` iterations.  Reductions use a fixed grid, a fixed per-thread stride order
// and a fixed shuffle tree, so the solution is bitwise reproducible.
#include "iga_common.cuh"

namespace iga {
namespace cg {

constexpr int kBlocks = 296, kThreads = 256;  // 2 CTAs per SM on 148 SMs

struct State {
  double rr[2];     // r.r entering iteration i (slot i & 1)
  double tol;       // rtol ||b||
  int32_t conv[2];  // converged before iteration i (slot i & 1)
  int64_t iters;    // iterations done when convergence was reached (-1: not yet)
};

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double part[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) part[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) s += part[i];
  return s;  // valid in thread 0
}

// every block sums the kBlocks partials in the same order (thread 0's result broadcast)
__device__ __forceinline__ double sum_partials(const double* part) {
  __shared__ double tot;
  double v = 0.0;
  for (int i = threadIdx.x; i < kBlocks; i += kThreads) v += part[i];
  const double s = block_sum(v);
  if (threadIdx.x == 0) tot = s;
  __syncthreads();
  return tot;
}

// r = b - Ap, p = r; partials of r.r and b.b
__global__ void __launch_bounds__(kThreads) k_cg_init(int64_t n, const double* b, const double* Ap,
                                                      double* r, double* p, double* prr,
                                                      double* pbb) {
  double rr = 0.0, bb = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)kBlocks * kThreads) {
    const double bi = b[i], ri = bi - Ap[i];
    r[i] = ri;
    p[i] = ri;
    rr = fma(ri, ri, rr);
    bb = fma(bi, bi, bb);
  }
  const double s0 = block_sum(rr);
  __syncthreads();
  const double s1 = block_sum(bb);
  if (threadIdx.x == 0) {
    prr[blockIdx.x] = s0;
    pbb[blockIdx.x] = s1;
  }
}

__global__ void __launch_bounds__(kThreads) k_cg_init_fin(const double* prr, const double* pbb,
                                                          double rtol, State* st) {
  const double rr = sum_partials(prr);
  const double bb = sum_partials(pbb);
  if (threadIdx.x == 0) {
    st->rr[0] = rr;
    st->tol = rtol * sqrt(bb);
    st->conv[0] = sqrt(rr) <= st->tol;
    st->conv[1] = 0;
    st->iters = st->conv[0] ? 0 : -1;
  }
}

__global__ void __launch_bounds__(kThreads) k_cg_dot(int64_t n, const double* p, const double* Ap,
                                                     double* ppap, const State* st, int slot) {
  if (st->conv[slot]) return;
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)kBlocks * kThreads)
    v = fma(p[i], Ap[i], v);
  const double s = block_sum(v);
  if (threadIdx.x == 0) ppap[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_cg_step(int64_t n, const double* p, const double* Ap,
                                                      double* x, double* r, const double* ppap,
                                                      double* prr, const State* st, int slot) {
  if (st->conv[slot]) return;
  const double alpha = st->rr[slot] / sum_partials(ppap);
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)kBlocks * kThreads) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    v = fma(ri, ri, v);
  }
  const double s = block_sum(v);
  if (threadIdx.x == 0) prr[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) k_cg_dir(int64_t n, const double* r, double* p,
                                                     const double* prr, State* st, int slot,
                                                     int64_t it) {
  const int next = slot ^ 1;
  if (st->conv[slot]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->conv[next] = 1;
      st->rr[next] = st->rr[slot];
    }
    return;
  }
  const double rr_new = sum_partials(prr);
  const double beta = rr_new / st->rr[slot];
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n; i += (int64_t)kBlocks * kThreads)
    p[i] = fma(beta, p[i], r[i]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rr[next] = rr_new;
    const int c = sqrt(rr_new) <= st->tol;
    st->conv[next] = c;
    if (c) st->iters = it + 1;
  }
}

}  // namespace cg
}  // namespace iga

using namespace iga;

extern "C" {

int64_t iga_cg_work_size(int64_t n) { return n < 1 ? -1 : 3 * n + 3 * cg::kBlocks + 8; }

int32_t iga_cg(int32_t dim, int32_t K, int32_t p, const double* values, const iga_problem* prob,
               double alpha, double beta, int64_t n, const double* b, double* x, double* work,
               double rtol, int64_t maxiter, int32_t check_every, int64_t* iters, void* stream) {
  if (n < 1) return fail_einval("system size must be >= 1");
  if (!b || !x || !work || !iters) return fail_einval("null pointer");
  if (!values && !prob) return fail_einval("need assembled values or a matrix-free problem");
  if (rtol < 0.0) return fail_einval("rtol must be >= 0");
  if (maxiter < 0) return fail_einval("maxiter must be >= 0");
  if (check_every < 1) return fail_einval("check_every must be >= 1");
  {
    const int d = values ? dim : 3;
    const int64_t N = values ? (int64_t)K + p : (int64_t)prob->K + prob->p;
    int64_t want = 1;
    for (int i = 0; i < d; ++i) want *= N;
    if ((d != 2 && d != 3) || N < 1 || n != want)
      return fail_einval("system size %lld does not match the operator's %lld dofs", (long long)n,
                         (long long)want);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* r = work;
  double* pv = r + n;
  double* Ap = pv + n;
  double* parts = Ap + n;
  double* ppap = parts;
  double* prr = ppap + cg::kBlocks;
  double* pbb = prr + cg::kBlocks;
  cg::State* st = reinterpret_cast<cg::State*>(pbb + cg::kBlocks);
  static_assert(sizeof(cg::State) <= 8 * sizeof(double), "state fits the work tail");
  auto apply = [&](const double* v, double* out) -> int32_t {
    if (values) return iga_spmv(dim, K, p, values, v, out, stream);
    return iga_apply(prob, alpha, beta, v, out, stream);
  };
  int32_t rc = apply(x, Ap);
  if (rc) return rc;
  cg::k_cg_init<<<cg::kBlocks, cg::kThreads, 0, s>>>(n, b, Ap, r, pv, prr, pbb);
  cg::k_cg_init_fin<<<1, cg::kThreads, 0, s>>>(prr, pbb, rtol, st);
  rc = check_cuda(cudaGetLastError(), "iga_cg init");
  if (rc) return rc;
  cg::State h{};
  for (int64_t it = 0;; ++it) {
    if (it % check_every == 0 || it == maxiter) {
      rc = check_cuda(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s), "iga_cg state");
      if (rc) return rc;
      rc = check_cuda(cudaStreamSynchronize(s), "iga_cg sync");
      if (rc) return rc;
      if (h.iters >= 0) {
        *iters = h.iters;
        return IGA_OK;
      }
      if (it == maxiter) {
        *iters = maxiter;
        set_error("conjugate gradients did not converge in %lld iterations", (long long)maxiter);
        return IGA_ENOCONV;
      }
    }
    const int slot = (int)(it & 1);
    rc = apply(pv, Ap);
    if (rc) return rc;
    cg::k_cg_dot<<<cg::kBlocks, cg::kThreads, 0, s>>>(n, pv, Ap, ppap, st, slot);
    cg::k_cg_step<<<cg::kBlocks, cg::kThreads, 0, s>>>(n, pv, Ap, x, r, ppap, prr, st, slot);
    cg::k_cg_dir<<<cg::kBlocks, cg::kThreads, 0, s>>>(n, r, pv, prr, st, slot, it);
    rc = check_cuda(cudaGetLastError(), "iga_cg iteration");
    if (rc) return rc;
  }
}

}  // extern "C"
