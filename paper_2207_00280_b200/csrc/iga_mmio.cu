// Matrix Market export of the assembled matrix, streamed
// from the device in row blocks: the replacement of assembly.write_matrix_market
// (assembly.py:118-120, scipy.io.mmwrite(path, coo, symmetry="symmetric"), called by
// cli.cmd_export, cli.py:292-297) without materialising the host CSR.
//
// Output is byte-identical to scipy 1.18's mmwrite of the same matrix: the header
// "%%MatrixMarket matrix coordinate real symmetric", a "%" line, "n n nnz_lower",
// then the lower-triangle entries (column <= row) in CSR order as "i j v" (1-based),
// v in shortest round-trip digits, scientific "d.dddE<exp>" with the exponent dropped
// when it is 0 ("2", "-0", "1.235E2", "5E-1").
//
// Pipeline: row blocks of ~4M values are copied device->host into two pinned
// buffers (one cudaMemcpyAsync each) while the previous block is formatted by a pool
// of host threads into per-thread text buffers, which are written in order.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "iga_dispatch.cuh"

namespace iga {
namespace mm {

// shortest round-trip value in scipy/fast_matrix_market style
inline char* put_value(char* o, double v) {
  char tmp[40];
  auto r = std::to_chars(tmp, tmp + sizeof(tmp), v, std::chars_format::scientific);
  const char* e = static_cast<const char*>(std::memchr(tmp, 'e', r.ptr - tmp));
  if (!e) {  // inf / nan
    std::memcpy(o, tmp, r.ptr - tmp);
    return o + (r.ptr - tmp);
  }
  std::memcpy(o, tmp, e - tmp);
  o += e - tmp;
  int ex = 0;
  std::from_chars(e + 1 + (e[1] == '+'), r.ptr, ex);
  if (ex != 0) {
    *o++ = 'E';
    auto r2 = std::to_chars(o, o + 8, ex);
    o = r2.ptr;
  }
  return o;
}

inline char* put_int(char* o, int64_t v) { return std::to_chars(o, o + 24, v).ptr; }

struct Shape {
  int dim, K, p;
  int64_t N, rows;
};

// lower-triangle entries of global row `row` whose values start at vals (CSR order)
inline char* format_row(const Shape& s, int64_t row, const double* vals, char* o) {
  const int64_t N = s.N;
  int64_t I[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, c[3] = {1, 1, 1};
  if (s.dim == 3) {
    I[0] = row / (N * N); I[1] = (row / N) % N; I[2] = row % N;
  } else {
    I[1] = row / N; I[2] = row % N;
  }
  for (int d = 3 - s.dim; d < 3; ++d) {
    lo[d] = band_lo(I[d], s.p);
    c[d] = band_cnt(I[d], s.p, N);
  }
  int64_t j = 0;
  for (int64_t a = 0; a < c[0]; ++a)
    for (int64_t b = 0; b < c[1]; ++b)
      for (int64_t k = 0; k < c[2]; ++k, ++j) {
        const int64_t col = s.dim == 3 ? ((lo[0] + a) * N + lo[1] + b) * N + lo[2] + k
                                       : (lo[1] + b) * N + lo[2] + k;
        if (col > row) continue;
        o = put_int(o, row + 1);
        *o++ = ' ';
        o = put_int(o, col + 1);
        *o++ = ' ';
        o = put_value(o, vals[j]);
        *o++ = '\n';
      }
  return o;
}

constexpr size_t kMaxLine = 2 * 21 + 32 + 3;  // two int64, one value, separators

// Format rows [r0, r1) whose values start at `vals` (value index v0 = rowptr(r0)) with
// `threads` host threads, append to f in row order.
int format_block(const Shape& s, int64_t r0, int64_t r1, const double* vals, int64_t v0,
                 int threads, std::vector<std::vector<char>>& bufs, FILE* f) {
  const int64_t nr = r1 - r0;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(threads, nr));
  std::vector<std::thread> pool;
  std::vector<size_t> used(T, 0);
  bufs.resize(T);
  auto work = [&](int t) {
    const int64_t a = r0 + nr * t / T, b = r0 + nr * (t + 1) / T;
    const int64_t va = rowptr(s.dim, a, s.p, s.N), vb = rowptr(s.dim, b, s.p, s.N);
    std::vector<char>& buf = bufs[t];
    const size_t need = (size_t)(vb - va) * kMaxLine + 64;
    if (buf.size() < need) buf.resize(need);
    char* o = buf.data();
    int64_t v = va;
    for (int64_t r = a; r < b; ++r) {
      const int64_t vn = rowptr(s.dim, r + 1, s.p, s.N);
      o = format_row(s, r, vals + (v - v0), o);
      v = vn;
    }
    used[t] = (size_t)(o - buf.data());
  };
  for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int t = 0; t < T; ++t)
    if (used[t] && std::fwrite(bufs[t].data(), 1, used[t], f) != used[t]) return -1;
  return 0;
}

int write_header(const Shape& s, FILE* f) {
  const int64_t nnz = rowptr(s.dim, s.rows, s.p, s.N);
  const int64_t lower = (nnz + s.rows) / 2;  // symmetric pattern: diagonal + half the rest
  return std::fprintf(f, "%%%%MatrixMarket matrix coordinate real symmetric\n%%\n%lld %lld %lld\n",
                      (long long)s.rows, (long long)s.rows, (long long)lower) > 0
             ? 0
             : -1;
}

int check_shape(int dim, int K, int p, Shape& s) {
  if (dim != 2 && dim != 3) return fail_einval("dim must be 2 or 3");
  if (K < 1 || p < 0) return fail_einval("mesh must be >= 1 and degree >= 0");
  s.dim = dim; s.K = K; s.p = p;
  s.N = (int64_t)K + p;
  s.rows = dim == 3 ? s.N * s.N * s.N : s.N * s.N;
  return IGA_OK;
}

}  // namespace mm
}  // namespace iga

using namespace iga;

extern "C" int32_t iga_write_matrix_market_host(int32_t dim, int32_t K, int32_t p,
                                                const double* values, const char* path,
                                                int32_t threads) {
  mm::Shape s;
  int rc = mm::check_shape(dim, K, p, s);
  if (rc) return rc;
  if (!values || !path) return fail_einval("null pointer");
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail_einval("cannot open %s for writing", path);
  std::vector<std::vector<char>> bufs;
  rc = mm::write_header(s, f);
  const int64_t step = std::max<int64_t>(1, (int64_t)(4 << 20) / ((2 * p + 1) * (2 * p + 1) * (dim == 3 ? 2 * p + 1 : 1)));
  for (int64_t r0 = 0; rc == 0 && r0 < s.rows; r0 += step) {
    const int64_t r1 = std::min(s.rows, r0 + step);
    const int64_t v0 = rowptr(dim, r0, p, s.N);
    rc = mm::format_block(s, r0, r1, values + v0, v0, threads > 0 ? threads : 1, bufs, f);
  }
  if (std::fclose(f) != 0) rc = -1;
  if (rc) return fail_einval("write to %s failed", path);
  return IGA_OK;
}

extern "C" int32_t iga_write_matrix_market(int32_t dim, int32_t K, int32_t p, const double* values,
                                           const char* path, int32_t threads, void* stream) {
  mm::Shape s;
  int rc = mm::check_shape(dim, K, p, s);
  if (rc) return rc;
  if (!values || !path) return fail_einval("null pointer");
  cudaStream_t st = as_stream(stream);
  const int64_t per_row = (int64_t)(2 * p + 1) * (2 * p + 1) * (dim == 3 ? 2 * p + 1 : 1);
  const int64_t step = std::max<int64_t>(1, (int64_t)(4 << 20) / per_row);  // rows per block
  const size_t cap = (size_t)(step * per_row);
  double* host[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    rc = check_cuda(cudaMallocHost(&host[b], cap * sizeof(double)), "pinned staging");
    if (!rc) rc = check_cuda(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
    if (rc) break;
  }
  FILE* f = rc ? nullptr : std::fopen(path, "wb");
  if (!rc && !f) rc = fail_einval("cannot open %s for writing", path);
  std::vector<std::vector<char>> bufs;
  if (!rc && mm::write_header(s, f)) rc = fail_einval("write to %s failed", path);
  const int64_t nblk = (s.rows + step - 1) / step;
  auto enqueue = [&](int64_t blk) {
    const int64_t r0 = blk * step, r1 = std::min(s.rows, r0 + step);
    const int64_t v0 = rowptr(dim, r0, p, s.N), v1 = rowptr(dim, r1, p, s.N);
    int e = check_cuda(cudaMemcpyAsync(host[blk & 1], values + v0, (size_t)(v1 - v0) * sizeof(double),
                                       cudaMemcpyDeviceToHost, st),
                       "D2H block");
    if (!e) e = check_cuda(cudaEventRecord(ev[blk & 1], st), "event record");
    return e;
  };
  if (!rc && nblk > 0) rc = enqueue(0);
  for (int64_t blk = 0; !rc && blk < nblk; ++blk) {
    // the copy of block blk+1 overlaps the formatting of block blk
    if (blk + 1 < nblk) rc = enqueue(blk + 1);
    if (!rc) rc = check_cuda(cudaEventSynchronize(ev[blk & 1]), "D2H wait");
    if (rc) break;
    const int64_t r0 = blk * step, r1 = std::min(s.rows, r0 + step);
    const int64_t v0 = rowptr(dim, r0, p, s.N);
    if (mm::format_block(s, r0, r1, host[blk & 1], v0, threads > 0 ? threads : 1, bufs, f))
      rc = fail_einval("write to %s failed", path);
  }
  if (f && std::fclose(f) != 0 && !rc) rc = fail_einval("write to %s failed", path);
  cudaStreamSynchronize(st);  // no copy may still target the staging buffers
  for (int b = 0; b < 2; ++b) {
    if (host[b]) cudaFreeHost(host[b]);
    if (ev[b]) cudaEventDestroy(ev[b]);
  }
  return rc;
}
