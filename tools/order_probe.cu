// Does the ORDER in which a persistent grid writes a large array set its DRAM write rate?
// memset_probe.cu found many short-lived CTAs (each a 40 KB contiguous range, ~16+ waves)
// reach 7.0 TB/s while one persistent wave of contiguous per-CTA ranges tops out at 6.0 TB/s.
// Here one persistent wave of TMA bulk-store CTAs writes chunks of C bytes either as one
// contiguous range per CTA, dealt round-robin (chunk c -> CTA c mod G), or claimed from a
// global atomic counter (all CTAs move through the array together).  C3 CSR size, L2 flushed.
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_next;

template <int MODE>  // 0 contiguous, 1 round-robin, 2 atomic counter
__global__ void tma_fill(double* v, size_t n, int U, size_t nchunks) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long claim;
  for (int i = threadIdx.x; i < U; i += blockDim.x) sm[i] = 1.5;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sm);
  auto store = [&](size_t c) {
    const size_t u = c * U, cnt = n - u < (size_t)U ? n - u : U;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(v + u), "r"(sa),
                 "r"((unsigned)(cnt * 8)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  };
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      const size_t lo = nchunks * blockIdx.x / gridDim.x, hi = nchunks * (blockIdx.x + 1) / gridDim.x;
      for (size_t c = lo; c < hi; ++c) store(c);
    }
  } else if (MODE == 1) {
    if (threadIdx.x == 0)
      for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) store(c);
  } else {
    if (threadIdx.x == 0)
      for (;;) {
        const unsigned long long c = atomicAdd(&g_next, 1ull);
        if (c >= nchunks) break;
        store(c);
      }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  (void)claim;
}

int main() {
  const size_t bytes = 763551944ull / 32 * 32, n = bytes / 8;
  double* d;
  void* flush;
  cudaMalloc(&d, bytes);
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto fn) {
    float sum = 0;
    for (int i = 0; i < 23; ++i) {
      cudaMemsetAsync(flush, i, 256 << 20);
      unsigned long long z = 0;
      cudaMemcpyToSymbolAsync(g_next, &z, 8);
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 3) sum += ms;
    }
    printf("%-44s %.4f ms  %.1f GB/s\n", name, sum / 20, bytes / (sum / 20) / 1e6);
  };
  run("cudaMemset", [&] { cudaMemsetAsync(d, 0x3f, bytes); });
  char nm[96];
  const char* mn[3] = {"contiguous", "round-robin", "atomic"};
  for (int U : {2048, 5120, 13312})
    for (int g : {148, 296, 592})
      for (int mode = 0; mode < 3; ++mode) {
        const size_t nch = (n + U - 1) / U;
        snprintf(nm, 96, "TMA %-11s chunk %6dB grid %d", mn[mode], U * 8, g);
        auto f0 = tma_fill<0>, f1 = tma_fill<1>, f2 = tma_fill<2>;
        auto f = mode == 0 ? f0 : mode == 1 ? f1 : f2;
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, U * 8);
        run(nm, [&] { f<<<g, 32, U * 8>>>(d, n, U, nch); });
      }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
