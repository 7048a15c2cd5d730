// What store pattern reaches cudaMemset's write rate (7.0 TB/s at the C3 size, 764 MB)?
// Kernel fills by store width, grid shape and address order (grid-stride vs one contiguous
// range per CTA), against memset with a nonzero value (so not zero compression); L2
// flushed between launches.  Results: profiles/r01h_write_patterns.log.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void fill_gs(double2* p, size_t n, double v) {
  const double2 x = make_double2(v, v);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = x;
}
__global__ void fill_gs256(double* p, size_t n4, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(p + 4 * i), "d"(v) : "memory");
}
// one contiguous range per CTA, 16-byte stores, warps interleaved over it
__global__ void fill_blk(double2* p, size_t n, double v) {
  const double2 x = make_double2(v, v);
  const size_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = x;
}
// one contiguous range per CTA, 32-byte stores
__global__ void fill_blk256(double* p, size_t n4, double v) {
  const size_t lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    asm volatile("st.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(p + 4 * i), "d"(v) : "memory");
}

// one contiguous range per CTA written by TMA bulk stores of U doubles from one smem chunk
__global__ void tma_blk(double* v, size_t n, int U) {
  extern __shared__ __align__(128) double sm[];
  for (int i = threadIdx.x; i < U; i += blockDim.x) sm[i] = 1.5;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t lo = n * blockIdx.x / gridDim.x / 2 * 2, hi = n * (blockIdx.x + 1) / gridDim.x / 2 * 2;
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sm);
    for (size_t u = lo; u < hi; u += U) {
      const size_t cnt = hi - u < (size_t)U ? hi - u : U;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(v + u), "r"(sa),
                   "r"((unsigned)(cnt * 8)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const size_t bytes = 763551944ull / 32 * 32;
  void* d;
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
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 3) sum += ms;
    }
    printf("%-40s %.4f ms  %.1f GB/s\n", name, sum / 20, bytes / (sum / 20) / 1e6);
  };
  const size_t n16 = bytes / 16, n32 = bytes / 32;
  run("cudaMemset 0x3f", [&] { cudaMemsetAsync(d, 0x3f, bytes); });
  char nm[64];
  for (int g : {296, 1184, 4736, 9472, 18944})
    for (int U : {2048, 5488}) {
      snprintf(nm, 64, "blk TMA U=%dB %dx128", U * 8, g);
      cudaFuncSetAttribute(tma_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, U * 8);
      run(nm, [&] { tma_blk<<<g, 128, U * 8>>>((double*)d, bytes / 8, U); });
    }
  for (int g : {296, 1184, 4736, 9472}) {
    snprintf(nm, 64, "blk STG.128 %dx352", g);
    run(nm, [&] { fill_blk<<<g, 352>>>((double2*)d, n16, 1.5); });
  }
  for (int g : {296, 592, 1184, 2368, 4736})
    for (int t : {256, 512, 1024}) {
      snprintf(nm, 64, "gs STG.128 %dx%d", g, t);
      run(nm, [&] { fill_gs<<<g, t>>>((double2*)d, n16, 1.5); });
      snprintf(nm, 64, "gs STG.256 %dx%d", g, t);
      run(nm, [&] { fill_gs256<<<g, t>>>((double*)d, n32, 1.5); });
    }
  for (int g : {148, 296, 592, 1184, 2368, 4736, 9472})
    for (int t : {256, 512, 1024}) {
      snprintf(nm, 64, "blk STG.128 %dx%d", g, t);
      run(nm, [&] { fill_blk<<<g, t>>>((double2*)d, n16, 1.5); });
      snprintf(nm, 64, "blk STG.256 %dx%d", g, t);
      run(nm, [&] { fill_blk256<<<g, t>>>((double*)d, n32, 1.5); });
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
