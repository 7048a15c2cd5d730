// Write-bandwidth ceiling for the C3 value array (95.4M doubles, 764 MB): how fast can
// a kernel fill it, by store width and by TMA bulk stores, against cudaMemset.
#include <cstdio>
#include <cstdlib>

__global__ void f64(double* v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] = 1.0;
}
__global__ void f128(double2* v, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    v[i] = make_double2(1.0, 1.0);
}
__global__ void f256(double* v, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    double* p = v + 4 * i;
    asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p), "d"(1.0) : "memory");
  }
}
// each CTA fills a smem chunk once, then bulk-stores it to successive units (round robin)
__global__ void tma(double* v, long long n, int U) {
  extern __shared__ __align__(128) double s[];
  for (int i = threadIdx.x; i < U; i += blockDim.x) s[i] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    for (long long u = blockIdx.x; u * U < n; u += gridDim.x) {
      const long long cnt = n - u * U < U ? n - u * U : U;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(v + u * U), "r"(sa),
                   "r"((unsigned)(cnt * 8))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 95443993LL;
  double* d;
  cudaMalloc(&d, (n + 64) * 8);
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    f();
    float tot = 0;
    const int R = 10;
    for (int i = 0; i < R; ++i) {
      cudaMemsetAsync(flush, i, 256 << 20);
      cudaEventRecord(a);
      f();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      tot += ms;
    }
    const double ms = tot / R;
    printf("%-36s %8.4f ms %7.1f GB/s\n", name, ms, n * 8 / (ms * 1e-3) / 1e9);
  };
  run("cudaMemset", [&] { cudaMemsetAsync(d, 0, n * 8); });
  for (int bpsm : {2, 4, 8}) {
    char nm[96];
    snprintf(nm, sizeof nm, "STG.64  grid-stride %dx148x256", bpsm);
    run(nm, [&] { f64<<<148 * bpsm, 256>>>(d, n); });
    snprintf(nm, sizeof nm, "STG.128 grid-stride %dx148x256", bpsm);
    run(nm, [&] { f128<<<148 * bpsm, 256>>>((double2*)d, n / 2); });
    snprintf(nm, sizeof nm, "STG.256 grid-stride %dx148x256", bpsm);
    run(nm, [&] { f256<<<148 * bpsm, 256>>>(d, n / 4); });
  }
  for (int U : {2048, 4096, 8192}) {
    cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, U * 8);
    for (int bpsm : {1, 2, 4}) {
      char nm[96];
      snprintf(nm, sizeof nm, "TMA bulk U=%d B %dx148", U * 8, bpsm);
      run(nm, [&] { tma<<<148 * bpsm, 128, U * 8>>>(d, n, U); });
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
