// Fixed cost of a launch after an L2 flush: empty kernels with and without a large
// dynamic shared-memory footprint (SM L1/shared carveout change), alone and behind a
// tiny latency-bound kernel (the K1 -> k_kron3 pair of a separable step).
#include <cstdio>

__global__ void empty_k(int x) {
  extern __shared__ double s[];
  if (x == 12345) s[threadIdx.x] = 0;
}
__global__ void tiny_k(double* v) {
  double x = threadIdx.x;
  for (int i = 0; i < 40; ++i) x = 1.0 / (x + 1.0);
  v[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  double* v;
  cudaMalloc(&v, 1 << 20);
  const int big = 102848;
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    f();
    float tot = 0;
    const int R = 20;
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
    printf("%-52s %7.2f us\n", name, tot / R * 1e3);
  };
  run("empty 296x352, no smem", [&] { empty_k<<<296, 352, 0>>>(0); });
  run("empty 296x352, 102.8 KB smem", [&] { empty_k<<<296, 352, big>>>(0); });
  run("tiny 2x128", [&] { tiny_k<<<2, 128>>>(v); });
  run("tiny 2x128 + empty 102.8 KB", [&] {
    tiny_k<<<2, 128>>>(v);
    empty_k<<<296, 352, big>>>(0);
  });
  cudaFuncSetAttribute(tiny_k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  run("tiny (carveout 100) + empty 102.8 KB", [&] {
    tiny_k<<<2, 128>>>(v);
    empty_k<<<296, 352, big>>>(0);
  });
  cudaFuncSetAttribute(empty_k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  run("empty 102.8 KB (carveout 100)", [&] { empty_k<<<296, 352, big>>>(0); });
  run("empty 102.8 KB x2 back to back", [&] {
    empty_k<<<296, 352, big>>>(0);
    empty_k<<<296, 352, big>>>(0);
  });
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
