// Timing harness for k_kron3 (C3 shape, or K from argv[1]): random tables, CUDA events.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2207_00280_b200/csrc/iga_kron.cu"
#include "../paper_2207_00280_b200/csrc/iga_abi.cu"


__global__ void fill_kernel(double* v, long long n, double x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) v[i] = x;
}

int main(int argc, char** argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 64, P = 3, Q = 4, M = 4;
  std::vector<double> V(K * M * Q), D(K * M * Q), w = {0.347854845137454, 0.652145154862546, 0.652145154862546, 0.347854845137454};
  for (auto& x : V) x = rand() / (double)RAND_MAX;
  for (auto& x : D) x = rand() / (double)RAND_MAX - 0.5;
  double *dV, *dD, *dw, *dval;
  cudaMalloc(&dV, V.size() * 8); cudaMalloc(&dD, D.size() * 8); cudaMalloc(&dw, 32);
  const long long N = K + P;
  const long long nnz = iga::rowptr3(N, 0, 0, P, N);
  cudaMalloc(&dval, nnz * 8);
  cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, D.data(), D.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), 32, cudaMemcpyHostToDevice);
  iga::KronArgs a{};
  a.K = K; a.op = 1; a.el_begin = 0; a.el_end = K; a.plane_begin = 0; a.plane_end = K + P;
  a.base = 0; a.jc = 1.0 / (8.0 * K * K * K); a.weights = dw; a.V = dV; a.D = dD; a.values = dval;
  void* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) iga::launch_kron(a, 3, 4, 0);
  float tot = 0; const int R = 10;
  for (int it = 0; it < R; ++it) {
    cudaMemsetAsync(flush, it, 256 << 20);
    cudaEventRecord(e0);
    iga::launch_kron(a, 3, 4, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
  }
  const double ms = tot / R;
  printf("K=%d nnz=%lld kernel %.4f ms  %.1f GB/s  err=%s\n", K, nnz, ms, nnz * 8 / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  // write-only bandwidth references on the same buffer
  for (int it = 0; it < 2; ++it) cudaMemsetAsync(dval, 0, nnz * 8);
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) cudaMemsetAsync(dval, it, nnz * 8);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float mms; cudaEventElapsedTime(&mms, e0, e1);
  printf("memset: %.1f GB/s\n", 5.0 * nnz * 8 / (mms * 1e-3) / 1e9);
  fill_kernel<<<148 * 8, 256>>>(dval, nnz, 1.0);
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) fill_kernel<<<148 * 8, 256>>>(dval, nnz, (double)it);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&mms, e0, e1);
  printf("fill STG.64 grid-stride: %.1f GB/s\n", 5.0 * nnz * 8 / (mms * 1e-3) / 1e9);
  return 0;
}
