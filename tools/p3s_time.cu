// Timing harness for k_gsf3_p3 variants (C3 shape, c = 1): build with -D overrides of
// the kernel's tuning macros (P3_NWB, P3_NWS, ...) and print the mean launch time of 20
// launches after warm-up, plus a checksum so variants can be compared for equality.
#include <cstdio>
#include <vector>
#include <cstdlib>
#include "../paper_2207_00280_b200/csrc/iga_gsf_p3s.cu"
#include "../paper_2207_00280_b200/csrc/iga_abi.cu"

int main() {
  const int K = 64, P = 3, Q = 4, M = 4;
  std::vector<double> V(K * M * Q), D(K * M * Q);
  std::vector<double> w = {0.347854845137454, 0.652145154862546, 0.652145154862546, 0.347854845137454};
  srand(1);
  for (auto& x : V) x = rand() / (double)RAND_MAX;
  for (auto& x : D) x = rand() / (double)RAND_MAX - 0.5;
  double *dV, *dD, *dw, *dval;
  cudaMalloc(&dV, V.size() * 8); cudaMalloc(&dD, D.size() * 8); cudaMalloc(&dw, 32);
  const long long nnz = 95443993;
  cudaMalloc(&dval, nnz * 8);
  cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dD, D.data(), D.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, w.data(), 32, cudaMemcpyHostToDevice);
  iga::GsfArgs a{};
  a.K = K; a.op = 1; a.el_begin = 0; a.el_end = K; a.plane_begin = 0; a.plane_end = K + P; a.segs = 1; a.seg_len = K;
  a.base = 0; a.jac = 1.0 / (8.0 * K * K * K); a.coef_scalar = 1.0; a.coef = nullptr;
  a.weights = dw; a.V = dV; a.D = dD; a.values = dval;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) iga::launch_gsf_p3s(a, 0);
  const int n = 20;
  cudaEventRecord(e0);
  for (int it = 0; it < n; ++it) iga::launch_gsf_p3s(a, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> h(nnz);
  cudaMemcpy(h.data(), dval, nnz * 8, cudaMemcpyDeviceToHost);
  double cs = 0; for (long long i = 0; i < nnz; i += 7) cs += h[i] * (1 + (i % 13));
  printf("%s kernel %.4f ms  checksum %.17g err=%s\n", VARIANT, ms / n, cs, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
