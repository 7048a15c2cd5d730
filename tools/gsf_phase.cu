// Phase timing harness for k_gsf3_p3 (C3 shape): builds the kernel with
// IGA_PHASE_TIMING=<block> and prints per-warp phase durations of steps 8..11.
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <algorithm>
#ifndef GSF_NOPHASE
#define IGA_PHASE_TIMING 300
#endif
#include "../paper_2207_00280_b200/csrc/iga_gsf_p3.cu"
#include "../paper_2207_00280_b200/csrc/iga_abi.cu"


int main() {
  const int K = 64, P = 3, Q = 4, M = 4;
  std::vector<double> V(K * M * Q), D(K * M * Q), w = {0.347854845137454, 0.652145154862546, 0.652145154862546, 0.347854845137454};
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
  for (int it = 0; it < 3; ++it) iga::launch_gsf_p3(a, 0);
  cudaEventRecord(e0);
  iga::launch_gsf_p3(a, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("kernel %.3f ms  err=%s\n", ms, cudaGetErrorString(cudaGetLastError()));
#ifdef GSF_NOPHASE
  return 0;
#else
  long long ph[4][16][3];
  cudaMemcpyFromSymbol(ph, iga::p3::g_phase, sizeof(ph));
  for (int s = 0; s < 4; ++s) {
    long long t0 = ph[s][0][2];
    long long amax = 0, bmax = 0, smid = 0, send = 0;
    for (int w = 0; w < 4; ++w) amax = std::max(amax, ph[s][w][0] - t0);
    for (int w = 4; w < 8; ++w) bmax = std::max(bmax, ph[s][w][0] - t0);
    for (int w = 8; w < 16; ++w) { smid = std::max(smid, ph[s][w][0] - t0); send = std::max(send, ph[s][w][1] - t0); }
    printf("iter %d: A_end %lld  B_end %lld  S_dmma_end %lld  S_flush_end %lld", s + 8, amax, bmax, smid, send);
    if (s < 3) printf("  | iteration %lld", ph[s + 1][0][2] - t0);
    printf("\n");
  }
  return 0;
#endif
}
