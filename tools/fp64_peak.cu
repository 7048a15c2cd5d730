// FP64 peak microbenchmark for B200 (sm_100a): DFMA loop and DMMA.8x8x4 loop.
// Results go to MEASURED_FP64.json (via tools/fp64_peak.py) and DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 123.456) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = k; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      dfma_loop<8><<<blocks, tpb>>>(d, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, tpb>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)blocks * tpb;
      printf("{\"kind\":\"dfma\",\"tpb\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", tpb, blocks, ms, flops / ms / 1e9);
    }
    for (int tpb : {128, 256, 512}) {
      int blocks = sms * (2048 / tpb);
      dmma_loop<4><<<blocks, tpb>>>(d, 100);
      cudaEventRecord(e0);
      dmma_loop<4><<<blocks, tpb>>>(d, iters / 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 4 * (iters / 4) * (double)blocks * (tpb / 32);
      printf("{\"kind\":\"dmma\",\"tpb\":%d,\"blocks\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", tpb, blocks, ms, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
