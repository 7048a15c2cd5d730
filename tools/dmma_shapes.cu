// FP64 tensor-core throughput per mma.sync shape on B200 (sm_100a): m8n8k4 (the shape every
// DMMA kernel here uses) against the sm_90+ shapes m16n8k4 / m16n8k8 / m16n8k16, with CHAINS
// independent accumulators per warp and W warps per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes tools/dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE, int CHAINS>
__global__ void loop(double* out, int iters) {
  const double x = threadIdx.x * 1e-3, y = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      if constexpr (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(x), "d"(y));
      } else if constexpr (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(x), "d"(y), "d"(y));
      } else if constexpr (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(x), "d"(y), "d"(x), "d"(y), "d"(y), "d"(x));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(x), "d"(y), "d"(x), "d"(y), "d"(x), "d"(y), "d"(x), "d"(y), "d"(y), "d"(x), "d"(y), "d"(x));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 123.456) out[0] = s;
}

template <int SHAPE, int CHAINS>
void run(const char* name, int warps_per_sm, double* d) {
  constexpr double flop[4] = {2.0 * 8 * 8 * 4, 2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8, 2.0 * 16 * 8 * 16};
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  const int threads = 32 * warps_per_sm;
  loop<SHAPE, CHAINS><<<sms, threads>>>(d, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  loop<SHAPE, CHAINS><<<sms, threads>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double tf = flop[SHAPE] * CHAINS * iters * (double)sms * warps_per_sm / (ms * 1e-3) / 1e12;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double clk_per_inst = ms * 1e-3 * clk * 1e3 / ((double)iters * CHAINS * warps_per_sm / 4);
  printf("%-10s chains %d warps/SM %2d: %6.2f TFLOP/s  %5.1f clk per instruction per sub-partition  %s\n", name,
         CHAINS, warps_per_sm, tf, clk_per_inst, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  for (int w : {4, 8, 16}) {
    run<0, 8>("m8n8k4", w, d);
    run<1, 8>("m16n8k4", w, d);
    run<2, 8>("m16n8k8", w, d);
    run<3, 4>("m16n8k16", w, d);
    run<3, 8>("m16n8k16", w, d);
  }
  return 0;
}
