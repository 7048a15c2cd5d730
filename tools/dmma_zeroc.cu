// Validate the zero-C DMMA rate: event-timed whole-GPU throughput + result check.
#include <cstdio>
#include <cmath>
template <int ZC>
__global__ void k(int iters, double* out) {
  const int lane = threadIdx.x & 31;
  double A[8], B[8], C[16];
  for (int i = 0; i < 8; ++i) { A[i] = 1.0 + i * 1e-3 + lane * 1e-6; B[i] = 0.5 + i * 1e-4 + lane * 1e-7; }
  for (int i = 0; i < 16; ++i) C[i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (ZC) {
        double d0, d1;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                     : "=d"(d0), "=d"(d1) : "d"(A[j]), "d"(B[j]), "d"(0.0), "d"(0.0));
        C[2 * j] += d0; C[2 * j + 1] += d1;
        if (ZC == 2) A[j] = A[j] + 1e-12;
      } else {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(C[2 * j]), "+d"(C[2 * j + 1]) : "d"(A[j]), "d"(B[j]));
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += C[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 512 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double res[3];
  for (int zc = 0; zc < 3; ++zc) {
    const int iters = 4000;
    if (zc == 2) k<2><<<148, 512>>>(10, d); else if (zc) k<1><<<148, 512>>>(10, d); else k<0><<<148, 512>>>(10, d);
    cudaEventRecord(e0);
    if (zc == 2) k<2><<<148, 512>>>(iters, d); else if (zc) k<1><<<148, 512>>>(iters, d); else k<0><<<148, 512>>>(iters, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8.0 * iters * 148 * 16;
    double h; cudaMemcpy(&h, d + 5, 8, cudaMemcpyDeviceToHost);
    res[zc] = h;
    printf("zeroC=%d: %.3f ms  %.1f TFLOP/s  sample=%.12e\n", zc, ms, flops / ms / 1e9, h);
  }
  printf("relative diff %.3e\n", std::fabs(res[0] - res[1]) / std::fabs(res[0]));
}
