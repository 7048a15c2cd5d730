// DMMA.8x8x4 issue rate vs operand reuse: A/B constant or varying, C in place or zero.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
template <int MODE>
__global__ void k(int iters, long long* cyc, double* out) {
  const int lane = threadIdx.x & 31;
  double A[8], B[8], C[16];
  for (int i = 0; i < 8; ++i) { A[i] = 1.0 + i * 1e-3 + lane * 1e-6; B[i] = 0.5 + i * 1e-4; }
  for (int i = 0; i < 16; ++i) C[i] = i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double a = (MODE & 1) ? A[j] : A[0];
      const double b = (MODE & 2) ? B[j] : B[0];
      if (MODE & 4) { double d0, d1; dmma(d0, d1, a, b, 0.0, 0.0); C[2 * j] += d0; C[2 * j + 1] += d1; }
      else dmma(C[2 * j], C[2 * j + 1], a, b, C[2 * j], C[2 * j + 1]);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += C[i];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int M>
void run(int warps, long long* dc, double* d) {
  const int iters = 1000;
  k<M><<<148, warps * 32>>>(10, dc, d);
  k<M><<<148, warps * 32>>>(iters, dc, d);
  cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("A %s B %s C %s warps/SM=%2d : %6.1f clk per DMMA per SMSP\n", (M & 1) ? "vary" : "same", (M & 2) ? "vary" : "same",
         (M & 4) ? "fresh+DADD" : "in-place", warps, (double)cyc / (iters * 8.0 * warps / 4.0));
}
int main() {
  long long* dc; double* d; cudaMalloc(&dc, 8); cudaMalloc(&d, 8);
  for (int w : {4, 16}) { run<0>(w, dc, d); run<1>(w, dc, d); run<2>(w, dc, d); run<3>(w, dc, d); run<7>(w, dc, d); }
}
