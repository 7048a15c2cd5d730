// DMMA.8x8x4 issue rate of one warp per SM sub-partition for the operand patterns of the p = 3
// kernel's stages: which operand changes between consecutive DMMAs (A, B, both) and how ptxas
// orders them. Each pattern: 8 independent accumulators, unrolled; prints clk per DMMA per SMSP.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(int iters, long long* cyc, double* out) {
  const int lane = threadIdx.x & 31;
  double A[8], B[8], C[16];
  for (int i = 0; i < 8; ++i) { A[i] = 1.0 + i * 1e-3 + lane * 1e-6; B[i] = 0.5 + i * 1e-4 + lane * 1e-7; }
  for (int i = 0; i < 16; ++i) C[i] = i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double a, b;
      if (MODE == 0) { a = A[j]; b = B[0]; }           // A varies, B same
      if (MODE == 1) { a = A[0]; b = B[j]; }           // A same, B varies
      if (MODE == 2) { a = A[j >> 1]; b = B[j & 1]; }  // stage-S pattern: A pairs, B alternating
      if (MODE == 3) { a = A[j & 3]; b = B[j >> 2]; }  // B runs of 4, A cycling
      if (MODE == 4) { a = A[j]; b = B[j]; }           // both vary
      dmma(C[2 * j], C[2 * j + 1], a, b);
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
  const int iters = 2000;
  k<M><<<148, warps * 32>>>(10, dc, d);
  k<M><<<148, warps * 32>>>(iters, dc, d);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"A vary, B same", "A same, B vary", "A pairs, B alternating", "B runs of 4, A cycling", "A vary, B vary"};
  printf("%-26s warps/SM=%2d : %6.1f clk per DMMA per SMSP\n", nm[M], warps, (double)cyc / (iters * 8.0 * warps / 4.0));
}
int main() {
  long long* dc; double* d;
  cudaMalloc(&dc, 8); cudaMalloc(&d, 8);
  for (int w : {4, 8}) { run<0>(w, dc, d); run<1>(w, dc, d); run<2>(w, dc, d); run<3>(w, dc, d); run<4>(w, dc, d); }
}
