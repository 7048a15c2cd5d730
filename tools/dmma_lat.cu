// DMMA.8x8x4 latency/throughput vs independent chains per warp and warps per SM.
#include <cstdio>
template <int CHAINS>
__global__ void k(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS][2];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) { c[j][0] = j; c[j][1] = 0; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int warps, double* d, long long* dc) {
  const int iters = 2000;
  k<C><<<148, warps * 32>>>(d, 100, dc);
  k<C><<<148, warps * 32>>>(d, iters, dc);
  cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double per_dmma_smsp = (double)cyc / ((double)iters * C * warps / 4.0);
  printf("chains=%d warps/SM=%2d : %6.1f clk per DMMA per SMSP, chain latency %.1f clk\n", C, warps,
         per_dmma_smsp, (double)cyc / iters);
}
int main() {
  double* d; long long* dc; cudaMalloc(&d, 8); cudaMalloc(&dc, 8);
  for (int w : {4, 8, 16, 32}) { run<1>(w, d, dc); run<2>(w, d, dc); run<4>(w, d, dc); run<8>(w, d, dc); }
  return 0;
}
