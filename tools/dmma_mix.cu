// Does DADD / DFMA / LDS traffic slow DMMA.8x8x4 issue?  (pipe-sharing probe)
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters, long long* cyc) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2], x[4] = {1, 2, 3, 4};
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = j; c[j][1] = 0; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
      if (MODE == 1) { asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[j]) : "d"(a)); asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[(j+1)&3]) : "d"(b)); }
      if (MODE == 2) { for (int q = 0; q < 4; ++q) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[q]) : "d"(a)); }
      if (MODE == 3) { a += sm[(threadIdx.x + i * 4 + j) & 1023] * 1e-30; }
    }
  }
  long long t1 = clock64();
  double s = x[0] + x[1] + x[2] + x[3] + a;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int M>
void run(int warps, double* d, long long* dc, const char* name) {
  const int iters = 2000;
  k<M><<<148, warps * 32>>>(d, 100, dc);
  k<M><<<148, warps * 32>>>(d, iters, dc);
  cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-22s warps/SM=%2d : %6.1f clk per DMMA per SMSP\n", name, warps, (double)cyc / (iters * 4.0 * warps / 4.0));
}
int main() {
  double* d; long long* dc; cudaMalloc(&d, 8); cudaMalloc(&dc, 8);
  for (int w : {8, 16}) {
    run<0>(w, d, dc, "dmma only");
    run<1>(w, d, dc, "dmma + 2 DADD");
    run<2>(w, d, dc, "dmma + 4 DADD");
    run<3>(w, d, dc, "dmma + LDS + DFMA");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
