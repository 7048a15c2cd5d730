// Stage-B-like DMMA microbenchmark: per unit 14 LDS, 30 DMMA into 32 in-place
// accumulators, 40 DADD (group sums), 16 STS.  Reports clk per DMMA per SMSP.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
template <int MODE>
__global__ void k(int iters, long long* cyc, double* out) {
  __shared__ double X[4096];
  __shared__ double Ys[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) X[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double bv[10], bd[10];
  for (int i = 0; i < 10; ++i) { bv[i] = 1.0 + i * 1e-3 + lane * 1e-5; bd[i] = 0.5 - i * 1e-3; }
  long long t0 = clock64();
  double tot = 0;
  for (int it = 0; it < iters; ++it) {
    double y[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = 0;
    double xv[7], xd[7];
#pragma unroll
    for (int l = 0; l < 7; ++l) { xv[l] = X[(warp * 64 + l * 8 + lane + it) & 4095]; xd[l] = X[(warp * 64 + l * 8 + lane + 7 + it) & 4095]; }
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int l = (i * 7) / 10;
      dmma(y[(2 * i) & 31], y[(2 * i + 1) & 31], xd[l], bv[i], y[(2 * i) & 31], y[(2 * i + 1) & 31]);
      dmma(y[(2 * i + 16) & 31], y[(2 * i + 17) & 31], xv[l], bv[i], y[(2 * i + 16) & 31], y[(2 * i + 17) & 31]);
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      const int l = (i * 7) / 10;
      dmma(y[(2 * i) & 31], y[(2 * i + 1) & 31], xv[l], bd[i], y[(2 * i) & 31], y[(2 * i + 1) & 31]);
    }
    if (MODE >= 1) {
      double s = 0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) { double p = y[i] + y[i + 1]; p = p + y[i + 2]; s += p + y[i + 3]; Ys[(warp * 32 + i + lane) & 4095] = p; }
      tot += s;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) tot += y[i] * 0.0;
    }
  }
  long long t1 = clock64();
  if (tot == 1.2345) out[0] = tot;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int M>
void run(int warps, long long* dc, double* d, const char* nm) {
  const int iters = 500;
  k<M><<<148, warps * 32>>>(10, dc, d);
  k<M><<<148, warps * 32>>>(iters, dc, d);
  cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-26s warps/SM=%2d : %6.1f clk per DMMA per SMSP\n", nm, warps, (double)cyc / (iters * 30.0 * warps / 4.0));
}
int main() {
  long long* dc; double* d; cudaMalloc(&dc, 8); cudaMalloc(&d, 8);
  for (int w : {4, 8, 16}) { run<0>(w, dc, d, "30 dmma + 14 lds"); run<1>(w, dc, d, "+ group sums + 8 sts"); }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
