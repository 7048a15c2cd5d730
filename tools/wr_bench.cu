// Write-pattern microbenchmark: what limits a 148-stream sequential CSR fill?
#include <cstdio>
#include <cstdlib>
// each CTA writes its own contiguous chunk [c*L, (c+1)*L) in steps of blockDim doubles
__global__ void chunked(double* v, long long L, int nchunks) {
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    double* p = v + (long long)c * L;
    for (long long i = threadIdx.x; i < L; i += blockDim.x) p[i] = 1.0;
  }
}
// round-robin: unit u of U doubles goes to CTA u % grid (coherent write front)
__global__ void rr(double* v, long long n, int U) {
  for (long long u = blockIdx.x; u * U < n; u += gridDim.x) {
    double* p = v + u * U;
    for (int i = threadIdx.x; i < U && u * U + i < n; i += blockDim.x) p[i] = 1.0;
  }
}
int main() {
  const long long n = 741217625LL;  // C3 K=128 nnz
  double* d; cudaMalloc(&d, n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    f(); cudaEventRecord(a); for (int i = 0; i < 3; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("%-40s %7.1f GB/s\n", name, 3.0 * n * 8 / (ms * 1e-3) / 1e9);
  };
  for (int bpsm : {1, 2, 4}) for (int nt : {352, 1024}) {
    if (nt * bpsm > 2048) continue;
    for (long long L : {23023LL, 88837LL, 2000000LL}) {
      const int nch = (int)(n / L);
      char nm[128]; snprintf(nm, sizeof nm, "chunked L=%lld nt=%d ctas/sm=%d", L, nt, bpsm);
      run(nm, [&] { chunked<<<148 * bpsm, nt>>>(d, L, nch); });
    }
    for (int U : {1372, 5488, 21952}) {
      char nm[128]; snprintf(nm, sizeof nm, "round-robin U=%d nt=%d ctas/sm=%d", U, nt, bpsm);
      run(nm, [&] { rr<<<148 * bpsm, nt>>>(d, n, U); });
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
