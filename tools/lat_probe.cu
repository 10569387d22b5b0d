// Dependent-chain latency of DFMA / DMUL / MUFU.RCP64H / SHFL on this GPU (one warp), and
// MUFU.RCP64H throughput.
#include <cstdio>
__global__ void chain_dfma(double* o, int n, double a, double b) {
  double x = threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64(); if (threadIdx.x == 0) printf("DFMA dep latency: %.2f cycles\n", (double)(t1 - t0) / (4.0 * n)); o[threadIdx.x] = x;
}
__global__ void chain_rcp(double* o, int n) {
  double x = 1.0 + threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
  long long t1 = clock64(); if (threadIdx.x == 0) printf("MUFU.RCP64H dep latency: %.2f cycles\n", (double)(t1 - t0) / n); o[threadIdx.x] = x;
}
__global__ void chain_shfl(double* o, int n) {
  double x = threadIdx.x; long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_down_sync(0xffffffffu, x, 1) + 1.0; }
  long long t1 = clock64(); if (threadIdx.x == 0) printf("SHFL.64+DADD dep latency: %.2f cycles\n", (double)(t1 - t0) / n); o[threadIdx.x] = x;
}
__global__ void tput_rcp(double* o, int n) {
  double x0 = 1.0 + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < n; ++i) {
#define R(x) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
    R(x0) R(x1) R(x2) R(x3) R(x4) R(x5) R(x6) R(x7)
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* o; cudaMalloc(&o, 1 << 24);
  chain_dfma<<<1, 32>>>(o, 10000, 0.999, 1e-3); cudaDeviceSynchronize();
  chain_rcp<<<1, 32>>>(o, 10000); cudaDeviceSynchronize();
  chain_shfl<<<1, 32>>>(o, 10000); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  tput_rcp<<<148 * 8, 256>>>(o, 100);
  cudaEventRecord(e0); tput_rcp<<<148 * 8, 256>>>(o, 2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 148.0 * 8 * 256 * 2000 * 8;
  printf("MUFU.RCP64H throughput: %.1f per SM per clk (at 1.965 GHz)\n", n / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}
