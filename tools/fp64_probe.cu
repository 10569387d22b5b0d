// Micro-probe: sustained DFMA throughput, IEEE division throughput, sqrt; and HBM copy GB/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ddiv_loop(double* out, int iters, double a) {
  double x0 = 1.0 + threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = __ddiv_rn(a, x0) + 1.0; x1 = __ddiv_rn(a, x1) + 1.0; x2 = __ddiv_rn(a, x2) + 1.0; x3 = __ddiv_rn(a, x3) + 1.0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d clock %d kHz l2 %d MB smem/blk optin %zu regs/SM %d\n", p.name, p.multiProcessorCount, p.clockRate, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / threads);
    int iters = 4000;
    dfma_loop<<<blocks, threads>>>(out, 10, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 16 * 8;
    printf("DFMA threads/blk %d: %.2f TFMA/s = %.2f TFLOP/s; per SM per clk @%.0f MHz nominal: %.1f\n", threads, fmas / ms / 1e9, 2 * fmas / ms / 1e9,
           p.clockRate / 1e3, fmas / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  }
  {
    int threads = 512, blocks = p.multiProcessorCount * 4, iters = 2000;
    ddiv_loop<<<blocks, threads>>>(out, 10, 3.0);
    cudaEventRecord(e0);
    ddiv_loop<<<blocks, threads>>>(out, iters, 3.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters * 8 * 4;
    printf("DDIV: %.2f Gdiv/s (%.1f per SM per clk)\n", n / ms / 1e6, n / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  }
  {
    size_t bytes = size_t(4) << 30; double2 *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes); size_t n = bytes / 16;
    for (int r = 0; r < 3; ++r) copy_k<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) copy_k<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s (read+write)\n", 2.0 * bytes * 10 / ms / 1e6);
  }
  cudaError_t err = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
