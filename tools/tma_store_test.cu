// standalone check of a 2D TMA tensor store with a 62-wide box (fp64)
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap map, int x, int y, int variant) {
  __shared__ __align__(128) double buf[192];
  for (int t = threadIdx.x; t < 186; t += 32) buf[t] = 1000.0 + t;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x == 0) {
    if (variant == 0)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&map), "r"(x), "r"(y), "r"(su32(buf)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" :: "l"(&map), "r"(x), "r"(y), "r"(su32(buf)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const int P = 160, rows = 12; double* d; cudaMalloc(&d, P * rows * 8); cudaMemset(d, 0, P * rows * 8);
  void* fn; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  for (int box : {64, 62}) {
    CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)P, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)P * 8};
    cuuint32_t bx[2] = {(cuuint32_t)box, 3}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int x : {0, 3, 63}) {
      k<<<1, 32>>>(m, x, 3, 0);
      cudaError_t e = cudaDeviceSynchronize();
      printf("box %d enc %d x %d -> %s\n", box, (int)r, x, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  double h[P * rows]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("row3: %g %g %g ... row4[63]=%g\n", h[3 * P + 62], h[3 * P + 63], h[3 * P + 64], h[4 * P + 63]);
  return 0;
}
