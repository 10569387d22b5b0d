// Probe of the TMA-store epilogue's building blocks on sm_100a: a 2D f64
// tensor map with an inner extent clipped below the pitch, box 30 x 12,
// stores at an even and an odd inner coordinate.  Prints OK / the CUDA error.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void k_store(const __grid_constant__ CUtensorMap map, int x, int y) {
    extern __shared__ __align__(128) double sm[];
    for (int k = threadIdx.x; k < 30 * 12; k += blockDim.x) sm[k] = 1000.0 * (k / 30) + (k % 30);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&map), "r"(x),
                     "r"(y), "r"(smem_u32(sm)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    const int P = 288, rows = 60, nx = 270, R = 1;
    double* d;
    cudaMalloc(&d, sizeof(double) * P * rows);
    cudaMemset(d, 0, sizeof(double) * P * rows);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap map;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(R + nx), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(P) * 8};
    const cuuint32_t box[2] = {30, 12}, estr[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", static_cast<int>(r));
    for (int x : {30, 31, 241, 259}) {
        k_store<<<1, 128, 30 * 12 * 8>>>(map, x, 12);
        cudaError_t e = cudaDeviceSynchronize();
        printf("store at x=%d: %s\n", x, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    std::vector<double> h(P * rows);
    cudaMemcpy(h.data(), d, sizeof(double) * P * rows, cudaMemcpyDeviceToHost);
    printf("row 12: x=30 -> %g, x=31 -> %g, x=259 -> %g, x=270 -> %g, x=271 -> %g (clipped: 0)\n", h[12 * P + 30],
           h[12 * P + 31], h[12 * P + 259], h[12 * P + 270], h[12 * P + 271]);
    return 0;
}
