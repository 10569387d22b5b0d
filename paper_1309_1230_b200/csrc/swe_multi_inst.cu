// swe_multi_inst.cu — instantiations of the multi-step kernel (swe_step.cuh,
// swe_multi_kernel) for small grids, one (arithmetic mode, smoothing) slice
// per translation unit: flat / both slopes / dz/dx-only bed x frictionless /
// Manning, both sweep directions inside each kernel.
//
// Compiled 4 times (see __graft_entry__.build): SWE_EXACT_TU = 1 / 0,
// SWE_SMOOTH = 1 / 0.
#include <cstdio>

#include "swe_launch.h"
#include "swe_step.cuh"

#ifndef SWE_EXACT_TU
#define SWE_EXACT_TU 1
#endif
#ifndef SWE_SMOOTH
#define SWE_SMOOTH 0
#endif

#define SWE_CAT2(a, b) a##b
#define SWE_CAT(a, b) SWE_CAT2(a, b)
#define SWE_MNAME(x) SWE_CAT(SWE_CAT(x, SWE_SMOOTH), SWE_CAT(_, SWE_EXACT_TU))

namespace SWE_MNAME(swe_multi) {

constexpr int kWPB = SWE_STEP_WPB;
constexpr bool kExact = SWE_EXACT_TU != 0;
constexpr bool kSmooth = SWE_SMOOTH != 0;

template <int BED, bool MANNING>
cudaError_t launch_one(int grid, cudaStream_t s, const StepParams& p, int nsteps) {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, kSmooth, BED, kExact, MANNING, false>();
    auto k = swe_dev::swe_multi_kernel<kWPB, kSmooth, BED, MANNING, kExact>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    // cooperative: the grid barrier needs every CTA resident
    StepParams pc = p;
    void* args[] = {&pc, &nsteps};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(kWPB * 32), args, smem, s);
}

template <int BED, bool MANNING>
int occupancy_one() {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, kSmooth, BED, kExact, MANNING, false>();
    auto k = swe_dev::swe_multi_kernel<kWPB, kSmooth, BED, MANNING, kExact>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kWPB * 32, smem) != cudaSuccess) return 0;
    return n;
}

using LaunchFn = cudaError_t (*)(int, cudaStream_t, const StepParams&, int);
using OccFn = int (*)();
struct Entry {
    LaunchFn launch;
    OccFn occ;
};
#define SWE_V(B, M) {launch_one<B, M>, occupancy_one<B, M>}
// index: bed (0 flat, 1 both slopes, 2 dz/dx only) * 2 + manning
const Entry kTable[6] = {SWE_V(0, false), SWE_V(0, true), SWE_V(1, false), SWE_V(1, true), SWE_V(2, false),
                         SWE_V(2, true)};
#undef SWE_V

}  // namespace swe_multi<smooth>_<mode>

// swe_step_variant bits: smooth 4, flat 2, manning 1, xonly 32
static int multi_index(int variant) {
    const int bed = (variant & 2) ? 0 : (variant & 32) ? 2 : 1;
    return bed * 2 + (variant & 1);
}
cudaError_t SWE_MNAME(swe_multi_launch)(int variant, int grid, cudaStream_t s, const StepParams& p, int nsteps) {
    return SWE_MNAME(swe_multi)::kTable[multi_index(variant)].launch(grid, s, p, nsteps);
}
int SWE_MNAME(swe_multi_occ)(int variant) { return SWE_MNAME(swe_multi)::kTable[multi_index(variant)].occ(); }
