// swe_step_inst.cu — instantiations of the fused step kernel and a launcher
// table indexed by (sweep parity, smoothing, flat bed, Manning friction).
//
// Compiled twice (see __graft_entry__.build):
//   SWE_EXACT_TU=1 with -fmad=false: expression trees are never contracted, so
//     the step is bit-identical to the reference built with -ffp-contract=off;
//   SWE_EXACT_TU=0 with -fmad=true: FMA contraction + shared reciprocals
//     (tolerance parity).
#include <cstdio>

#include "swe_launch.h"
#include "swe_step.cuh"

#ifndef SWE_EXACT_TU
#define SWE_EXACT_TU 1
#endif

namespace {

constexpr int kWPB = SWE_STEP_WPB;  // warps (independent workers) per CTA
constexpr bool kExact = SWE_EXACT_TU != 0;

template <bool FWD, bool SMOOTH, bool FLAT, bool MANNING>
cudaError_t launch_one(int grid, cudaStream_t s, const StepParams& p) {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, SMOOTH, FLAT>();
    auto k = swe_dev::swe_step_kernel<kWPB, FWD, SMOOTH, FLAT, MANNING, kExact>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    k<<<grid, kWPB * 32, smem, s>>>(p);
    return cudaGetLastError();
}

template <bool FWD, bool SMOOTH, bool FLAT, bool MANNING>
int occupancy_one() {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, SMOOTH, FLAT>();
    auto k = swe_dev::swe_step_kernel<kWPB, FWD, SMOOTH, FLAT, MANNING, kExact>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kWPB * 32, smem) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

using LaunchFn = cudaError_t (*)(int, cudaStream_t, const StepParams&);
using OccFn = int (*)();

struct Entry {
    LaunchFn launch;
    OccFn occ;
};
#define SWE_V(F, S, Z, M) {launch_one<F, S, Z, M>, occupancy_one<F, S, Z, M>}
const Entry kTable[16] = {
    SWE_V(false, false, false, false), SWE_V(false, false, false, true),
    SWE_V(false, false, true, false),  SWE_V(false, false, true, true),
    SWE_V(false, true, false, false),  SWE_V(false, true, false, true),
    SWE_V(false, true, true, false),   SWE_V(false, true, true, true),
    SWE_V(true, false, false, false),  SWE_V(true, false, false, true),
    SWE_V(true, false, true, false),   SWE_V(true, false, true, true),
    SWE_V(true, true, false, false),   SWE_V(true, true, false, true),
    SWE_V(true, true, true, false),    SWE_V(true, true, true, true),
};
#undef SWE_V

}  // namespace

#if SWE_EXACT_TU
cudaError_t swe_launch_step_exact(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return kTable[variant & 15].launch(grid, stream, p);
}
int swe_step_occupancy_exact(int variant) { return kTable[variant & 15].occ(); }

__global__ void swe_finalize_kernel(const __grid_constant__ StepParams p) {
    SweCtl* c = p.ctl;
    const volatile SweCtl* vc = c;
    if (vc->done) return;
    double dt, tc;
    if (vc->mode == 1) {
        const double t = vc->t, te = vc->t_end, dr = vc->dt_raw;
        if (!(t < te)) return;
        const double remaining = te - t;
        const bool landing = dr >= remaining;
        dt = landing ? remaining : dr;
        tc = landing ? te : t + dt;
    } else {
        dt = vc->dt_req;
        tc = vc->tcommit_req;
    }
    swe_dev::finalize_step(p, c, dt, tc);
}

cudaError_t swe_launch_finalize(cudaStream_t stream, const StepParams& p) {
    swe_finalize_kernel<<<1, 1, 0, stream>>>(p);
    return cudaGetLastError();
}
#else
cudaError_t swe_launch_step_fast(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return kTable[variant & 15].launch(grid, stream, p);
}
int swe_step_occupancy_fast(int variant) { return kTable[variant & 15].occ(); }
#endif
