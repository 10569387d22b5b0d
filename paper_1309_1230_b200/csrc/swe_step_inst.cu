// swe_step_inst.cu — instantiations of the fused step kernel and a launcher
// table indexed by (sweep parity, smoothing, flat bed, Manning friction).
//
// Compiled twice (see __graft_entry__.build):
//   SWE_EXACT_TU=1 with -fmad=false: expression trees are never contracted, so
//     the step is bit-identical to the reference built with -ffp-contract=off;
//   SWE_EXACT_TU=0 with -fmad=true: FMA contraction + shared reciprocals
//     (tolerance parity).
#include <algorithm>
#include <cstdio>

#include "swe_launch.h"
#include "swe_step.cuh"

#ifndef SWE_EXACT_TU
#define SWE_EXACT_TU 1
#endif

namespace {

constexpr int kWPB = SWE_STEP_WPB;  // warps (independent workers) per CTA
constexpr bool kExact = SWE_EXACT_TU != 0;

template <bool FWD, bool SMOOTH, bool FLAT, bool MANNING, bool EARLY = false>
cudaError_t launch_one(int grid, cudaStream_t s, const StepParams& p) {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, SMOOTH, FLAT>();
    auto k = swe_dev::swe_step_kernel<kWPB, FWD, SMOOTH, FLAT, MANNING, kExact, EARLY>;
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

template <bool FWD, bool SMOOTH, bool FLAT, bool MANNING, bool EARLY = false>
int occupancy_one() {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, SMOOTH, FLAT>();
    auto k = swe_dev::swe_step_kernel<kWPB, FWD, SMOOTH, FLAT, MANNING, kExact, EARLY>;
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
// early-exit variants exist for a flat bed only (variant bit 16)
#define SWE_E(F, S, M) {launch_one<F, S, true, M, true>, occupancy_one<F, S, true, M, true>}
const Entry kTableEarly[8] = {
    SWE_E(false, false, false), SWE_E(false, false, true), SWE_E(false, true, false), SWE_E(false, true, true),
    SWE_E(true, false, false),  SWE_E(true, false, true),  SWE_E(true, true, false),  SWE_E(true, true, true),
};
#undef SWE_E
#undef SWE_V

static const Entry& entry(int variant) {
    if (variant & 16) return kTableEarly[((variant >> 1) & 4) | ((variant >> 1) & 2) | (variant & 1)];
    return kTable[variant & 15];
}

}  // namespace

static cudaError_t launch_schedule(cudaStream_t stream, const StepParams& p) {
    const int items = p.ntiles * p.nchunks;
    const int grid = std::max(1, std::min((items + 255) / 256, 148 * 4));
    swe_dev::swe_schedule_kernel<kExact><<<grid, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

#if SWE_EXACT_TU
cudaError_t swe_launch_schedule_exact(cudaStream_t stream, const StepParams& p) { return launch_schedule(stream, p); }
cudaError_t swe_launch_step_exact(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return entry(variant).launch(grid, stream, p);
}
int swe_step_occupancy_exact(int variant) { return entry(variant).occ(); }

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
cudaError_t swe_launch_schedule_fast(cudaStream_t stream, const StepParams& p) { return launch_schedule(stream, p); }
cudaError_t swe_launch_step_fast(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return entry(variant).launch(grid, stream, p);
}
int swe_step_occupancy_fast(int variant) { return entry(variant).occ(); }
#endif
