// swe_launch.h — internal launcher interface between the host runtime and the
// step-kernel instantiations (swe_step_inst.cu, compiled once per mode).
#pragma once

#include <cuda_runtime.h>

#include "swe_types.h"

#ifndef SWE_STEP_WPB
#define SWE_STEP_WPB 4   // warps per CTA; every warp is an independent row-march worker
#endif
#define SWE_TILE_W(R) (32 - 2 * (R))  // output columns per warp window
// Rows per TMA request (state box 32 x 3G, slope box 32 x 2G): 4 in fast mode
// (fewer request and ring-bookkeeping instructions per cell: 3-5 % faster),
// 2 in exact mode (its larger kernels spill with the deeper ring) and for the
// early-exit kernels (short 32-row items).
#ifndef SWE_EXACT_ROW_GROUP
#define SWE_EXACT_ROW_GROUP 2
#endif
#ifndef SWE_EARLY_ROW_GROUP
#define SWE_EARLY_ROW_GROUP 2
#endif
constexpr int swe_row_group(bool exact, bool early = false) {
    return early ? (exact ? 2 : SWE_EARLY_ROW_GROUP) : exact ? SWE_EXACT_ROW_GROUP : 4;
}

// bit 16: early-exit instantiation (flat bed only); bit 32: sloped bed whose
// dz/dy is +0.0 everywhere (only the dz/dx rows are read)
inline int swe_step_variant(bool fwd, bool smooth, bool flat, bool manning, bool early = false, bool xonly = false) {
    return (fwd ? 8 : 0) | (smooth ? 4 : 0) | (flat ? 2 : 0) | (manning ? 1 : 0) | ((early && flat) ? 16 : 0) |
           ((xonly && !flat) ? 32 : 0);
}
cudaError_t swe_launch_step_exact(int variant, int grid, cudaStream_t stream, const StepParams& p);
cudaError_t swe_launch_step_fast(int variant, int grid, cudaStream_t stream, const StepParams& p);
int swe_step_occupancy_exact(int variant);
int swe_step_occupancy_fast(int variant);
cudaError_t swe_launch_schedule_exact(cudaStream_t stream, const StepParams& p);
cudaError_t swe_launch_schedule_fast(cudaStream_t stream, const StepParams& p);
cudaError_t swe_launch_finalize(cudaStream_t stream, const StepParams& p);

// multi-step kernel (small grids, one rank, no early exit): per (smooth, mode) TU
cudaError_t swe_multi_launch0_0(int variant, int grid, cudaStream_t s, const StepParams& p, int nsteps);
cudaError_t swe_multi_launch0_1(int variant, int grid, cudaStream_t s, const StepParams& p, int nsteps);
cudaError_t swe_multi_launch1_0(int variant, int grid, cudaStream_t s, const StepParams& p, int nsteps);
cudaError_t swe_multi_launch1_1(int variant, int grid, cudaStream_t s, const StepParams& p, int nsteps);
int swe_multi_occ0_0(int variant);
int swe_multi_occ0_1(int variant);
int swe_multi_occ1_0(int variant);
int swe_multi_occ1_1(int variant);
inline cudaError_t swe_launch_multi(bool exact, bool smooth, int variant, int grid, cudaStream_t s,
                                    const StepParams& p, int nsteps) {
    if (smooth) return exact ? swe_multi_launch1_1(variant, grid, s, p, nsteps) : swe_multi_launch1_0(variant, grid, s, p, nsteps);
    return exact ? swe_multi_launch0_1(variant, grid, s, p, nsteps) : swe_multi_launch0_0(variant, grid, s, p, nsteps);
}
inline int swe_multi_occupancy(bool exact, bool smooth, int variant) {
    if (smooth) return exact ? swe_multi_occ1_1(variant) : swe_multi_occ1_0(variant);
    return exact ? swe_multi_occ0_1(variant) : swe_multi_occ0_0(variant);
}

inline cudaError_t swe_launch_step(bool exact, int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return exact ? swe_launch_step_exact(variant, grid, stream, p) : swe_launch_step_fast(variant, grid, stream, p);
}
inline cudaError_t swe_launch_schedule(bool exact, cudaStream_t stream, const StepParams& p) {
    return exact ? swe_launch_schedule_exact(stream, p) : swe_launch_schedule_fast(stream, p);
}
inline int swe_step_occupancy(bool exact, int variant) {
    return exact ? swe_step_occupancy_exact(variant) : swe_step_occupancy_fast(variant);
}
