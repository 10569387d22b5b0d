// swe_launch.h — internal launcher interface between the host runtime and the
// step-kernel instantiations.
#pragma once

#include <cuda_runtime.h>

#include "swe_types.h"

#ifndef SWE_STEP_NT
#define SWE_STEP_NT 128
#endif

int swe_step_variant(bool fwd, bool smooth, bool flat, bool manning);
cudaError_t swe_launch_step(int variant, int grid, cudaStream_t stream, const StepParams& p);
int swe_step_occupancy(int variant);
cudaError_t swe_launch_finalize(cudaStream_t stream, const StepParams& p);
