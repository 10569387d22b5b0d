// swe_step_inst.cu — instantiations of the fused step kernel, one slice of the
// variant space per translation unit so the build runs in parallel.
//
// Compiled 8 times (see __graft_entry__.build):
//   SWE_EXACT_TU = 1 / 0   exact (IEEE expression trees, bit-identical to the
//                          reference built with -ffp-contract=off) / fast
//                          (explicit FMA + shared reciprocals, tolerance parity)
//                          -- both with -fmad=false; fast mode writes its FMAs
//                          explicitly;
//   SWE_PART = 0..3        sweep parity (bit 1) x smoothing (bit 0).
// Each part instantiates flat/sloped x frictionless/Manning, plus the
// early-exit kernels (flat bed only).  Part 0 also carries the schedule and
// finalize kernels of its mode.
#include <algorithm>
#include <cstdio>

#include "swe_launch.h"
#include "swe_step.cuh"

#ifndef SWE_EXACT_TU
#define SWE_EXACT_TU 1
#endif
#ifndef SWE_PART
#define SWE_PART 0
#endif

#define SWE_CAT2(a, b) a##b
#define SWE_CAT(a, b) SWE_CAT2(a, b)
#define SWE_MODE_NAME(x) SWE_CAT(SWE_CAT(x, SWE_PART), SWE_CAT(_, SWE_EXACT_TU))

// One uniquely named namespace per (part, mode): the same source is compiled
// 8 times, and nvcc names an anonymous namespace after the file, so internal
// helpers of different TUs would otherwise share (and merge) symbol names.
namespace SWE_MODE_NAME(swe_inst) {

constexpr int kWPB = SWE_STEP_WPB;  // warps (independent workers) per CTA
constexpr bool kExact = SWE_EXACT_TU != 0;
constexpr bool kFwd = (SWE_PART & 2) != 0;
constexpr bool kSmooth = (SWE_PART & 1) != 0;

template <int BED, bool MANNING, bool EARLY>
cudaError_t launch_one(int grid, cudaStream_t s, const StepParams& p) {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, kSmooth, BED, kExact, MANNING, EARLY>();
    auto k = swe_dev::swe_step_kernel<kWPB, kFwd, kSmooth, BED, MANNING, kExact, EARLY>;
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

template <int BED, bool MANNING, bool EARLY>
int occupancy_one() {
    constexpr size_t smem = swe_dev::step_smem_bytes<kWPB, kSmooth, BED, kExact, MANNING, EARLY>();
    auto k = swe_dev::swe_step_kernel<kWPB, kFwd, kSmooth, BED, MANNING, kExact, EARLY>;
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
#define SWE_V(B, M, E) {launch_one<B, M, E>, occupancy_one<B, M, E>}
// index: flat (bit 1) | manning (bit 0); bed 0 flat, 1 both slopes, 2 dz/dx only;
// early-exit kernels exist for a flat bed only
const Entry kTable[4] = {SWE_V(1, false, false), SWE_V(1, true, false), SWE_V(0, false, false), SWE_V(0, true, false)};
const Entry kXonly[2] = {SWE_V(2, false, false), SWE_V(2, true, false)};
const Entry kEarly[2] = {SWE_V(0, false, true), SWE_V(0, true, true)};
#undef SWE_V

const Entry& entry(int variant) {
    if (variant & 16) return kEarly[variant & 1];
    if ((variant & 32) && !(variant & 2)) return kXonly[variant & 1];
    return kTable[variant & 3];
}

}  // namespace swe_inst<part>_<mode>
using namespace SWE_MODE_NAME(swe_inst);

// per-part entry points, dispatched by swe_launch_step_{exact,fast} below
cudaError_t SWE_MODE_NAME(swe_part_launch)(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return entry(variant).launch(grid, stream, p);
}
int SWE_MODE_NAME(swe_part_occ)(int variant) { return entry(variant).occ(); }

#if SWE_PART == 0
// declarations of the other parts of this mode
#define SWE_DECL(k)                                                                                         \
    cudaError_t SWE_CAT(SWE_CAT(swe_part_launch, k), SWE_CAT(_, SWE_EXACT_TU))(int, int, cudaStream_t,      \
                                                                               const StepParams&);         \
    int SWE_CAT(SWE_CAT(swe_part_occ, k), SWE_CAT(_, SWE_EXACT_TU))(int);
SWE_DECL(1)
SWE_DECL(2)
SWE_DECL(3)
#undef SWE_DECL

namespace SWE_MODE_NAME(swe_inst) {
using PartLaunch = cudaError_t (*)(int, int, cudaStream_t, const StepParams&);
using PartOcc = int (*)(int);
const PartLaunch kPartLaunch[4] = {SWE_CAT(swe_part_launch0_, SWE_EXACT_TU), SWE_CAT(swe_part_launch1_, SWE_EXACT_TU),
                                   SWE_CAT(swe_part_launch2_, SWE_EXACT_TU), SWE_CAT(swe_part_launch3_, SWE_EXACT_TU)};
const PartOcc kPartOcc[4] = {SWE_CAT(swe_part_occ0_, SWE_EXACT_TU), SWE_CAT(swe_part_occ1_, SWE_EXACT_TU),
                             SWE_CAT(swe_part_occ2_, SWE_EXACT_TU), SWE_CAT(swe_part_occ3_, SWE_EXACT_TU)};
// swe_step_variant bits: fwd 8, smooth 4, flat 2, manning 1, early 16
int part_of(int variant) { return ((variant >> 3) & 1) * 2 + ((variant >> 2) & 1); }

cudaError_t launch_schedule(cudaStream_t stream, const StepParams& p) {
    const int items = p.ntiles * p.nchunks;
    const int grid = std::max(1, std::min((items + 255) / 256, 148 * 4));
    swe_dev::swe_schedule_kernel<kExact><<<grid, 256, 0, stream>>>(p);
    return cudaGetLastError();
}
}  // namespace swe_inst<part>_<mode>

#if SWE_EXACT_TU
cudaError_t swe_launch_step_exact(int variant, int grid, cudaStream_t stream, const StepParams& p) {
    return kPartLaunch[part_of(variant)](variant, grid, stream, p);
}
int swe_step_occupancy_exact(int variant) { return kPartOcc[part_of(variant)](variant); }
cudaError_t swe_launch_schedule_exact(cudaStream_t stream, const StepParams& p) { return launch_schedule(stream, p); }

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
    return kPartLaunch[part_of(variant)](variant, grid, stream, p);
}
int swe_step_occupancy_fast(int variant) { return kPartOcc[part_of(variant)](variant); }
cudaError_t swe_launch_schedule_fast(cudaStream_t stream, const StepParams& p) { return launch_schedule(stream, p); }
#endif
#endif  // SWE_PART == 0
