// swe_step.cuh — the fused MacCormack step (plan kernels K1-K6 + smoothing)
// as ONE sm_100a kernel per time step.
//
// Reference plan (executor.hpp:113-148, naive strategy 846-911):
//   K1 ghost fill (committed) -> K2 predictor -> K3 ghost fill (U*) ->
//   K4 corrector [+ ghost fill + 5-point smoothing] -> K5 guard -> K6 CFL min.
// Here:
//   K1   ghosts of the committed state are written by the previous step's
//        epilogue (or the load kernel) into the padded buffer, so the
//        predictor reads them as ordinary cells.
//   K2+K4 fused per warp with row marching: a warp owns a 32-column window
//        (30 output columns, 28 with smoothing) and walks a contiguous run of
//        rows in the sweep direction, independently of every other warp (no
//        CTA barriers).  Each state's fluxes F/G are evaluated once per cell
//        and shared: x-neighbours through warp shuffles, y-neighbours in
//        registers.  Interface fluxes
//        H_{i+1/2} are evaluated once per interface (the reference computes
//        them twice, bit-identically: README.md:191-196).
//   K3   U* ghosts are formed in-thread at domain edges only.
//   K5/K6 fused into the epilogue: guard offenders and dry-U* consumers go to
//        atomicMax(~index) words (row-major first offender wins); the CFL
//        reduction keeps max sx / max sy because min_k RN(dx/sx_k) =
//        RN(dx / max_k sx_k) (correctly rounded division is monotone).
//   Finalize: the last CTA to finish turns the reduction words into
//        StepResult / errors and commits by flipping the ping-pong selector
//        in the device control block (executor.hpp:836-840).
// Committed rows arrive through a per-warp cp.async.bulk (TMA bulk copy)
// ring with mbarrier completion; stores are coalesced 8-byte STG.
#pragma once

#include <cooperative_groups.h>

#include "swe_device.cuh"
#include "swe_launch.h"

namespace swe_dev {

// Resident CTAs per SM (4 warps each) the register allocation must allow:
// 4 (16 warps, 128 registers) where the extra warps pay -- exact mode and the
// flat frictionless step -- and 3 (12 warps, 168 registers) for the fast steps
// with bathymetry or friction, which run at the board power cap and lose clock
// with more warps (measured).  SWE_MINB forces one value.
template <bool EXACT, bool FLAT, bool MANNING>
constexpr int step_min_blocks() {
#ifdef SWE_MINB
    return SWE_MINB;
#else
    return (EXACT || (FLAT && !MANNING)) ? 4 : 3;
#endif
}

// Ring depth in row groups per warp: 8 rows in flight with groups of 2; with
// groups of 4, as many as fit 227 KB of shared memory at the variant's
// occupancy (3 stages, 2 for 16 warps on a sloped bed).
template <bool EXACT, bool FLAT, bool MANNING, bool EARLY>
constexpr int step_stages() {
#ifdef SWE_STAGES
    return SWE_STAGES;
#else
    return swe_row_group(EXACT, EARLY) == 2 ? 4 : (FLAT || step_min_blocks<EXACT, FLAT, MANNING>() == 3) ? 3 : 2;
#endif
}

// Ring slot of one row group: the state box ([3G][BW] doubles) and the slope
// box ([(NF-3)G][BW]), each padded to 128 bytes (TMA destination alignment).
constexpr int swe_pad16(int n) { return (n + 15) / 16 * 16; }
constexpr int step_slot_doubles(int NF, int G, int R) {
    return swe_pad16(3 * G * swe_box_w(R)) + swe_pad16((NF - 3) * G * swe_box_w(R));
}

// Output staging for a TMA-store epilogue: per warp two buffers of one row
// group ([3G field rows][TW doubles], padded to 128 B), for the variants whose
// ring + staging fit the SM's 228 KB at their occupancy.  OFF: a TMA tensor
// store must start on a 16-byte-aligned inner coordinate
// (tools/tma_store_probe.cu: an odd double offset is an illegal instruction),
// and with R = 1 the output columns of every window start at an odd padded
// column; enabling it needs an even column offset for the windows (padding
// 2 instead of R and a 34-wide load box).  The coalesced STG epilogue is used.
#ifndef SWE_TMA_STORE
#define SWE_TMA_STORE 0
#endif
template <bool EXACT, bool EARLY, int TW>
constexpr int step_stage_doubles() {
    return ((3 * swe_row_group(EXACT, EARLY) * TW * 8 + 127) / 128) * 128 / 8;
}
// staging buffers per warp for the TMA-store epilogue: 2 (the next group is
// staged while the previous store reads), 1 if two do not fit, 0 = STG epilogue
template <int WPB, bool SMOOTH, int BED, bool EXACT, bool MANNING, bool EARLY>
constexpr int step_tma_buffers() {
    constexpr int NF = BED == 0 ? 3 : BED == 2 ? 4 : 5;
    constexpr int G = swe_row_group(EXACT, EARLY);
    constexpr int D = step_stages<EXACT, BED == 0, MANNING, EARLY>();
    constexpr int TW = SMOOTH ? 28 : 30;
    constexpr long ring = static_cast<long>(D) * step_slot_doubles(NF, G, SMOOTH ? 2 : 1) * 8;
    constexpr long stage = static_cast<long>(step_stage_doubles<EXACT, EARLY, TW>()) * 8;
    constexpr int blocks = step_min_blocks<EXACT, BED == 0, MANNING>();
    // + static smem and the per-CTA reserve
    constexpr long cta2 = WPB * (ring + 2 * stage + D * 8) + 1536, cta1 = WPB * (ring + stage + D * 8) + 1536;
    if (SWE_TMA_STORE == 0) return 0;
    return cta2 * blocks <= 228L * 1024 ? 2 : cta1 * blocks <= 228L * 1024 ? 1 : 0;
}
template <int WPB, bool SMOOTH, int BED, bool EXACT, bool MANNING, bool EARLY>
constexpr bool step_tma_store() {
    return step_tma_buffers<WPB, SMOOTH, BED, EXACT, MANNING, EARLY>() > 0;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
                 "r"(y), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Rows per TMA request (swe_row_group): one 2D box carries G consecutive rows
// (state box 32 x 3G, slope box 32 x 2G), so the per-request issue cost
// (uniform-register setup, mbarrier arm/wait, ring bookkeeping) is paid once
// per G rows.

// ------------------------------------------------------------ work partition
// Worker w (one warp) owns units [w*U/G, (w+1)*U/G) of the unit space
// u = tile*nloc + row.  A unit run is split into segments at tile boundaries.
struct Seg {
    int tile, ra, rb;
};

__device__ __forceinline__ int seg_list(const StepParams& p, long long w, long long nw, Seg* segs,
                                        int maxseg) {
    const long long total = static_cast<long long>(p.ntiles) * p.nloc;
    long long u = total * w / nw;
    const long long u1 = total * (w + 1) / nw;
    int n = 0;
    while (u < u1 && n < maxseg) {
        const int tile = static_cast<int>(u / p.nloc);
        const int ra = static_cast<int>(u % p.nloc);
        const long long left = u1 - u;
        const int rb = static_cast<int>(left < (p.nloc - ra) ? ra + left : p.nloc);
        segs[n++] = {tile, ra, rb};
        u += rb - ra;
    }
    return n;
}

// --------------------------------------------------------------- finalize
// executor.hpp:889-903 (K5/K6 outcome) + 1091-1104 (finish_dt) + 836-840 (commit).
struct StepOutcome {
    int status, kind, ei, ej, dflags;
    double et, edt, dt_next, msx, msy;
};

__device__ __forceinline__ StepOutcome finalize_compute(const StepParams& p, const volatile unsigned long long* red,
                                                        double tc) {
    const unsigned long long e2 = red[RED_E2], e4 = red[RED_E4], e5 = red[RED_E5];
    const unsigned long long dg = red[RED_DIAG], dry = red[RED_DRY];
    StepOutcome o{0, 0, -1, -1, 0, 0.0, 0.0, 0.0, 0.0, 0.0};
    o.msx = __longlong_as_double(static_cast<long long>(red[RED_SX]));
    o.msy = __longlong_as_double(static_cast<long long>(red[RED_SY]));
    // plan order (executor.hpp:846-911): K2 precondition, K4 dry U*, K5 guard, K6
    if (e2) {
        o.status = SWE_ERR_INSTABILITY; o.kind = 2;
    } else if (dry) {
        // an interior window saw a dry U*: the host finds the row-major first
        // consumer over the whole grid (dry_scan_kernel), then K5/K6
        o.status = SWE_STATUS_DIAG;
        o.dflags = 2 | (e5 ? 1 : 0);
    } else if (e4) {
        const unsigned long long idx = ~e4;
        o.status = SWE_ERR_INSTABILITY; o.kind = 4;
        o.ei = static_cast<int>(idx % static_cast<unsigned long long>(p.nx));
        o.ej = static_cast<int>(idx / static_cast<unsigned long long>(p.nx));
        o.et = tc;
    } else if (e5 || dg || p.always_diag || !(o.msx < p.tz_x) || !(o.msy < p.tz_y)) {
        // guard screen failed (first offender and values from the exact scan)
        // or dx/sx may round to 0 / overflow: exact per-cell K5 + K6 scan
        o.status = SWE_STATUS_DIAG;
        o.dflags = e5 ? 1 : 0;
    } else {
        const double a = __ddiv_rn(p.dx, o.msx);
        const double b = __ddiv_rn(p.dy, o.msy);
        const double core = (b < a) ? b : a;
        const double dt_raw = std_min(p.cfl * core, p.dt_max);
        o.dt_next = dt_raw;
        if (dt_raw < p.dt_min) {
            o.status = SWE_ERR_STEP_COLLAPSE; o.kind = 6; o.edt = dt_raw; o.et = tc;
        }
    }
    return o;
}

// The launch's results into the control block (the host reads them).
__device__ __forceinline__ void write_outcome(SweCtl* c, const StepOutcome& o, double dt, double tc) {
    c->diag_flags = o.dflags;
    c->max_sx = o.msx;
    c->max_sy = o.msy;
    c->dt_used = dt;
    c->t_commit = tc;
    c->dt_next = o.dt_next;
    c->status = o.status;
    c->err_kind = o.kind;
    c->err_i = o.ei;
    c->err_j = o.ej;
    c->err_t = o.et;
    c->err_dt = o.edt;
}

__device__ __forceinline__ void finalize_step(const StepParams& p, SweCtl* c, double dt, double tc) {
    volatile unsigned long long* red = c->red;
    const StepOutcome o = finalize_compute(p, red, tc);
    write_outcome(c, o, dt, tc);
    if (o.status == 0) {
        c->sel ^= 1;
        c->t = tc;
        c->step_index += 1ull;
        c->dt_raw = o.dt_next;
        c->steps_done += 1ull;
        c->done = (c->mode == 1) ? (!(tc < c->t_end) || tc >= c->t_mark) : 0;
    } else {
        c->done = 1;
    }
    for (int k = 0; k < RED_N; ++k) red[k] = 0ull;
    c->finish = 0u;
    c->work[0] = 0u;
    c->work[1] = 0u;
    c->nactive = 0u;
    __threadfence();
}

// --------------------------------------------------------------- the kernel
// One warp = one worker.  Lane t owns column i = x0 - R + t of a 32-column
// window; lanes R..31-R are output columns.  Iteration k of the row march
// works on two consecutive rows (march direction S):
//   stage 1  row b+S : committed row from the warp's TMA ring; F/G/S(U)
//   stage 2  row b   : predictor U*, F/G/S(U*), interface fluxes, boundary
//                      faces, dry-U* detection -- then, once the neighbour
//                      lane's x face is shuffled in, the corrector of row b
//                      (+ smoothing of row b-S), guard, CFL, store
// Stage 1 of the next row is independent of row b's stage 2, so the two
// dependency chains interleave; x neighbours are exchanged with shuffles, so
// warps never wait for each other.  (Running the corrector one iteration
// later, as a third stage, gave more overlap but carried 11 more doubles per
// lane and spilled: the two-stage march is 5 % faster.)  The steady state is
// unrolled by two with the pipeline registers ping-ponging between two carry
// sets, so no register moves are needed to advance the march.

// Pipeline registers between iterations (the c_* members hand row b's stage-2
// results to its corrector within the same iteration).
struct Carry {
    CellVec U;                 // committed state of the stage-2 row b
    Flux FU;                   // its fluxes
    double srx, sry, zx, zy;   // its source term and bed slopes
    CellVec Hyp;               // y face (b-S, b)
    CellVec Uc;                // committed state of the corrector row
    double c_sx, c_sy;         // S(U) + S(U*) of that row (summed as the corrector does)
    CellVec c_dy;              // (dt/dy) * (H_north - H_south) of that row (its y-face term)
    CellVec c_hx;              // its own x face (the other one comes from the neighbour lane)
    CellVec Cp, Cpp;           // corrector output of rows b-S, b-2S (smoothing)
    // fast mode (classic corrector form, see iter()): G(U*) of the stage-2 row,
    // carried to the next iteration, and row b's own stage-2 results
    CellVec Gs;                // G(U*) of row b
    CellVec c_fs;              // F(U*) of row b (shuffled to the corrector neighbour)
    CellVec c_sum;             // U + U* of row b
    double c_ssx, c_ssy;       // S(U*) of row b
};

struct WarpRing {  // per-warp TMA ring state (warp-uniform)
    int d;         // stage of the next request to consume
    unsigned ph;   // its mbarrier phase parity
};

// BED: 0 flat (no bed reads), 1 both slopes, 2 dz/dx only (dz/dy is +0.0
// everywhere, e.g. a channel sloping along x: the dz/dy rows are not read)
#ifndef SWE_FAST_CLASSIC
#define SWE_FAST_CLASSIC 0
#endif
// SWE_ABL (measurement only, wrong results): 1 no output stores, 2 no guard /
// dry checks, 4 no CFL speeds, 8 no friction on U*, 16 no friction on U
#ifndef SWE_ABL
#define SWE_ABL 0
#endif
#ifndef SWE_LATE_SRC
#define SWE_LATE_SRC 0
#endif
#ifndef SWE_EMIT_MASKED
#define SWE_EMIT_MASKED 0
#endif
#ifndef SWE_CFL_DEFER
#define SWE_CFL_DEFER 0
#endif
// interior windows store all 32 lanes: the two halo lanes' stores go to a
// pitch-padding column (never read), so the row's epilogue has no branch and
// the warp no reconvergence point between rows
// (0 off, 1 every kernel, 2 the fast Manning and the exact frictionless
// kernels: measured -2.5 % on C3 fast, -0.8 % on C3f / flat exact; +1 % on
// the fast frictionless and flat configs, whose steps are closer to the HBM
// bound, +2 % on C3 exact and +2.6 % on C5)
#ifndef SWE_EMIT_PAD
#define SWE_EMIT_PAD 2
#endif
// refill the ring right before the next group's wait instead of after the
// last row of a group: one divergent region (refill + wait) per group
// (2: the fast Manning kernels, with the padding-column epilogue, and the
// early-exit kernels: C5 -1.7 % fast, -1.6 % exact; +0.4-1.5 % elsewhere)
#ifndef SWE_LATE_PRODUCE
#define SWE_LATE_PRODUCE 2
#endif
#ifndef SWE_MIRROR_BWD
#define SWE_MIRROR_BWD 1  // backward sweeps take their items top-down (see prod_seg)
#endif
#ifndef SWE_MULTI_COMPACT
#define SWE_MULTI_COMPACT 1  // multi-step kernels: two-iteration march trips (see march())
#endif

// ONE_MARCH: every segment runs the edge march (a superset of the interior
// one), so the kernel holds one march body per sweep direction
template <int WPB, bool FWD, bool SMOOTH, int BED, bool MANNING, bool EXACT, bool EARLY, bool ONE_MARCH = false>
struct Marcher {
    static constexpr bool CLASSIC = SWE_FAST_CLASSIC != 0;  // fast-mode corrector form (see iter())
    static constexpr bool COMPACT = ONE_MARCH && SWE_MULTI_COMPACT != 0;
    static constexpr bool PAD =
        SWE_EMIT_PAD == 1 || (SWE_EMIT_PAD == 2 && !EARLY && (EXACT ? !MANNING : MANNING));
    static constexpr bool FLAT = BED == 0;
    static constexpr bool XONLY = BED == 2;
    using A = Arith<EXACT>;
    using Rc = typename A::Rc;
    static constexpr int R = SMOOTH ? 2 : 1;
    static constexpr int S = FWD ? 1 : -1;
    static constexpr int NF = FLAT ? 3 : XONLY ? 4 : 5;  // doubles per cell in the ring
    static constexpr int D = step_stages<EXACT, FLAT, MANNING, EARLY>();
    // late refill: needs D >= 3, or the refill at a segment's last group never
    // reaches the next segment's claim (with D = 2 the warp's queue runs dry
    // and it stops early -- caught by the C3 parity check of a 16-warp build)
    static constexpr bool LATE =
        (SWE_LATE_PRODUCE == 1 || (SWE_LATE_PRODUCE == 2 && ((MANNING && !EXACT) || EARLY))) && D >= 3;
    static constexpr int G = swe_row_group(EXACT, EARLY);
    static_assert((G & (G - 1)) == 0, "row groups are powers of two");
    static constexpr int BW = swe_box_w(R);   // load box width (32, or 34 for R = 1: see swe_types.h)
    static constexpr int BO = swe_box_off(R); // lane 0's column in the box
    static constexpr int ST_D = swe_pad16(3 * G * BW);         // state box doubles in a slot (padded)
    static constexpr int SLOT = step_slot_doubles(NF, G, R);     // doubles per ring slot: state, then slopes
    static constexpr unsigned TX_BYTES = NF * G * BW * 8;        // bytes the slot's TMA loads deliver
    static constexpr int TW = 32 - 2 * R;
    static constexpr unsigned FULL = 0xffffffffu;
    static constexpr int NB = step_tma_buffers<WPB, SMOOTH, BED, EXACT, MANNING, EARLY>();  // staging buffers
    static constexpr bool TSTORE = NB > 0;
    static constexpr int SD = step_stage_doubles<EXACT, EARLY, TW>();  // doubles per staging buffer

    const StepParams& p;
    double* stage;
    unsigned long long* bars;
    Seg* segq;      // per-warp queue of claimed work items (ring of QN)
    int qhead, qtail;  // consumer / producer positions (warp-uniform)
    int lane;
    const double* cur;
    double* nxt;
    int P;
    double dt, dtdx, dtdy, half_dt, cx, cy;
    // physics constants are read from the kernel parameters (constant-bank
    // operands, no registers): p.h_min, p.half_g, p.neg_g, p.gnn
    // producer state (warp-uniform): row groups left in the current segment,
    // TMA coordinates of the next request, committed buffer
    int pleft;
    bool pdone;
    int px, py, sel;
    int pn, req;  // row groups requested / fully consumed
    WarpRing ring;
    // per-segment constants
    int i, L, r_start;
    bool in_x, out_x, star_ok, xedge;
    double* orow;  // output row of the next emit (this lane's column; STG epilogue)
    // TMA-store epilogue: this warp's two staging buffers, groups issued so
    // far (parity = buffer), the current segment's tile, first output row in
    // march order and completed groups
    double* sstage;
    unsigned sgrp;
    int seg_tile, erow0, egrp;
    // reductions
    double mx, my;
    int e2;
    unsigned long long e4;  // ~ first dry-U* consumer found in an edge window / row (exact)
    // screens whose exact first offender the host finds only when they fail:
    // g_ok = every emitted cell passed the guard screen (h >= h_min and finite
    // CFL speeds, which is finite h, qx, qy); d_ok = no interior U* was dry
    bool g_ok, d_ok;
    // quiet-item tracking of the current segment (early exit): with
    // mom = bits(qx) | bits(qy) per output cell, qo |= bits(h) | mom and
    // qn &= bits(h) & ~mom end equal iff every cell is (H, +0, +0), same H
    unsigned long long qo, qn;
    unsigned nitems;  // items of this launch (all, or the active list)
    unsigned* wctr;   // the step's work-item counter (null: static assignment from sclaim)
    unsigned sclaim;
    bool pushed;      // this lane stored halo rows into a neighbour's buffer (fused halo push)
    CellVec pend;     // SWE_CFL_DEFER: output cell whose CFL speeds are pending
    bool pvalid;

    __device__ __forceinline__ double shf_nb(double x) const {
        return FWD ? __shfl_down_sync(FULL, x, 1) : __shfl_up_sync(FULL, x, 1);
    }
    __device__ __forceinline__ double shf_back(double x) const {
        return FWD ? __shfl_up_sync(FULL, x, 1) : __shfl_down_sync(FULL, x, 1);
    }
    // Interface flux 0.5*(F(U) + F(U*)) (scheme.hpp:153-161).  FAST mode keeps
    // the plain sum and folds the 0.5 into the corrector coefficients cx/cy.
    static __device__ __forceinline__ double avg(double a, double b) {
        if constexpr (EXACT) return 0.5 * (a + b);
        else return a + b;
    }

    static constexpr int QN = 4;
    // Producer: claim the next work item (tile, row chunk) from the step's
    // atomic counter, queue it for the consumer and point this lane at its
    // first row.  Dynamic claiming balances the cheaper interior windows
    // against the boundary windows and any per-SM speed differences.
    // With EARLY the items come from the active list the schedule kernel
    // built for this step (quiet items already accounted for).
    __device__ __forceinline__ void prod_seg() {
        unsigned item = 0;
        if (wctr) {
            if (lane == 0) item = atomicAdd(wctr, 1u);
            item = __shfl_sync(FULL, item, 0);
        } else {  // static assignment (multi-step launches): items w, w + W, ...
            item = sclaim;
            sclaim += gridDim.x * WPB;
        }
        if (item >= nitems) {
            pleft = 0;
            pdone = true;
            return;
        }
        // (fast backward sweeps walk the active list from its end: it is built
        // in item order, so they start on the rows the step before wrote last:
        // C5 fast -0.7 %; exact +3 %, so not there)
        if constexpr (EARLY) item = p.active[(FWD || !SWE_MIRROR_BWD || EXACT) ? item : nitems - 1u - item];
        SWE_DCHECK(item < static_cast<unsigned>(p.ntiles) * static_cast<unsigned>(p.nchunks));
        const int rc = static_cast<int>(item / p.ntiles);   // row-chunk major: neighbouring
        const int tile = static_cast<int>(item % p.ntiles); // windows share halo sectors in L2
        Seg sg;
        sg.tile = tile;
        // rows of this launch: [row_lo, row_hi) in chunks; row_gap jumps from the
        // first chunk to the second (the strip-edge launch: bottom and top band)
        // (guided: chunks rc >= tier_rc are chunk2 rows, so the last items are short)
        if (rc < p.tier_rc) {
            sg.ra = p.row_lo + rc * p.chunk + (rc > 0 ? p.row_gap : 0);
            sg.rb = min(sg.ra + p.chunk, p.row_hi);
        } else {
            sg.ra = p.row_lo + p.tier_rc * p.chunk + (rc - p.tier_rc) * p.chunk2;
            sg.rb = min(sg.ra + p.chunk2, p.row_hi);
        }
        if constexpr (SWE_MIRROR_BWD && !FWD && !EARLY) {
            // backward sweeps hand out the rows top-down (the same items,
            // mirrored): the forward sweep before wrote the top rows last, so
            // the first reads of this step hit what is still in L2, and the
            // next forward sweep starts on the rows this one wrote last
            if (p.row_gap == 0) {
                const int a = sg.ra, b = sg.rb;
                sg.ra = p.row_lo + p.row_hi - b;
                sg.rb = p.row_lo + p.row_hi - a;
            }
        }
        SWE_DCHECK(sg.tile >= 0 && sg.tile < p.ntiles && sg.ra >= p.row_lo && sg.ra < sg.rb && sg.rb <= p.row_hi);
        segq[qtail % QN] = sg;
        ++qtail;
        pleft = ((sg.rb - sg.ra) + 2 * R + G - 1) / G;
        const int row = FWD ? sg.ra - R : sg.rb - 1 + R;  // first row in march order
        px = sg.tile * TW - R + SWE_XO - BO;              // load box start (lane 0's column - BO, even)
        py = (FWD ? row : row - (G - 1)) + R;             // lowest padded row of the first group
    }
    __device__ __forceinline__ void produce() {
        while (pn < req + D - 1) {
            if (pleft == 0 && !(pdone || qtail - qhead >= QN - 1)) prod_seg();
            if (pleft == 0) return;
            const int d = pn % D;
            // the box may run past the buffer at a strip end (TMA fills zeros there,
            // never consumed), but it must overlap it
            SWE_DCHECK(px >= 0 && (px & 1) == 0 && px + BW <= P && py + G > 0 && py < p.nloc + 2 * R);
            if (lane == 0) {
                mbar_expect_tx(&bars[d], TX_BYTES);
                tma_load_2d(stage + d * SLOT, &p.tmap_state[sel], px, py * 3, &bars[d]);
                if constexpr (XONLY) tma_load_2d(stage + d * SLOT + ST_D, &p.tmap_slopex, px, py, &bars[d]);
                else if constexpr (!FLAT) tma_load_2d(stage + d * SLOT + ST_D, &p.tmap_slope, px, py * 2, &bars[d]);
            }
            py += S * G;
            --pleft;
            ++pn;
        }
    }
    // Row GI (in march order) of the current group.  Groups never span two
    // segments; the group row of each march iteration is static (see march()).
    // GI < 0: the group row is the run-time gi (COMPACT marches)
    template <int GI>
    __device__ __forceinline__ void consume(CellVec& u, double& zx, double& zy, int gi = 0) {
        SWE_DCHECK(ring.d >= 0 && ring.d < D && req < pn);
        if constexpr (GI >= 0) gi = GI;
        if (GI == 0 || (GI < 0 && gi == 0)) {
            if constexpr (LATE) {
                __syncwarp();  // every lane is done with the released slot
                produce();
            }
            mbar_wait(&bars[ring.d], ring.ph);
        }
        const int g = FWD ? gi : G - 1 - gi;  // row within the box (boxes ascend in y)
        const double* st = stage + ring.d * SLOT;
        u.h = st[g * 3 * BW + lane + BO];
        u.qx = st[g * 3 * BW + BW + lane + BO];
        u.qy = st[g * 3 * BW + 2 * BW + lane + BO];
        if constexpr (XONLY) {
            zx = st[ST_D + g * BW + lane + BO];
            zy = 0.0;  // the bed's dz/dy bit patterns are all +0.0
        } else if constexpr (!FLAT) {
            zx = st[ST_D + g * 2 * BW + lane + BO];
            zy = st[ST_D + g * 2 * BW + BW + lane + BO];
        } else {
            zx = 0.0;
            zy = 0.0;
        }
        if (GI == G - 1 || (GI < 0 && gi == G - 1)) next_group();
    }
    __device__ __forceinline__ void next_group() {
        if (++ring.d == D) {
            ring.d = 0;
            ring.ph ^= 1u;
        }
        ++req;
        if constexpr (!LATE) {
            __syncwarp();
            produce();
        }
    }

    // output cell: guard (K5), CFL (K6), store, ghosts for the next step (K1)
    // on = false (SWE_EMIT_MASKED, lanes outside the output columns): the
    // arithmetic runs, the reductions and stores are masked.  SLOT: the row's
    // position in its output group (TMA-store epilogue; -1 = STG)
    template <bool EDGE, int SLOT = -1>
    __device__ __forceinline__ void emit(const CellVec& o, int rr, bool on = true) {
        const int jj = p.j0 + rr;
        double sx, sy;  // executor.hpp:560-580
        bool cfl_ok = true;
        if constexpr (EXACT) {
            double u, v;
            const Rc rc = A::recip(o.h);
            const double c = A::sqrt_(p.g * o.h);
            A::template div2<!EARLY>(o.qx, o.qy, rc, u, v);
            sx = fabs(u) + c;
            sy = fabs(v) + c;
        } else if constexpr (SWE_CFL_DEFER) {
            // the speeds of this row's cell are formed in the next emit (or at
            // the end of the segment), off this iteration's dependency chain
            cfl_speeds_fast(pend.h, pend.qx, pend.qy, p.sqrt_g, sx, sy);
            cfl_ok = pvalid;
            pend = o;
            pvalid = true;
        } else if constexpr ((SWE_ABL & 4) != 0) {
            sx = o.h;
            sy = o.qx;
        } else {
            cfl_speeds_fast(o.h, o.qx, o.qy, p.sqrt_g, sx, sy);
        }
        // guard (executor.hpp:543-558): a non-finite h, qx or qy always makes
        // sx + sy non-finite, so one test screens the cell; the exact test
        // runs only for the rare cell that fails the screen.
        // predicated: no branch splits the iteration's basic block
        {
            // h >= h_min also rejects NaN h; the speeds are NaN for a NaN qx, qy
            // or an infinite h, and an infinite qx makes the CFL maximum
            // infinite, which sends the step to the exact scan as well
            const bool ok = (o.h >= p.h_min) & !isnan(sx) & !isnan(sy);
            if (!(SWE_ABL & 2)) g_ok = g_ok & (ok | !on);
        }
        // CFL maxima; a NaN speed (only in a guarded cell) never replaces them
        cfl_ok = cfl_ok && on;
        mx = (cfl_ok && sx > mx) ? sx : mx;
        my = (cfl_ok && sy > my) ? sy : my;
        if constexpr (EARLY) {
            const unsigned long long hb = dbits(o.h), mom = dbits(o.qx) | dbits(o.qy);
            qo |= on ? (hb | mom) : 0ull;
            qn &= on ? (hb & ~mom) : ~0ull;
        }
        if constexpr (TSTORE && SLOT >= 0) {  // stage the row for the warp's TMA store of its group
            constexpr int gr = FWD ? SLOT : G - 1 - SLOT;  // row within the box (boxes ascend in y)
            double* sb = sstage + (NB == 2 ? (sgrp & 1u) * SD : 0) + gr * 3 * TW + (lane - R);
            if (on && !(SWE_ABL & 1)) {
                sb[0] = o.h;
                sb[TW] = o.qx;
                sb[2 * TW] = o.qy;
            }
        }
        double* row = orow;  // == nxt + (rr + R) * 3P + (i + SWE_XO)
        orow += S * 3 * P;
        SWE_DCHECK(!on || (row == nxt + (static_cast<long long>(rr + R) * 3 * P + (i + SWE_XO)) && rr >= 0 && rr < p.nloc &&
                           i >= 0 && i < p.nx));
        // (PAD: a halo lane of an interior window stores to its padding column)
        if (!(TSTORE && SLOT >= 0) && (on || (PAD && !EDGE)) && !(SWE_ABL & 1)) {
            row[0] = o.h;
            row[P] = o.qx;
            row[2 * P] = o.qy;
        }
        if constexpr (!EDGE) return;
        if (!on) return;
        double* q = nullptr;  // the neighbour's copy of this cell (fused halo push), if any
        if (p.p2p) {
            // fused halo push: this strip's R edge rows -- with their x ghosts,
            // below -- go straight into the neighbours' halo rows of the same
            // (candidate) buffer, over NVLink peer memory; the step's allreduce
            // orders them before the neighbours' next step (no send/recv)
            if (rr < R && p.peer_dn[sel ^ 1])
                q = p.peer_dn[sel ^ 1] + static_cast<size_t>(p.nloc_dn + rr + R) * 3 * P + (i + SWE_XO);
            else if (rr >= p.nloc - R && p.peer_up[sel ^ 1])
                q = p.peer_up[sel ^ 1] + static_cast<size_t>(rr - p.nloc + R) * 3 * P + (i + SWE_XO);
            if (q) {
                q[0] = o.h;
                q[P] = o.qx;
                q[2 * P] = o.qy;
                pushed = true;
            }
        }
        if (!(xedge || jj == 0 || jj == p.ny - 1)) return;
        SWE_DCHECK(row - nxt >= 3 * P && row - nxt + 2 * P + 1 < p.buf_doubles - 3 * P && rr + R < p.nloc + 2 * R);
        if (i == 0) {
            const CellVec g = edge_ghost(SWE_EDGE_W, p.bc[SWE_EDGE_W], o, p.z_w[rr + R], p.h_min);
            row[-1] = g.h;
            row[P - 1] = g.qx;
            row[2 * P - 1] = g.qy;
            if (q) {
                q[-1] = g.h;
                q[P - 1] = g.qx;
                q[2 * P - 1] = g.qy;
            }
        }
        if (i == p.nx - 1) {
            const CellVec g = edge_ghost(SWE_EDGE_E, p.bc[SWE_EDGE_E], o, p.z_e[rr + R], p.h_min);
            row[1] = g.h;
            row[P + 1] = g.qx;
            row[2 * P + 1] = g.qy;
            if (q) {
                q[1] = g.h;
                q[P + 1] = g.qx;
                q[2 * P + 1] = g.qy;
            }
        }
        if (jj == 0) {
            const CellVec g = edge_ghost(SWE_EDGE_S, p.bc[SWE_EDGE_S], o, p.z_s[i], p.h_min);
            double* gr = row - 3 * P;
            gr[0] = g.h;
            gr[P] = g.qx;
            gr[2 * P] = g.qy;
        }
        if (jj == p.ny - 1) {
            const CellVec g = edge_ghost(SWE_EDGE_N, p.bc[SWE_EDGE_N], o, p.z_n[i], p.h_min);
            double* gr = row + 3 * P;
            gr[0] = g.h;
            gr[P] = g.qx;
            gr[2 * P] = g.qy;
        }
    }

    // TMA-store epilogue, warp-uniform: before the first row of a group is
    // staged, the store issued from the same buffer two groups ago must have
    // finished reading it; after the last row, every lane's staged values are
    // made visible to the async proxy and lane 0 stores the group's box
    // (G rows x h/qx/qy x TW columns; the tensor map ends at column R + nx, so
    // the last window's out-of-domain lanes are clipped).
    __device__ __forceinline__ void group_begin() {
        if (lane == 0) {
            if constexpr (NB == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
        }
        __syncwarp();
    }
    __device__ __forceinline__ void group_flush() {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
            const int y0 = FWD ? erow0 + egrp * G : erow0 - (egrp + 1) * G;  // lowest row of the group
            SWE_DCHECK(y0 >= 0 && y0 + G <= p.nloc);
            tma_store_2d(&p.tmap_out[sel ^ 1], seg_tile * TW + SWE_XO, (y0 + R) * 3,
                         sstage + (NB == 2 ? (sgrp & 1u) * SD : 0));
            bulk_commit();
        }
        ++sgrp;
        ++egrp;
    }

    // boundary faces of row b (executor.hpp:471-514): walls carry pressure only,
    // inflow the flux of the pump states, the other kinds use U* ghosts.
    // Updates the own x face Hx and the y faces; returns the x face that belongs
    // to the neighbouring out-of-domain lane (handed over by the caller).
    __device__ __forceinline__ void boundary_faces(int b, int jb, const CellVec& U, const Flux& FU, const CellVec& Us,
                                                const Flux& FS, CellVec& Hx, CellVec& hy_a, CellVec& hy_b,
                                                CellVec& xo, int& give) {
        give = 0;
        if (!(i >= 0 && i < p.nx && jb >= 0 && jb < p.ny)) return;
        const unsigned long long idx = static_cast<unsigned long long>(jb) * p.nx + i;
        if (i == 0) {
            const SweBC& bc = p.bc[SWE_EDGE_W];
            CellVec w = Hx;
            bool set = true;
            if (bc.type == SWE_BC_WALL) {
                w = {0.0, avg(FU.fxx, FS.fxx), 0.0};
            } else if (bc.type == SWE_BC_INFLOW) {
                const CellVec a = flux_x_plain(pump_state(SWE_EDGE_W, bc.q_n, U), p.half_g);
                const CellVec c = flux_x_plain(pump_state(SWE_EDGE_W, bc.q_n, Us), p.half_g);
                w = {avg(a.h, c.h), avg(a.qx, c.qx), avg(a.qy, c.qy)};
            } else if (FWD) {
                const CellVec g = edge_ghost(SWE_EDGE_W, bc, Us, p.z_w[b + R], p.h_min);
                if (!(g.h >= p.h_min)) e4 = max(e4, ~idx);
                const CellVec c = flux_x_plain(g, p.half_g);
                w = {avg(U.qx, c.h), avg(FU.fxx, c.qx), avg(FU.fxy, c.qy)};
            } else {
                set = false;
            }
            if (set) {
                if (FWD) { xo = w; give = 1; }  // the west face is lane t-1's
                else Hx = w;
            }
        }
        if (i == p.nx - 1) {
            const SweBC& bc = p.bc[SWE_EDGE_E];
            CellVec e = Hx;
            bool set = true;
            if (bc.type == SWE_BC_WALL) {
                e = {0.0, avg(FU.fxx, FS.fxx), 0.0};
            } else if (bc.type == SWE_BC_INFLOW) {
                const CellVec a = flux_x_plain(pump_state(SWE_EDGE_E, bc.q_n, U), p.half_g);
                const CellVec c = flux_x_plain(pump_state(SWE_EDGE_E, bc.q_n, Us), p.half_g);
                e = {avg(a.h, c.h), avg(a.qx, c.qx), avg(a.qy, c.qy)};
            } else if (!FWD) {
                const CellVec g = edge_ghost(SWE_EDGE_E, bc, Us, p.z_e[b + R], p.h_min);
                if (!(g.h >= p.h_min)) e4 = max(e4, ~idx);
                const CellVec c = flux_x_plain(g, p.half_g);
                e = {avg(U.qx, c.h), avg(FU.fxx, c.qx), avg(FU.fxy, c.qy)};
            } else {
                set = false;
            }
            if (set) {
                if (FWD) Hx = e;
                else { xo = e; give = 1; }  // the east face is lane t+1's
            }
        }
        if (jb == 0) {
            const SweBC& bc = p.bc[SWE_EDGE_S];
            CellVec f = {0.0, 0.0, 0.0};
            bool set = true;
            if (bc.type == SWE_BC_WALL) {
                f = {0.0, 0.0, avg(FU.gyy, FS.gyy)};
            } else if (bc.type == SWE_BC_INFLOW) {
                const CellVec a = flux_y_plain(pump_state(SWE_EDGE_S, bc.q_n, U), p.half_g);
                const CellVec c = flux_y_plain(pump_state(SWE_EDGE_S, bc.q_n, Us), p.half_g);
                f = {avg(a.h, c.h), avg(a.qx, c.qx), avg(a.qy, c.qy)};
            } else if (FWD) {
                const CellVec g = edge_ghost(SWE_EDGE_S, bc, Us, p.z_s[i], p.h_min);
                if (!(g.h >= p.h_min)) e4 = max(e4, ~idx);
                const CellVec c = flux_y_plain(g, p.half_g);
                f = {avg(U.qy, c.h), avg(FU.fxy, c.qx), avg(FU.gyy, c.qy)};
            } else {
                set = false;
            }
            if (set) {
                if (FWD) hy_a = f;
                else hy_b = f;
            }
        }
        if (jb == p.ny - 1) {
            const SweBC& bc = p.bc[SWE_EDGE_N];
            CellVec f = {0.0, 0.0, 0.0};
            bool set = true;
            if (bc.type == SWE_BC_WALL) {
                f = {0.0, 0.0, avg(FU.gyy, FS.gyy)};
            } else if (bc.type == SWE_BC_INFLOW) {
                const CellVec a = flux_y_plain(pump_state(SWE_EDGE_N, bc.q_n, U), p.half_g);
                const CellVec c = flux_y_plain(pump_state(SWE_EDGE_N, bc.q_n, Us), p.half_g);
                f = {avg(a.h, c.h), avg(a.qx, c.qx), avg(a.qy, c.qy)};
            } else if (!FWD) {
                const CellVec g = edge_ghost(SWE_EDGE_N, bc, Us, p.z_n[i], p.h_min);
                if (!(g.h >= p.h_min)) e4 = max(e4, ~idx);
                const CellVec c = flux_y_plain(g, p.half_g);
                f = {avg(U.qy, c.h), avg(FU.fxy, c.qx), avg(FU.gyy, c.qy)};
            } else {
                set = false;
            }
            if (set) {
                if (FWD) hy_b = f;
                else hy_a = f;
            }
        }
    }

    // One iteration k of the march: `in` -> `out`.
    // EDGE = false: the segment touches no domain edge (interior window, rows
    // clear of j = 0 and j = ny-1), so every boundary test is compiled out.
    template <bool EDGE, bool DO12, bool DO3, bool EMIT, int GI = 0, int SLOT = -1>
    __device__ __forceinline__ void iter(int k, const Carry& in, Carry& out, int gi = 0) {
        const int b = r_start + S * k;  // stage-2 row (local)
        if constexpr (TSTORE && EMIT && SLOT == 0) group_begin();
        if constexpr (DO12) {
            // ======== stage 1: committed row b+S
            consume<GI>(out.U, out.zx, out.zy, gi);
            const Rc rcN = A::recip(out.U.h);
            out.FU = A::template flux<MANNING, !EARLY>(out.U, rcN, p.half_g);
            // SWE_LATE_SRC: row b+S's source term (Manning friction) is only
            // carried to the next iteration; placed after the predictor in the
            // source so the scheduler overlaps it with the U* chain
            if constexpr (!SWE_LATE_SRC)
                source_of<EXACT, MANNING && !(SWE_ABL & 16), FLAT, FLAT || XONLY>(out.U, out.FU, rcN, out.zx, out.zy, p.neg_g, p.gnn, out.srx, out.sry);

            // ======== stage 2: predictor at (i, b)   scheme.hpp:100-113
            const CellVec& U = in.U;
            const Flux& FU = in.FU;
            const CellVec& Un = out.U;
            const Flux& FN = out.FU;
            const double fn_h = shf_nb(U.qx);
            const double fn_qx = shf_nb(FU.fxx);
            const double fn_qy = shf_nb(FU.fxy);
            double df_h, df_qx, df_qy, dg_h, dg_qx, dg_qy;
            if constexpr (FWD) {
                df_h = fn_h - U.qx; df_qx = fn_qx - FU.fxx; df_qy = fn_qy - FU.fxy;
                dg_h = Un.qy - U.qy; dg_qx = FN.fxy - FU.fxy; dg_qy = FN.gyy - FU.gyy;
            } else {
                df_h = U.qx - fn_h; df_qx = FU.fxx - fn_qx; df_qy = FU.fxy - fn_qy;
                dg_h = U.qy - Un.qy; dg_qx = FU.fxy - FN.fxy; dg_qy = FU.gyy - FN.gyy;
            }
            CellVec Us;
            if constexpr (EXACT) {
                Us.h = (U.h - (dtdx * df_h + dtdy * dg_h)) + 0.0;
                Us.qx = (U.qx - (dtdx * df_qx + dtdy * dg_qx)) + dt * in.srx;
                Us.qy = (U.qy - (dtdx * df_qy + dtdy * dg_qy)) + dt * in.sry;
            } else {
                Us.h = U.h - __fma_rn(dtdx, df_h, dtdy * dg_h);
                Us.qx = __fma_rn(dt, in.srx, U.qx - __fma_rn(dtdx, df_qx, dtdy * dg_qx));
                Us.qy = __fma_rn(dt, in.sry, U.qy - __fma_rn(dtdx, df_qy, dtdy * dg_qy));
            }

            const int jb = p.j0 + b;
            // dry U* -> row-major first consumer (executor.hpp:429-436, 459-513)
            if constexpr (!EDGE) {  // interior rows: jb >= 1, consumer is the row-major next cell
                // every lane's U* is a real interior U* here, consumed by some
                // corrector cell: a flag, the host finds the first consumer
                if (!(SWE_ABL & 2)) d_ok = d_ok & (Us.h >= p.h_min);
            } else if (!(Us.h >= p.h_min) && star_ok && (!EDGE || (in_x && jb >= 0 && jb < p.ny))) {
                unsigned long long cons;
                if (FWD) cons = static_cast<unsigned long long>(jb) * p.nx + i;
                else if (jb >= 1) cons = static_cast<unsigned long long>(jb - 1) * p.nx + i;
                else if (i >= 1) cons = static_cast<unsigned long long>(jb) * p.nx + (i - 1);
                else cons = static_cast<unsigned long long>(jb) * p.nx + i;
                e4 = max(e4, ~cons);
            }
            // K2 precondition on the committed state (scheme.hpp:35-39)
            if constexpr (!EDGE) {
                // interior windows: every lane and march row is a domain cell
                // the reference's predictor reads
                if (!(SWE_ABL & 2)) e2 |= static_cast<int>(!(U.h >= p.h_min));
            } else {
                e2 |= static_cast<int>(!(U.h >= p.h_min) & (k >= 0) & (k < L) & out_x);
            }

            const Rc rcS = A::recip(Us.h);
            const Flux FS = A::template flux<MANNING, !EARLY>(Us, rcS, p.half_g);
            double ssx, ssy;
            source_of<EXACT, MANNING && !(SWE_ABL & 8), FLAT, FLAT || XONLY>(Us, FS, rcS, in.zx, in.zy, p.neg_g, p.gnn, ssx, ssy);
            if constexpr (SWE_LATE_SRC)
                source_of<EXACT, MANNING && !(SWE_ABL & 16), FLAT, FLAT || XONLY>(out.U, out.FU, rcN, out.zx, out.zy, p.neg_g, p.gnn, out.srx, out.sry);

            if constexpr (EXACT || !CLASSIC) {
                // own x face (FWD: east, BWD: west) and y face (b, b+S)   scheme.hpp:153-161
                CellVec Hx = {avg(fn_h, Us.qx), avg(fn_qx, FS.fxx), avg(fn_qy, FS.fxy)};
                out.Hyp = {avg(Un.qy, Us.qy), avg(FN.fxy, FS.fxy), avg(FN.gyy, FS.gyy)};
                CellVec hy_a = in.Hyp, hy_b = out.Hyp;  // faces (b-S, b) and (b, b+S)
                if (EDGE && (xedge || jb == 0 || jb == p.ny - 1)) {  // warp-uniform
                    CellVec xo = {0.0, 0.0, 0.0};
                    int give = 0;
                    boundary_faces(b, jb, U, FU, Us, FS, Hx, hy_a, hy_b, xo, give);
                    if (xedge) {  // hand the boundary face to the out-of-domain lane that owns it
                        const double gh = shf_nb(xo.h), gqx = shf_nb(xo.qx), gqy = shf_nb(xo.qy);
                        const int gv = FWD ? __shfl_down_sync(FULL, give, 1) : __shfl_up_sync(FULL, give, 1);
                        if (gv && i == (FWD ? -1 : p.nx)) Hx = {gh, gqx, gqy};
                    }
                }
                // the corrector's y-face term and source sum are formed here, so row c
                // carries 8 doubles less into stage 3 (same operations, same order)
                {
                    const CellVec& hs = FWD ? hy_a : hy_b;
                    const CellVec& hn = FWD ? hy_b : hy_a;
                    out.c_dy = {cy * (hn.h - hs.h), cy * (hn.qx - hs.qx), cy * (hn.qy - hs.qy)};
                }
                out.c_hx = Hx;
                out.Uc = U;
                out.c_sx = in.srx + ssx;
                out.c_sy = in.sry + ssy;
            } else {
                // FAST: the classic MacCormack corrector (see stage 3) needs F(U*)
                // and G(U*) of row b, U + U* and S(U*); the face form runs only
                // for cells with a boundary face (EDGE windows / rows)
                out.Gs = {Us.qy, FS.fxy, FS.gyy};
                out.c_fs = {Us.qx, FS.fxx, FS.fxy};
                out.c_sum = {U.h + Us.h, U.qx + Us.qx, U.qy + Us.qy};
                out.c_ssx = ssx;
                out.c_ssy = ssy;
                if (EDGE && (xedge || jb == 0 || jb == p.ny - 1)) {  // warp-uniform
                    CellVec Hx = {avg(fn_h, Us.qx), avg(fn_qx, FS.fxx), avg(fn_qy, FS.fxy)};
                    // face (b-S, b) from G(U_b) and G(U*_{b-S}) (bit-identical to
                    // the exact path's carried face), face (b, b+S)
                    CellVec hy_a = {avg(U.qy, in.Gs.h), avg(FU.fxy, in.Gs.qx), avg(FU.gyy, in.Gs.qy)};
                    CellVec hy_b = {avg(Un.qy, Us.qy), avg(FN.fxy, FS.fxy), avg(FN.gyy, FS.gyy)};
                    CellVec xo = {0.0, 0.0, 0.0};
                    int give = 0;
                    boundary_faces(b, jb, U, FU, Us, FS, Hx, hy_a, hy_b, xo, give);
                    if (xedge) {
                        const double gh = shf_nb(xo.h), gqx = shf_nb(xo.qx), gqy = shf_nb(xo.qy);
                        const int gv = FWD ? __shfl_down_sync(FULL, give, 1) : __shfl_up_sync(FULL, give, 1);
                        if (gv && i == (FWD ? -1 : p.nx)) Hx = {gh, gqx, gqy};
                    }
                    const CellVec& hs = FWD ? hy_a : hy_b;
                    const CellVec& hn = FWD ? hy_b : hy_a;
                    out.c_dy = {cy * (hn.h - hs.h), cy * (hn.qx - hs.qx), cy * (hn.qy - hs.qy)};
                    out.c_hx = Hx;
                    out.Uc = U;
                    out.c_sx = in.srx + ssx;
                    out.c_sy = in.sry + ssy;
                }
            }
        }

        if constexpr (DO3) {
            // ======== stage 3: corrector of row b   scheme.hpp:185-191
            const Carry& cc = out;  // row b's own stage-2 results (two-stage march)
            CellVec C;
            if constexpr (EXACT || !CLASSIC) {
                const CellVec ot = {shf_back(cc.c_hx.h), shf_back(cc.c_hx.qx), shf_back(cc.c_hx.qy)};
                const CellVec hw = FWD ? ot : cc.c_hx, he = FWD ? cc.c_hx : ot;
                if constexpr (EXACT) {
                    // cx = dt/dx, cy = dt/dy (scheme.hpp:185-191 evaluation order)
                    const double fs_h = cx * (he.h - hw.h) + cc.c_dy.h;
                    const double fs_qx = cx * (he.qx - hw.qx) + cc.c_dy.qx;
                    const double fs_qy = cx * (he.qy - hw.qy) + cc.c_dy.qy;
                    C.h = (cc.Uc.h - fs_h) + 0.0;
                    C.qx = (cc.Uc.qx - fs_qx) + half_dt * cc.c_sx;
                    C.qy = (cc.Uc.qy - fs_qy) + half_dt * cc.c_sy;
                } else {  // faces are plain sums, cx = dt/(2dx), cy = dt/(2dy)
                    const double fs_h = __fma_rn(cx, he.h - hw.h, cc.c_dy.h);
                    const double fs_qx = __fma_rn(cx, he.qx - hw.qx, cc.c_dy.qx);
                    const double fs_qy = __fma_rn(cx, he.qy - hw.qy, cc.c_dy.qy);
                    C.h = cc.Uc.h - fs_h;
                    C.qx = __fma_rn(half_dt, cc.c_sx, cc.Uc.qx - fs_qx);
                    C.qy = __fma_rn(half_dt, cc.c_sy, cc.Uc.qy - fs_qy);
                }
            } else {
                // FAST: with the interface fluxes H = (F(U) + F(U*))/2 expanded,
                // the face differences are the predictor's own differences plus
                // those of F(U*), G(U*), and the update collapses to the classic
                // MacCormack corrector
                //   U^{n+1} = (U + U*)/2 - cx dF* - cy dG* + (dt/2) S(U*)
                // (cx = dt/(2dx), cy = dt/(2dy); dF* the difference of F(U*) in
                // the corrector's direction).  Cells with a boundary face keep the
                // face form (boundary_faces), so every cell's arithmetic depends
                // only on its position, not on the work decomposition.
                const CellVec fb = {shf_back(cc.c_fs.h), shf_back(cc.c_fs.qx), shf_back(cc.c_fs.qy)};
                const CellVec& gp = in.Gs;  // G(U*) of row b - S
                CellVec dF, dG;
                if constexpr (FWD) {
                    dF = {cc.c_fs.h - fb.h, cc.c_fs.qx - fb.qx, cc.c_fs.qy - fb.qy};
                    dG = {cc.Gs.h - gp.h, cc.Gs.qx - gp.qx, cc.Gs.qy - gp.qy};
                } else {
                    dF = {fb.h - cc.c_fs.h, fb.qx - cc.c_fs.qx, fb.qy - cc.c_fs.qy};
                    dG = {gp.h - cc.Gs.h, gp.qx - cc.Gs.qx, gp.qy - cc.Gs.qy};
                }
                const double t_h = __fma_rn(cx, dF.h, cy * dG.h);
                const double t_qx = __fma_rn(cx, dF.qx, cy * dG.qx);
                const double t_qy = __fma_rn(cx, dF.qy, cy * dG.qy);
                C.h = __fma_rn(0.5, cc.c_sum.h, -t_h);
                C.qx = __fma_rn(0.5, cc.c_sum.qx, __fma_rn(half_dt, cc.c_ssx, -t_qx));
                C.qy = __fma_rn(0.5, cc.c_sum.qy, __fma_rn(half_dt, cc.c_ssy, -t_qy));
                if constexpr (EDGE) {
                    const int jb = p.j0 + b;
                    if (xedge || jb == 0 || jb == p.ny - 1) {  // warp-uniform
                        const CellVec ot = {shf_back(cc.c_hx.h), shf_back(cc.c_hx.qx), shf_back(cc.c_hx.qy)};
                        const CellVec hw = FWD ? ot : cc.c_hx, he = FWD ? cc.c_hx : ot;
                        if (i == 0 || i == p.nx - 1 || jb == 0 || jb == p.ny - 1) {
                            const double fs_h = __fma_rn(cx, he.h - hw.h, cc.c_dy.h);
                            const double fs_qx = __fma_rn(cx, he.qx - hw.qx, cc.c_dy.qx);
                            const double fs_qy = __fma_rn(cx, he.qy - hw.qy, cc.c_dy.qy);
                            C.h = cc.Uc.h - fs_h;
                            C.qx = __fma_rn(half_dt, cc.c_sx, cc.Uc.qx - fs_qx);
                            C.qy = __fma_rn(half_dt, cc.c_sy, cc.Uc.qy - fs_qy);
                        }
                    }
                }
            }
            const int c_row = b;
            if constexpr (!SMOOTH) {
                if constexpr (SWE_EMIT_MASKED || (PAD && !EDGE)) {
                    if (EMIT) emit<EDGE, SLOT>(C, c_row, out_x);
                } else {
                    if (EMIT && out_x) emit<EDGE, SLOT>(C, c_row);
                }
            } else {
                // smoothing of row q = c - S   (executor.hpp:533-540, scheme.hpp:197-204)
                const CellVec& Cp = in.Cp;
                if constexpr (EMIT) {
                    CellVec ce = {__shfl_down_sync(FULL, Cp.h, 1), __shfl_down_sync(FULL, Cp.qx, 1),
                                  __shfl_down_sync(FULL, Cp.qy, 1)};
                    CellVec cw = {__shfl_up_sync(FULL, Cp.h, 1), __shfl_up_sync(FULL, Cp.qx, 1),
                                  __shfl_up_sync(FULL, Cp.qy, 1)};
                    if (out_x) {
                        const int q = c_row - S;
                        const int jq = p.j0 + q;
                        CellVec cn = FWD ? C : in.Cpp;
                        CellVec cs = FWD ? in.Cpp : C;
                        if (EDGE && (xedge || jq == 0 || jq == p.ny - 1)) {
                            if (i == 0) cw = edge_ghost(SWE_EDGE_W, p.bc[SWE_EDGE_W], Cp, p.z_w[q + R], p.h_min);
                            if (i == p.nx - 1) ce = edge_ghost(SWE_EDGE_E, p.bc[SWE_EDGE_E], Cp, p.z_e[q + R], p.h_min);
                            if (jq == 0) cs = edge_ghost(SWE_EDGE_S, p.bc[SWE_EDGE_S], Cp, p.z_s[i], p.h_min);
                            if (jq == p.ny - 1) cn = edge_ghost(SWE_EDGE_N, p.bc[SWE_EDGE_N], Cp, p.z_n[i], p.h_min);
                        }
                        const double nu = p.nu;
                        CellVec o;
                        if constexpr (EXACT) {
                            o.h = Cp.h + nu * (((ce.h - Cp.h) + (cw.h - Cp.h)) + ((cn.h - Cp.h) + (cs.h - Cp.h)));
                            o.qx = Cp.qx + nu * (((ce.qx - Cp.qx) + (cw.qx - Cp.qx)) + ((cn.qx - Cp.qx) + (cs.qx - Cp.qx)));
                            o.qy = Cp.qy + nu * (((ce.qy - Cp.qy) + (cw.qy - Cp.qy)) + ((cn.qy - Cp.qy) + (cs.qy - Cp.qy)));
                        } else {  // U + nu (E + W + N + S - 4U), contracted
                            o.h = __fma_rn(nu, __fma_rn(-4.0, Cp.h, (ce.h + cw.h) + (cn.h + cs.h)), Cp.h);
                            o.qx = __fma_rn(nu, __fma_rn(-4.0, Cp.qx, (ce.qx + cw.qx) + (cn.qx + cs.qx)), Cp.qx);
                            o.qy = __fma_rn(nu, __fma_rn(-4.0, Cp.qy, (ce.qy + cw.qy) + (cn.qy + cs.qy)), Cp.qy);
                        }
                        emit<EDGE, SLOT>(o, q);
                    }
                }
                out.Cpp = Cp;
                out.Cp = C;
            }
        }
        if constexpr (TSTORE && EMIT && SLOT == G - 1) group_flush();
    }

    // March one segment: output rows [ra, rb) of one 32-column window.
    __device__ __forceinline__ void segment(const Seg& sg) {
        L = sg.rb - sg.ra;
        const int xw0 = sg.tile * TW - R;  // global column of lane 0
        i = xw0 + lane;
        in_x = (i >= 0) && (i < p.nx);
        out_x = in_x && lane >= R && lane < 32 - R;
        star_ok = FWD ? (lane < 31) : (lane > 0);
        xedge = (xw0 <= 0) || (xw0 + 31 >= p.nx - 1);
        r_start = FWD ? sg.ra : sg.rb - 1;
        seg_tile = sg.tile;
        erow0 = FWD ? sg.ra : sg.rb;
        egrp = 0;

        orow = nxt + static_cast<size_t>(r_start + R) * 3 * P + (i + SWE_XO);  // first output row
        qo = 0ull;
        qn = ~0ull;
        const int jlo = p.j0 + sg.ra - R - 1, jhi = p.j0 + sg.rb + R;  // rows the march touches, padded
        // segments with strip edge rows run the edge march too (fused halo push)
        const bool pedge = p.p2p && (sg.ra < R || sg.rb > p.nloc - R);
        const bool edge_march = xedge || jlo <= 0 || jhi >= p.ny - 1 || pedge;
        if constexpr (ONE_MARCH) {
            march<true>();
        } else {
            if (PAD && !edge_march && !out_x)  // lanes 0 and 31 of an interior window
                orow = nxt + static_cast<size_t>(r_start + R) * 3 * P +
                       (SWE_XO + p.nx + 2 + (2 * sg.tile + (lane != 0)) % 30);
            if (edge_march) march<true>();
            else march<false>();
        }
        if (pedge && __any_sync(FULL, pushed)) __threadfence_system();  // the peer stores, system-wide
        if constexpr (!EXACT && SWE_CFL_DEFER) {  // the segment's last pending cell
            double sx, sy;
            cfl_speeds_fast(pend.h, pend.qx, pend.qy, p.sqrt_g, sx, sy);
            mx = (pvalid && sx > mx) ? sx : mx;
            my = (pvalid && sy > my) ? sy : my;
            pvalid = false;
        }
        if constexpr (EARLY) {
            // quiet flag of this item in the candidate buffer: the depth bits
            // H when every output cell is (H, +0, +0) with H >= p.h_min, else 0
            const unsigned long long ref = __shfl_sync(FULL, qo, R);  // lane R is always an output lane
            const bool ok = !out_x || (qo == qn && qo == ref);
            const double H = __longlong_as_double(static_cast<long long>(ref));
            const bool quiet = __all_sync(FULL, ok) && H >= p.h_min && finite_d(H);
            if (lane == 0) {
                SWE_DCHECK((sg.ra / p.chunk) * p.ntiles + sg.tile < p.ntiles * p.nchunks);
                p.qflag[sel ^ 1][(sg.ra / p.chunk) * p.ntiles + sg.tile] = quiet ? ref : 0ull;
            }
        }
    }

    template <bool EDGE>
    __device__ __forceinline__ void march() {
        Carry A, B;
        // pre-iteration: committed row r_start - S*R
        consume<0>(A.U, A.zx, A.zy);  // march row 0
        {
            const Rc rc = A::recip(A.U.h);
            A.FU = A::template flux<MANNING, !EARLY>(A.U, rc, p.half_g);
            source_of<EXACT, MANNING, FLAT, FLAT || XONLY>(A.U, A.FU, rc, A.zx, A.zy, p.neg_g, p.gnn, A.srx, A.sry);
        }
        A.Hyp = {0.0, 0.0, 0.0};
        A.Gs = {0.0, 0.0, 0.0};
        A.Cp = {0.0, 0.0, 0.0};
        A.Cpp = {0.0, 0.0, 0.0};
        // corrector of row b in the same iteration as its predictor.  Row GI of
        // a group is static: the prologue consumes 2 (R = 1) or 4 (R = 2) rows.
        constexpr int GI0 = (SMOOTH ? 4 : 2) % G;  // group row of the first steady iteration
        int k;
        if constexpr (!SMOOTH) {
            iter<EDGE, true, false, false, 1>(-1, A, B);  // U* of the halo row
            k = 0;                                         // 0..L-1: full iterations
        } else {
            iter<EDGE, true, false, false, 1>(-2, A, B);      // U* of the outer halo row
            iter<EDGE, true, true, false, 2 % G>(-1, B, A);   // corrector of the halo row
            iter<EDGE, true, true, false, 3 % G>(0, A, B);    // first own row: its smoothing waits a row
            k = 1;                                             // 1..L: smooth + emit row b - S
        }
        const int k_last = SMOOTH ? L : L - 1;
        const int k_first = k;
        // carries enter the steady state in B and alternate (B->A, A->B, ...)
        if constexpr (COMPACT) {
            // two iterations per trip with run-time group rows: the
            // instruction footprint of a small-grid step (4-row items, no
            // trip runs twice) is two iteration bodies, not G
            int gi = GI0;
            for (; k + 1 <= k_last; k += 2) {
                iter<EDGE, true, true, true, -1>(k, B, A, gi);
                gi = (gi + 1) & (G - 1);
                iter<EDGE, true, true, true, -1>(k + 1, A, B, gi);
                gi = (gi + 1) & (G - 1);
            }
            if (k <= k_last) iter<EDGE, true, true, true, -1>(k, B, A, gi);
            k = k_last + 1;
        }
        for (; k + G - 1 <= k_last; k += G) {
            iter<EDGE, true, true, true, (GI0 + 0) % G, 0>(k, B, A);
            iter<EDGE, true, true, true, (GI0 + 1) % G, 1>(k + 1, A, B);
            if constexpr (G == 4) {
                iter<EDGE, true, true, true, (GI0 + 2) % G, 2>(k + 2, B, A);
                iter<EDGE, true, true, true, (GI0 + 3) % G, 3>(k + 3, A, B);
            }
        }
        const int rem = k_last - k + 1;  // 0 .. G-1 tail iterations
        if (rem > 0) {  // a segment's partial last group: plain STG stores
            iter<EDGE, true, true, true, (GI0 + 0) % G>(k, B, A);
            if constexpr (G == 4) {
                if (rem > 1) {
                    iter<EDGE, true, true, true, (GI0 + 1) % G>(k + 1, A, B);
                    if (rem > 2) iter<EDGE, true, true, true, (GI0 + 2) % G>(k + 2, B, A);
                }
            }
        }
        // release a half-consumed last group
        if ((GI0 + (k_last - k_first + 1) - 1) % G != G - 1) next_group();
    }
};

template <int WPB, bool FWD, bool SMOOTH, int BED, bool MANNING, bool EXACT, bool EARLY>
__global__ void __launch_bounds__(WPB * 32, (step_min_blocks<EXACT, BED == 0, MANNING>())) swe_step_kernel(const __grid_constant__ StepParams p) {
    using M = Marcher<WPB, FWD, SMOOTH, BED, MANNING, EXACT, EARLY>;
    constexpr int D = M::D;
    constexpr int NF = M::NF;
    constexpr unsigned FULL = 0xffffffffu;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    __shared__ Seg segq_all[WPB][M::QN];
    __shared__ int s_skip, s_sel, s_last;
    __shared__ unsigned s_nact;
    __shared__ double s_dt, s_tc;
    __shared__ double s_red[2][WPB];
    SweCtl* ctl = p.ctl;
    double* stage = reinterpret_cast<double*>(smem_raw) + warp * (D * M::SLOT);  // [D][SLOT]
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<double*>(smem_raw) + WPB * D * M::SLOT) + warp * D;
    // TMA-store staging: after the rings and barriers, 128-byte aligned
    constexpr size_t kStageOff = (static_cast<size_t>(WPB) * D * M::SLOT * 8 + WPB * D * 8 + 127) / 128 * 128;
    double* sstage = reinterpret_cast<double*>(smem_raw + kStageOff) + warp * M::NB * M::SD;

    if (tid == 0) {
        const volatile SweCtl* vc = ctl;
        int skip = vc->done;
        double dt = 0.0, tc = 0.0;
        if (!skip) {
            if (vc->mode == 1) {
                const double t = vc->t, te = vc->t_end, dr = vc->dt_raw;
                const double remaining = te - t;  // run.hpp:150-153
                const bool landing = dr >= remaining;
                dt = landing ? remaining : dr;
                tc = landing ? te : t + dt;
                if (!(t < te)) skip = 1;
            } else {
                dt = vc->dt_req;
                tc = vc->tcommit_req;
            }
        }
        s_skip = skip;
        s_dt = dt;
        s_tc = tc;
        s_sel = vc->sel;
        s_nact = EARLY ? vc->nactive : 0u;
    }
    if (lane == 0) {
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (s_skip) return;

    M m{p};
    m.stage = stage;
    m.bars = bars;
    m.segq = segq_all[warp];
    m.qhead = 0;
    m.qtail = 0;
    m.lane = lane;
    m.cur = p.buf[s_sel];
    m.sel = s_sel;
    m.px = 0;
    m.py = 0;
    m.nxt = p.buf[s_sel ^ 1];
    m.P = p.pitch;
    m.dt = s_dt;
    m.dtdx = m.dt / p.dx;  // scheme.hpp:110, 188-190
    m.dtdy = m.dt / p.dy;
    m.half_dt = 0.5 * m.dt;
    m.cx = EXACT ? m.dtdx : 0.5 * m.dtdx;
    m.cy = EXACT ? m.dtdy : 0.5 * m.dtdy;
    m.pleft = 0;
    m.pdone = false;
    m.pn = 0;
    m.req = 0;
    m.ring = {0, 0u};
    m.mx = 0.0;
    m.my = 0.0;
    m.e2 = 0;
    m.e4 = 0ull;
    m.g_ok = true;
    m.d_ok = true;
    m.nitems = EARLY ? s_nact : static_cast<unsigned>(p.ntiles) * static_cast<unsigned>(p.nchunks);  // this launch's items
    m.wctr = &ctl->work[p.wslot];
    m.qo = 0ull;
    m.qn = ~0ull;
    m.pend = {1.0, 0.0, 0.0};
    m.pvalid = false;
    m.pushed = false;
    m.sstage = sstage;
    m.sgrp = 0u;
    m.produce();
    while (m.qhead < m.qtail) {  // the producer keeps the queue ahead of the consumer
        const Seg sg = m.segq[m.qhead % M::QN];
        ++m.qhead;
        m.segment(sg);
    }
    SWE_DCHECK(m.pdone);  // the queue ran dry only after the last claim
    if constexpr (M::TSTORE) {  // this warp's bulk stores complete before the step is finalized
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }

    // ---- CTA reduction of the CFL maxima and error words
    double mx = m.mx, my = m.my;
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        my = fmax(my, __shfl_xor_sync(FULL, my, o));
    }
    if (lane == 0) {
        s_red[0][warp] = mx;
        s_red[1][warp] = my;
    }
    if (m.e2) atomicMax(&ctl->red[RED_E2], 1ull);
    if (m.e4) atomicMax(&ctl->red[RED_E4], m.e4);
    if (!m.g_ok) atomicMax(&ctl->red[RED_E5], 1ull);
    if (!m.d_ok) atomicMax(&ctl->red[RED_DRY], 1ull);
    __syncthreads();
    if (tid == 0) {
        double a = s_red[0][0], b = s_red[1][0];
        for (int w = 1; w < WPB; ++w) {
            a = fmax(a, s_red[0][w]);
            b = fmax(b, s_red[1][w]);
        }
        atomicMax(&ctl->red[RED_SX], dbits(a));
        atomicMax(&ctl->red[RED_SY], dbits(b));
        if (p.finalize) {
            __threadfence();
            const unsigned prev = atomicAdd(&ctl->finish, 1u);
            s_last = (prev == static_cast<unsigned>(gridDim.x) - 1u);
        } else {
            s_last = 0;
        }
    }
    __syncthreads();
    if (s_last && tid == 0) {
        __threadfence();
        finalize_step(p, ctl, s_dt, s_tc);
    }
}

// ------------------------------------------------------------ early exit
// Schedule kernel (Brodtkorb-style early-exit tiles), run
// before each early-exit step.  An eligible item (interior, flat bed over its
// 3x3 item neighbourhood; see item_elig_kernel) is skipped when all 9 items
// its output depends on (dependency radius R + 1 <= 3 < item size) are quiet
// with the same depth H in the committed buffer -- a flat bed at rest, a
// bit-exact fixed point of the step -- and the candidate buffer already holds
// that same quiet item.  Skipped items contribute their CFL speed
// sqrt(g H) (u = v = 0, exactly as the step's epilogue computes it) to the
// reduction words; the others are appended to the step's active list.
template <bool EXACT>
__global__ void __launch_bounds__(256) swe_schedule_kernel(const __grid_constant__ StepParams p) {
    SweCtl* ctl = p.ctl;
    __shared__ int s_go, s_sel;
    __shared__ double s_max[8];
    __shared__ unsigned long long s_cells[8];
    if (threadIdx.x == 0) {
        const volatile SweCtl* vc = ctl;
        int go = !vc->done;
        if (go && vc->mode == 1 && !(vc->t < vc->t_end)) go = 0;  // same no-op rule as the step
        s_go = go;
        s_sel = vc->sel;
    }
    __syncthreads();
    if (!s_go) return;
    const int sel = s_sel;
    const unsigned nitems = static_cast<unsigned>(p.ntiles) * static_cast<unsigned>(p.nchunks);
    const int tw = 32 - 2 * (p.nu > 0.0 ? 2 : 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double smax = 0.0;
    unsigned long long cells = 0ull;
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned base = blockIdx.x * blockDim.x; base < nitems; base += stride) {
        const unsigned item = base + threadIdx.x;
        bool skip = false;
        if (item < nitems && p.elig[item]) {
            const int rc = static_cast<int>(item / p.ntiles), tile = static_cast<int>(item % p.ntiles);
            const unsigned long long c = p.qflag[sel][item];
            skip = c != 0ull && p.qflag[sel ^ 1][item] == c;
            for (int d = 0; skip && d < 9; ++d)
                skip = p.qflag[sel][(rc + d / 3 - 1) * p.ntiles + tile + d % 3 - 1] == c;
            if (skip) {
                const double H = __longlong_as_double(static_cast<long long>(c));
                double s;  // the epilogue's own arithmetic for sqrt(g H)
                if constexpr (EXACT) {
                    s = Arith<EXACT>::sqrt_(p.g * H);
                } else {
                    s = cfl_quiet_fast(H, p.sqrt_g);
                }
                smax = (s > smax) ? s : smax;
                const int ra = rc * p.chunk, rb = min(ra + p.chunk, p.nloc);
                const int x0 = tile * tw, x1 = min(x0 + tw, p.nx);
                cells += static_cast<unsigned long long>(rb - ra) * static_cast<unsigned long long>(x1 - x0);
            }
        }
        const bool act = item < nitems && !skip;
        const unsigned ball = __ballot_sync(0xffffffffu, act);
        unsigned pos = 0;
        if (lane == 0 && ball) pos = atomicAdd(&ctl->nactive, static_cast<unsigned>(__popc(ball)));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (act) p.active[pos + __popc(ball & ((1u << lane) - 1u))] = item;
    }
    for (int o = 16; o > 0; o >>= 1) {
        smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
        cells += __shfl_xor_sync(0xffffffffu, cells, o);
    }
    if (lane == 0) {
        s_max[warp] = smax;
        s_cells[warp] = cells;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        unsigned long long n = 0ull;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            m = fmax(m, s_max[w]);
            n += s_cells[w];
        }
        if (n) {  // sx = sy = sqrt(g H) for a quiet cell
            atomicMax(&ctl->red[RED_SX], dbits(m));
            atomicMax(&ctl->red[RED_SY], dbits(m));
            atomicAdd(&p.stats[0], n);
        }
    }
}

// ------------------------------------------------------------ multi-step launch
// Small grids (C1 256^2, C2 512^2: the state sits in L2) are bound by per-launch
// latency -- launch gaps, an instruction cache refilled for the other sweep
// parity's kernel, TMA descriptor fetches, ring fill -- not by the step's
// work.  swe_multi_kernel runs up to `nsteps` steps of the device-resident
// run loop (mode 1, run.hpp:149-163) in ONE cooperative launch: both sweep
// directions are in the kernel, every CTA keeps the committed scalars (t,
// dt_raw, selector, step index) in shared memory and recomputes the finalize
// from the step's reduction words after a grid barrier, so the arithmetic,
// the landing clamp and the error outcome are those of the one-step kernel
// (finalize_compute), bit for bit.  Work counters and reduction words are
// triple-buffered by step (the buffer of step s+1 is cleared during step s:
// every CTA stopped reading it before the barrier of step s-1).  A failed
// step stops every CTA; the host resolves it as after a one-step launch.
#ifndef SWE_MULTI_ONE_MARCH
#define SWE_MULTI_ONE_MARCH 1  // multi-step kernels: one march body per direction (instruction cache)
#endif
#ifndef SWE_CG_GRID_SYNC
#define SWE_CG_GRID_SYNC 1  // cooperative_groups grid sync (C1 8.6 -> 6.8 us/step against grid_barrier)
#endif
#ifndef SWE_MULTI_STATIC
#define SWE_MULTI_STATIC 1  // static item assignment in multi-step launches (no per-item atomics)
#endif
__device__ __forceinline__ void grid_barrier(SweCtl* c, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = &c->bar_gen;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(&c->bar_count, 1u) == nblocks - 1u) {
            c->bar_count = 0u;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int WPB, bool FWD, bool SMOOTH, int BED, bool MANNING, bool EXACT>
__device__ __forceinline__ void multi_step_body(const StepParams& p, double* stage, unsigned long long* bars,
                                                Seg* segq, double* sstage, int lane, int warp, int sel, double dt,
                                                unsigned* wctr, unsigned long long* red, WarpRing& ring,
                                                double (*s_red)[WPB]) {
    using M = Marcher<WPB, FWD, SMOOTH, BED, MANNING, EXACT, false, SWE_MULTI_ONE_MARCH != 0>;
    constexpr unsigned FULL = 0xffffffffu;
    M m{p};
    m.stage = stage;
    m.bars = bars;
    m.segq = segq;
    m.qhead = 0;
    m.qtail = 0;
    m.lane = lane;
    m.cur = p.buf[sel];
    m.sel = sel;
    m.px = 0;
    m.py = 0;
    m.nxt = p.buf[sel ^ 1];
    m.P = p.pitch;
    m.dt = dt;
    m.dtdx = dt / p.dx;  // scheme.hpp:110, 188-190
    m.dtdy = dt / p.dy;
    m.half_dt = 0.5 * dt;
    m.cx = EXACT ? m.dtdx : 0.5 * m.dtdx;
    m.cy = EXACT ? m.dtdy : 0.5 * m.dtdy;
    m.pleft = 0;
    m.pdone = false;
    m.ring = ring;  // the ring continues across steps: slot pn % D == ring.d
    m.pn = ring.d;
    m.req = ring.d;
    m.mx = 0.0;
    m.my = 0.0;
    m.e2 = 0;
    m.e4 = 0ull;
    m.g_ok = true;
    m.d_ok = true;
    m.nitems = static_cast<unsigned>(p.ntiles) * static_cast<unsigned>(p.nchunks);
    m.wctr = SWE_MULTI_STATIC ? nullptr : wctr;
    m.sclaim = blockIdx.x * WPB + warp;
    m.qo = 0ull;
    m.qn = ~0ull;
    m.pend = {1.0, 0.0, 0.0};
    m.pvalid = false;
    m.pushed = false;
    m.sstage = sstage;
    m.sgrp = 0u;
    m.produce();
    while (m.qhead < m.qtail) {
        const Seg sg = m.segq[m.qhead % M::QN];
        ++m.qhead;
        m.segment(sg);
    }
    SWE_DCHECK(m.pdone);
    if constexpr (M::TSTORE) {
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    ring = m.ring;
    double mx = m.mx, my = m.my;
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        my = fmax(my, __shfl_xor_sync(FULL, my, o));
    }
    if (lane == 0) {
        s_red[0][warp] = mx;
        s_red[1][warp] = my;
    }
    if (m.e2) atomicMax(&red[RED_E2], 1ull);
    if (m.e4) atomicMax(&red[RED_E4], m.e4);
    if (!m.g_ok) atomicMax(&red[RED_E5], 1ull);
    if (!m.d_ok) atomicMax(&red[RED_DRY], 1ull);
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = s_red[0][0], b = s_red[1][0];
        for (int w = 1; w < WPB; ++w) {
            a = fmax(a, s_red[0][w]);
            b = fmax(b, s_red[1][w]);
        }
        atomicMax(&red[RED_SX], dbits(a));
        atomicMax(&red[RED_SY], dbits(b));
    }
}

template <int WPB, bool SMOOTH, int BED, bool MANNING, bool EXACT>
__global__ void __launch_bounds__(WPB * 32, (step_min_blocks<EXACT, BED == 0, MANNING>()))
    swe_multi_kernel(const __grid_constant__ StepParams p, int nsteps) {
    using MF = Marcher<WPB, true, SMOOTH, BED, MANNING, EXACT, false>;
    constexpr int D = MF::D;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    __shared__ Seg segq_all[WPB][MF::QN];
    __shared__ double s_red[2][WPB];
    __shared__ double s_t, s_dtraw, s_dt, s_tc, s_te, s_tm;
    __shared__ unsigned long long s_idx, s_steps;
    __shared__ int s_sel, s_done, s_go;
    SweCtl* ctl = p.ctl;
    double* stage = reinterpret_cast<double*>(smem_raw) + warp * (D * MF::SLOT);
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<double*>(smem_raw) + WPB * D * MF::SLOT) + warp * D;
    constexpr size_t kStageOff = (static_cast<size_t>(WPB) * D * MF::SLOT * 8 + WPB * D * 8 + 127) / 128 * 128;
    double* sstage = reinterpret_cast<double*>(smem_raw + kStageOff) + warp * MF::NB * MF::SD;
    if (tid == 0) {
        const volatile SweCtl* vc = ctl;
        s_t = vc->t;
        s_dtraw = vc->dt_raw;
        s_te = vc->t_end;
        s_tm = vc->t_mark;
        s_idx = vc->step_index;
        s_steps = vc->steps_done;
        s_sel = vc->sel;
        s_done = vc->done;
    }
    if (lane == 0) {
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncthreads();
    WarpRing ring{0, 0u};
    StepOutcome last{0, 0, -1, -1, 0, 0.0, 0.0, 0.0, 0.0, 0.0};
    double last_dt = 0.0, last_tc = 0.0;
    bool ran = false;
    for (int s = 0; s < nsteps; ++s) {
        if (tid == 0) {
            const double t = s_t, te = s_te, dr = s_dtraw;
            const double remaining = te - t;  // run.hpp:150-153
            const bool landing = dr >= remaining;
            s_dt = landing ? remaining : dr;
            s_tc = landing ? te : t + s_dt;
            s_go = !s_done && (t < te);
        }
        __syncthreads();
        if (!s_go) break;  // identical in every CTA: the state is
        const int b3 = s % 3, n3 = (s + 1) % 3;
        if (blockIdx.x == 0) {  // clear the next step's buffers (see above)
            if (tid < RED_N) ctl->mred[n3][tid] = 0ull;
            if (tid == 0) ctl->mwork[n3] = 0u;
        }
        if (s > 0 && lane == 0)  // the previous step's STG outputs are this step's TMA inputs
            asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if ((s_idx % 2ull) == 0ull)  // scheme.hpp:86-88
            multi_step_body<WPB, true, SMOOTH, BED, MANNING, EXACT>(p, stage, bars, segq_all[warp], sstage, lane,
                                                                   warp, s_sel, s_dt, &ctl->mwork[b3],
                                                                   ctl->mred[b3], ring, s_red);
        else
            multi_step_body<WPB, false, SMOOTH, BED, MANNING, EXACT>(p, stage, bars, segq_all[warp], sstage, lane,
                                                                    warp, s_sel, s_dt, &ctl->mwork[b3],
                                                                    ctl->mred[b3], ring, s_red);
        __threadfence();
        if constexpr (SWE_CG_GRID_SYNC != 0) cooperative_groups::this_grid().sync();
        else grid_barrier(ctl, gridDim.x);
        if (tid == 0) {
            const StepOutcome o = finalize_compute(p, ctl->mred[b3], s_tc);
            last = o;
            last_dt = s_dt;
            last_tc = s_tc;
            ran = true;
            if (o.status == 0) {
                s_sel ^= 1;
                s_t = s_tc;
                s_idx += 1ull;
                s_dtraw = o.dt_next;
                s_steps += 1ull;
                s_done = (!(s_tc < s_te) || s_tc >= s_tm) ? 1 : 0;
            } else {
                s_done = 1;
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) {  // the run's state for the host (every CTA holds the same)
        if (ran) write_outcome(ctl, last, last_dt, last_tc);
        ctl->sel = s_sel;
        ctl->t = s_t;
        ctl->step_index = s_idx;
        ctl->dt_raw = s_dtraw;
        ctl->steps_done = s_steps;
        ctl->done = s_done;
        __threadfence();
    }
}

template <int WPB, bool SMOOTH, int BED, bool EXACT, bool MANNING, bool EARLY>
constexpr size_t step_smem_bytes() {
    constexpr int D = step_stages<EXACT, BED == 0, MANNING, EARLY>();
    constexpr int NF = BED == 0 ? 3 : BED == 2 ? 4 : 5;
    constexpr size_t ring_bars =
        static_cast<size_t>(WPB) * D * step_slot_doubles(NF, swe_row_group(EXACT, EARLY), SMOOTH ? 2 : 1) * 8 +
        WPB * D * 8;
    if constexpr (!step_tma_store<WPB, SMOOTH, BED, EXACT, MANNING, EARLY>()) return ring_bars;
    // + per-warp TMA-store staging (one or two buffers), 128-byte aligned
    return (ring_bars + 127) / 128 * 128 + static_cast<size_t>(WPB) *
                                               step_tma_buffers<WPB, SMOOTH, BED, EXACT, MANNING, EARLY>() *
                                               step_stage_doubles<EXACT, EARLY, SMOOTH ? 28 : 30>() * 8;
}

}  // namespace swe_dev
