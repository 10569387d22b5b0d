// swe_common.cuh — shared pieces of the fused step kernel (swe_step2.cuh):
// PTX helpers (mbarrier, TMA tensor loads/stores), work items, finalize,
// boundary faces and ghost writes.
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

#include "swe_device.cuh"

namespace swe_dev {

#ifndef SWE_STAGES
#define SWE_STAGES 8
#endif
constexpr int kStages = SWE_STAGES;
#ifndef SWE_MINB
#define SWE_MINB 2
#endif

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

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y) : "memory");
}

#ifndef SWE_PF
#define SWE_PF 0  // rows of L2 prefetch ahead of the TMA ring (0 = off; measured no gain)
#endif

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
__device__ __forceinline__ void finalize_step(const StepParams& p, SweCtl* c, double dt, double tc) {
    volatile unsigned long long* red = c->red;
    const unsigned long long e2 = red[RED_E2], e4 = red[RED_E4], e5 = red[RED_E5];
    const unsigned long long dg = red[RED_DIAG];
    const double msx = __longlong_as_double(static_cast<long long>(red[RED_SX]));
    const double msy = __longlong_as_double(static_cast<long long>(red[RED_SY]));
    int status = 0, kind = 0, ei = -1, ej = -1;
    double et = 0.0, edt = 0.0, dt_next = 0.0;
    if (e2) {
        status = SWE_ERR_INSTABILITY; kind = 2;
    } else if (e4) {
        const unsigned long long idx = ~e4;
        status = SWE_ERR_INSTABILITY; kind = 4;
        ei = static_cast<int>(idx % static_cast<unsigned long long>(p.nx));
        ej = static_cast<int>(idx / static_cast<unsigned long long>(p.nx));
        et = tc;
    } else if (e5) {
        const unsigned long long idx = ~e5;
        status = SWE_ERR_INSTABILITY; kind = 5;
        ei = static_cast<int>(idx % static_cast<unsigned long long>(p.nx));
        ej = static_cast<int>(idx / static_cast<unsigned long long>(p.nx));
        et = tc;
    } else if (dg || p.always_diag || !(msx < p.tz_x) || !(msy < p.tz_y)) {
        status = SWE_STATUS_DIAG;
    } else {
        const double a = __ddiv_rn(p.dx, msx);
        const double b = __ddiv_rn(p.dy, msy);
        const double core = (b < a) ? b : a;
        const double dt_raw = std_min(p.cfl * core, p.dt_max);
        dt_next = dt_raw;
        if (dt_raw < p.dt_min) {
            status = SWE_ERR_STEP_COLLAPSE; kind = 6; edt = dt_raw; et = tc;
        }
    }
    c->max_sx = msx;
    c->max_sy = msy;
    c->dt_used = dt;
    c->t_commit = tc;
    c->dt_next = dt_next;
    c->status = status;
    c->err_kind = kind;
    c->err_i = ei;
    c->err_j = ej;
    c->err_t = et;
    c->err_dt = edt;
    if (status == 0) {
        c->sel ^= 1;
        c->t = tc;
        c->step_index += 1ull;
        c->dt_raw = dt_next;
        c->steps_done += 1ull;
        c->done = (c->mode == 1) ? !(tc < c->t_end) : 0;
    } else {
        c->done = 1;
    }
    for (int k = 0; k < RED_N; ++k) red[k] = 0ull;
    c->finish = 0u;
    c->work = 0u;
    __threadfence();
}

// --------------------------------------------------------------- the kernel
// One warp = one worker.  Lane t owns column i = x0 - R + t of a 32-column
// window; lanes R..31-R are output columns.  Iteration k of the row march is
// a 3-stage software pipeline over consecutive rows (march direction S):
//   stage 1  row b+S : committed row from the warp's TMA ring; F/G/S(U)
//   stage 2  row b   : predictor U*, F/G/S(U*), interface fluxes, boundary
//                      faces, dry-U* detection
//   stage 3  row b-S : corrector (+ smoothing of row b-2S), guard, CFL, store
// The three dependency chains interleave within the warp; x neighbours are
// exchanged with shuffles, so warps never wait for each other.  The steady
// state is unrolled by two with the pipeline registers ping-ponging between
// two carry sets, so no register moves are needed to advance the march.

struct WarpRing {  // per-warp TMA ring state (warp-uniform)
    int d;         // stage of the next request to consume
    unsigned ph;   // its mbarrier phase parity
};

// Inputs of the boundary-face construction (executor.hpp:471-514).
struct EdgeIn {
    CellVec U, Us;
    double fu_xx, fu_xy, fu_yy, fs_xx, fs_xy, fs_yy;
    CellVec Hx, hy_a, hy_b;  // faces before the override
};
struct EdgeOut {
    CellVec Hx, hy_a, hy_b, xo;  // overridden faces; xo: face handed to the neighbour lane
    int give;
    unsigned long long e4;
};

// Boundary faces of one cell at a domain edge: walls carry pressure only,
// inflow the flux of the pump states, the other kinds use U* ghosts.  Out of
// line: only edge windows/rows call it.  `sum` selects fast-mode face sums
// (the 0.5 of iface_flux is folded into the corrector's dt/dx there).
template <bool FWD>
static __device__ __noinline__ EdgeOut boundary_faces(const EdgeIn in, int i, int jb, int nx, int ny,
                                                    const SweBC* bc, double zw, double ze, double zs, double zn,
                                                    double h_min, double half_g, unsigned long long e4,
                                                    bool sum) {
    EdgeOut o;
    o.Hx = in.Hx;
    o.hy_a = in.hy_a;
    o.hy_b = in.hy_b;
    o.xo = {0.0, 0.0, 0.0};
    o.give = 0;
    o.e4 = e4;
    auto fc = [sum](double a, double b) { return sum ? (a + b) : 0.5 * (a + b); };
    const unsigned long long idx = static_cast<unsigned long long>(jb) * nx + i;
    const CellVec& U = in.U;
    const CellVec& Us = in.Us;
    if (i == 0) {
        const SweBC& w = bc[SWE_EDGE_W];
        CellVec f;
        bool set = true;
        if (w.type == SWE_BC_WALL) {
            f = {0.0, fc(in.fu_xx, in.fs_xx), 0.0};
        } else if (w.type == SWE_BC_INFLOW) {
            const CellVec a = flux_x_plain(pump_state(SWE_EDGE_W, w.q_n, U), half_g);
            const CellVec c = flux_x_plain(pump_state(SWE_EDGE_W, w.q_n, Us), half_g);
            f = {fc(a.h, c.h), fc(a.qx, c.qx), fc(a.qy, c.qy)};
        } else if (FWD) {
            const CellVec g = edge_ghost(SWE_EDGE_W, w, Us, zw, h_min);
            if (!(g.h >= h_min)) o.e4 = max(o.e4, ~idx);
            const CellVec c = flux_x_plain(g, half_g);
            f = {fc(U.qx, c.h), fc(in.fu_xx, c.qx), fc(in.fu_xy, c.qy)};
        } else {
            set = false;
        }
        if (set) {
            if (FWD) { o.xo = f; o.give = 1; }  // the west face is lane t-1's
            else o.Hx = f;
        }
    }
    if (i == nx - 1) {
        const SweBC& e = bc[SWE_EDGE_E];
        CellVec f;
        bool set = true;
        if (e.type == SWE_BC_WALL) {
            f = {0.0, fc(in.fu_xx, in.fs_xx), 0.0};
        } else if (e.type == SWE_BC_INFLOW) {
            const CellVec a = flux_x_plain(pump_state(SWE_EDGE_E, e.q_n, U), half_g);
            const CellVec c = flux_x_plain(pump_state(SWE_EDGE_E, e.q_n, Us), half_g);
            f = {fc(a.h, c.h), fc(a.qx, c.qx), fc(a.qy, c.qy)};
        } else if (!FWD) {
            const CellVec g = edge_ghost(SWE_EDGE_E, e, Us, ze, h_min);
            if (!(g.h >= h_min)) o.e4 = max(o.e4, ~idx);
            const CellVec c = flux_x_plain(g, half_g);
            f = {fc(U.qx, c.h), fc(in.fu_xx, c.qx), fc(in.fu_xy, c.qy)};
        } else {
            set = false;
        }
        if (set) {
            if (FWD) o.Hx = f;
            else { o.xo = f; o.give = 1; }  // the east face is lane t+1's
        }
    }
    if (jb == 0) {
        const SweBC& sb = bc[SWE_EDGE_S];
        CellVec f;
        bool set = true;
        if (sb.type == SWE_BC_WALL) {
            f = {0.0, 0.0, fc(in.fu_yy, in.fs_yy)};
        } else if (sb.type == SWE_BC_INFLOW) {
            const CellVec a = flux_y_plain(pump_state(SWE_EDGE_S, sb.q_n, U), half_g);
            const CellVec c = flux_y_plain(pump_state(SWE_EDGE_S, sb.q_n, Us), half_g);
            f = {fc(a.h, c.h), fc(a.qx, c.qx), fc(a.qy, c.qy)};
        } else if (FWD) {
            const CellVec g = edge_ghost(SWE_EDGE_S, sb, Us, zs, h_min);
            if (!(g.h >= h_min)) o.e4 = max(o.e4, ~idx);
            const CellVec c = flux_y_plain(g, half_g);
            f = {fc(U.qy, c.h), fc(in.fu_xy, c.qx), fc(in.fu_yy, c.qy)};
        } else {
            set = false;
        }
        if (set) {
            if (FWD) o.hy_a = f;
            else o.hy_b = f;
        }
    }
    if (jb == ny - 1) {
        const SweBC& nb = bc[SWE_EDGE_N];
        CellVec f;
        bool set = true;
        if (nb.type == SWE_BC_WALL) {
            f = {0.0, 0.0, fc(in.fu_yy, in.fs_yy)};
        } else if (nb.type == SWE_BC_INFLOW) {
            const CellVec a = flux_y_plain(pump_state(SWE_EDGE_N, nb.q_n, U), half_g);
            const CellVec c = flux_y_plain(pump_state(SWE_EDGE_N, nb.q_n, Us), half_g);
            f = {fc(a.h, c.h), fc(a.qx, c.qx), fc(a.qy, c.qy)};
        } else if (!FWD) {
            const CellVec g = edge_ghost(SWE_EDGE_N, nb, Us, zn, h_min);
            if (!(g.h >= h_min)) o.e4 = max(o.e4, ~idx);
            const CellVec c = flux_y_plain(g, half_g);
            f = {fc(U.qy, c.h), fc(in.fu_xy, c.qx), fc(in.fu_yy, c.qy)};
        } else {
            set = false;
        }
        if (set) {
            if (FWD) o.hy_b = f;
            else o.hy_a = f;
        }
    }
    return o;
}

// Ghost cells of an output cell for the next step's K1 (executor.hpp:384-408),
// written next to it in the padded buffer.  Out of line: edge cells only.
static __device__ __noinline__ void write_ghosts(double* row, int P, CellVec o, int i, int jj, int nx, int ny,
                                                const SweBC* bc, double zw, double ze, double zs, double zn,
                                                double h_min) {
    if (i == 0) {
        const CellVec g = edge_ghost(SWE_EDGE_W, bc[SWE_EDGE_W], o, zw, h_min);
        row[-1] = g.h;
        row[P - 1] = g.qx;
        row[2 * P - 1] = g.qy;
    }
    if (i == nx - 1) {
        const CellVec g = edge_ghost(SWE_EDGE_E, bc[SWE_EDGE_E], o, ze, h_min);
        row[1] = g.h;
        row[P + 1] = g.qx;
        row[2 * P + 1] = g.qy;
    }
    if (jj == 0) {
        const CellVec g = edge_ghost(SWE_EDGE_S, bc[SWE_EDGE_S], o, zs, h_min);
        double* gr = row - 3 * P;
        gr[0] = g.h;
        gr[P] = g.qx;
        gr[2 * P] = g.qy;
    }
    if (jj == ny - 1) {
        const CellVec g = edge_ghost(SWE_EDGE_N, bc[SWE_EDGE_N], o, zn, h_min);
        double* gr = row + 3 * P;
        gr[0] = g.h;
        gr[P] = g.qx;
        gr[2 * P] = g.qy;
    }
}

}  // namespace swe_dev
