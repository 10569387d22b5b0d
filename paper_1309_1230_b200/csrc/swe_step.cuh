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
//   K2+K4 fused per CTA with row marching: a CTA owns a 128-column window and
//        walks a contiguous run of rows in the sweep direction.  Each state's
//        fluxes F/G are evaluated once per cell and shared: x-neighbours
//        through shared memory, y-neighbours in registers.  Interface fluxes
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
// Committed rows arrive through a 4-stage cp.async.bulk (TMA bulk copy)
// ring with mbarrier completion; stores are coalesced 8-byte STG.
#pragma once

#include "swe_device.cuh"

namespace swe_dev {

constexpr int kStages = 4;

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

// ------------------------------------------------------------ work partition
// CTA b owns units [b*U/G, (b+1)*U/G) of the unit space u = tile*nloc + row.
// A unit run is split into segments at tile boundaries.
struct Seg {
    int tile, ra, rb;
};

__device__ __forceinline__ int seg_list(const StepParams& p, int b, Seg* segs, int maxseg) {
    const long long total = static_cast<long long>(p.ntiles) * p.nloc;
    long long u = total * b / p.ncta;
    const long long u1 = total * (b + 1) / p.ncta;
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
    __threadfence();
}

// --------------------------------------------------------------- the kernel
// Block = NT compute threads (one column each) + one producer warp that
// streams committed rows into the shared-memory ring with TMA bulk copies.
template <int NT, bool FWD, bool SMOOTH, bool FLAT, bool MANNING>
__global__ void __launch_bounds__(NT + 32, 3) swe_step_kernel(const __grid_constant__ StepParams p) {
    constexpr int R = SMOOTH ? 2 : 1;
    constexpr int S = FWD ? 1 : -1;
    constexpr int NF = FLAT ? 3 : 5;
    constexpr int D = kStages;
    constexpr int MAXSEG = 8;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* stage = reinterpret_cast<double*>(smem_raw);  // [D][NF][NT]
    double* xF = stage + D * NF * NT;                     // [2][3][NT] committed F (qx, fxx, fxy)
    double* xH = xF + 2 * 3 * NT;                         // [2][3][NT] x-interface fluxes
    double* xC = xH + 2 * 3 * NT;                         // [2][3][NT] corrector output (SMOOTH)
    unsigned long long* bars =  // [D] full, [D] empty
        reinterpret_cast<unsigned long long*>(xC + (SMOOTH ? 2 * 3 * NT : 0));
    unsigned long long* ebars = bars + D;

    __shared__ Seg segs[MAXSEG];
    __shared__ int s_nseg, s_skip, s_sel, s_last;
    __shared__ double s_dt, s_tc;
    __shared__ double s_red[2][NT / 32];

    const int tid = threadIdx.x;
    SweCtl* ctl = p.ctl;

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
        s_nseg = seg_list(p, blockIdx.x, segs, MAXSEG);
        for (int d = 0; d < D; ++d) {
            mbar_init(&bars[d], 1);
            mbar_init(&ebars[d], NT / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (s_skip) return;

    const double dt = s_dt, tc = s_tc;
    const double dtdx = dt / p.dx, dtdy = dt / p.dy, half_dt = 0.5 * dt;
    const double* __restrict__ cur = p.buf[s_sel];
    double* __restrict__ nxt = p.buf[s_sel ^ 1];
    const int P = p.pitch;
    const int nseg = s_nseg;
    const double h_min = p.h_min, half_g = p.half_g, neg_g = p.neg_g, gnn = p.gnn;

    int req = 0;  // next request to consume
    double mx = 0.0, my = 0.0;
    unsigned long long e2 = 0, e4 = 0, e5 = 0;

    if (tid >= NT) {
        // ---- producer warp: request n = (segment, row), L + 2R per segment, in
        // consumption order; stage n % D is refilled once every compute warp
        // has released request n - D (empty barrier).
        if (tid == NT) {
            int n = 0;
            for (int k = 0; k < nseg; ++k) {
                const int cnt = (segs[k].rb - segs[k].ra) + 2 * R;
                const size_t col0 = static_cast<size_t>(segs[k].tile) * (NT - 2 * R);  // padded x0-R
                for (int m = 0; m < cnt; ++m, ++n) {
                    const int row = FWD ? segs[k].ra - R + m : segs[k].rb - 1 + R - m;
                    const int d = n % D;
                    if (n >= D) mbar_wait(&ebars[d], static_cast<unsigned>(((n / D) - 1) & 1));
                    double* dst = stage + d * NF * NT;
                    const double* src = cur + static_cast<size_t>(row + R) * 3 * P + col0;
                    mbar_expect_tx(&bars[d], NF * NT * 8);
                    bulk_g2s(dst, src, NT * 8, &bars[d]);
                    bulk_g2s(dst + NT, src + P, NT * 8, &bars[d]);
                    bulk_g2s(dst + 2 * NT, src + 2 * P, NT * 8, &bars[d]);
                    if constexpr (!FLAT) {
                        const double* ss = p.slope + static_cast<size_t>(row + R) * 2 * P + col0;
                        bulk_g2s(dst + 3 * NT, ss, NT * 8, &bars[d]);
                        bulk_g2s(dst + 4 * NT, ss + P, NT * 8, &bars[d]);
                    }
                }
            }
        }
    } else {

    const unsigned lane = tid & 31u;
    auto consume = [&](CellVec& u, double& zx, double& zy) {
        const int d = req % D;
        mbar_wait(&bars[d], static_cast<unsigned>((req / D) & 1));
        const double* st = stage + d * NF * NT;
        u.h = st[tid];
        u.qx = st[NT + tid];
        u.qy = st[2 * NT + tid];
        if constexpr (!FLAT) {
            zx = st[3 * NT + tid];
            zy = st[4 * NT + tid];
        } else {
            zx = 0.0;
            zy = 0.0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ebars[d]);
    };
    auto csync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };

    for (int sgi = 0; sgi < nseg; ++sgi) {
        const Seg sg = segs[sgi];
        const int L = sg.rb - sg.ra;
        const int i = sg.tile * (NT - 2 * R) - R + tid;  // global column of this thread
        const bool in_x = (i >= 0) && (i < p.nx);
        const bool out_x = in_x && tid >= R && tid < NT - R;
        const bool corr_x = tid >= 1 && tid < NT - 1;
        const bool star_ok = FWD ? (tid < NT - 1) : (tid > 0);
        const int r_start = FWD ? sg.ra : sg.rb - 1;
        // CTA-uniform: does this window touch the west/east domain edge?
        const int xw0 = sg.tile * (NT - 2 * R) - R;
        const bool xedge_cta = (xw0 <= 0) || (xw0 + NT - 1 >= p.nx - 1);
        constexpr int E = R;             // warm-up rows
        constexpr int X = SMOOTH ? 1 : 0;  // extra trailing iteration
        constexpr int KC = SMOOTH ? -1 : 0;

        // ---- pre-iteration: row r_start - S*E
        CellVec U;
        double zx, zy;
        consume(U, zx, zy);
        ++req;
        Recip rcU = make_recip(U.h);
        Flux FU = flux_of(U, rcU, half_g);
        double srx, sry;
        source_of<MANNING>(U, FU, rcU, zx, zy, neg_g, gnn, srx, sry);
        int par = 0;
        xF[(par * 3 + 0) * NT + tid] = U.qx;
        xF[(par * 3 + 1) * NT + tid] = FU.fxx;
        xF[(par * 3 + 2) * NT + tid] = FU.fxy;
        csync();

        CellVec Hyp = {0.0, 0.0, 0.0};
        CellVec Cp = {0.0, 0.0, 0.0}, Cpp = {0.0, 0.0, 0.0};

        for (int k = -E; k <= L - 1 + X; ++k) {
            const int r = r_start + S * k;  // local row of this iteration
            const int j = p.j0 + r;         // global row
            // 1. lookahead row r+S
            CellVec Un;
            double zxn, zyn;
            consume(Un, zxn, zyn);
            ++req;
            const Recip rcN = make_recip(Un.h);
            const Flux FN = flux_of(Un, rcN, half_g);
            double srxn, sryn;
            source_of<MANNING>(Un, FN, rcN, zxn, zyn, neg_g, gnn, srxn, sryn);

            // 2. predictor U* at (i, r)   scheme.hpp:100-113
            const int tn = FWD ? (tid + 1 < NT ? tid + 1 : tid) : (tid > 0 ? tid - 1 : tid);
            const double fn_h = xF[(par * 3 + 0) * NT + tn];
            const double fn_qx = xF[(par * 3 + 1) * NT + tn];
            const double fn_qy = xF[(par * 3 + 2) * NT + tn];
            double df_h, df_qx, df_qy, dg_h, dg_qx, dg_qy;
            if constexpr (FWD) {
                df_h = fn_h - U.qx; df_qx = fn_qx - FU.fxx; df_qy = fn_qy - FU.fxy;
                dg_h = Un.qy - U.qy; dg_qx = FN.fxy - FU.fxy; dg_qy = FN.gyy - FU.gyy;
            } else {
                df_h = U.qx - fn_h; df_qx = FU.fxx - fn_qx; df_qy = FU.fxy - fn_qy;
                dg_h = U.qy - Un.qy; dg_qx = FU.fxy - FN.fxy; dg_qy = FU.gyy - FN.gyy;
            }
            CellVec Us;
            Us.h = (U.h - (dtdx * df_h + dtdy * dg_h)) + 0.0;
            Us.qx = (U.qx - (dtdx * df_qx + dtdy * dg_qx)) + dt * srx;
            Us.qy = (U.qy - (dtdx * df_qy + dtdy * dg_qy)) + dt * sry;

            // dry U* -> first consumer (executor.hpp:429-436, 459-513)
            const bool row_in = (j >= 0) && (j < p.ny);
            if (star_ok && in_x && row_in && !(Us.h >= h_min)) {
                unsigned long long cons;
                if (FWD) cons = static_cast<unsigned long long>(j) * p.nx + i;
                else if (j >= 1) cons = static_cast<unsigned long long>(j - 1) * p.nx + i;
                else if (i >= 1) cons = static_cast<unsigned long long>(j) * p.nx + (i - 1);
                else cons = static_cast<unsigned long long>(j) * p.nx + i;
                e4 = max(e4, ~cons);
            }
            const Recip rcS = make_recip(Us.h);
            const Flux FS = flux_of(Us, rcS, half_g);
            double ssx, ssy;
            source_of<MANNING>(Us, FS, rcS, zx, zy, neg_g, gnn, ssx, ssy);

            // 3. interface fluxes  scheme.hpp:153-161
            CellVec Hxo;  // FWD: i+1/2 ; BWD: i-1/2
            Hxo.h = 0.5 * (fn_h + Us.qx);
            Hxo.qx = 0.5 * (fn_qx + FS.fxx);
            Hxo.qy = 0.5 * (fn_qy + FS.fxy);
            CellVec Hyn;  // FWD: j+1/2 ; BWD: j-1/2
            Hyn.h = 0.5 * (Un.qy + Us.qy);
            Hyn.qx = 0.5 * (FN.fxy + FS.fxy);
            Hyn.qy = 0.5 * (FN.gyy + FS.gyy);
            xH[(par * 3 + 0) * NT + tid] = Hxo.h;
            xH[(par * 3 + 1) * NT + tid] = Hxo.qx;
            xH[(par * 3 + 2) * NT + tid] = Hxo.qy;
            xF[((par ^ 1) * 3 + 0) * NT + tid] = Un.qx;
            xF[((par ^ 1) * 3 + 1) * NT + tid] = FN.fxx;
            xF[((par ^ 1) * 3 + 2) * NT + tid] = FN.fxy;
            csync();

            // 4. corrector  executor.hpp:451-519, scheme.hpp:185-191
            CellVec C = {0.0, 0.0, 0.0};
            const bool do_corr = (k >= KC) && corr_x;
            if (do_corr) {
                const int to = tid - S;
                CellVec Hxx;
                Hxx.h = xH[(par * 3 + 0) * NT + to];
                Hxx.qx = xH[(par * 3 + 1) * NT + to];
                Hxx.qy = xH[(par * 3 + 2) * NT + to];
                CellVec hw = FWD ? Hxx : Hxo, he = FWD ? Hxo : Hxx;
                CellVec hs = FWD ? Hyp : Hyn, hn = FWD ? Hyn : Hyp;
                const bool yedge_row = (j == 0) || (j == p.ny - 1);
                if ((xedge_cta || yedge_row) && in_x && row_in) {
                    const bool west = (i == 0), east = (i == p.nx - 1);
                    const bool south = (j == 0), north = (j == p.ny - 1);
                    if (west | east | south | north) {
                        const unsigned long long idx = static_cast<unsigned long long>(j) * p.nx + i;
                        if (west) {
                            const SweBC& bc = p.bc[SWE_EDGE_W];
                            if (bc.type == SWE_BC_WALL) {
                                hw = {0.0, 0.5 * (FU.fxx + FS.fxx), 0.0};
                            } else if (bc.type == SWE_BC_INFLOW) {
                                const CellVec a = flux_x_plain(pump_state(SWE_EDGE_W, bc.q_n, U), half_g);
                                const CellVec b = flux_x_plain(pump_state(SWE_EDGE_W, bc.q_n, Us), half_g);
                                hw = {0.5 * (a.h + b.h), 0.5 * (a.qx + b.qx), 0.5 * (a.qy + b.qy)};
                            } else if (FWD) {
                                const CellVec g = edge_ghost(SWE_EDGE_W, bc, Us, p.z_w[r + R], h_min);
                                if (!(g.h >= h_min)) e4 = max(e4, ~idx);
                                const CellVec b = flux_x_plain(g, half_g);
                                hw = {0.5 * (U.qx + b.h), 0.5 * (FU.fxx + b.qx), 0.5 * (FU.fxy + b.qy)};
                            }
                        }
                        if (east) {
                            const SweBC& bc = p.bc[SWE_EDGE_E];
                            if (bc.type == SWE_BC_WALL) {
                                he = {0.0, 0.5 * (FU.fxx + FS.fxx), 0.0};
                            } else if (bc.type == SWE_BC_INFLOW) {
                                const CellVec a = flux_x_plain(pump_state(SWE_EDGE_E, bc.q_n, U), half_g);
                                const CellVec b = flux_x_plain(pump_state(SWE_EDGE_E, bc.q_n, Us), half_g);
                                he = {0.5 * (a.h + b.h), 0.5 * (a.qx + b.qx), 0.5 * (a.qy + b.qy)};
                            } else if (!FWD) {
                                const CellVec g = edge_ghost(SWE_EDGE_E, bc, Us, p.z_e[r + R], h_min);
                                if (!(g.h >= h_min)) e4 = max(e4, ~idx);
                                const CellVec b = flux_x_plain(g, half_g);
                                he = {0.5 * (U.qx + b.h), 0.5 * (FU.fxx + b.qx), 0.5 * (FU.fxy + b.qy)};
                            }
                        }
                        if (south) {
                            const SweBC& bc = p.bc[SWE_EDGE_S];
                            if (bc.type == SWE_BC_WALL) {
                                hs = {0.0, 0.0, 0.5 * (FU.gyy + FS.gyy)};
                            } else if (bc.type == SWE_BC_INFLOW) {
                                const CellVec a = flux_y_plain(pump_state(SWE_EDGE_S, bc.q_n, U), half_g);
                                const CellVec b = flux_y_plain(pump_state(SWE_EDGE_S, bc.q_n, Us), half_g);
                                hs = {0.5 * (a.h + b.h), 0.5 * (a.qx + b.qx), 0.5 * (a.qy + b.qy)};
                            } else if (FWD) {
                                const CellVec g = edge_ghost(SWE_EDGE_S, bc, Us, p.z_s[i], h_min);
                                if (!(g.h >= h_min)) e4 = max(e4, ~idx);
                                const CellVec b = flux_y_plain(g, half_g);
                                hs = {0.5 * (U.qy + b.h), 0.5 * (FU.fxy + b.qx), 0.5 * (FU.gyy + b.qy)};
                            }
                        }
                        if (north) {
                            const SweBC& bc = p.bc[SWE_EDGE_N];
                            if (bc.type == SWE_BC_WALL) {
                                hn = {0.0, 0.0, 0.5 * (FU.gyy + FS.gyy)};
                            } else if (bc.type == SWE_BC_INFLOW) {
                                const CellVec a = flux_y_plain(pump_state(SWE_EDGE_N, bc.q_n, U), half_g);
                                const CellVec b = flux_y_plain(pump_state(SWE_EDGE_N, bc.q_n, Us), half_g);
                                hn = {0.5 * (a.h + b.h), 0.5 * (a.qx + b.qx), 0.5 * (a.qy + b.qy)};
                            } else if (!FWD) {
                                const CellVec g = edge_ghost(SWE_EDGE_N, bc, Us, p.z_n[i], h_min);
                                if (!(g.h >= h_min)) e4 = max(e4, ~idx);
                                const CellVec b = flux_y_plain(g, half_g);
                                hn = {0.5 * (U.qy + b.h), 0.5 * (FU.fxy + b.qx), 0.5 * (FU.gyy + b.qy)};
                            }
                        }
                    }
                }
                const double fs_h = dtdx * (he.h - hw.h) + dtdy * (hn.h - hs.h);
                const double fs_qx = dtdx * (he.qx - hw.qx) + dtdy * (hn.qx - hs.qx);
                const double fs_qy = dtdx * (he.qy - hw.qy) + dtdy * (hn.qy - hs.qy);
                C.h = (U.h - fs_h) + 0.0;
                C.qx = (U.qx - fs_qx) + half_dt * (srx + ssx);
                C.qy = (U.qy - fs_qy) + half_dt * (sry + ssy);
            }

            // K2 precondition on the committed state (scheme.hpp:35-39)
            if (k >= 0 && k < L && out_x && !(U.h >= h_min)) e2 = 1;

            // 5. output row (guard, CFL, store, next-step ghosts)
            auto emit = [&](const CellVec& o, int rr) {
                const int jj = p.j0 + rr;
                const unsigned long long idx = static_cast<unsigned long long>(jj) * p.nx + i;
                const bool ok = finite_d(o.h) && finite_d(o.qx) && finite_d(o.qy) && o.h >= h_min;
                if (!ok) e5 = max(e5, ~idx);
                // K6 executor.hpp:560-580
                const Recip rc = make_recip(o.h);
                const double c = __dsqrt_rn(p.g * o.h);
                double u, v;
                div2(o.qx, o.qy, rc, u, v);
                const double sx = fabs(u) + c;
                const double sy = fabs(v) + c;
                mx = fmax(mx, sx);
                my = fmax(my, sy);
                const size_t rb = static_cast<size_t>(rr + R) * 3;
                const size_t col = static_cast<size_t>(i + R);
                nxt[(rb + 0) * P + col] = o.h;
                nxt[(rb + 1) * P + col] = o.qx;
                nxt[(rb + 2) * P + col] = o.qy;
                // K1 of the next step: ghosts of the committed candidate
                if (!(xedge_cta || jj == 0 || jj == p.ny - 1)) return;
                if (i == 0) {
                    const CellVec g = edge_ghost(SWE_EDGE_W, p.bc[SWE_EDGE_W], o, p.z_w[rr + R], h_min);
                    nxt[(rb + 0) * P + col - 1] = g.h;
                    nxt[(rb + 1) * P + col - 1] = g.qx;
                    nxt[(rb + 2) * P + col - 1] = g.qy;
                }
                if (i == p.nx - 1) {
                    const CellVec g = edge_ghost(SWE_EDGE_E, p.bc[SWE_EDGE_E], o, p.z_e[rr + R], h_min);
                    nxt[(rb + 0) * P + col + 1] = g.h;
                    nxt[(rb + 1) * P + col + 1] = g.qx;
                    nxt[(rb + 2) * P + col + 1] = g.qy;
                }
                if (jj == 0) {
                    const CellVec g = edge_ghost(SWE_EDGE_S, p.bc[SWE_EDGE_S], o, p.z_s[i], h_min);
                    const size_t gb = static_cast<size_t>(rr - 1 + R) * 3;
                    nxt[(gb + 0) * P + col] = g.h;
                    nxt[(gb + 1) * P + col] = g.qx;
                    nxt[(gb + 2) * P + col] = g.qy;
                }
                if (jj == p.ny - 1) {
                    const CellVec g = edge_ghost(SWE_EDGE_N, p.bc[SWE_EDGE_N], o, p.z_n[i], h_min);
                    const size_t gb = static_cast<size_t>(rr + 1 + R) * 3;
                    nxt[(gb + 0) * P + col] = g.h;
                    nxt[(gb + 1) * P + col] = g.qx;
                    nxt[(gb + 2) * P + col] = g.qy;
                }
            };

            if constexpr (!SMOOTH) {
                if (k >= 0 && out_x) emit(C, r);
            } else {
                // smoothing of row q = r - S   (executor.hpp:533-540, scheme.hpp:197-204)
                if (k >= 1 && out_x) {
                    const int q = r - S;
                    const int jq = p.j0 + q;
                    const int pp = par ^ 1;
                    CellVec Ce, Cw, Cn, Cs;
                    Ce = {xC[(pp * 3 + 0) * NT + tid + 1], xC[(pp * 3 + 1) * NT + tid + 1],
                          xC[(pp * 3 + 2) * NT + tid + 1]};
                    Cw = {xC[(pp * 3 + 0) * NT + tid - 1], xC[(pp * 3 + 1) * NT + tid - 1],
                          xC[(pp * 3 + 2) * NT + tid - 1]};
                    Cn = FWD ? C : Cpp;
                    Cs = FWD ? Cpp : C;
                    if (xedge_cta || jq == 0 || jq == p.ny - 1) {
                    if (i == 0) Cw = edge_ghost(SWE_EDGE_W, p.bc[SWE_EDGE_W], Cp, p.z_w[q + R], h_min);
                    if (i == p.nx - 1) Ce = edge_ghost(SWE_EDGE_E, p.bc[SWE_EDGE_E], Cp, p.z_e[q + R], h_min);
                    if (jq == 0) Cs = edge_ghost(SWE_EDGE_S, p.bc[SWE_EDGE_S], Cp, p.z_s[i], h_min);
                    if (jq == p.ny - 1) Cn = edge_ghost(SWE_EDGE_N, p.bc[SWE_EDGE_N], Cp, p.z_n[i], h_min);
                    }
                    const double nu = p.nu;
                    CellVec o;
                    o.h = Cp.h + nu * (((Ce.h - Cp.h) + (Cw.h - Cp.h)) + ((Cn.h - Cp.h) + (Cs.h - Cp.h)));
                    o.qx = Cp.qx + nu * (((Ce.qx - Cp.qx) + (Cw.qx - Cp.qx)) + ((Cn.qx - Cp.qx) + (Cs.qx - Cp.qx)));
                    o.qy = Cp.qy + nu * (((Ce.qy - Cp.qy) + (Cw.qy - Cp.qy)) + ((Cn.qy - Cp.qy) + (Cs.qy - Cp.qy)));
                    emit(o, q);
                }
                xC[(par * 3 + 0) * NT + tid] = C.h;
                xC[(par * 3 + 1) * NT + tid] = C.qx;
                xC[(par * 3 + 2) * NT + tid] = C.qy;
                Cpp = Cp;
                Cp = C;
            }

            // 6. shift the march
            U = Un;
            FU = FN;
            srx = srxn;
            sry = sryn;
            zx = zxn;
            zy = zyn;
            Hyp = Hyn;
            par ^= 1;
        }
        csync();  // smem exchange slots are reused by the next segment
    }
    }  // compute threads

    // ---- CTA reduction of the CFL maxima and error words
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        my = fmax(my, __shfl_xor_sync(0xffffffffu, my, o));
    }
    if ((tid & 31) == 0 && tid < NT) {
        s_red[0][tid >> 5] = mx;
        s_red[1][tid >> 5] = my;
    }
    if (e2) atomicMax(&ctl->red[RED_E2], 1ull);
    if (e4) atomicMax(&ctl->red[RED_E4], e4);
    if (e5) atomicMax(&ctl->red[RED_E5], e5);
    __syncthreads();
    if (tid == 0) {
        double a = s_red[0][0], b = s_red[1][0];
        for (int w = 1; w < NT / 32; ++w) {
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
        finalize_step(p, ctl, dt, tc);
    }
}

template <int NT, bool FWD, bool SMOOTH, bool FLAT>
constexpr size_t step_smem_bytes() {
    return static_cast<size_t>(kStages) * (FLAT ? 3 : 5) * NT * 8 + 2 * 3 * NT * 8 * (SMOOTH ? 3 : 2) +
           2 * kStages * 8;
}

}  // namespace swe_dev
