// swe_step.cuh — the fused MacCormack step (plan K1-K6 + smoothing) as one
// sm_100a kernel per time step.  Every lane owns TWO adjacent columns, a
// warp a 64-column window (2 halo + 60 output + 2 halo columns).  Same numerics and plan as swe_step.cuh (merged
// schedule: stage 1 load+fluxes of row b+S, stage 2 predictor of row b,
// stage 3 corrector/smoothing/guard/CFL/store), but the per-row costs of a
// lane (ring wait, TMA issue, bookkeeping, votes, row addressing) are shared
// by two cells, the x exchange needs one shuffle per pair instead of one per
// cell, and the two cells give the scheduler independent dependency chains.
#pragma once

#include "swe_common.cuh"

namespace swe_dev {

// Registers carried from one row to the next.  The committed state and bed
// slopes of row b are NOT carried: they are re-read from row b's TMA ring slot,
// which is only refilled at the end of the iteration that consumes row b+S.
// The source term is recomputed from them (carried only with Manning friction,
// whose pow/rcbrt is too expensive to repeat).
struct Carry {
    Flux FU[2];
    double srx[2], sry[2];   // S(U) of row b (Manning only)
    CellVec Hyp[2];          // y face (b-S, b)
    CellVec Cp[2], Cpp[2];   // corrector rows b-S, b-2S (smoothing)
};

template <int WPB, bool FWD, bool SMOOTH, bool FLAT, bool MANNING, bool EXACT>
struct Marcher {
    using A = Arith<EXACT>;
    using Rc = typename A::Rc;
    static constexpr int R = SMOOTH ? 2 : 1;
    static constexpr int S = FWD ? 1 : -1;
    static constexpr int NF = FLAT ? 3 : 5;
    static constexpr int D = kStages;
    static constexpr int W = 64;           // window columns
    static constexpr int XH = SWE_XOFF;    // halo columns per side (2: keeps TMA boxes 16-byte aligned)
    static constexpr int TW = W - 2 * XH;  // output columns per window
    static constexpr int QN = 4;
    static constexpr unsigned FULL = 0xffffffffu;

    static constexpr int NO = 3;  // output staging buffers (TMA store ring)
    static constexpr int OB = (3 * TW + 15) / 16 * 16;  // doubles per staging buffer (128-byte aligned)
    const StepParams& p;
    double* stage;
    double* ostage;  // [NO][3][TW] staged output rows
    int obuf;        // next output staging buffer
    unsigned long long* bars;
    Seg* segq;
    int qhead, qtail;
    int lane;
    double* nxt;
    int P;
    double dt, dtdx, dtdy, half_dt, h_min, half_g, neg_g, gnn, cx, cy;
    int pleft;
    bool pdone;
    int px, py, pzy, sel;
    int pn, req;
    WarpRing ring;
    int dprev;           // ring slot of the previously consumed row (row b during iteration k)
    int i0, L, r_start;  // i0: global column of the lane's first cell
    int tile_x;
    bool in_x[2], out_x[2], star_ok[2], xedge;
    double mx, my;
    unsigned long long e4, e5;
    int e2;

    static __device__ __forceinline__ double face(double a, double b) {
        if constexpr (EXACT) return 0.5 * (a + b);
        else return a + b;
    }
    // value of the neighbouring lane towards +x (down) / -x (up)
    static __device__ __forceinline__ double from_right(double x) { return __shfl_down_sync(FULL, x, 1); }
    static __device__ __forceinline__ double from_left(double x) { return __shfl_up_sync(FULL, x, 1); }

    __device__ __forceinline__ void prod_seg() {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(&p.ctl->work, 1u);
        item = __shfl_sync(FULL, item, 0);
        const unsigned nitems = static_cast<unsigned>(p.ntiles) * static_cast<unsigned>(p.nchunks);
        if (item >= nitems) {
            pleft = 0;
            pdone = true;
            return;
        }
        const int rc = static_cast<int>(item / p.ntiles);
        const int tile = static_cast<int>(item % p.ntiles);
        Seg sg;
        sg.tile = tile;
        sg.ra = rc * p.chunk;
        sg.rb = min(sg.ra + p.chunk, p.nloc);
        segq[qtail % QN] = sg;
        ++qtail;
        pleft = (sg.rb - sg.ra) + 2 * R;
        const int row = FWD ? sg.ra - R : sg.rb - 1 + R;
        px = tile * TW;  // padded column of the window start
        py = (row + R) * 3;
        pzy = (row + R) * 2;
    }
    __device__ __forceinline__ void produce() {
#ifdef SWE_COMPUTEONLY
        if (pleft == 0 && !(pdone || qtail - qhead >= QN - 1)) prod_seg();
        if (pleft > 0) {
            --pleft;
            ++pn;
        }
        return;
#endif
        while (pn < req + D - 2) {  // keep the slots of rows b and b+S resident
            if (pleft == 0 && !(pdone || qtail - qhead >= QN - 1)) prod_seg();
            if (pleft == 0) return;
            const int d = pn % D;
            if (lane == 0) {
                mbar_expect_tx(&bars[d], NF * W * 8);
                tma_load_2d(stage + d * NF * W, &p.tmap_state[sel], px, py, &bars[d]);
                if constexpr (!FLAT) tma_load_2d(stage + d * NF * W + 3 * W, &p.tmap_slope, px, pzy, &bars[d]);
                if constexpr (SWE_PF > 0) {  // warm L2 for the row SWE_PF requests later (same window)
                    if (pleft > SWE_PF) {
                        tma_prefetch_2d(&p.tmap_state[sel], px, py + S * 3 * SWE_PF);
                        if constexpr (!FLAT) tma_prefetch_2d(&p.tmap_slope, px, pzy + S * 2 * SWE_PF);
                    }
                }
            }
            py += S * 3;
            pzy += S * 2;
            --pleft;
            ++pn;
        }
    }
    // read the two cells of a resident ring slot
    __device__ __forceinline__ void read_slot(int d, CellVec (&u)[2], double (&zx)[2], double (&zy)[2]) const {
#ifdef SWE_COMPUTEONLY
        {
            const double r = 1e-6 * static_cast<double>(d);
            u[0] = {1.0 + r + 1e-5 * lane, 0.01 + r, 0.002 - r};
            u[1] = {1.0 - r + 2e-5 * lane, 0.012 - r, 0.001 + r};
            zx[0] = zx[1] = FLAT ? 0.0 : 1e-5;
            zy[0] = zy[1] = 0.0;
            return;
        }
#endif
        const double* st = stage + d * NF * W + 2 * lane;
        const double2 h = *reinterpret_cast<const double2*>(st);
        const double2 qx = *reinterpret_cast<const double2*>(st + W);
        const double2 qy = *reinterpret_cast<const double2*>(st + 2 * W);
        u[0] = {h.x, qx.x, qy.x};
        u[1] = {h.y, qx.y, qy.y};
        if constexpr (!FLAT) {
            const double2 a = *reinterpret_cast<const double2*>(st + 3 * W);
            const double2 c = *reinterpret_cast<const double2*>(st + 4 * W);
            zx[0] = a.x;
            zx[1] = a.y;
            zy[0] = c.x;
            zy[1] = c.y;
        } else {
            zx[0] = zx[1] = zy[0] = zy[1] = 0.0;
        }
    }
    __device__ __forceinline__ void consume(CellVec (&u)[2], double (&zx)[2], double (&zy)[2]) {
#ifdef SWE_COMPUTEONLY
        {
            const double r = 1e-6 * static_cast<double>(req & 15);
            u[0] = {1.0 + r + 1e-5 * lane, 0.01 + r, 0.002 - r};
            u[1] = {1.0 - r + 2e-5 * lane, 0.012 - r, 0.001 + r};
            zx[0] = zx[1] = FLAT ? 0.0 : 1e-5;
            zy[0] = zy[1] = 0.0;
            dprev = ring.d;
            if (++ring.d == D) {
                ring.d = 0;
                ring.ph ^= 1u;
            }
            ++req;
            return;
        }
#endif
        mbar_wait(&bars[ring.d], ring.ph);
        dprev = ring.d;
        const double* st = stage + ring.d * NF * W + 2 * lane;
        const double2 h = *reinterpret_cast<const double2*>(st);
        const double2 qx = *reinterpret_cast<const double2*>(st + W);
        const double2 qy = *reinterpret_cast<const double2*>(st + 2 * W);
        u[0] = {h.x, qx.x, qy.x};
        u[1] = {h.y, qx.y, qy.y};
        if constexpr (!FLAT) {
            const double2 a = *reinterpret_cast<const double2*>(st + 3 * W);
            const double2 c = *reinterpret_cast<const double2*>(st + 4 * W);
            zx[0] = a.x;
            zx[1] = a.y;
            zy[0] = c.x;
            zy[1] = c.y;
        } else {
            zx[0] = zx[1] = zy[0] = zy[1] = 0.0;
        }
        if (++ring.d == D) {
            ring.d = 0;
            ring.ph ^= 1u;
        }
        ++req;
    }
    __device__ __forceinline__ void fluxes(const CellVec& u, double zx, double zy, Flux& f, double& sx,
                                           double& sy) const {
        const Rc rc = A::recip(u.h);
        f = A::flux(u, rc, half_g);
        source_of<EXACT, MANNING>(u, f, rc, zx, zy, neg_g, gnn, sx, sy);
    }

    // guard + CFL + store of the lane's two cells of row rr (executor.hpp:543-580)
    __device__ __forceinline__ void emit2(const CellVec (&o)[2], int rr) {
        bool bad[2];
        double* row = nxt + static_cast<size_t>(rr + R) * 3 * P + (i0 + XH);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const bool ok = finite_d(o[c].h) && finite_d(o[c].qx) && finite_d(o[c].qy) && o[c].h >= h_min;
            const Rc rc = A::recip(o[c].h);
            const double cc = A::sqrt_(p.g * o[c].h);
            double u, v;
            A::div2(o[c].qx, o[c].qy, rc, u, v);
            const double sx = fabs(u) + cc, sy = fabs(v) + cc;
            if (out_x[c]) {
                mx = fmax(mx, sx);
                my = fmax(my, sy);
            }
            bad[c] = out_x[c] && !ok;
        }
#if defined(SWE_COMPUTEONLY) && !defined(SWE_KEEPSTORES) || defined(SWE_NOSTORES)
        if (o[0].h == -12345.0) row[0] = o[1].qx + o[0].qy;  // never true: keeps the values live
        if (true) return;
#endif
        if (!xedge) {  // stage the row and hand it to the TMA engine (asynchronous)
            bulk_wait_read<NO - 1>();  // the buffer reused now has been read by its store
            __syncwarp();
            double* ob = ostage + obuf * OB;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int t = 2 * lane + c - XH;  // output column within the window
                if (out_x[c]) {
                    ob[t] = o[c].h;
                    ob[TW + t] = o[c].qx;
                    ob[2 * TW + t] = o[c].qy;
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_2d(&p.tmap_out[sel ^ 1], tile_x, (rr + R) * 3, ob);
                bulk_commit();
            }
            if (++obuf == NO) obuf = 0;
        } else if (out_x[0] && out_x[1]) {  // 16-byte stores (the column pair is 16-byte aligned)
            *reinterpret_cast<double2*>(row) = make_double2(o[0].h, o[1].h);
            *reinterpret_cast<double2*>(row + P) = make_double2(o[0].qx, o[1].qx);
            *reinterpret_cast<double2*>(row + 2 * P) = make_double2(o[0].qy, o[1].qy);
        } else {
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if (out_x[c]) {
                    row[c] = o[c].h;
                    row[P + c] = o[c].qx;
                    row[2 * P + c] = o[c].qy;
                }
        }
        const int jj = p.j0 + rr;
        if (__any_sync(FULL, bad[0] || bad[1])) {
            for (int c = 1; c >= 0; --c)
                if (bad[c]) e5 = max(e5, ~(static_cast<unsigned long long>(jj) * p.nx + (i0 + c)));
        }
        if (xedge || jj == 0 || jj == p.ny - 1) {
            for (int c = 0; c < 2; ++c) {
                const int ic = i0 + c;
                if (out_x[c] && (ic == 0 || ic == p.nx - 1 || jj == 0 || jj == p.ny - 1))
                    write_ghosts(row + c, P, o[c], ic, jj, p.nx, p.ny, p.bc, p.z_w[rr + R], p.z_e[rr + R],
                                 p.z_s[ic], p.z_n[ic], h_min);
            }
        }
    }

    template <bool DO3, bool EMIT>
    __device__ __forceinline__ void iter(int k, const Carry& in, Carry& out) {
        const int b = r_start + S * k;
        const int jb = p.j0 + b;
        const int dslot_b = dprev;  // row b's ring slot
        CellVec Un[2];
        double zxn[2], zyn[2];
        consume(Un, zxn, zyn);
        // row b, re-read from its resident slot
        CellVec Ub[2];
        double zxb[2], zyb[2];
        read_slot(dslot_b, Ub, zxb, zyb);
        // ---- stage 1: fluxes (and Manning source) of row b+S
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const Rc rc = A::recip(Un[c].h);
            out.FU[c] = A::flux(Un[c], rc, half_g);
            if constexpr (MANNING)
                source_of<EXACT, MANNING>(Un[c], out.FU[c], rc, zxn[c], zyn[c], neg_g, gnn, out.srx[c], out.sry[c]);
        }
        // source of row b: carried (Manning) or recomputed (scheme.hpp:54-63, fr = 0)
        double srxb[2], sryb[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if constexpr (MANNING) {
                srxb[c] = in.srx[c];
                sryb[c] = in.sry[c];
            } else {
                const double gh = neg_g * Ub[c].h;
                srxb[c] = gh * zxb[c] - 0.0 * Ub[c].qx;
                sryb[c] = gh * zyb[c] - 0.0 * Ub[c].qy;
            }
        }
        // ---- stage 2: predictor of row b   scheme.hpp:100-113
        // F of the x neighbour each cell differences with
        double fn_h[2], fn_qx[2], fn_qy[2];
        if constexpr (FWD) {
            fn_h[0] = Ub[1].qx;
            fn_qx[0] = in.FU[1].fxx;
            fn_qy[0] = in.FU[1].fxy;
            fn_h[1] = from_right(Ub[0].qx);
            fn_qx[1] = from_right(in.FU[0].fxx);
            fn_qy[1] = from_right(in.FU[0].fxy);
        } else {
            fn_h[1] = Ub[0].qx;
            fn_qx[1] = in.FU[0].fxx;
            fn_qy[1] = in.FU[0].fxy;
            fn_h[0] = from_left(Ub[1].qx);
            fn_qx[0] = from_left(in.FU[1].fxx);
            fn_qy[0] = from_left(in.FU[1].fxy);
        }
        CellVec Us[2], Hx[2], hs[2], hn[2];
        Flux FS[2];
        double ssx[2], ssy[2];
        bool dry[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const CellVec& U = Ub[c];
            const Flux& FU = in.FU[c];
            const Flux& FN = out.FU[c];
            double df_h, df_qx, df_qy, dg_h, dg_qx, dg_qy;
            if constexpr (FWD) {
                df_h = fn_h[c] - U.qx; df_qx = fn_qx[c] - FU.fxx; df_qy = fn_qy[c] - FU.fxy;
                dg_h = Un[c].qy - U.qy; dg_qx = FN.fxy - FU.fxy; dg_qy = FN.gyy - FU.gyy;
            } else {
                df_h = U.qx - fn_h[c]; df_qx = FU.fxx - fn_qx[c]; df_qy = FU.fxy - fn_qy[c];
                dg_h = U.qy - Un[c].qy; dg_qx = FU.fxy - FN.fxy; dg_qy = FU.gyy - FN.gyy;
            }
            if constexpr (EXACT) {
                Us[c].h = (U.h - (dtdx * df_h + dtdy * dg_h)) + 0.0;
                Us[c].qx = (U.qx - (dtdx * df_qx + dtdy * dg_qx)) + dt * srxb[c];
                Us[c].qy = (U.qy - (dtdx * df_qy + dtdy * dg_qy)) + dt * sryb[c];
            } else {
                Us[c].h = U.h - __fma_rn(dtdx, df_h, dtdy * dg_h);
                Us[c].qx = __fma_rn(dt, srxb[c], U.qx - __fma_rn(dtdx, df_qx, dtdy * dg_qx));
                Us[c].qy = __fma_rn(dt, sryb[c], U.qy - __fma_rn(dtdx, df_qy, dtdy * dg_qy));
            }
            dry[c] = !(Us[c].h >= h_min) && star_ok[c] && in_x[c];
            if (!(U.h >= h_min) && k >= 0 && k < L && out_x[c]) e2 = 1;
            fluxes(Us[c], zxb[c], zyb[c], FS[c], ssx[c], ssy[c]);
            Hx[c] = {face(fn_h[c], Us[c].qx), face(fn_qx[c], FS[c].fxx), face(fn_qy[c], FS[c].fxy)};
            out.Hyp[c] = {face(Un[c].qy, Us[c].qy), face(FN.fxy, FS[c].fxy), face(FN.gyy, FS[c].gyy)};
            hs[c] = FWD ? in.Hyp[c] : out.Hyp[c];
            hn[c] = FWD ? out.Hyp[c] : in.Hyp[c];
        }
        if (__any_sync(FULL, dry[0] || dry[1])) {  // dry U* -> first consumer (executor.hpp:459-513)
            for (int c = 0; c < 2; ++c) {
                const int ic = i0 + c;
                if (dry[c] && jb >= 0 && jb < p.ny) {
                    unsigned long long cons;
                    if (FWD) cons = static_cast<unsigned long long>(jb) * p.nx + ic;
                    else if (jb >= 1) cons = static_cast<unsigned long long>(jb - 1) * p.nx + ic;
                    else if (ic >= 1) cons = static_cast<unsigned long long>(jb) * p.nx + (ic - 1);
                    else cons = static_cast<unsigned long long>(jb) * p.nx + ic;
                    e4 = max(e4, ~cons);
                }
            }
        }
        // boundary faces (edge windows / rows only); FWD hands the west face of i=0
        // to the cell at i=-1, BWD the east face of i=nx-1 to the cell at i=nx
        if (xedge || jb == 0 || jb == p.ny - 1) {
            CellVec give_f[2] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
            int give[2] = {0, 0};
            for (int c = 0; c < 2; ++c) {
                const int ic = i0 + c;
                if (in_x[c] && jb >= 0 && jb < p.ny && (ic == 0 || ic == p.nx - 1 || jb == 0 || jb == p.ny - 1)) {
                    EdgeIn ei;
                    ei.U = Ub[c];
                    ei.Us = Us[c];
                    ei.fu_xx = in.FU[c].fxx;
                    ei.fu_xy = in.FU[c].fxy;
                    ei.fu_yy = in.FU[c].gyy;
                    ei.fs_xx = FS[c].fxx;
                    ei.fs_xy = FS[c].fxy;
                    ei.fs_yy = FS[c].gyy;
                    ei.Hx = Hx[c];
                    ei.hy_a = FWD ? hs[c] : hn[c];
                    ei.hy_b = FWD ? hn[c] : hs[c];
                    const EdgeOut eo = boundary_faces<FWD>(ei, ic, jb, p.nx, p.ny, p.bc, p.z_w[b + R], p.z_e[b + R],
                                                           p.z_s[ic], p.z_n[ic], h_min, half_g, e4, !EXACT);
                    Hx[c] = eo.Hx;
                    hs[c] = FWD ? eo.hy_a : eo.hy_b;
                    hn[c] = FWD ? eo.hy_b : eo.hy_a;
                    e4 = eo.e4;
                    give[c] = eo.give;
                    give_f[c] = eo.xo;
                }
            }
            if (xedge) {
                if constexpr (FWD) {  // face of cell c goes to cell c-1 (lane-1's cell 1 for c = 0)
                    if (give[1]) Hx[0] = give_f[1];
                    const double gh = from_right(give_f[0].h), gqx = from_right(give_f[0].qx),
                                 gqy = from_right(give_f[0].qy);
                    const int gv = __shfl_down_sync(FULL, give[0], 1);
                    if (gv) Hx[1] = {gh, gqx, gqy};
                } else {              // face of cell c goes to cell c+1 (lane+1's cell 0 for c = 1)
                    if (give[0]) Hx[1] = give_f[0];
                    const double gh = from_left(give_f[1].h), gqx = from_left(give_f[1].qx),
                                 gqy = from_left(give_f[1].qy);
                    const int gv = __shfl_up_sync(FULL, give[1], 1);
                    if (gv) Hx[0] = {gh, gqx, gqy};
                }
            }
        }
        // ---- stage 3: corrector of row b   scheme.hpp:185-191
        if constexpr (DO3) {
            CellVec hw[2], he[2];
            if constexpr (FWD) {  // own face is the east face
                he[0] = Hx[0];
                he[1] = Hx[1];
                hw[1] = Hx[0];
                hw[0] = {from_left(Hx[1].h), from_left(Hx[1].qx), from_left(Hx[1].qy)};
            } else {              // own face is the west face
                hw[0] = Hx[0];
                hw[1] = Hx[1];
                he[0] = Hx[1];
                he[1] = {from_right(Hx[0].h), from_right(Hx[0].qx), from_right(Hx[0].qy)};
            }
            CellVec C[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const CellVec& U = Ub[c];
                const double sx_ = srxb[c] + ssx[c], sy_ = sryb[c] + ssy[c];
                if constexpr (EXACT) {
                    const double fs_h = dtdx * (he[c].h - hw[c].h) + dtdy * (hn[c].h - hs[c].h);
                    const double fs_qx = dtdx * (he[c].qx - hw[c].qx) + dtdy * (hn[c].qx - hs[c].qx);
                    const double fs_qy = dtdx * (he[c].qy - hw[c].qy) + dtdy * (hn[c].qy - hs[c].qy);
                    C[c].h = (U.h - fs_h) + 0.0;
                    C[c].qx = (U.qx - fs_qx) + half_dt * sx_;
                    C[c].qy = (U.qy - fs_qy) + half_dt * sy_;
                } else {
                    const double fs_h = __fma_rn(cx, he[c].h - hw[c].h, cy * (hn[c].h - hs[c].h));
                    const double fs_qx = __fma_rn(cx, he[c].qx - hw[c].qx, cy * (hn[c].qx - hs[c].qx));
                    const double fs_qy = __fma_rn(cx, he[c].qy - hw[c].qy, cy * (hn[c].qy - hs[c].qy));
                    C[c].h = U.h - fs_h;
                    C[c].qx = __fma_rn(half_dt, sx_, U.qx - fs_qx);
                    C[c].qy = __fma_rn(half_dt, sy_, U.qy - fs_qy);
                }
            }
            if constexpr (!SMOOTH) {
                if constexpr (EMIT) emit2(C, b);
            } else {
                if constexpr (EMIT) {  // smoothing of row q = b - S (executor.hpp:533-540)
                    const CellVec* Cp = in.Cp;
                    CellVec ce[2], cw[2];
                    ce[0] = Cp[1];
                    cw[1] = Cp[0];
                    ce[1] = {from_right(Cp[0].h), from_right(Cp[0].qx), from_right(Cp[0].qy)};
                    cw[0] = {from_left(Cp[1].h), from_left(Cp[1].qx), from_left(Cp[1].qy)};
                    const int q = b - S;
                    const int jq = p.j0 + q;
                    CellVec o[2];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        CellVec cn = FWD ? C[c] : in.Cpp[c];
                        CellVec cs = FWD ? in.Cpp[c] : C[c];
                        CellVec e = ce[c], w = cw[c];
                        if (xedge || jq == 0 || jq == p.ny - 1) {
                            const int ic = i0 + c;
                            if (ic == 0) w = edge_ghost(SWE_EDGE_W, p.bc[SWE_EDGE_W], Cp[c], p.z_w[q + R], h_min);
                            if (ic == p.nx - 1)
                                e = edge_ghost(SWE_EDGE_E, p.bc[SWE_EDGE_E], Cp[c], p.z_e[q + R], h_min);
                            if (jq == 0) cs = edge_ghost(SWE_EDGE_S, p.bc[SWE_EDGE_S], Cp[c], p.z_s[ic], h_min);
                            if (jq == p.ny - 1)
                                cn = edge_ghost(SWE_EDGE_N, p.bc[SWE_EDGE_N], Cp[c], p.z_n[ic], h_min);
                        }
                        const double nu = p.nu;
                        const CellVec& u = Cp[c];
                        o[c].h = u.h + nu * (((e.h - u.h) + (w.h - u.h)) + ((cn.h - u.h) + (cs.h - u.h)));
                        o[c].qx = u.qx + nu * (((e.qx - u.qx) + (w.qx - u.qx)) + ((cn.qx - u.qx) + (cs.qx - u.qx)));
                        o[c].qy = u.qy + nu * (((e.qy - u.qy) + (w.qy - u.qy)) + ((cn.qy - u.qy) + (cs.qy - u.qy)));
                    }
                    emit2(o, q);
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    out.Cpp[c] = in.Cp[c];
                    out.Cp[c] = C[c];
                }
            }
        }
        produce();
    }

    __device__ __forceinline__ void segment(const Seg& sg) {
        L = sg.rb - sg.ra;
        const int xw0 = sg.tile * TW - XH;  // global column of lane 0's first cell
        tile_x = sg.tile * TW + XH;         // padded column of the first output column
        i0 = xw0 + 2 * lane;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int ic = i0 + c;
            const int t = 2 * lane + c;  // column within the window
            in_x[c] = (ic >= 0) && (ic < p.nx);
            out_x[c] = in_x[c] && t >= XH && t < W - XH;
            star_ok[c] = FWD ? (t < W - 1) : (t > 0);
        }
        xedge = (xw0 <= 0) || (xw0 + W - 1 >= p.nx - 1);
        r_start = FWD ? sg.ra : sg.rb - 1;
        Carry A, B;
        {
            CellVec u[2];
            double zx[2], zy[2];
            consume(u, zx, zy);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const Rc rc = A::recip(u[c].h);
                A.FU[c] = A::flux(u[c], rc, half_g);
                A.srx[c] = A.sry[c] = 0.0;
                if constexpr (MANNING)
                    source_of<EXACT, MANNING>(u[c], A.FU[c], rc, zx[c], zy[c], neg_g, gnn, A.srx[c], A.sry[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            A.Hyp[c] = {0.0, 0.0, 0.0};
            A.Cp[c] = {0.0, 0.0, 0.0};
            A.Cpp[c] = {0.0, 0.0, 0.0};
        }
        produce();
        int k = -R;
        if constexpr (SMOOTH) {
            iter<false, false>(k++, A, B);  // row -2: predictor only
            A = B;
            iter<true, false>(k++, A, B);   // rows -1, 0: correctors feeding the first smoothed row
            A = B;
            iter<true, false>(k++, A, B);
            A = B;
        } else {
            iter<false, false>(k++, A, B);  // row -1: predictor only
            A = B;
        }
        const int k_last = SMOOTH ? L : L - 1;
        for (; k + 1 <= k_last; k += 2) {
            iter<true, true>(k, A, B);
            iter<true, true>(k + 1, B, A);
        }
        if (k <= k_last) iter<true, true>(k, A, B);
    }
};

template <int WPB, bool FWD, bool SMOOTH, bool FLAT, bool MANNING, bool EXACT>
__global__ void __launch_bounds__(WPB * 32, SWE_MINB) swe_step_kernel(const __grid_constant__ StepParams p) {
    using M = Marcher<WPB, FWD, SMOOTH, FLAT, MANNING, EXACT>;
    constexpr int D = kStages;
    constexpr int NF = M::NF;
    constexpr int W = M::W;
    constexpr unsigned FULL = 0xffffffffu;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    __shared__ Seg segq_all[WPB][M::QN];
    __shared__ int s_skip, s_sel, s_last;
    __shared__ double s_dt, s_tc;
    __shared__ double s_red[2][WPB];
    SweCtl* ctl = p.ctl;
    double* stage = reinterpret_cast<double*>(smem_raw) + warp * (D * NF * W);  // [D][NF][64]
    double* ostage = reinterpret_cast<double*>(smem_raw) + WPB * D * NF * W + warp * (M::NO * M::OB);
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<double*>(smem_raw) + WPB * D * NF * W +
                                              WPB * M::NO * M::OB) +
        warp * D;

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
    }
    if (lane == 0) {
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (s_skip) return;

    M m{p};
    m.stage = stage;
    m.ostage = ostage;
    m.obuf = 0;
    m.bars = bars;
    m.segq = segq_all[warp];
    m.qhead = 0;
    m.qtail = 0;
    m.lane = lane;
    m.sel = s_sel;
    m.nxt = p.buf[s_sel ^ 1];
    m.P = p.pitch;
    m.dt = s_dt;
    m.dtdx = m.dt / p.dx;
    m.dtdy = m.dt / p.dy;
    m.half_dt = 0.5 * m.dt;
    m.cx = EXACT ? m.dtdx : 0.5 * m.dtdx;
    m.cy = EXACT ? m.dtdy : 0.5 * m.dtdy;
    m.h_min = p.h_min;
    m.half_g = p.half_g;
    m.neg_g = p.neg_g;
    m.gnn = p.gnn;
    m.pleft = 0;
    m.pdone = false;
    m.px = m.py = m.pzy = 0;
    m.pn = 0;
    m.req = 0;
    m.ring = {0, 0u};
    m.dprev = 0;
    m.mx = 0.0;
    m.my = 0.0;
    m.e2 = 0;
    m.e4 = m.e5 = 0ull;
    m.produce();
    while (m.qhead < m.qtail) {
        const Seg sg = m.segq[m.qhead % M::QN];
        ++m.qhead;
        m.segment(sg);
    }

    bulk_wait_all();  // this warp's TMA row stores are complete
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
    if (m.e5) atomicMax(&ctl->red[RED_E5], m.e5);
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

template <int WPB, bool SMOOTH, bool FLAT>
constexpr size_t step_smem_bytes() {
    return static_cast<size_t>(WPB) * kStages * (FLAT ? 3 : 5) * 64 * 8 +
           WPB * 3 * ((3 * (64 - 2 * SWE_XOFF) + 15) / 16 * 16) * 8 + WPB * kStages * 8;
}

}  // namespace swe_dev
