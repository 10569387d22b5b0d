// swe_aux.cu — auxiliary kernels of the host runtime: buffer set-up, the K1
// ghosts after a load, bed slopes / edge values / clamp diagnostic, on-device
// initial conditions, early-exit tables, the exact CFL/guard scan, the
// division self-test and the local-group allreduce.  Compiled -fmad=false.
#include "swe_runtime.h"

namespace swe_rt {

using swe_dev::CellVec;
constexpr int swe_dev_edge_n = SWE_EDGE_N, swe_dev_edge_s = SWE_EDGE_S, swe_dev_edge_e = SWE_EDGE_E,
              swe_dev_edge_w = SWE_EDGE_W;

__device__ __forceinline__ size_t pidx(int P, int R, int lr, int f, int i) {
    return (static_cast<size_t>(lr + R) * 3 + f) * P + static_cast<size_t>(i + SWE_XO);
}

// Fill the whole padded buffer (every field row, all columns) with a benign
// wet state so never-consumed padding cells stay finite.
__global__ void fill_benign_kernel(double* buf, size_t rows3, int P) {
    const size_t n = rows3 * static_cast<size_t>(P);
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t row = k / P;
        buf[k] = (row % 3 == 0) ? 1.0 : 0.0;
    }
}

// K1 (executor.hpp:384-408) on the committed buffer after load: x ghosts of
// own rows, y ghost rows where this rank owns a domain edge.
__global__ void ghost_fill_rows_kernel(double* b, int P, int R, int nx, int nloc, int j0, int ny,
                                       SweBC w, SweBC e, SweBC s, SweBC n, const double* z_w,
                                       const double* z_e, const double* z_s, const double* z_n,
                                       double h_min) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nloc) {
        const int lr = t;
        CellVec u0 = {b[pidx(P, R, lr, 0, 0)], b[pidx(P, R, lr, 1, 0)], b[pidx(P, R, lr, 2, 0)]};
        CellVec g = swe_dev::edge_ghost(SWE_EDGE_W, w, u0, z_w[lr + R], h_min);
        b[pidx(P, R, lr, 0, -1)] = g.h;
        b[pidx(P, R, lr, 1, -1)] = g.qx;
        b[pidx(P, R, lr, 2, -1)] = g.qy;
        CellVec u1 = {b[pidx(P, R, lr, 0, nx - 1)], b[pidx(P, R, lr, 1, nx - 1)],
                      b[pidx(P, R, lr, 2, nx - 1)]};
        g = swe_dev::edge_ghost(SWE_EDGE_E, e, u1, z_e[lr + R], h_min);
        b[pidx(P, R, lr, 0, nx)] = g.h;
        b[pidx(P, R, lr, 1, nx)] = g.qx;
        b[pidx(P, R, lr, 2, nx)] = g.qy;
    }
    if (t < nx) {
        const int i = t;
        if (j0 == 0) {
            CellVec u = {b[pidx(P, R, 0, 0, i)], b[pidx(P, R, 0, 1, i)], b[pidx(P, R, 0, 2, i)]};
            CellVec g = swe_dev::edge_ghost(SWE_EDGE_S, s, u, z_s[i], h_min);
            b[pidx(P, R, -1, 0, i)] = g.h;
            b[pidx(P, R, -1, 1, i)] = g.qx;
            b[pidx(P, R, -1, 2, i)] = g.qy;
        }
        if (j0 + nloc == ny) {
            const int lr = nloc - 1;
            CellVec u = {b[pidx(P, R, lr, 0, i)], b[pidx(P, R, lr, 1, i)], b[pidx(P, R, lr, 2, i)]};
            CellVec g = swe_dev::edge_ghost(SWE_EDGE_N, n, u, z_n[i], h_min);
            b[pidx(P, R, lr + 1, 0, i)] = g.h;
            b[pidx(P, R, lr + 1, 1, i)] = g.qx;
            b[pidx(P, R, lr + 1, 2, i)] = g.qy;
        }
    }
}

// make_domain_ctx slopes (executor.hpp:351-376) for local rows [-R, nloc+R)
// that lie inside the domain; zp holds z for local rows [-R-1, nloc+R+1)
// (compact, nx per row; rows outside the domain unused).  Output rows use the
// padded 2-field layout.  flags[0] |= 1 when any slope bit pattern is not +0.0.
__global__ void slopes_kernel(const double* zp, double* slope, int P, int R, int nx, int nloc,
                              int j0, int ny, double two_dx, double two_dy, double scale, unsigned* flags) {
    // one row per block iteration, columns across the threads (coalesced);
    // the flat / dz/dy flags are OR-ed per warp, then once per block
    __shared__ unsigned s_any, s_y;
    if (threadIdx.x == 0) s_any = s_y = 0u;
    __syncthreads();
    unsigned any = 0u, anyy = 0u;
    const int rows = nloc + 2 * R;
    for (int rr = blockIdx.x; rr < rows; rr += gridDim.x) {
        const int lr = rr - R;
        const int j = j0 + lr;
        const bool own = j >= 0 && j < ny;
        const double* zr = zp + static_cast<size_t>(lr + R + 1) * nx;  // bed row j
        const int js = max(j - 1, 0) - j, jn = min(j + 1, ny - 1) - j;    // clamped row offsets
        double* sxr = slope + (static_cast<size_t>(rr) * 2 + 0) * P + SWE_XO;
        double* syr = slope + (static_cast<size_t>(rr) * 2 + 1) * P + SWE_XO;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            double sx = 0.0, sy = 0.0;
            if (own) {  // make_domain_ctx (executor.hpp:351-376): clamped central differences
                const int iw = max(i - 1, 0), ie = min(i + 1, nx - 1);
                sx = (zr[ie] - zr[iw]) / two_dx;
                sy = (zr[static_cast<ptrdiff_t>(jn) * nx + i] - zr[static_cast<ptrdiff_t>(js) * nx + i]) / two_dy;
            }
            const bool nzx = swe_dev::dbits(sx) != 0ull, nzy = swe_dev::dbits(sy) != 0ull;
            any |= static_cast<unsigned>(nzx || nzy);
            anyy |= static_cast<unsigned>(nzy);
            // fast mode stores -g * slope (one FMA for the bed source term);
            // +0.0 stays +0.0 so flat items are recognised by their bit patterns
            sxr[i] = nzx ? sx * scale : sx;
            syr[i] = nzy ? sy * scale : sy;
        }
    }
    any = __any_sync(0xffffffffu, any);
    anyy = __any_sync(0xffffffffu, anyy);
    if ((threadIdx.x & 31) == 0) {
        if (any) atomicOr(&s_any, 1u);
        if (anyy) atomicOr(&s_y, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_any) atomicOr(flags, 1u);
        if (s_y) atomicOr(flags + 2, 1u);
    }
}

// Early exit, static part: an item (32-column window x row chunk, the step
// kernel's unit of work) is eligible when its dependency region -- its cells
// widened by R + 1 <= 3 -- lies inside this rank's own rows and the domain's
// columns (no ghost or strip-halo cell involved) and the bed slopes of the 3x3
// block of items around it are all +0.0 (a flat bed, so the rest state
// (H, +0, +0) is a fixed point of the step).
__global__ void item_flat_kernel(const double* slope, int P, int R, int nx, int nloc, int TW, int chunk,
                                 int ntiles, int nitems, unsigned char* flat) {
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int rc = item / ntiles, tile = item % ntiles;
        const int x0 = tile * TW, x1 = min(x0 + TW, nx), y0 = rc * chunk, y1 = min(y0 + chunk, nloc);
        const int w = x1 - x0;
        int bad = 0;
        for (int k = threadIdx.x; k < (y1 - y0) * w; k += blockDim.x) {
            const int lr = y0 + k / w, i = x0 + k % w;
            const size_t o = (static_cast<size_t>(lr + R) * 2) * P + (i + SWE_XO);
            bad |= (swe_dev::dbits(slope[o]) | swe_dev::dbits(slope[o + P])) != 0ull;
        }
        bad = __syncthreads_or(bad);
        if (threadIdx.x == 0) flat[item] = bad ? 0 : 1;
    }
}

__global__ void item_elig_kernel(const unsigned char* flat, int nx, int nloc, int TW, int chunk, int ntiles,
                                 int nchunks, int R, unsigned char* elig, unsigned long long* count) {
    const int nitems = ntiles * nchunks;
    for (int item = blockIdx.x * blockDim.x + threadIdx.x; item < nitems; item += gridDim.x * blockDim.x) {
        const int rc = item / ntiles, tile = item % ntiles;
        const int x0 = tile * TW, x1 = min(x0 + TW, nx), y0 = rc * chunk, y1 = min(y0 + chunk, nloc);
        const int rad = R + 1;
        bool ok = x0 - rad >= 0 && x1 + rad <= nx && y0 - rad >= 0 && y1 + rad <= nloc && tile >= 1 &&
                  tile + 1 < ntiles && rc >= 1 && rc + 1 < nchunks && chunk >= rad && TW >= rad;
        for (int d = 0; ok && d < 9; ++d) ok = flat[(rc + d / 3 - 1) * ntiles + tile + d % 3 - 1] != 0;
        elig[item] = ok ? 1 : 0;
        if (ok) atomicAdd(count, 1ull);
    }
}

// Bed edge values for the K1 ghosts: z_w / z_e of own rows (local rows
// [0, nloc) at offset R), from the compact bed rows zp (row lr at lr + R + 1).
__global__ void edge_z_kernel(const double* zp, int R, int nx, int nloc, double* zw, double* ze) {
    for (int lr = blockIdx.x * blockDim.x + threadIdx.x; lr < nloc; lr += gridDim.x * blockDim.x) {
        const double* row = zp + static_cast<size_t>(lr + R + 1) * nx;
        zw[lr + R] = row[0];
        ze[lr + R] = row[nx - 1];
    }
}


// Fixed-elevation clamp diagnostic (grid.hpp:256-263): any fixed-eta edge
// cell of this rank whose ghost depth eta - z falls below h_min.
__global__ void clamp_kernel(const double* zp, int R, int nx, int nloc, int own_s, int own_n, BcSet b,
                             double h_min, unsigned* flag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    int hit = 0;
    if (t < nloc) {
        const double* row = zp + static_cast<size_t>(t + R + 1) * nx;
        if (b.bc[SWE_EDGE_W].type == SWE_BC_FIXED_ETA && b.bc[SWE_EDGE_W].eta_out - row[0] < h_min) hit = 1;
        if (b.bc[SWE_EDGE_E].type == SWE_BC_FIXED_ETA && b.bc[SWE_EDGE_E].eta_out - row[nx - 1] < h_min) hit = 1;
    }
    if (t < nx) {
        if (own_s && b.bc[SWE_EDGE_S].type == SWE_BC_FIXED_ETA &&
            b.bc[SWE_EDGE_S].eta_out - zp[static_cast<size_t>(R + 1) * nx + t] < h_min)
            hit = 1;
        if (own_n && b.bc[SWE_EDGE_N].type == SWE_BC_FIXED_ETA &&
            b.bc[SWE_EDGE_N].eta_out - zp[static_cast<size_t>(R + nloc) * nx + t] < h_min)
            hit = 1;
    }
    if (hit) atomicOr(flag, 1u);
}

// build_initial_state (scenarios.hpp:95-171) on the device for the kinds
// without transcendental functions: flat_pool, channel_slope, dam_break.
// Same expression trees (the TU is compiled -fmad=false), so the state is
// bit-identical to the reference's; own rows only (strip-local).
__global__ void initial_kernel(swe_initial ic, double dx, int nx, int nloc, int P, int R, double* buf, double* zp) {
    const size_t n = static_cast<size_t>(nloc) * nx;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int lr = static_cast<int>(k / nx), i = static_cast<int>(k % nx);
        double z = 0.0, h = ic.depth;
        if (ic.kind == SWE_IC_CHANNEL_SLOPE) {
            z = ic.slope * dx * static_cast<double>(nx - 1 - i);
            h = ic.depth - z;
        } else if (ic.kind == SWE_IC_DAM_BREAK) {
            const double x = (i + 0.5) * dx;
            h = (x < ic.split_x) ? ic.h_left : ic.h_right;
        }
        buf[pidx(P, R, lr, 0, i)] = h;
        buf[pidx(P, R, lr, 1, i)] = 0.0;
        buf[pidx(P, R, lr, 2, i)] = 0.0;
        zp[static_cast<size_t>(lr + R + 1) * nx + i] = z;
    }
}


// K6 exact per-cell scan (timestep.hpp:83-105 / executor.hpp:560-580) and K5
// guard (timestep.hpp:64-78) over own rows of buffer b.
__global__ void scan_kernel(const double* b, int P, int R, int nx, int nloc, int j0, double g,
                            double dx, double dy, double h_min, int cfl, unsigned long long* out) {
    // one row per block iteration, columns across the threads (coalesced).
    // cfl = 0: the stability guard only (load, Stepper::stability_guard).
    // The CFL part needs min over cells of r = min(dx/sx, dy/sy).  Correctly
    // rounded division by a positive number is monotone, so over the cells
    // whose quotients are certainly positive and finite (sx, sy within 2^1000
    // of dx, dy in exponent) that minimum is min(dx / max sx, dy / max sy),
    // formed on the host from the two maxima; only the other cells take the
    // per-cell quotients (executor.hpp:560-580), exactly as the reference.
    // u = qx/h, v = qy/h use the step kernels' shared-reciprocal division
    // under its range test (IEEE quotients), __ddiv_rn outside it.
    unsigned long long bad = 0, minr = 0, guard = 0, mxs = 0, mys = 0;
    const unsigned ex = swe_dev::dexp(dx), ey = swe_dev::dexp(dy);
    const bool normal_d = ex - 1u < 2046u && ey - 1u < 2046u;  // else every cell takes the per-cell path
    for (int lr = blockIdx.x; lr < nloc; lr += gridDim.x) {
        const double* hr = b + pidx(P, R, lr, 0, 0);
        const unsigned long long row0 = static_cast<unsigned long long>(j0 + lr) * nx;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            const double h = hr[i], qx = hr[P + i], qy = hr[2 * P + i];
            const unsigned long long idx = row0 + i;
            // stability guard (executor.hpp:543-556)
            const bool ok = swe_dev::finite_d(h) && swe_dev::finite_d(qx) && swe_dev::finite_d(qy) &&
                            h >= h_min;
            if (!ok) guard = max(guard, ~idx);
            if (!cfl) continue;
            // K6 (executor.hpp:560-580)
            const double c = __dsqrt_rn(g * h);
            double u, v;
            if (swe_dev::h_safe(h) && swe_dev::q_safe(qx) && swe_dev::q_safe(qy)) {
                const swe_dev::Recip rc = swe_dev::make_recip(h);
                u = swe_dev::quot_checked(qx, rc, swe_dev::is_zero(qx));
                v = swe_dev::quot_checked(qy, rc, swe_dev::is_zero(qy));
            } else {
                u = __ddiv_rn(qx, h);
                v = __ddiv_rn(qy, h);
            }
            const double sx = fabs(u) + c;
            const double sy = fabs(v) + c;
            const unsigned esx = swe_dev::dexp(sx), esy = swe_dev::dexp(sy);
            // sx, sy positive normal within 2^1000 of dx, dy: dx/sx, dy/sy in
            // (2^-1001, 2^1002), positive and finite
            if (normal_d && sx > 0.0 && sy > 0.0 && esx - 1u < 2046u && esy - 1u < 2046u &&
                esx + 1000u - ex < 2000u && esy + 1000u - ey < 2000u) {
                mxs = max(mxs, swe_dev::dbits(sx));
                mys = max(mys, swe_dev::dbits(sy));
                continue;
            }
            const double r = swe_dev::std_min(__ddiv_rn(dx, sx), __ddiv_rn(dy, sy));
            if (!(r > 0.0) || !swe_dev::finite_d(r)) {
                bad = max(bad, ~idx);
                continue;
            }
            minr = max(minr, ~swe_dev::dbits(r));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        bad = max(bad, __shfl_xor_sync(0xffffffffu, bad, o));
        minr = max(minr, __shfl_xor_sync(0xffffffffu, minr, o));
        guard = max(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        mxs = max(mxs, __shfl_xor_sync(0xffffffffu, mxs, o));
        mys = max(mys, __shfl_xor_sync(0xffffffffu, mys, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicMax(&out[SCAN_BAD], bad);
        if (minr) atomicMax(&out[SCAN_MINR], minr);
        if (guard) atomicMax(&out[SCAN_GUARD], guard);
        if (mxs) atomicMax(&out[SCAN_MAXSX], mxs);
        if (mys) atomicMax(&out[SCAN_MAXSY], mys);
    }
}

// K4's dry-U* check (executor.hpp:429-436, 451-513) for every corrector cell
// of this rank's rows, from the committed buffer: U*.h needs only h of the
// cell and the momenta of its sweep neighbours (scheme.hpp:100-113), formed
// with the step kernel's arithmetic for the mode.  Reports the row-major first
// consumer whose own U* or a neighbour U* its corrector reads is dry (NaN
// counts as dry).  Run only after a step whose interior windows flagged one.
__global__ void dry_scan_kernel(const double* b, int P, int R, int nx, int ny, int nloc, int j0, double dt,
                                double dx, double dy, int fwd, int exact, BcSet bs, const double* z_w,
                                const double* z_e, const double* z_s, const double* z_n, double h_min,
                                unsigned long long* out) {
    const double dtdx = dt / dx, dtdy = dt / dy;
    const int s = fwd ? 1 : -1;
    auto star_h = [&](int lr, int i) {  // U*.h of interior cell (i, local row lr)
        const double h = b[pidx(P, R, lr, 0, i)], qx = b[pidx(P, R, lr, 1, i)], qy = b[pidx(P, R, lr, 2, i)];
        const double qxn = b[pidx(P, R, lr, 1, i + s)], qyn = b[pidx(P, R, lr + s, 2, i)];
        const double df = fwd ? qxn - qx : qx - qxn, dg = fwd ? qyn - qy : qy - qyn;
        if (exact) return (h - (dtdx * df + dtdy * dg)) + 0.0;
        return h - __fma_rn(dtdx, df, dtdy * dg);
    };
    auto wet = [&](double x) { return x >= h_min; };
    unsigned long long first = 0;
    for (int lr = blockIdx.x; lr < nloc; lr += gridDim.x) {
        const int j = j0 + lr;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            const double own = star_h(lr, i);
            bool dry = !wet(own);
            // faces whose U* is the neighbour's (FWD: west and south; BWD: east
            // and north); wall and inflow faces read no neighbour U*; an edge
            // face of another kind reads the U* ghost of this cell
            auto face = [&](int edge, bool at_edge, int di, int dj) {
                const SweBC& bc = bs.bc[edge];
                if (at_edge) {
                    if (bc.type == SWE_BC_WALL || bc.type == SWE_BC_INFLOW) return true;
                    const double zin = edge == swe_dev_edge_w ? z_w[lr + R] : edge == swe_dev_edge_e ? z_e[lr + R]
                                       : edge == swe_dev_edge_s ? z_s[i] : z_n[i];
                    const CellVec us = {own, 0.0, 0.0};
                    return wet(swe_dev::edge_ghost(edge, bc, us, zin, h_min).h);
                }
                return wet(star_h(lr + dj, i + di));
            };
            if (!dry && fwd) dry = !face(swe_dev_edge_w, i == 0, -1, 0);
            if (!dry && !fwd) dry = !face(swe_dev_edge_e, i == nx - 1, 1, 0);
            if (!dry && fwd) dry = !face(swe_dev_edge_s, j == 0, 0, -1);
            if (!dry && !fwd) dry = !face(swe_dev_edge_n, j == ny - 1, 0, 1);
            if (dry) first = max(first, ~(static_cast<unsigned long long>(j) * nx + i));
        }
    }
    for (int o = 16; o > 0; o >>= 1) first = max(first, __shfl_xor_sync(0xffffffffu, first, o));
    if ((threadIdx.x & 31) == 0 && first) atomicMax(&out[SCAN_DRY], first);
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// swe_cuda_state_digest: sum over owned cells of mix(h, qx, qy, global index).
__global__ void digest_kernel(const double* b, int P, int R, int nx, int nloc, int j0, unsigned long long* out) {
    unsigned long long acc = 0;
    for (int lr = blockIdx.x; lr < nloc; lr += gridDim.x) {
        const double* hr = b + pidx(P, R, lr, 0, 0);
        const unsigned long long row0 = static_cast<unsigned long long>(j0 + lr) * nx;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            unsigned long long x = splitmix64(row0 + i);
            x = splitmix64(x ^ swe_dev::dbits(hr[i]));
            x = splitmix64(x ^ swe_dev::dbits(hr[P + i]));
            acc += splitmix64(x ^ swe_dev::dbits(hr[2 * P + i]));
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// Shared-reciprocal division of the step kernels (swe_device.cuh), exposed for
// the parity self-test.  Compiled with -fmad=false like the exact kernels.
__global__ void selftest_div_kernel(const double* a, const double* b, size_t n, int exact, double* out) {
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (exact == 2) {  // the per-state range test (SWE_EXACT_STATE_CHECK) with a as the momentum
            const swe_dev::Recip rc = swe_dev::make_recip(b[k]);
            out[k] = (swe_dev::h_safe(b[k]) && swe_dev::q_safe(a[k]))
                         ? swe_dev::quot_checked(a[k], rc, swe_dev::is_zero(a[k]))
                         : __ddiv_rn(a[k], b[k]);
        } else if (exact) {
            const swe_dev::Recip rc = swe_dev::make_recip(b[k]);
            out[k] = swe_dev::div_rn(a[k], rc);
        } else {
            out[k] = a[k] * swe_dev::make_recip_fast(b[k]).y;
        }
    }
}

__global__ void max_reduce_kernel(RedPtrs in, int nranks, int n, unsigned long long* out) {
    const int k = threadIdx.x;
    if (k >= n) return;
    unsigned long long m = 0ull;
    for (int r = 0; r < nranks; ++r) m = max(m, in.p[r][k]);
    out[k] = m;
}

}  // namespace swe_rt
