// swe_capi.cu — host runtime behind include/swe_cuda.h (libswe_cuda.so).
//
// Owns the device state of one swe::Stepper replacement (executor.hpp:726-1116):
// ping-pong padded buffers, bed slopes, the device control block, CUDA graphs
// for the device-resident run loop, and (for row strips) its transport
// (swe_transport.cu).  The auxiliary kernels live in swe_aux.cu.  Compiled
// with -fmad=false like the kernels.
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "swe_runtime.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

using namespace swe_rt;

namespace swe_rt {

int set_status(swe_status* st, int code, int i, int j, double t, const char* fmt, ...) {
    if (st) {
        std::memset(st, 0, sizeof *st);
        st->code = code;
        st->i = i;
        st->j = j;
        st->t = t;
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(st->msg, sizeof st->msg, fmt, ap);
        va_end(ap);
    }
    return code;
}

int ok_status(swe_status* st) {
    if (st) std::memset(st, 0, sizeof *st);
    return SWE_OK;
}

}  // namespace swe_rt

namespace swe_rt {

// ---------------------------------------------------------------- device allocations
// Product build: cudaMalloc / cudaFree.  SWE_CHECKED build: every allocation
// gets 64 KiB guard bands of a fixed byte pattern on both sides;
// swe_cuda_debug_guard_check() reports corrupted guard bytes (a stray write
// past any buffer the kernels touch).
#if SWE_CHECKED
namespace {
constexpr size_t kGuard = 64 * 1024;
constexpr unsigned char kGuardByte = 0xA5;
std::mutex g_alloc_m;
std::map<void*, std::pair<char*, size_t>> g_allocs;  // user pointer -> (base, user bytes)
}  // namespace
cudaError_t dev_alloc(void** p, size_t bytes) {
    char* base = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    e = cudaMemset(base, kGuardByte, kGuard);
    if (e == cudaSuccess) e = cudaMemset(base + kGuard + bytes, kGuardByte, kGuard);
    if (e != cudaSuccess) return e;
    *p = base + kGuard;
    std::lock_guard<std::mutex> lk(g_alloc_m);
    g_allocs[*p] = {base, bytes};
    return cudaSuccess;
}
void dev_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_alloc_m);
    auto it = g_allocs.find(p);
    if (it == g_allocs.end()) return;
    cudaFree(it->second.first);
    g_allocs.erase(it);
}
#else
cudaError_t dev_alloc(void** p, size_t bytes) { return cudaMalloc(p, bytes); }
void dev_free(void* p) { cudaFree(p); }
#endif

// ---------------------------------------------------------------- TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool encode_rows(CUtensorMap* map, double* base, int P, long long field_rows, int box_rows, std::string& err,
                 int box_cols, int row_stride) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            err = "cuTensorMapEncodeTiled unavailable";
            return false;
        }
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(field_rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride > 0 ? row_stride : P) * sizeof(double)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        err = "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")";
        return false;
    }
    return true;
}

}  // namespace swe_rt

namespace {

// ---------------------------------------------------------------- helpers
double std_min(double a, double b) { return (b < a) ? b : a; }

// Smallest positive double s with RN(a / s) == 0 (the dt reduction's "r > 0"
// test fails for sx >= this); found by bisection on bit patterns using the
// host's IEEE division (identical to the device's).
double zero_threshold(double a) {
    unsigned long long lo = 0x0000000000000001ull, hi = 0x7ff0000000000000ull;  // inf
    auto q0 = [&](unsigned long long bits) {
        double s;
        std::memcpy(&s, &bits, 8);
        return a / s == 0.0;
    };
    if (!q0(hi)) return std::numeric_limits<double>::infinity();
    while (hi - lo > 1) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        if (q0(mid)) hi = mid;
        else lo = mid;
    }
    double s;
    std::memcpy(&s, &hi, 8);
    return s;
}

// Largest double s with RN(a / s) == +inf (0 when none).
double inf_threshold(double a) {
    unsigned long long lo = 0x0000000000000001ull, hi = 0x7ff0000000000000ull;
    auto qi = [&](unsigned long long bits) {
        double s;
        std::memcpy(&s, &bits, 8);
        return std::isinf(a / s);
    };
    if (!qi(lo)) return 0.0;
    while (hi - lo > 1) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        if (qi(mid)) lo = mid;
        else hi = mid;
    }
    double s;
    std::memcpy(&s, &lo, 8);
    return s;
}

std::vector<std::pair<int, int>> partition_scanlines(int ny, int workers) {
    std::vector<std::pair<int, int>> bands;
    const int base = ny / workers, rem = ny % workers;
    int j = 0;
    for (int w = 0; w < workers; ++w) {
        const int rows = base + (w < rem ? 1 : 0);
        bands.push_back({j, j + rows});
        j += rows;
    }
    return bands;
}

}  // namespace

namespace {


bool is_fin(double x) { return std::isfinite(x); }

SweBC to_bc(const swe_boundary& b) {
    SweBC o;
    o.type = b.type;
    o.q_n = b.q_n;
    o.eta_out = b.eta_out;
    return o;
}

// validate_physics / validate_policy / validate_boundary (scheme.hpp:22-32,
// timestep.hpp:26-39, grid.hpp:177-193) and GridSpec (grid.hpp:28-37).
int validate(const swe_grid* g, const swe_physics* p, const swe_policy* pol,
             const swe_boundary_set* b, swe_status* st) {
    if (g->nx < 3 || g->ny < 3)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "GridSpec: nx and ny must be at least 3, got %dx%d",
                          g->nx, g->ny);
    if (!(g->dx > 0.0) || !(g->dy > 0.0) || !is_fin(g->dx) || !is_fin(g->dy))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "GridSpec: dx and dy must be positive and finite");
    if (!(p->g > 0.0) || !is_fin(p->g))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "physics: g must be positive and finite");
    if (!(p->manning_n >= 0.0))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "physics: manning_n must be >= 0");
    if (!(p->nu_art >= 0.0) || !(p->nu_art < 0.5))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "physics: nu_art must lie in [0, 0.5)");
    if (!(pol->cfl > 0.0) || !(pol->cfl <= 1.0))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "policy: cfl must lie in (0, 1]");
    if (!(pol->dt_min > 0.0))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "policy: dt_min must be > 0");
    if (!(pol->dt_max >= pol->dt_min))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "policy: dt_max must be >= dt_min");
    if (!(pol->h_min > 0.0))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "policy: h_min must be > 0");
    const swe_boundary* bs[4] = {&b->north, &b->south, &b->east, &b->west};
    const char* names[4] = {"north", "south", "east", "west"};
    for (int k = 0; k < 4; ++k) {
        if (bs[k]->type < 0 || bs[k]->type > 3)
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "%s: unknown boundary type %d", names[k], bs[k]->type);
        if (bs[k]->type == SWE_BC_INFLOW && (!(bs[k]->h_in >= pol->h_min) || !is_fin(bs[k]->q_n)))
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "%s: inflow requires finite q_n and h_in >= h_min",
                              names[k]);
        if (bs[k]->type == SWE_BC_FIXED_ETA && !is_fin(bs[k]->eta_out))
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "%s: fixed elevation must be finite", names[k]);
    }
    return SWE_OK;
}

double* row_ptr(swe_ctx* c, int which, int lr) {
    return c->d_buf[which] + static_cast<size_t>(lr + c->R) * 3 * c->pitch;
}

// Exchange R committed rows with the strip neighbours:
// own top rows -> rank+1's lower halo, own bottom rows -> rank-1's upper halo.
// (c->halo_x rows: R, or fewer under the SWE_DEBUG_HALO_ROWS test hook, which
// must then break the strips' equality with one domain: the halo-mutation
// check of test_executor.cpp:246-303.)
int halo_exchange(swe_ctx* c, int which, cudaStream_t s, swe_status* st) {
    if (c->ex.nranks <= 1) return SWE_OK;
    const int rows = c->halo_x;
    const size_t bytes = static_cast<size_t>(rows) * 3 * c->pitch * sizeof(double);
    const int rk = c->ex.rank, nr = c->ex.nranks;
    const bool up = rk + 1 < nr, down = rk > 0;
    return c->tr->sendrecv(c, s, up ? row_ptr(c, which, c->nloc - rows) : nullptr,
                           up ? row_ptr(c, which, c->nloc) : nullptr, down ? row_ptr(c, which, 0) : nullptr,
                           down ? row_ptr(c, which, -rows) : nullptr, bytes, st);
}

// Enqueue one step on the stream (no host sync).  `fwd` = sweep parity,
// `cand` = candidate buffer as assumed by the host (used for the strip halo
// exchange only).
int enqueue_step(swe_ctx* c, bool fwd, int cand, swe_status* st) {
    const int v = swe_step_variant(fwd, c->smooth, c->flat, c->manning, c->early, c->xonly);
    if (c->p2p) {
        // Strips with the fused halo push: the step kernel stores its edge rows
        // into the neighbours' halos itself; one allreduce of the reduction
        // words (which also orders those stores before every rank's next
        // step), then the finalize.
        if (c->prm.early) {
            CUDA_TRY(swe_launch_schedule(c->exact, c->stream, c->prm));
            ++c->launches;
        }
        CUDA_TRY(swe_launch_step(c->exact, v, c->ncta, c->stream, c->prm));
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[2], c->stream));
        int rc = c->tr->allreduce_max(c, c->stream, c->d_ctl->red, RED_N, st);
        if (rc) return rc;
        if (c->time_exchange) {
            CUDA_TRY(cudaEventRecord(c->ev_x[3], c->stream));
            CUDA_TRY(cudaEventRecord(c->ev_x[0], c->stream));  // no separate exchange (not counted)
            CUDA_TRY(cudaEventRecord(c->ev_x[1], c->stream));
        }
        CUDA_TRY(swe_launch_finalize(c->stream, c->prm));
        c->launches += 2 + (c->tr->capturable() ? 0 : 1);  // step + finalize (+ local max kernel)
        return SWE_OK;
    }
    if (c->overlap) {
        // Strips, overlapped: the edge launch (the bands whose rows the
        // neighbours need) runs on a high-priority stream and its halo
        // send/recv follows it there, while the interior launch runs on the
        // main stream; the allreduce and the finalize wait for both.
        CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->stream_edge, c->ev_fork, 0));
        CUDA_TRY(swe_launch_step(c->exact, v, c->ncta_edge, c->stream_edge, c->prm_edge));
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[0], c->stream_edge));
        int rc = halo_exchange(c, cand, c->stream_edge, st);
        if (rc) return rc;
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[1], c->stream_edge));
        CUDA_TRY(cudaEventRecord(c->ev_join, c->stream_edge));
        CUDA_TRY(swe_launch_step(c->exact, v, c->ncta, c->stream, c->prm_int));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[2], c->stream));
        rc = c->tr->allreduce_max(c, c->stream, c->d_ctl->red, RED_N, st);
        if (rc) return rc;
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[3], c->stream));
        CUDA_TRY(swe_launch_finalize(c->stream, c->prm));
        c->launches += 3 + (c->tr->capturable() ? 0 : 1);  // edge + interior + finalize (+ local max kernel)
        return SWE_OK;
    }
    if (c->prm.early) {
        CUDA_TRY(swe_launch_schedule(c->exact, c->stream, c->prm));
        ++c->launches;
    }
    CUDA_TRY(swe_launch_step(c->exact, v, c->ncta, c->stream, c->prm));
    ++c->launches;
    if (c->ex.nranks > 1) {
        // same collective order as the overlapped path (send/recv, then the
        // allreduce): ranks may take different paths (strip heights differ
        // by one row, early exit depends on the local bed) and NCCL requires
        // every rank to issue a communicator's operations in the same order
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[0], c->stream));
        int rc = halo_exchange(c, cand, c->stream, st);
        if (rc) return rc;
        if (c->time_exchange) {
            CUDA_TRY(cudaEventRecord(c->ev_x[1], c->stream));
            CUDA_TRY(cudaEventRecord(c->ev_x[2], c->stream));
        }
        rc = c->tr->allreduce_max(c, c->stream, c->d_ctl->red, RED_N, st);
        if (rc) return rc;
        if (c->time_exchange) CUDA_TRY(cudaEventRecord(c->ev_x[3], c->stream));
        CUDA_TRY(swe_launch_finalize(c->stream, c->prm));
        c->launches += 1 + (c->tr->capturable() ? 0 : 1);  // finalize (+ local max kernel)
    }
    return SWE_OK;
}

int read_ctl(swe_ctx* c, swe_status* st) {
    CUDA_TRY(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(SweCtl), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SWE_OK;
}

int write_ctl(swe_ctx* c, swe_status* st) {
    CUDA_TRY(cudaMemcpyAsync(c->d_ctl, c->h_ctl, sizeof(SweCtl), cudaMemcpyHostToDevice, c->stream));
    return SWE_OK;
}

// min over cells of min(dx/sx, dy/sy) (executor.hpp:560-580) from the scan
// words: the quotients of the two speed maxima of the cells whose quotients
// are certainly finite (correctly rounded division is monotone, so the
// minimum quotient is the quotient of the maximum), and the per-cell minimum
// of the other cells; +inf for no cells.
double scan_core(const swe_ctx* c, const unsigned long long sc[SCAN_N]) {
    auto as_double = [](unsigned long long b) {
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    };
    double core = std::numeric_limits<double>::infinity();
    if (sc[SCAN_MAXSX]) core = std_min(core, c->g.dx / as_double(sc[SCAN_MAXSX]));
    if (sc[SCAN_MAXSY]) core = std_min(core, c->g.dy / as_double(sc[SCAN_MAXSY]));
    if (sc[SCAN_MINR]) core = std_min(core, as_double(~sc[SCAN_MINR]));
    return core;
}

// Run the exact scan over own rows of buffer `which`; results all-reduced.
// cfl = false: the stability guard only.
int run_scan(swe_ctx* c, int which, unsigned long long out[SCAN_N], swe_status* st, bool cfl = true) {
    CUDA_TRY(cudaMemsetAsync(c->d_scan, 0, SCAN_N * sizeof(unsigned long long), c->stream));
    const size_t n = static_cast<size_t>(c->nloc) * c->g.nx;
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16));
    scan_kernel<<<std::max(blocks, 1), 256, 0, c->stream>>>(c->d_buf[which], c->pitch, c->R, c->g.nx,
                                                            c->nloc, c->j0, c->ph.g, c->g.dx, c->g.dy,
                                                            c->pol.h_min, cfl ? 1 : 0, c->d_scan);
    CUDA_TRY(cudaGetLastError());
    if (c->ex.nranks > 1) {
        int rc = c->tr->allreduce_max(c, c->stream, c->d_scan, SCAN_N, st);
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(out, c->d_scan, SCAN_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return SWE_OK;
}

// First row-major corrector cell consuming a dry U* (dry_scan_kernel over
// this rank's rows of the committed buffer), all-reduced; 0 = none.
int run_dry_scan(swe_ctx* c, double dt, bool fwd, unsigned long long* first, swe_status* st) {
    CUDA_TRY(cudaMemsetAsync(c->d_scan, 0, SCAN_N * sizeof(unsigned long long), c->stream));
    BcSet b;
    for (int e = 0; e < 4; ++e) b.bc[e] = c->prm.bc[e];
    dry_scan_kernel<<<std::max(1, std::min(c->nloc, 148 * 8)), 256, 0, c->stream>>>(
        c->d_buf[c->sel], c->pitch, c->R, c->g.nx, c->g.ny, c->nloc, c->j0, dt, c->g.dx, c->g.dy, fwd ? 1 : 0,
        c->exact ? 1 : 0, b, c->d_zw, c->d_ze, c->d_zs, c->d_zn, c->pol.h_min, c->d_scan);
    CUDA_TRY(cudaGetLastError());
    if (c->ex.nranks > 1) {
        int rc = c->tr->allreduce_max(c, c->stream, c->d_scan, SCAN_N, st);
        if (rc) return rc;
    }
    unsigned long long sc[SCAN_N];
    CUDA_TRY(cudaMemcpyAsync(sc, c->d_scan, sizeof sc, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *first = sc[SCAN_DRY];
    return SWE_OK;
}

// Values of global cell idx from buffer `which` (the owning rank answers;
// others return NaN).
void cell_values(swe_ctx* c, int which, unsigned long long idx, double* h, double* qx, double* qy) {
    const int j = static_cast<int>(idx / c->g.nx), i = static_cast<int>(idx % c->g.nx);
    *h = *qx = *qy = std::numeric_limits<double>::quiet_NaN();
    const int lr = j - c->j0;
    if (lr < 0 || lr >= c->nloc) return;
    double v[3];
    for (int f = 0; f < 3; ++f)
        cudaMemcpy(&v[f], c->d_buf[which] + (static_cast<size_t>(lr + c->R) * 3 + f) * c->pitch + (i + SWE_XO), 8,
                   cudaMemcpyDeviceToHost);
    *h = v[0];
    *qx = v[1];
    *qy = v[2];
}

// Depth of the dry predicted state that failed the corrector's check at
// consumer (i, j) (executor.hpp:429-436, 451-513: own U* first, then the
// west, east, south and north U* the corrector reads).  U*.h only needs
// h of the cell and the momenta of its sweep neighbours
// (scheme.hpp:100-113), so the host recomputes it from the intact committed
// buffer with the kernel's arithmetic.  NaN when a needed row is not held by
// this rank.
double dry_star_depth(swe_ctx* c, int i, int j, double dt, bool fwd) {
    const int nx = c->g.nx, ny = c->g.ny, R = c->R, P = c->pitch;
    const int lj = j - c->j0;
    if (lj - 1 < -R || lj + 1 >= c->nloc + R) return std::numeric_limits<double>::quiet_NaN();
    // rows lj-1 .. lj+1, padded columns i-1 .. i+1 of h, qx, qy
    double v[3][3][3];  // [row][field][col]
    for (int r = 0; r < 3; ++r)
        for (int f = 0; f < 3; ++f)
            cudaMemcpy(v[r][f], c->d_buf[c->sel] + (static_cast<size_t>(lj - 1 + r + R) * 3 + f) * P + (i - 1 + SWE_XO),
                       3 * sizeof(double), cudaMemcpyDeviceToHost);
    const double dtdx = dt / c->g.dx, dtdy = dt / c->g.dy;
    const int s = fwd ? 1 : -1;
    auto star_h = [&](int di, int dj) {  // U*.h of cell (i+di, j+dj), |di|,|dj| <= 1
        const int r = 1 + dj, col = 1 + di;
        const double hh = v[r][0][col], qx = v[r][1][col], qy = v[r][2][col];
        const double qxn = v[r][1][col + s], qyn = v[r + s][2][col];
        const double df = fwd ? qxn - qx : qx - qxn, dg = fwd ? qyn - qy : qy - qyn;
        if (c->exact) return (hh - (dtdx * df + dtdy * dg)) + 0.0;
        return hh - std::fma(dtdx, df, dtdy * dg);
    };
    const double h_min = c->pol.h_min;
    auto dry = [&](double x) { return !(x >= h_min); };
    const double own = star_h(0, 0);
    if (dry(own)) return own;
    auto face = [&](bool at_edge, int type, int di, int dj, bool uses_nbr) -> double {
        // wall / inflow faces read no neighbour U*; other edge faces read a ghost
        // of U*(i, j), which already passed (fixed-elevation ghosts are >= h_min)
        if (at_edge && (type == SWE_BC_WALL || type == SWE_BC_INFLOW)) return h_min;
        if (at_edge || !uses_nbr) return h_min;
        return star_h(di, dj);
    };
    const double cand[4] = {face(i == 0, c->bnd.west.type, -1, 0, fwd), face(i == nx - 1, c->bnd.east.type, 1, 0, !fwd),
                            face(j == 0, c->bnd.south.type, 0, -1, fwd),
                            face(j == ny - 1, c->bnd.north.type, 0, 1, !fwd)};
    for (double x : cand)
        if (dry(x)) return x;
    return own;
}

// Translate the control block after a launch into the reference's outcome.
// Returns SWE_OK (committed), an error, or resolves a diagnosis request.
int resolve(swe_ctx* c, swe_status* st) {
    SweCtl& h = *c->h_ctl;
    if (h.status == SWE_OK) return SWE_OK;
    if (h.status == SWE_STATUS_DIAG) {
        const int cand = h.sel ^ 1;
        const bool fwd = (h.step_index % 2) == 0;
        if (h.diag_flags & 2) {  // K4: an interior window saw a dry U*
            unsigned long long first = 0;
            int rc = run_dry_scan(c, h.dt_used, fwd, &first, st);
            if (rc) return rc;
            if (first) {
                const unsigned long long idx = ~first;
                const int i = static_cast<int>(idx % c->g.nx), j = static_cast<int>(idx / c->g.nx);
                h.status = SWE_ERR_INSTABILITY;
                h.err_kind = 4;
                h.done = 1;
                write_ctl(c, st);
                const double hd = dry_star_depth(c, i, j, h.dt_used, fwd);
                int r = set_status(st, SWE_ERR_INSTABILITY, i, j, h.t_commit,
                                   "predicted depth %f below dry threshold at cell (%d, %d)", hd, i, j);
                if (st) st->h = hd;
                return r;
            }
        }
        // Exact per-cell guard (K5, executor.hpp:543-556) and CFL (K6,
        // executor.hpp:560-580) scan of the candidate.
        unsigned long long sc[SCAN_N];
        int rc = run_scan(c, cand, sc, st);
        if (rc) return rc;
        if (sc[SCAN_GUARD]) {
            const unsigned long long idx = ~sc[SCAN_GUARD];
            const int i = static_cast<int>(idx % c->g.nx), j = static_cast<int>(idx / c->g.nx);
            h.status = SWE_ERR_INSTABILITY;
            h.err_kind = 5;
            h.done = 1;
            write_ctl(c, st);
            double vh, vqx, vqy;
            cell_values(c, cand, idx, &vh, &vqx, &vqy);
            int r = set_status(st, SWE_ERR_INSTABILITY, i, j, h.t_commit,
                               "instability: cell (%d, %d) at t=%f: h=%f qx=%f qy=%f", i, j, h.t_commit, vh, vqx,
                               vqy);
            if (st) {
                st->h = vh;
                st->qx = vqx;
                st->qy = vqy;
            }
            return r;
        }
        if (sc[SCAN_BAD]) {
            const unsigned long long idx = ~sc[SCAN_BAD];
            h.status = SWE_ERR_INSTABILITY;
            h.done = 1;
            write_ctl(c, st);
            return set_status(st, SWE_ERR_INSTABILITY, static_cast<int>(idx % c->g.nx),
                              static_cast<int>(idx / c->g.nx), h.t_commit,
                              "non-finite wave speed in dt reduction");
        }
        const double core = scan_core(c, sc);
        const double dt_raw = std_min(c->pol.cfl * core, c->pol.dt_max);
        if (dt_raw < c->pol.dt_min) {
            h.status = SWE_ERR_STEP_COLLAPSE;
            h.done = 1;
            write_ctl(c, st);
            int r = set_status(st, SWE_ERR_STEP_COLLAPSE, -1, -1, h.t_commit,
                               "next step size %f collapsed below dt_min %f", dt_raw, c->pol.dt_min);
            if (st) st->dt = dt_raw;
            return r;
        }
        // commit on the host's behalf
        h.status = SWE_OK;
        h.dt_next = dt_raw;
        h.sel ^= 1;
        h.t = h.t_commit;
        h.step_index += 1;
        h.dt_raw = dt_raw;
        h.steps_done += 1;
        h.done = (h.mode == 1) ? (!(h.t < h.t_end) || h.t >= h.t_mark) : 0;
        return write_ctl(c, st);
    }
    if (h.status == SWE_ERR_INSTABILITY) {
        if (h.err_kind == 2)
            return set_status(st, SWE_ERR_INSTABILITY, -1, -1, 0.0, "depth below dry threshold");
        if (h.err_kind == 4) {  // require_wet_at's message (executor.hpp:429-436)
            const double hd = dry_star_depth(c, h.err_i, h.err_j, h.dt_used, (h.step_index % 2) == 0);
            int r = set_status(st, SWE_ERR_INSTABILITY, h.err_i, h.err_j, h.err_t,
                               "predicted depth %f below dry threshold at cell (%d, %d)", hd, h.err_i, h.err_j);
            if (st) st->h = hd;
            return r;
        }
        // guard (executor.hpp:889-897): values come from the candidate buffer
        double vh, vqx, vqy;
        cell_values(c, h.sel ^ 1, static_cast<unsigned long long>(h.err_j) * c->g.nx + h.err_i, &vh, &vqx, &vqy);
        int r = set_status(st, SWE_ERR_INSTABILITY, h.err_i, h.err_j, h.err_t,
                           "instability: cell (%d, %d) at t=%f: h=%f qx=%f qy=%f", h.err_i, h.err_j,
                           h.err_t, vh, vqx, vqy);
        if (st) {
            st->h = vh;
            st->qx = vqx;
            st->qy = vqy;
        }
        return r;
    }
    if (h.status == SWE_ERR_STEP_COLLAPSE) {
        int r = set_status(st, SWE_ERR_STEP_COLLAPSE, -1, -1, h.err_t,
                           "next step size %f collapsed below dt_min %f", h.err_dt, c->pol.dt_min);
        if (st) st->dt = h.err_dt;
        return r;
    }
    return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "unexpected device status %d", h.status);
}

int destroy_graphs(swe_ctx* c) {
    for (auto& kv : c->graphs)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    c->graphs.clear();
    return 0;
}

// The graph of `len` steps whose first step has sweep parity `parity` and
// finds the committed selector at `sel` (only strips depend on sel).
// A step graph that cannot be captured or instantiated (e.g. a transport's
// collectives refusing capture on some system) is not an error of the run:
// get_graph returns kGraphUnavailable once, and advance() launches the steps
// plainly from then on (same kernels, same order).
constexpr int kGraphUnavailable = -100;
constexpr long long kL2BandBytes = 48ll << 20;  // rows in flight of the persistent step (see finish_load)

int get_graph(swe_ctx* c, int len, int parity, int sel, swe_ctx::Graph** out, swe_status* st) {
    if (c->ex.nranks == 1) sel = 0;  // one rank: the kernels read the selector on the device
    const int key = (len << 2) | (parity << 1) | sel;
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
        const unsigned long long before = c->launches;
        cudaGraph_t gph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int rc = SWE_OK;
        for (int k = 0; k < len && rc == SWE_OK; ++k)
            rc = enqueue_step(c, ((parity + k) % 2) == 0, (sel + k + 1) & 1, st);
        cudaError_t e = cudaStreamEndCapture(c->stream, &gph);
        const unsigned long long captured = c->launches - before;
        c->launches = before;  // captured (or discarded), not launched
        if (rc) {
            if (gph) cudaGraphDestroy(gph);
            return rc;
        }
        swe_ctx::Graph g;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&g.exec, gph, 0);
        if (const char* f = std::getenv("SWE_DEBUG_GRAPH_FAIL"); f && f[0] == '1' && e == cudaSuccess) {
            cudaGraphExecDestroy(g.exec);  // test hook: the fallback below
            e = cudaErrorStreamCaptureUnsupported;
        }
        if (gph) cudaGraphDestroy(gph);
        if (e != cudaSuccess) {
            cudaGetLastError();  // capture errors are not sticky
            std::fprintf(stderr, "swe-b200: CUDA graph of %d steps unavailable (%s); launching steps without graphs\n",
                         len, cudaGetErrorString(e));
            c->graph_failed = true;
            return kGraphUnavailable;
        }
        g.kernels = captured;
        it = c->graphs.emplace(key, g).first;
    }
    *out = &it->second;
    return SWE_OK;
}

// Graph chunks for `left` steps: powers of two of at most 64 steps
// (20 = 16 + 4), so any step count runs from a handful of cached graphs.
std::vector<int> chunk_plan(uint64_t left) {
    std::vector<int> v;
    while (left) {
        int n = 64;
        while (static_cast<uint64_t>(n) > left) n >>= 1;
        v.push_back(n);
        left -= static_cast<uint64_t>(n);
    }
    return v;
}

}  // namespace

// ======================================================================= API

EXPORT const char* swe_cuda_version(void) { return "swe-b200 1.0 (sm_100a, ABI 1)"; }

EXPORT int swe_cuda_nccl_unique_id(void* out, swe_status* st) { return nccl_unique_id(out, st); }

// The row strip of `rank` (executor.hpp:189-208 partition_scanlines, with the
// decomposed executor's >= 4-row band rule); host only, no CUDA call.
EXPORT int swe_cuda_strip_rows(int32_t ny, int32_t nranks, int32_t rank, int32_t* row_begin, int32_t* row_end,
                               swe_status* st) {
    if (!row_begin || !row_end) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "strip_rows: null output");
    if (nranks < 1) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "partition_scanlines: workers must be >= 1");
    if (rank < 0 || rank >= nranks)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: rank %d outside [0, %d)", rank, nranks);
    if (ny < nranks)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0,
                          "partition_scanlines: %d workers need at least as many rows, grid has %d", nranks, ny);
    const auto bands = partition_scanlines(ny, nranks);
    if (nranks > 1)
        for (const auto& b : bands)
            if (b.second - b.first < 4)
                return set_status(st, SWE_ERR_CONFIG, -1, -1, 0,
                                  "executor: decomposed bands need at least 4 rows; %d workers on %d rows "
                                  "leaves a band with %d",
                                  nranks, ny, b.second - b.first);
    *row_begin = bands[rank].first;
    *row_end = bands[rank].second;
    return ok_status(st);
}

EXPORT int swe_cuda_create(const swe_grid* grid, const swe_physics* phys, const swe_policy* pol,
                           const swe_boundary_set* bnd, const swe_exec* exec, swe_ctx** out,
                           swe_status* st) {
    *out = nullptr;
    int rc = validate(grid, phys, pol, bnd, st);
    if (rc) return rc;
    swe_exec ex{};
    if (exec) ex = *exec;
    if (ex.nranks < 1) ex.nranks = 1;
    if (ex.rank < 0 || ex.rank >= ex.nranks)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: rank %d outside [0, %d)", ex.rank, ex.nranks);
    int32_t band_b = 0, band_e = 0;
    if (int rc = swe_cuda_strip_rows(grid->ny, ex.nranks, ex.rank, &band_b, &band_e, st)) return rc;
    CUDA_TRY(cudaSetDevice(ex.device));

    swe_ctx* c = new swe_ctx();
    c->g = *grid;
    c->ph = *phys;
    c->pol = *pol;
    c->bnd = *bnd;
    c->ex = ex;
    c->ex.nccl_id = nullptr;
    c->exact = (ex.flags & SWE_EXEC_EXACT) != 0;
    c->early = (ex.flags & SWE_EXEC_EARLY_EXIT) != 0;
    c->smooth = phys->nu_art > 0.0;  // StepPlan::standard(nu_art > 0), executor.hpp:730
    c->manning = phys->manning_n > 0.0;
    c->R = c->smooth ? 2 : 1;
    c->halo_x = c->R;
    if (const char* hx = std::getenv("SWE_DEBUG_HALO_ROWS"))  // test hook (halo mutation)
        c->halo_x = std::max(0, std::min(c->R, std::atoi(hx)));
    c->j0 = band_b;
    c->nloc = band_e - band_b;
    const int out_w = SWE_TILE_W(c->R);
    c->ntiles = (grid->nx + out_w - 1) / out_w;
    // columns touched: the last window's load box ends at ntiles*TW - R + SWE_XO + 33
    c->pitch = ((c->ntiles * out_w + SWE_XO + 34) + 31) / 32 * 32;
    const size_t rows = static_cast<size_t>(c->nloc + 2 * c->R);
    c->buf_doubles = rows * 3 * c->pitch;
    *out = c;

    CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    if (ex.nranks > 1) {
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_TRY(cudaStreamCreateWithPriority(&c->stream_edge, cudaStreamNonBlocking, hi));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        for (auto& e : c->ev_x) CUDA_TRY(cudaEventCreate(&e));
    }
    CUDA_TRY(cudaEventCreate(&c->ev0));
    CUDA_TRY(cudaEventCreate(&c->ev1));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_buf[k]), c->buf_doubles * sizeof(double)));
        fill_benign_kernel<<<148 * 8, 256, 0, c->stream>>>(c->d_buf[k], rows * 3, c->pitch);
        CUDA_TRY(cudaGetLastError());
    }
    const size_t zrows = rows;
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_zw), zrows * sizeof(double)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_ze), zrows * sizeof(double)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_zs), grid->nx * sizeof(double)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_zn), grid->nx * sizeof(double)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_zp), static_cast<size_t>(c->nloc + 2 * c->R + 2) * grid->nx * sizeof(double)));
    CUDA_TRY(cudaMemsetAsync(c->d_zw, 0, zrows * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_ze, 0, zrows * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_zs, 0, grid->nx * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_zn, 0, grid->nx * sizeof(double), c->stream));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_scan), SCAN_N * sizeof(unsigned long long)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_flags), 4 * sizeof(unsigned)));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_stats), 4 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(c->d_stats, 0, 4 * sizeof(unsigned long long), c->stream));
    CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_ctl), sizeof(SweCtl)));
    CUDA_TRY(cudaMallocHost(&c->h_ctl, sizeof(SweCtl)));
    std::memset(c->h_ctl, 0, sizeof(SweCtl));
    CUDA_TRY(cudaMemcpyAsync(c->d_ctl, c->h_ctl, sizeof(SweCtl), cudaMemcpyHostToDevice, c->stream));

    if (ex.nranks > 1) {
        if (!exec->nccl_id)
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: nranks > 1 requires nccl_id");
        CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_xr), 16 * sizeof(unsigned long long)));
        const int trc = create_transport(c, ex, exec->nccl_id, st);
        if (trc) return trc;
        // fused halo push: map the strip neighbours' buffers; used only if every
        // rank could (an allreduce agrees), else the halo goes by send/recv
        const char* pe = std::getenv("SWE_P2P");
        double *dn[2] = {nullptr, nullptr}, *up[2] = {nullptr, nullptr};
        int nloc_dn = 0;
        if (!(pe && pe[0] == '0')) {
            int rc2 = c->tr->peer_buffers(c, dn, up, &nloc_dn, st);
            if (rc2) return rc2;
        }
        const bool mine_ok = (ex.rank == 0 || dn[0]) && (ex.rank + 1 == ex.nranks || up[0]);
        unsigned long long bad = mine_ok ? 0ull : 1ull;
        CUDA_TRY(cudaMemcpyAsync(c->d_scan, &bad, sizeof bad, cudaMemcpyHostToDevice, c->stream));
        int rc3 = c->tr->allreduce_max(c, c->stream, c->d_scan, 1, st);
        if (rc3) return rc3;
        CUDA_TRY(cudaMemcpyAsync(&bad, c->d_scan, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        c->p2p = bad == 0ull;
        if (c->p2p) {
            for (int k = 0; k < 2; ++k) {
                c->prm.peer_dn[k] = dn[k];
                c->prm.peer_up[k] = up[k];
            }
            c->prm.nloc_dn = nloc_dn;
            c->prm.p2p = 1;
        }
    }

    // K6 diagnosis thresholds (see swe_step.cuh finalize_step)
    c->tz_x = zero_threshold(grid->dx);
    c->tz_y = zero_threshold(grid->dy);
    {
        const double cmin = std::sqrt(phys->g * pol->h_min);
        const double ti_x = inf_threshold(grid->dx), ti_y = inf_threshold(grid->dy);
        c->always_diag = !(cmin > ti_x || cmin > ti_y);
    }

    StepParams& p = c->prm;
    {
        std::string err;
        for (int k = 0; k < 2; ++k)
            if (!encode_rows(&p.tmap_state[k], c->d_buf[k], c->pitch, static_cast<long long>(rows) * 3,
                             3 * swe_row_group(c->exact), err, swe_box_w(c->R)))
                return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
    }
    p.buf[0] = c->d_buf[0];
    p.buf[1] = c->d_buf[1];
    p.slope = nullptr;
    p.z_w = c->d_zw;
    p.z_e = c->d_ze;
    p.z_s = c->d_zs;
    p.z_n = c->d_zn;
    p.ctl = c->d_ctl;
    p.nx = grid->nx;
    p.ny = grid->ny;
    p.nloc = c->nloc;
    p.j0 = c->j0;
    p.pitch = c->pitch;
    p.buf_doubles = static_cast<long long>(c->buf_doubles);
    p.ntiles = c->ntiles;
    p.finalize = ex.nranks > 1 ? 0 : 1;
    p.nranks = ex.nranks;
    p.dx = grid->dx;
    p.dy = grid->dy;
    p.g = phys->g;
    p.half_g = 0.5 * phys->g;
    p.sqrt_g = std::sqrt(phys->g);
    p.neg_g = -phys->g;
    p.gnn = phys->g * phys->manning_n * phys->manning_n;
    p.h_min = pol->h_min;
    p.nu = phys->nu_art;
    p.cfl = pol->cfl;
    p.dt_max = pol->dt_max;
    p.dt_min = pol->dt_min;
    p.tz_x = c->tz_x;
    p.tz_y = c->tz_y;
    p.always_diag = c->always_diag;
    p.bc[SWE_EDGE_N] = to_bc(bnd->north);
    p.bc[SWE_EDGE_S] = to_bc(bnd->south);
    p.bc[SWE_EDGE_E] = to_bc(bnd->east);
    p.bc[SWE_EDGE_W] = to_bc(bnd->west);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ok_status(st);
}

EXPORT void swe_cuda_destroy(swe_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->stream_edge) cudaStreamSynchronize(c->stream_edge);
    destroy_graphs(c);
    delete c->tr;
    dev_free(c->d_xr);
    for (auto& b : c->d_buf)
        if (b) dev_free(b);
    dev_free(c->d_slope);
    dev_free(c->d_zw);
    dev_free(c->d_zp);
    dev_free(c->d_ze);
    dev_free(c->d_zs);
    dev_free(c->d_zn);
    dev_free(c->d_scan);
    dev_free(c->d_flags);
    dev_free(c->d_stats);
    dev_free(c->d_qflag);
    dev_free(c->d_elig);
    dev_free(c->d_iflat);
    dev_free(c->d_active);
    dev_free(c->d_ctl);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream_edge) cudaStreamDestroy(c->stream_edge);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (auto& e : c->ev_x)
        if (e) cudaEventDestroy(e);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

namespace {

constexpr int kNcclSms = 2;  // SMs left free for NCCL kernels on strips
constexpr long long kMultiMaxCells = 1 << 20;  // multi-step launches up to 1024^2 cells

#ifndef SWE_ITEMS_PER_WORKER
#define SWE_ITEMS_PER_WORKER 0  // first-tier work items per persistent worker (warp); 0: by variant
#endif

// Guided chunking: the first ~80 % of a launch's rows go out in `chunk`-row
// items, the rest in quarter-size items, so the dynamic queue ends with short
// items and the last warps finish together.  SWE_GUIDED=0 keeps uniform chunks.
void guided_chunks(StepParams& p, int rows) {
    const char* env = std::getenv("SWE_GUIDED");
    if (env && env[0] == '0') return;
    int c1 = p.chunk, c2 = std::max(8, c1 / 4);
    int big_pct = 80;
    // A/B hooks: first-tier chunk, second-tier chunk, first-tier share of the rows
    if (const char* e = std::getenv("SWE_CHUNK1")) c1 = p.chunk = std::max(8, std::atoi(e));
    if (const char* e = std::getenv("SWE_CHUNK2")) c2 = std::max(4, std::atoi(e));
    if (const char* e = std::getenv("SWE_BIGPCT")) big_pct = std::max(0, std::min(100, std::atoi(e)));
    if (c1 < 32 || rows < 8 * c1) return;
    const int big = (rows * big_pct / 100) / c1;
    const int rest = rows - big * c1;
    p.tier_rc = big;
    p.chunk2 = c2;
    p.nchunks = big + (rest + c2 - 1) / c2;
}

// Everything Stepper::load derives from the bed and the committed state once
// both sit on the device (state in buffer 0, own bed rows in d_zp): strip
// halos of the bed, edge bed values, slopes and flat-bed detection, K1 ghosts,
// the fixed-elevation clamp diagnostic, the launch geometry, the early-exit
// tables, and the control block.
int finish_load(swe_ctx* c, double t, swe_status* st) {
    const int nx = c->g.nx, R = c->R, P = c->pitch, nloc = c->nloc;
    const size_t rowb = static_cast<size_t>(nx) * sizeof(double);
    c->sel = 0;
    double* d_zp = c->d_zp;
    if (c->ex.nranks > 1) {  // bed halo rows of the strip neighbours (R + 1 each side)
        const int rk = c->ex.rank, nr = c->ex.nranks, H = R + 1;
        const size_t bytes = static_cast<size_t>(H) * nx * sizeof(double);
        const bool up = rk + 1 < nr, down = rk > 0;
        int rc = c->tr->sendrecv(c, c->stream, up ? d_zp + static_cast<size_t>(R + 1 + nloc - H) * nx : nullptr,
                                 up ? d_zp + static_cast<size_t>(R + 1 + nloc) * nx : nullptr,
                                 down ? d_zp + static_cast<size_t>(R + 1) * nx : nullptr, down ? d_zp : nullptr,
                                 bytes, st);
        if (rc) return rc;
    }
    // edge z arrays (z_w/z_e for local rows [-R, nloc+R), z_s/z_n per column)
    CUDA_TRY(cudaMemsetAsync(c->d_zw, 0, (nloc + 2 * R) * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_ze, 0, (nloc + 2 * R) * sizeof(double), c->stream));
    edge_z_kernel<<<std::max(1, std::min((nloc + 255) / 256, 148 * 4)), 256, 0, c->stream>>>(d_zp, R, nx, nloc,
                                                                                             c->d_zw, c->d_ze);
    CUDA_TRY(cudaGetLastError());
    if (c->j0 == 0)
        CUDA_TRY(cudaMemcpyAsync(c->d_zs, d_zp + static_cast<size_t>(R + 1) * nx, rowb, cudaMemcpyDeviceToDevice,
                                 c->stream));
    if (c->j0 + nloc == c->g.ny)
        CUDA_TRY(cudaMemcpyAsync(c->d_zn, d_zp + static_cast<size_t>(R + nloc) * nx, rowb, cudaMemcpyDeviceToDevice,
                                 c->stream));

    // slopes + flat-bed detection
    if (!c->d_slope) CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_slope), static_cast<size_t>(nloc + 2 * R) * 2 * P * sizeof(double)));
    CUDA_TRY(cudaMemsetAsync(c->d_slope, 0, static_cast<size_t>(nloc + 2 * R) * 2 * P * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_flags, 0, 4 * sizeof(unsigned), c->stream));
    slopes_kernel<<<std::min(nloc + 2 * R, 148 * 8), 256, 0, c->stream>>>(
        d_zp, c->d_slope, P, R, nx, nloc, c->j0, c->g.ny, 2.0 * c->g.dx, 2.0 * c->g.dy, c->exact ? 1.0 : -c->ph.g,
        c->d_flags);
    CUDA_TRY(cudaGetLastError());
    // fixed-elevation clamp diagnostic (grid.hpp:256-263): depends on the bed only
    {
        BcSet b;
        for (int e = 0; e < 4; ++e) b.bc[e] = c->prm.bc[e];
        const int n = std::max(nloc, nx);
        clamp_kernel<<<(n + 255) / 256, 256, 0, c->stream>>>(d_zp, R, nx, nloc, c->j0 == 0, c->j0 + nloc == c->g.ny,
                                                            b, c->pol.h_min, c->d_flags + 1);
        CUDA_TRY(cudaGetLastError());
    }
    unsigned flags[3] = {0u, 0u, 0u};
    CUDA_TRY(cudaMemcpyAsync(flags, c->d_flags, sizeof flags, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->flat = (flags[0] == 0);
    c->xonly = !c->flat && flags[2] == 0;  // every dz/dy is +0.0: skip those rows
    int clamp = flags[1] ? 1 : 0;
    c->prm.slope = c->d_slope;
    {
        std::string err;
        // row-group boxes of the kernels this load selects (early exit needs a flat bed)
        const int G = swe_row_group(c->exact, c->early && c->flat);
        for (int k = 0; k < 2; ++k)
            if (!encode_rows(&c->prm.tmap_state[k], c->d_buf[k], P, static_cast<long long>(nloc + 2 * R) * 3, 3 * G,
                             err, swe_box_w(R)))
                return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        if (!encode_rows(&c->prm.tmap_slope, c->d_slope, P, static_cast<long long>(nloc + 2 * R) * 2, 2 * G, err,
                         swe_box_w(R)))
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        // TMA-store epilogue: inner extent SWE_XO + nx (the window's
        // out-of-domain columns are clipped), rows 3*(nloc+2R), pitch P
        const int TW = SWE_TILE_W(R);
        for (int k = 0; k < 2; ++k) {
            if (!encode_rows(&c->prm.tmap_out[k], c->d_buf[k], SWE_XO + nx, static_cast<long long>(nloc + 2 * R) * 3,
                             3 * G, err, TW, P))
                return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        }
        if (!encode_rows(&c->prm.tmap_slopex, c->d_slope, P, static_cast<long long>(nloc + 2 * R), G, err,
                         swe_box_w(R), 2 * P))
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
    }

    // K1 ghosts of the committed state + strip halos
    const int gthreads = std::max(nloc, nx);
    ghost_fill_rows_kernel<<<(gthreads + 127) / 128, 128, 0, c->stream>>>(
        c->d_buf[0], P, R, nx, nloc, c->j0, c->g.ny, c->prm.bc[SWE_EDGE_W], c->prm.bc[SWE_EDGE_E],
        c->prm.bc[SWE_EDGE_S], c->prm.bc[SWE_EDGE_N], c->d_zw, c->d_ze, c->d_zs, c->d_zn, c->pol.h_min);
    CUDA_TRY(cudaGetLastError());
    int rc = halo_exchange(c, 0, c->stream, st);
    if (rc) return rc;

    if (c->ex.nranks > 1) {
        unsigned long long v = static_cast<unsigned long long>(clamp);
        CUDA_TRY(cudaMemcpyAsync(c->d_scan, &v, sizeof v, cudaMemcpyHostToDevice, c->stream));
        rc = c->tr->allreduce_max(c, c->stream, c->d_scan, 1, st);
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(&v, c->d_scan, sizeof v, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        clamp = static_cast<int>(v);
    }
    c->clamp_any = clamp;

    // occupancy-sized persistent grid
    const int v = swe_step_variant(true, c->smooth, c->flat, c->manning, c->early, c->xonly);
    c->occ = swe_step_occupancy(c->exact, v);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->ex.device);
    // NCCL strips: leave two SMs to NCCL's send/recv and allreduce kernels so
    // the halo exchange runs beside the persistent interior launch instead of
    // after it (its CTAs never retire early)
    // (not with the fused halo push: no send/recv runs beside the step)
    if (c->ex.nranks > 1 && !c->p2p && !(c->ex.flags & SWE_EXEC_LOCAL_GROUP)) nsm = std::max(1, nsm - kNcclSms);
    // persistent grid: every resident warp is a worker; small grids keep at
    // least 4 rows per worker so the 2R warm-up rows stay amortised
    const long long units = static_cast<long long>(c->ntiles) * nloc;
    const long long want = std::max<long long>(1, units / (4 * SWE_STEP_WPB));
    long long ncta = std::min<long long>(static_cast<long long>(c->occ) * nsm, want);
    // every worker must span at most 7 tiles (MAXSEG = 8 segments)
    ncta = std::max<long long>(ncta, (c->ntiles + 7 * SWE_STEP_WPB - 1) / (7 * SWE_STEP_WPB));
    if (const char* e = std::getenv("SWE_NCTA"))  // A/B hook: persistent grid size
        ncta = std::max<long long>(1, std::min<long long>(std::atoll(e), static_cast<long long>(c->occ) * nsm));
    c->ncta = static_cast<int>(ncta);
    c->prm.ncta = c->ncta;
    // multi-step launches for small grids (latency-bound: launch gaps and a
    // cold instruction cache per step); the cooperative grid must be resident
    {
        const char* env = std::getenv("SWE_MULTI");
        const bool allow = !(env && env[0] == '0');
        const int vm = swe_step_variant(true, c->smooth, c->flat, c->manning, false, c->xonly);
        const int occm = allow ? swe_multi_occupancy(c->exact, c->smooth, vm) : 0;
        c->multi_ok = allow && occm > 0 && static_cast<long long>(nloc) * c->g.nx <= kMultiMaxCells;
        c->occ_multi = occm;
    }
    // dynamic work items: ~16 per worker, 16..128 rows each
    {
        const long long workers = ncta * SWE_STEP_WPB;
        // first-tier items per worker: 20 for the fast sloped-bed kernels (12
        // warps/SM: C3 -0.7 %, C3f -0.4 % against 16), 16 for the fast flat
        // ones, 12 in exact mode (C3 exact -0.7 %, flat exact -0.4 %; each
        // alternative measured +0.4-1.4 % on the others:
        // profiles/r2d_ab_items_per_worker.log)
        const long long ipw = SWE_ITEMS_PER_WORKER ? SWE_ITEMS_PER_WORKER : c->exact ? 12 : c->flat ? 16 : 20;
        long long ch = units / std::max<long long>(1, workers * ipw);
        // Item heights are multiples of the row group (4 rows per TMA request
        // in fast mode): a segment then marches whole groups with no tail
        // iterations (the 8192^2 C3 step: 79-row items 0.830 ms, 80-row
        // 0.789 ms; 59 -> 64 rows on the flat 8192^2 grid, 0.573 ms)
        if (ch >= 16) {
            // L2 residency: items go out row-chunk-major, so the rows in flight
            // are about one chunk across the whole width; kept within ~48 MB of
            // the 126 MB L2 the neighbouring windows' halo columns and the next
            // chunk's halo rows are L2 hits (C4 32768^2: 128-row items 9.9 ms,
            // 64-row 8.75 ms, profiles/r2d_ab_c4_item_rows.log)
            // (fast mode: exact mode, compute-heavier, keeps 128-row items:
            // 64 rows cost it 1-2 % on C4)
            const long long cell_b = 24 + (c->flat ? 0 : c->xonly ? 8 : 16);  // state + slope bytes
            const long long cap = c->exact ? 128
                                           : std::max<long long>(16, std::min<long long>(
                                                 128, (kL2BandBytes / (static_cast<long long>(nx) * cell_b)) / 16 * 16));
            ch = std::min<long long>(cap, (ch + 8) / 16 * 16);
        } else {
            // small grids are latency-bound: the shortest items (>= 4 rows) that
            // still give every worker at most one item (512^2: 28 -> 20 us/step)
            ch = std::max<long long>(4, std::min<long long>(16, (units + workers - 1) / workers));
            ch = (ch + 3) / 4 * 4;
        }
        // early exit: finer items (32 rows) so the active band is balanced
        // across workers and skipped at a finer grain
        if (c->early && c->flat) {
            ch = 32;
            if (const char* e = std::getenv("SWE_EARLY_CHUNK")) ch = std::max(8, std::atoi(e));  // A/B hook
        }
        ch = std::min<long long>(ch, nloc);
        c->prm.chunk = static_cast<int>(ch);
        c->prm.nchunks = static_cast<int>((nloc + ch - 1) / ch);
    }
    // multi-step launches: the shortest items that give every resident warp
    // at most one (a warp marches its item's rows serially, one dependent
    // chain per row: C1 256^2 with 1-row items on 576 CTAs 10.6 -> 8.6 us per
    // step; C2 keeps 4-row items, its 2368 resident warps being the limit)
    if (c->multi_ok) {
        const long long max_warps = static_cast<long long>(c->occ_multi) * nsm * SWE_STEP_WPB;
        long long mch = std::max<long long>(1, (units + max_warps - 1) / max_warps);
        if (const char* e = std::getenv("SWE_SMALL_CHUNK")) mch = std::max(1, std::atoi(e));  // A/B hook
        mch = std::min<long long>(mch, c->prm.chunk);
        c->multi_chunk = static_cast<int>(mch);
        c->multi_nchunks = static_cast<int>((nloc + mch - 1) / mch);
        const long long items = static_cast<long long>(c->ntiles) * c->multi_nchunks;
        c->ncta_multi = static_cast<int>(std::max<long long>(
            1, std::min<long long>(static_cast<long long>(c->occ_multi) * nsm, (items + SWE_STEP_WPB - 1) / SWE_STEP_WPB)));
        if (const char* e = std::getenv("SWE_MULTI_CTAS"))  // A/B hook
            c->ncta_multi = std::max(1, std::min(std::atoi(e), c->occ_multi * nsm));
    }
    c->prm.row_lo = 0;
    c->prm.row_hi = nloc;
    c->prm.row_gap = 0;
    c->prm.wslot = 0;
    c->prm.tier_rc = c->prm.nchunks;  // uniform (the early-exit flags index uniform chunks)
    c->prm.chunk2 = c->prm.chunk;
    destroy_graphs(c);  // variant may have changed

    // early-exit tables for this item geometry (flags of both buffers reset:
    // nothing is known about the candidate buffer after a load)
    c->prm.early = 0;
    c->prm.stats = c->d_stats;
    CUDA_TRY(cudaMemsetAsync(c->d_stats, 0, 4 * sizeof(unsigned long long), c->stream));
    if (c->early && c->flat) {  // early-exit kernels exist for a flat bed only
        const int nitems = c->ntiles * c->prm.nchunks;
        if (nitems != c->nitems_alloc) {
            dev_free(c->d_qflag);
            dev_free(c->d_elig);
            dev_free(c->d_iflat);
            dev_free(c->d_active);
            c->d_qflag = nullptr;
            c->d_elig = c->d_iflat = nullptr;
            c->d_active = nullptr;
            CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_active), static_cast<size_t>(nitems) * sizeof(unsigned)));
            CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_qflag), 2 * static_cast<size_t>(nitems) * sizeof(unsigned long long)));
            CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_elig), nitems));
            CUDA_TRY(dev_alloc(reinterpret_cast<void**>(&c->d_iflat), nitems));
            c->nitems_alloc = nitems;
        }
        CUDA_TRY(cudaMemsetAsync(c->d_qflag, 0, 2 * static_cast<size_t>(nitems) * sizeof(unsigned long long),
                                 c->stream));
        const int TW = SWE_TILE_W(R);
        item_flat_kernel<<<std::min(nitems, 148 * 16), 128, 0, c->stream>>>(c->d_slope, P, R, nx, nloc, TW,
                                                                             c->prm.chunk, c->ntiles, nitems,
                                                                             c->d_iflat);
        CUDA_TRY(cudaGetLastError());
        item_elig_kernel<<<std::min((nitems + 255) / 256, 148 * 4), 256, 0, c->stream>>>(
            c->d_iflat, nx, nloc, TW, c->prm.chunk, c->ntiles, c->prm.nchunks, R, c->d_elig, c->d_stats + 1);
        CUDA_TRY(cudaGetLastError());
        c->prm.early = 1;
        c->prm.qflag[0] = c->d_qflag;
        c->prm.qflag[1] = c->d_qflag + nitems;
        c->prm.elig = c->d_elig;
        c->prm.active = c->d_active;
    }

    // strips: overlap the halo exchange with the interior rows.  The edge
    // launch covers the kEdge rows at each end of the strip (>= R, the rows the
    // neighbours receive); the interior launch the rows in between.
    constexpr int kEdge = 8;
    c->overlap = c->ex.nranks > 1 && !c->p2p && !(c->early && c->flat) && nloc >= 2 * kEdge + 16;
    if (c->overlap) {
        c->prm_edge = c->prm;
        c->prm_edge.chunk = kEdge;
        c->prm_edge.nchunks = 2;
        c->prm_edge.row_gap = nloc - 2 * kEdge;
        c->prm_edge.wslot = 0;
        c->ncta_edge = std::max(1, std::min(c->ncta, (2 * c->ntiles + SWE_STEP_WPB - 1) / SWE_STEP_WPB));
        c->prm_int = c->prm;
        c->prm_int.row_lo = kEdge;
        c->prm_int.row_hi = nloc - kEdge;
        c->prm_int.nchunks = (nloc - 2 * kEdge + c->prm.chunk - 1) / c->prm.chunk;
        c->prm_int.tier_rc = c->prm_int.nchunks;
        c->prm_int.wslot = 1;
        c->prm_edge.tier_rc = 2;
        guided_chunks(c->prm_int, nloc - 2 * kEdge);
    } else if (!c->prm.early) {
        guided_chunks(c->prm, nloc);
    }
    std::memset(c->h_ctl, 0, sizeof(SweCtl));
    c->h_ctl->t = t;
    c->h_ctl->sel = 0;
    CUDA_TRY(cudaMemcpyAsync(c->d_ctl, c->h_ctl, sizeof(SweCtl), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->t = t;
    c->loaded = true;
    return ok_status(st);
}

}  // namespace

EXPORT int swe_cuda_load(swe_ctx* c, const double* z, const double* h, const double* qx,
                         const double* qy, double t, swe_status* st) {
    if (!c) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "null context");
    if (!z || !h || !qx || !qy) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::load: null field");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    c->loaded = false;
    const int nx = c->g.nx, R = c->R, P = c->pitch, nloc = c->nloc;
    const size_t rowb = static_cast<size_t>(nx) * sizeof(double);
    // committed state into buffer 0 (padded, row-interleaved), bed into d_zp
    const double* src[3] = {h, qx, qy};
    for (int f = 0; f < 3; ++f) {
        double* dst = c->d_buf[0] + (static_cast<size_t>(R) * 3 + f) * P + SWE_XO;
        CUDA_TRY(cudaMemcpy2DAsync(dst, 3 * P * sizeof(double), src[f], rowb, rowb, nloc,
                                   cudaMemcpyHostToDevice, c->stream));
    }
    CUDA_TRY(cudaMemsetAsync(c->d_zp, 0, static_cast<size_t>(nloc + 2 * R + 2) * rowb, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_zp + static_cast<size_t>(R + 1) * nx, z, static_cast<size_t>(nloc) * rowb,
                             cudaMemcpyHostToDevice, c->stream));
    return finish_load(c, t, st);
}

EXPORT int swe_cuda_load_initial(swe_ctx* c, const swe_initial* ic, double t, swe_status* st) {
    if (!c || !ic) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "null context or initial condition");
    if (ic->kind != SWE_IC_FLAT_POOL && ic->kind != SWE_IC_CHANNEL_SLOPE && ic->kind != SWE_IC_DAM_BREAK)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0,
                          "load_initial: kind %d is not generated on the device (drops/vortex use std::exp, "
                          "which is not bit-reproducible on CUDA); load a host FieldSet instead",
                          ic->kind);
    CUDA_TRY(cudaSetDevice(c->ex.device));
    c->loaded = false;
    const int nx = c->g.nx, R = c->R, nloc = c->nloc;
    CUDA_TRY(cudaMemsetAsync(c->d_zp, 0, static_cast<size_t>(nloc + 2 * R + 2) * nx * sizeof(double), c->stream));
    const size_t n = static_cast<size_t>(nloc) * nx;
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16));
    initial_kernel<<<std::max(blocks, 1), 256, 0, c->stream>>>(*ic, c->g.dx, nx, nloc, c->pitch, R, c->d_buf[0],
                                                               c->d_zp);
    CUDA_TRY(cudaGetLastError());
    int rc = finish_load(c, t, st);
    if (rc) return rc;
    // build_initial_state ends with the stability guard (scenarios.hpp:165-169)
    unsigned long long sc[SCAN_N];
    rc = run_scan(c, 0, sc, st, false);
    if (rc) return rc;
    if (sc[SCAN_GUARD]) {
        c->loaded = false;
        const unsigned long long idx = ~sc[SCAN_GUARD];
        return set_status(st, SWE_ERR_CONFIG, static_cast<int>(idx % nx), static_cast<int>(idx / nx), t,
                          "initial state fails the stability guard: cell (%d, %d)", static_cast<int>(idx % nx),
                          static_cast<int>(idx / nx));
    }
    return ok_status(st);
}

EXPORT int swe_cuda_state(swe_ctx* c, double* z, double* h, double* qx, double* qy, double* t,
                          swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::state: no state loaded");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    const int nx = c->g.nx, R = c->R, P = c->pitch;
    const size_t rowb = static_cast<size_t>(nx) * sizeof(double);
    double* dst[3] = {h, qx, qy};
    for (int f = 0; f < 3; ++f) {
        if (!dst[f]) continue;
        const double* src = c->d_buf[c->sel] + (static_cast<size_t>(R) * 3 + f) * P + SWE_XO;
        CUDA_TRY(cudaMemcpy2DAsync(dst[f], rowb, src, 3 * P * sizeof(double), rowb, c->nloc,
                                   cudaMemcpyDeviceToHost, c->stream));
    }
    if (z)
        CUDA_TRY(cudaMemcpyAsync(z, c->d_zp + static_cast<size_t>(R + 1) * nx, static_cast<size_t>(c->nloc) * rowb,
                                 cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (t) *t = c->t;
    return ok_status(st);
}

EXPORT int swe_cuda_step(swe_ctx* c, double dt, uint64_t step_index, double t_after,
                         swe_step_result* res, swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::step: no state loaded");
    if (!(dt > 0.0) || !is_fin(dt))
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::step: dt must be positive and finite");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    const double t_commit = is_fin(t_after) ? t_after : c->t + dt;  // executor.hpp:820
    const bool fwd = (step_index % 2) == 0;                          // scheme.hpp:86-88
    SweCtl& h = *c->h_ctl;
    h.mode = 0;
    h.done = 0;
    h.dt_req = dt;
    h.tcommit_req = t_commit;
    h.step_index = step_index;
    h.sel = c->sel;
    h.t = c->t;
    h.status = 0;
    h.finish = 0;
    std::memset(h.red, 0, sizeof h.red);
    int rc = write_ctl(c, st);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    c->time_exchange = c->ex.nranks > 1;
    rc = enqueue_step(c, fwd, c->sel ^ 1, st);
    c->time_exchange = false;
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    rc = read_ctl(c, st);
    if (rc) return rc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->timing.steps += 1;
    c->timing.step_seconds += ms * 1e-3;
    if (c->ex.nranks > 1) {
        float mx = 0.f, ma = 0.f;
        cudaEventElapsedTime(&mx, c->ev_x[0], c->ev_x[1]);
        cudaEventElapsedTime(&ma, c->ev_x[2], c->ev_x[3]);
        c->timing.exchange_steps += 1;
        if (!c->p2p) c->timing.exchange_seconds += mx * 1e-3;  // fused push: no separate exchange
        c->timing.allreduce_seconds += ma * 1e-3;
    }
    rc = resolve(c, st);
    if (rc) return rc;
    c->sel = h.sel;
    c->t = h.t;
    const int warn = c->clamp_any ? (c->smooth ? 3 : 2) : 0;  // K1 + K3 (+ smoothing) fills
    c->warnings_total += warn;
    if (res) {
        res->dt_used = dt;
        res->dt_next = h.dt_next;
        res->guard_warnings = warn;
    }
    return ok_status(st);
}

EXPORT int swe_cuda_compute_dt(swe_ctx* c, double t_end, double* dt, swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "compute_dt: no state loaded");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    unsigned long long sc[SCAN_N];
    int rc = run_scan(c, c->sel, sc, st);
    if (rc) return rc;
    if (sc[SCAN_BAD]) {
        const unsigned long long idx = ~sc[SCAN_BAD];
        return set_status(st, SWE_ERR_INSTABILITY, static_cast<int>(idx % c->g.nx), static_cast<int>(idx / c->g.nx),
                          c->t, "compute_dt: non-finite wave speed");
    }
    const double core = scan_core(c, sc);
    const double dt_raw = std_min(c->pol.cfl * core, c->pol.dt_max);  // timestep.hpp:170-177
    if (dt_raw < c->pol.dt_min) {
        int r = set_status(st, SWE_ERR_STEP_COLLAPSE, -1, -1, c->t,
                           "compute_dt: step size %f collapsed below dt_min %f", dt_raw, c->pol.dt_min);
        if (st) st->dt = dt_raw;
        return r;
    }
    *dt = std_min(dt_raw, t_end - c->t);
    return ok_status(st);
}

EXPORT int swe_cuda_guard(swe_ctx* c, swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "guard: no state loaded");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    unsigned long long sc[SCAN_N];
    int rc = run_scan(c, c->sel, sc, st, false);
    if (rc) return rc;
    if (!sc[SCAN_GUARD]) return ok_status(st);
    const unsigned long long idx = ~sc[SCAN_GUARD];
    double vh, vqx, vqy;
    cell_values(c, c->sel, idx, &vh, &vqx, &vqy);
    const int i = static_cast<int>(idx % c->g.nx), j = static_cast<int>(idx / c->g.nx);
    int r = set_status(st, SWE_ERR_INSTABILITY, i, j, c->t, "cell (%d, %d) at t=%f: h=%f qx=%f qy=%f", i, j, c->t,
                       vh, vqx, vqy);
    if (st) {
        st->h = vh;
        st->qx = vqx;
        st->qy = vqy;
    }
    return r;
}

EXPORT int swe_cuda_advance(swe_ctx* c, double t_end, uint64_t step_index0, double dt_first,
                            uint64_t max_steps, swe_run_result* res, swe_status* st) {
    return swe_cuda_advance_marked(c, t_end, std::numeric_limits<double>::infinity(), step_index0, dt_first,
                                   max_steps, res, st);
}

EXPORT int swe_cuda_advance_marked(swe_ctx* c, double t_end, double t_mark, uint64_t step_index0,
                                   double dt_first, uint64_t max_steps, swe_run_result* res, swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "advance: no state loaded");
    if (!is_fin(t_end)) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "advance: t_end must be finite");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    std::memset(res, 0, sizeof *res);
    res->step_index = step_index0;
    res->t_final = c->t;
    double dt_raw = 0.0;
    if (is_fin(dt_first)) {
        dt_raw = dt_first;
    } else if (c->t < t_end) {  // run.hpp:125-130
        int rc = swe_cuda_compute_dt(c, std::numeric_limits<double>::infinity(), &dt_raw, st);
        if (rc) return rc;
    }
    res->dt_next = dt_raw;
    SweCtl& h = *c->h_ctl;
    h.mode = 1;
    h.t = c->t;
    h.t_end = t_end;
    h.t_mark = t_mark;
    h.dt_raw = dt_raw;
    h.step_index = step_index0;
    h.steps_done = 0;
    h.sel = c->sel;
    // t_mark stops the run only after a committed step (the device finalize
    // and resolve() test it), like run_from's mark check after each step
    // (run.hpp:159-163): a mark that rounds to <= t still advances one step.
    h.done = !(c->t < t_end);
    h.status = 0;
    h.finish = 0;
    std::memset(h.red, 0, sizeof h.red);
    int rc = write_ctl(c, st);
    if (rc) return rc;
    bool use_graph = !(c->ex.flags & SWE_EXEC_NO_GRAPH) && (!c->tr || c->tr->capturable()) && !c->graph_failed;
    // small grids, one rank, no early exit: many steps per cooperative launch
    // (swe_multi_kernel) instead of one launch per step
    const int v_multi = swe_step_variant(true, c->smooth, c->flat, c->manning, false, c->xonly);
    const bool use_multi = c->multi_ok && c->ex.nranks == 1 && !c->prm.early;
    // one batch = the chunks covering the steps still to run (64 at a time
    // when the run is bounded only by t_end / t_mark), launched back to back
    // without a host sync; launches after a halting step are device no-ops
    auto batch_of = [&](uint64_t launched) {
        if (!max_steps) return std::vector<int>{64};
        return chunk_plan(max_steps - launched);
    };
    if (use_graph && !use_multi) {  // build the first batch's graphs before the timed region
        uint64_t par = h.step_index, sl = static_cast<uint64_t>(h.sel);
        for (int n : batch_of(0)) {
            swe_ctx::Graph* g;
            rc = get_graph(c, n, static_cast<int>(par % 2), static_cast<int>(sl % 2), &g, st);
            if (rc == kGraphUnavailable) {
                use_graph = false;
                break;
            }
            if (rc) return rc;
            par += n;
            sl += n;
        }
    }
    uint64_t launched = 0;
    unsigned long long committed_before = 0;
    int rc_final = SWE_OK;
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    while (true) {
        if (h.done) break;
        if (max_steps && launched >= max_steps) break;
        uint64_t par = h.step_index, sl = static_cast<uint64_t>(h.sel);
        if (use_multi) {
            const uint64_t left = max_steps ? max_steps - launched : 4096;
            const int n = static_cast<int>(std::min<uint64_t>(left, 4096));
            CUDA_TRY(cudaMemsetAsync(&c->d_ctl->mwork[0], 0,
                                     sizeof(SweCtl) - offsetof(SweCtl, mwork), c->stream));
            StepParams pm = c->prm;  // the multi-step launch's own item height
            pm.chunk = pm.chunk2 = c->multi_chunk;
            pm.nchunks = pm.tier_rc = c->multi_nchunks;
            CUDA_TRY(swe_launch_multi(c->exact, c->smooth, v_multi, c->ncta_multi, c->stream, pm, n));
            c->launches += 1;
        }
        for (int n : use_multi ? std::vector<int>{} : batch_of(launched)) {
            swe_ctx::Graph* g = nullptr;
            if (use_graph) {
                rc = get_graph(c, n, static_cast<int>(par % 2), static_cast<int>(sl % 2), &g, st);
                if (rc == kGraphUnavailable) use_graph = false;
                else if (rc) return rc;
            }
            if (use_graph) {
                CUDA_TRY(cudaGraphLaunch(g->exec, c->stream));
                c->launches += g->kernels;
            } else {
                for (int k = 0; k < n; ++k) {
                    rc = enqueue_step(c, ((par + k) % 2) == 0, static_cast<int>((sl + k + 1) & 1), st);
                    if (rc) return rc;
                }
            }
            par += n;
            sl += n;
        }
        rc = read_ctl(c, st);
        if (rc) return rc;
        // keep the host mirror of the committed selector/time in sync
        c->sel = h.sel;
        c->t = h.t;
        if (h.status != SWE_OK) {
            rc = resolve(c, st);
            c->sel = h.sel;
            c->t = h.t;
            if (rc) {
                rc_final = rc;
                break;
            }
            // diagnosis committed the step on the host: continue the run
            h.status = SWE_OK;
            if (!h.done) {
                rc = write_ctl(c, st);
                if (rc) return rc;
            }
        }
        // launches after a halted step were no-ops: count committed steps
        launched = h.steps_done;
    }
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->timing.steps += h.steps_done - committed_before;
    c->timing.step_seconds += ms * 1e-3;
    c->sel = h.sel;
    c->t = h.t;
    const int warn = c->clamp_any ? (c->smooth ? 3 : 2) : 0;
    res->steps = h.steps_done;
    res->step_index = h.step_index;
    res->t_final = h.t;
    res->dt_next = h.dt_raw;
    res->guard_warnings = static_cast<int32_t>(warn * h.steps_done);
    c->warnings_total += res->guard_warnings;
    if (rc_final) return rc_final;
    return ok_status(st);
}

EXPORT int swe_cuda_selftest_div(const double* a, const double* b, size_t n, int exact, double* out,
                                  swe_status* st) {
    double *da = nullptr, *db = nullptr, *dout = nullptr;
    CUDA_TRY(cudaMalloc(&da, n * 8 + 8));
    CUDA_TRY(cudaMalloc(&db, n * 8 + 8));
    CUDA_TRY(cudaMalloc(&dout, n * 8 + 8));
    CUDA_TRY(cudaMemcpy(da, a, n * 8, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(db, b, n * 8, cudaMemcpyHostToDevice));
    selftest_div_kernel<<<148 * 8, 256>>>(da, db, n, exact, dout);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out, dout, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(da);
    cudaFree(db);
    cudaFree(dout);
    return ok_status(st);
}

EXPORT int swe_cuda_debug_guard_check(uint64_t* corrupted_bytes, uint64_t* allocations, swe_status* st) {
#if SWE_CHECKED
    std::vector<unsigned char> g(kGuard);
    uint64_t bad = 0;
    std::lock_guard<std::mutex> lk(g_alloc_m);
    for (auto& kv : g_allocs) {
        char* base = kv.second.first;
        for (char* band : {base, base + kGuard + kv.second.second}) {
            CUDA_TRY(cudaMemcpy(g.data(), band, kGuard, cudaMemcpyDeviceToHost));
            for (unsigned char b : g) bad += (b != kGuardByte);
        }
    }
    *corrupted_bytes = bad;
    *allocations = g_allocs.size();
    return ok_status(st);
#else
    (void)corrupted_bytes;
    (void)allocations;
    return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "debug_guard_check: library built without SWE_CHECKED");
#endif
}

EXPORT double swe_cuda_time(const swe_ctx* c) { return c ? c->t : 0.0; }
EXPORT int32_t swe_cuda_guard_warnings(const swe_ctx* c) { return c ? c->warnings_total : 0; }
EXPORT int swe_cuda_timing(const swe_ctx* c, swe_timing* out) {
    if (!c || !out) return SWE_ERR_CONFIG;
    *out = c->timing;
    return SWE_OK;
}
EXPORT int swe_cuda_accounting(const swe_ctx* c, swe_accounting* out) {
    if (!c || !out) return SWE_ERR_CONFIG;
    std::memset(out, 0, sizeof *out);
    const int nb = (c->ex.rank > 0 ? 1 : 0) + (c->ex.rank + 1 < c->ex.nranks ? 1 : 0);
    out->halo_values_exchanged = static_cast<int64_t>(nb) * c->R * 3 * c->g.nx;
    if (c->loaded) {  // each work item's march starts R rows early and ends R rows late
        const int items_per_column = c->overlap ? c->prm_int.nchunks + c->prm_edge.nchunks : c->prm.nchunks;
        out->redundant_star_rows = items_per_column * 2 * c->R;
        out->redundant_corrector_rows = items_per_column * 2 * (c->R - 1);
    }
    return SWE_OK;
}

EXPORT void swe_cuda_rows(const swe_ctx* c, int32_t* row_begin, int32_t* row_end) {
    if (row_begin) *row_begin = c ? c->j0 : 0;
    if (row_end) *row_end = c ? c->j0 + c->nloc : 0;
}
EXPORT int swe_cuda_activity(swe_ctx* c, swe_activity* out) {
    swe_status* st = nullptr;
    if (!c || !out) return SWE_ERR_CONFIG;
    std::memset(out, 0, sizeof *out);
    if (!c->loaded) return SWE_OK;
    CUDA_TRY(cudaSetDevice(c->ex.device));
    unsigned long long v[4];
    CUDA_TRY(cudaMemcpyAsync(v, c->d_stats, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    out->cells_per_step = static_cast<uint64_t>(c->nloc) * c->g.nx;
    out->items_per_step = static_cast<uint64_t>(c->ntiles) * c->prm.nchunks;
    out->eligible_items = v[1];
    out->skipped_cells = v[0];
    return SWE_OK;
}
EXPORT int32_t swe_cuda_halo_rows(const swe_ctx* c) { return c ? c->R : 0; }
EXPORT int swe_cuda_state_digest(swe_ctx* c, uint64_t* digest, swe_status* st) {
    if (!c || !c->loaded) return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "state_digest: no state loaded");
    CUDA_TRY(cudaSetDevice(c->ex.device));
    CUDA_TRY(cudaMemsetAsync(c->d_scan, 0, sizeof(unsigned long long), c->stream));
    digest_kernel<<<std::max(1, std::min(c->nloc, 148 * 8)), 256, 0, c->stream>>>(
        c->d_buf[c->sel], c->pitch, c->R, c->g.nx, c->nloc, c->j0, c->d_scan);
    CUDA_TRY(cudaGetLastError());
    unsigned long long v = 0;
    CUDA_TRY(cudaMemcpyAsync(&v, c->d_scan, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *digest = v;
    return ok_status(st);
}
EXPORT uint64_t swe_cuda_launch_count(const swe_ctx* c) { return c ? c->launches : 0; }
