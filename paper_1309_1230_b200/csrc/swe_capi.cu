// swe_capi.cu — host runtime behind include/swe_cuda.h (libswe_cuda.so).
//
// Owns the device state of one swe::Stepper replacement (executor.hpp:726-1116):
// ping-pong padded buffers, bed slopes, the device control block, CUDA graphs
// for the device-resident run loop, and (for row strips) the NCCL
// communicator.  Compiled with -fmad=false like the kernels.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nccl.h>

#include "swe_device.cuh"
#include "swe_launch.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& err) {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            err = "cannot dlopen libnccl.so.2";
            return false;
        }
#define SWE_SYM(f) f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f))
        SWE_SYM(GetUniqueId);
        SWE_SYM(CommInitRank);
        SWE_SYM(CommDestroy);
        SWE_SYM(AllReduce);
        SWE_SYM(Send);
        SWE_SYM(Recv);
        SWE_SYM(GroupStart);
        SWE_SYM(GroupEnd);
        SWE_SYM(GetErrorString);
#undef SWE_SYM
        if (!GetUniqueId || !CommInitRank || !AllReduce || !Send || !Recv || !GroupStart ||
            !GroupEnd) {
            err = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;

// ---------------------------------------------------------------- aux kernels
using swe_dev::CellVec;

__device__ __forceinline__ size_t pidx(int P, int R, int lr, int f, int i) {
    return (static_cast<size_t>(lr + R) * 3 + f) * P + static_cast<size_t>(i + R);
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
                              int j0, int ny, double two_dx, double two_dy, unsigned* flags) {
    const int rows = nloc + 2 * R;
    const size_t n = static_cast<size_t>(rows) * nx;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int lr = static_cast<int>(k / nx) - R;
        const int i = static_cast<int>(k % nx);
        const int j = j0 + lr;
        double sx = 0.0, sy = 0.0;
        if (j >= 0 && j < ny) {
            auto zat = [&](int ii, int jj) {
                return zp[static_cast<size_t>(jj - j0 + R + 1) * nx + ii];
            };
            const int iw = max(i - 1, 0), ie = min(i + 1, nx - 1);
            const int js = max(j - 1, 0), jn = min(j + 1, ny - 1);
            sx = (zat(ie, j) - zat(iw, j)) / two_dx;
            sy = (zat(i, jn) - zat(i, js)) / two_dy;
            if (swe_dev::dbits(sx) != 0ull || swe_dev::dbits(sy) != 0ull) atomicOr(flags, 1u);
            if (swe_dev::dbits(sy) != 0ull) atomicOr(flags + 2, 1u);
        }
        slope[(static_cast<size_t>(lr + R) * 2 + 0) * P + (i + R)] = sx;
        slope[(static_cast<size_t>(lr + R) * 2 + 1) * P + (i + R)] = sy;
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
            const size_t o = (static_cast<size_t>(lr + R) * 2) * P + (i + R);
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

struct BcSet {
    SweBC bc[4];  // N, S, E, W
};

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

// Scan words (max-combined, like the step reduction).
enum { SCAN_BAD = 0, SCAN_MINR = 1, SCAN_GUARD = 2, SCAN_N = 4 };

// K6 exact per-cell scan (timestep.hpp:83-105 / executor.hpp:560-580) and K5
// guard (timestep.hpp:64-78) over own rows of buffer b.
__global__ void scan_kernel(const double* b, int P, int R, int nx, int nloc, int j0, double g,
                            double dx, double dy, double h_min, unsigned long long* out) {
    const size_t n = static_cast<size_t>(nloc) * nx;
    unsigned long long bad = 0, minr = 0, guard = 0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int lr = static_cast<int>(k / nx), i = static_cast<int>(k % nx);
        const double h = b[pidx(P, R, lr, 0, i)], qx = b[pidx(P, R, lr, 1, i)],
                     qy = b[pidx(P, R, lr, 2, i)];
        const unsigned long long idx = static_cast<unsigned long long>(j0 + lr) * nx + i;
        const bool ok = swe_dev::finite_d(h) && swe_dev::finite_d(qx) && swe_dev::finite_d(qy) &&
                        h >= h_min;
        if (!ok) guard = max(guard, ~idx);
        const double c = __dsqrt_rn(g * h);
        const double sx = fabs(__ddiv_rn(qx, h)) + c;
        const double sy = fabs(__ddiv_rn(qy, h)) + c;
        const double r = swe_dev::std_min(__ddiv_rn(dx, sx), __ddiv_rn(dy, sy));
        if (!(r > 0.0) || !swe_dev::finite_d(r)) {
            bad = max(bad, ~idx);
            continue;
        }
        minr = max(minr, ~swe_dev::dbits(r));
    }
    for (int o = 16; o > 0; o >>= 1) {
        bad = max(bad, __shfl_xor_sync(0xffffffffu, bad, o));
        minr = max(minr, __shfl_xor_sync(0xffffffffu, minr, o));
        guard = max(guard, __shfl_xor_sync(0xffffffffu, guard, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicMax(&out[SCAN_BAD], bad);
        if (minr) atomicMax(&out[SCAN_MINR], minr);
        if (guard) atomicMax(&out[SCAN_GUARD], guard);
    }
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// 2D map over field_rows rows of P doubles at row_stride doubles (P if 0); box
// box_cols x box_rows
bool encode_rows(CUtensorMap* map, double* base, int P, long long field_rows, int box_rows, std::string& err,
                 int box_cols = 32, int row_stride = 0) {
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

// Shared-reciprocal division of the step kernels (swe_device.cuh), exposed for
// the parity self-test.  Compiled with -fmad=false like the exact kernels.
__global__ void selftest_div_kernel(const double* a, const double* b, size_t n, int exact, double* out) {
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (exact) {
            const swe_dev::Recip rc = swe_dev::make_recip(b[k]);
            out[k] = swe_dev::div_rn(a[k], rc);
        } else {
            out[k] = a[k] * swe_dev::make_recip_fast(b[k]).y;
        }
    }
}

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

// ---------------------------------------------------------------- context
namespace {
struct Transport;
}
struct swe_ctx {
    swe_grid g{};
    swe_physics ph{};
    swe_policy pol{};
    swe_boundary_set bnd{};
    swe_exec ex{};
    int R = 1, nloc = 0, j0 = 0, pitch = 0, ntiles = 0;
    bool smooth = false, manning = false, flat = true, xonly = false, loaded = false, exact = true;
    int clamp_any = 0;
    int warnings_total = 0;
    double t = 0.0;
    int sel = 0;
    size_t buf_doubles = 0;
    double* d_buf[2] = {nullptr, nullptr};
    double* d_slope = nullptr;
    double *d_zw = nullptr, *d_ze = nullptr, *d_zs = nullptr, *d_zn = nullptr;
    unsigned long long* d_scan = nullptr;
    unsigned* d_flags = nullptr;
    // early exit: quiet flags per buffer, eligibility, per-item flat bits,
    // counters {skipped cells, eligible items}
    unsigned long long* d_qflag = nullptr;
    unsigned char* d_elig = nullptr;
    unsigned* d_active = nullptr;
    unsigned char* d_iflat = nullptr;
    unsigned long long* d_stats = nullptr;
    int nitems_alloc = 0;
    bool early = false;
    SweCtl* d_ctl = nullptr;
    SweCtl* h_ctl = nullptr;  // pinned mirror
    double* d_zp = nullptr;  // bed rows [-R-1, nloc+R+1) (compact, nx per row, strip halos): state() z, slopes
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    StepParams prm{};
    int ncta = 0;
    int occ = 1;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int graph_len = 0;
    unsigned long long graph_kernels = 0;  // our kernels in one captured graph
    Transport* tr = nullptr;  // row-strip collectives (NCCL or local group); null for one rank
    unsigned long long* d_xr = nullptr;  // local-group allreduce scratch
    // strips: halo exchange overlapped with the interior (edge + interior launches)
    bool overlap = false;
    StepParams prm_edge{}, prm_int{};
    int ncta_edge = 0;
    cudaStream_t stream_edge = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    unsigned long long launches = 0;
    swe_timing timing{};
    double tz_x = 0, tz_y = 0;
    int always_diag = 0;
};

namespace {

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

#define CUDA_TRY(x)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "CUDA error %s at %s:%d",        \
                              cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

#define NCCL_TRY(x)                                                                              \
    do {                                                                                         \
        ncclResult_t r_ = (x);                                                                   \
        if (r_ != ncclSuccess)                                                                   \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "NCCL error %d at %s:%d",        \
                              static_cast<int>(r_), __FILE__, __LINE__);                         \
    } while (0)

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

// ---------------------------------------------------------------- strip transport
// The row-strip protocol needs two collectives: an
// unsigned-max allreduce of the reduction words (error indices are stored
// complemented, so max = row-major first offender; non-negative doubles order
// like their bit patterns) and a send/recv of R halo rows with each strip
// neighbour.  Between GPUs NCCL carries them over NVLink.  The local group
// carries them between contexts of one process on one device (one host thread
// per rank, ordered by CUDA events, no kernel ever waits on another rank's):
// it lets the GPU tests check the whole strip path bit for bit on one B200.
struct Transport {
    virtual ~Transport() = default;
    virtual int allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) = 0;
    // send_up -> (rank+1).recv_down, send_down -> (rank-1).recv_up, `bytes` each;
    // null pointers where the neighbour does not exist
    virtual int sendrecv(swe_ctx* c, cudaStream_t s, const void* send_up, void* recv_up, const void* send_down,
                         void* recv_down, size_t bytes, swe_status* st) = 0;
    virtual bool capturable() const = 0;  // may be recorded into a CUDA graph
};

struct NcclTransport final : Transport {
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm && g_nccl.CommDestroy) g_nccl.CommDestroy(comm);
    }
    int allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) override;
    int sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd, size_t bytes,
                 swe_status* st) override;
    bool capturable() const override { return true; }
};

constexpr int kMaxLocalRanks = 16;
struct RedPtrs {
    const unsigned long long* p[kMaxLocalRanks];
};
__global__ void max_reduce_kernel(RedPtrs in, int nranks, int n, unsigned long long* out) {
    const int k = threadIdx.x;
    if (k >= n) return;
    unsigned long long m = 0ull;
    for (int r = 0; r < nranks; ++r) m = max(m, in.p[r][k]);
    out[k] = m;
}

struct LocalGroup {
    std::mutex m;
    std::condition_variable cv;
    int n = 0, arrived = 0, refs = 0;
    unsigned long long gen = 0;
    bool broken = false;
    cudaEvent_t ready[kMaxLocalRanks] = {}, done[kMaxLocalRanks] = {};
    const void* su[kMaxLocalRanks] = {};
    const void* sd[kMaxLocalRanks] = {};
    const unsigned long long* red[kMaxLocalRanks] = {};
    // all ranks arrive (or a 120 s timeout breaks the group, so a failing
    // test cannot hang the box)
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) return false;
        const unsigned long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; })) broken = true;
        if (broken) {
            cv.notify_all();
            return false;
        }
        return true;
    }
};
std::mutex g_groups_m;
std::map<std::string, LocalGroup*> g_groups;

struct LocalTransport final : Transport {
    LocalGroup* grp = nullptr;
    std::string key;
    int rank = 0;
    ~LocalTransport() override {
        std::lock_guard<std::mutex> lk(g_groups_m);
        if (grp && --grp->refs == 0) {
            for (int r = 0; r < grp->n; ++r) {
                if (grp->ready[r]) cudaEventDestroy(grp->ready[r]);
                if (grp->done[r]) cudaEventDestroy(grp->done[r]);
            }
            g_groups.erase(key);
            delete grp;
        }
    }
    int allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) override;
    int sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd, size_t bytes,
                 swe_status* st) override;
    bool capturable() const override { return false; }
};

double* row_ptr(swe_ctx* c, int which, int lr) {
    return c->d_buf[which] + static_cast<size_t>(lr + c->R) * 3 * c->pitch;
}

int NcclTransport::allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) {
    (void)c;
    NCCL_TRY(g_nccl.AllReduce(d, d, static_cast<size_t>(n), ncclUint64, ncclMax, comm, s));
    return SWE_OK;
}

int NcclTransport::sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd,
                            size_t bytes, swe_status* st) {
    const int rk = c->ex.rank;
    NCCL_TRY(g_nccl.GroupStart());
    if (su) NCCL_TRY(g_nccl.Send(su, bytes, ncclUint8, rk + 1, comm, s));
    if (ru) NCCL_TRY(g_nccl.Recv(ru, bytes, ncclUint8, rk + 1, comm, s));
    if (sd) NCCL_TRY(g_nccl.Send(sd, bytes, ncclUint8, rk - 1, comm, s));
    if (rd) NCCL_TRY(g_nccl.Recv(rd, bytes, ncclUint8, rk - 1, comm, s));
    NCCL_TRY(g_nccl.GroupEnd());
    return SWE_OK;
}

#define GROUP_SYNC()                                                                                   \
    do {                                                                                               \
        if (!grp->barrier())                                                                           \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "local strip group: a rank timed out"); \
    } while (0)

// post -> barrier -> read the neighbours' posts -> barrier -> wait for the
// neighbours' reads before the posted rows may change again
int LocalTransport::sendrecv(swe_ctx* c, cudaStream_t s, const void* su, void* ru, const void* sd, void* rd,
                             size_t bytes, swe_status* st) {
    (void)c;
    const int r = rank, n = grp->n;
    grp->su[r] = su;
    grp->sd[r] = sd;
    CUDA_TRY(cudaEventRecord(grp->ready[r], s));
    GROUP_SYNC();
    if (ru && r + 1 < n) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[r + 1], 0));
        CUDA_TRY(cudaMemcpyAsync(ru, grp->sd[r + 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (rd && r > 0) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[r - 1], 0));
        CUDA_TRY(cudaMemcpyAsync(rd, grp->su[r - 1], bytes, cudaMemcpyDeviceToDevice, s));
    }
    CUDA_TRY(cudaEventRecord(grp->done[r], s));
    GROUP_SYNC();
    if (r + 1 < n) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[r + 1], 0));
    if (r > 0) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[r - 1], 0));
    return SWE_OK;
}

int LocalTransport::allreduce_max(swe_ctx* c, cudaStream_t s, unsigned long long* d, int n, swe_status* st) {
    const int r = rank, nr = grp->n;
    grp->red[r] = d;
    CUDA_TRY(cudaEventRecord(grp->ready[r], s));
    GROUP_SYNC();
    RedPtrs in{};
    for (int k = 0; k < nr; ++k) {
        CUDA_TRY(cudaStreamWaitEvent(s, grp->ready[k], 0));
        in.p[k] = grp->red[k];
    }
    max_reduce_kernel<<<1, 32, 0, s>>>(in, nr, n, c->d_xr);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(grp->done[r], s));
    GROUP_SYNC();
    for (int k = 0; k < nr; ++k) CUDA_TRY(cudaStreamWaitEvent(s, grp->done[k], 0));
    CUDA_TRY(cudaMemcpyAsync(d, c->d_xr, static_cast<size_t>(n) * sizeof(unsigned long long),
                             cudaMemcpyDeviceToDevice, s));
    return SWE_OK;
}
#undef GROUP_SYNC

// Exchange R committed rows with the strip neighbours:
// own top rows -> rank+1's lower halo, own bottom rows -> rank-1's upper halo.
int halo_exchange(swe_ctx* c, int which, cudaStream_t s, swe_status* st) {
    if (c->ex.nranks <= 1) return SWE_OK;
    const size_t bytes = static_cast<size_t>(c->R) * 3 * c->pitch * sizeof(double);
    const int rk = c->ex.rank, nr = c->ex.nranks;
    const bool up = rk + 1 < nr, down = rk > 0;
    return c->tr->sendrecv(c, s, up ? row_ptr(c, which, c->nloc - c->R) : nullptr,
                           up ? row_ptr(c, which, c->nloc) : nullptr, down ? row_ptr(c, which, 0) : nullptr,
                           down ? row_ptr(c, which, -c->R) : nullptr, bytes, st);
}

// Enqueue one step on the stream (no host sync).  `fwd` = sweep parity,
// `cand` = candidate buffer as assumed by the host (used for the strip halo
// exchange only).
int enqueue_step(swe_ctx* c, bool fwd, int cand, swe_status* st) {
    const int v = swe_step_variant(fwd, c->smooth, c->flat, c->manning, c->early, c->xonly);
    if (c->overlap) {
        // Strips, overlapped: the edge launch (the bands whose rows the
        // neighbours need) runs on a high-priority stream and its halo
        // send/recv follows it there, while the interior launch runs on the
        // main stream; the allreduce and the finalize wait for both.
        CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->stream_edge, c->ev_fork, 0));
        CUDA_TRY(swe_launch_step(c->exact, v, c->ncta_edge, c->stream_edge, c->prm_edge));
        int rc = halo_exchange(c, cand, c->stream_edge, st);
        if (rc) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_join, c->stream_edge));
        CUDA_TRY(swe_launch_step(c->exact, v, c->ncta, c->stream, c->prm_int));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        rc = c->tr->allreduce_max(c, c->stream, c->d_ctl->red, RED_N, st);
        if (rc) return rc;
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
        int rc = halo_exchange(c, cand, c->stream, st);
        if (rc) return rc;
        rc = c->tr->allreduce_max(c, c->stream, c->d_ctl->red, RED_N, st);
        if (rc) return rc;
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

// Run the exact scan over own rows of buffer `which`; results all-reduced.
int run_scan(swe_ctx* c, int which, unsigned long long out[SCAN_N], swe_status* st) {
    CUDA_TRY(cudaMemsetAsync(c->d_scan, 0, SCAN_N * sizeof(unsigned long long), c->stream));
    const size_t n = static_cast<size_t>(c->nloc) * c->g.nx;
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16));
    scan_kernel<<<std::max(blocks, 1), 256, 0, c->stream>>>(c->d_buf[which], c->pitch, c->R, c->g.nx,
                                                            c->nloc, c->j0, c->ph.g, c->g.dx, c->g.dy,
                                                            c->pol.h_min, c->d_scan);
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

// Values of global cell idx from buffer `which` (the owning rank answers;
// others return NaN).
void cell_values(swe_ctx* c, int which, unsigned long long idx, double* h, double* qx, double* qy) {
    const int j = static_cast<int>(idx / c->g.nx), i = static_cast<int>(idx % c->g.nx);
    *h = *qx = *qy = std::numeric_limits<double>::quiet_NaN();
    const int lr = j - c->j0;
    if (lr < 0 || lr >= c->nloc) return;
    double v[3];
    for (int f = 0; f < 3; ++f)
        cudaMemcpy(&v[f], c->d_buf[which] + (static_cast<size_t>(lr + c->R) * 3 + f) * c->pitch + (i + c->R), 8,
                   cudaMemcpyDeviceToHost);
    *h = v[0];
    *qx = v[1];
    *qy = v[2];
}

// Translate the control block after a launch into the reference's outcome.
// Returns SWE_OK (committed), an error, or resolves a diagnosis request.
int resolve(swe_ctx* c, swe_status* st) {
    SweCtl& h = *c->h_ctl;
    if (h.status == SWE_OK) return SWE_OK;
    if (h.status == SWE_STATUS_DIAG) {
        // Exact per-cell CFL scan of the candidate (executor.hpp:560-580).
        const int cand = h.sel ^ 1;
        unsigned long long sc[SCAN_N];
        int rc = run_scan(c, cand, sc, st);
        if (rc) return rc;
        if (sc[SCAN_BAD]) {
            const unsigned long long idx = ~sc[SCAN_BAD];
            h.status = SWE_ERR_INSTABILITY;
            h.done = 1;
            write_ctl(c, st);
            return set_status(st, SWE_ERR_INSTABILITY, static_cast<int>(idx % c->g.nx),
                              static_cast<int>(idx / c->g.nx), h.t_commit,
                              "non-finite wave speed in dt reduction");
        }
        const unsigned long long b = ~sc[SCAN_MINR];
        double core;
        std::memcpy(&core, &b, 8);
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
        if (h.err_kind == 4)
            return set_status(st, SWE_ERR_INSTABILITY, h.err_i, h.err_j, h.err_t,
                              "predicted depth below dry threshold at cell (%d, %d)", h.err_i, h.err_j);
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
    for (auto& gph : c->graph)
        if (gph) {
            cudaGraphExecDestroy(gph);
            gph = nullptr;
        }
    c->graph_len = 0;
    return 0;
}

int build_graphs(swe_ctx* c, int len, swe_status* st) {
    destroy_graphs(c);
    const unsigned long long before = c->launches;
    for (int start = 0; start < 2; ++start) {  // start 0: first launch forward
        cudaGraph_t gph;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int rc = SWE_OK;
        for (int k = 0; k < len && rc == SWE_OK; ++k) {
            const bool fwd = ((start + k) % 2) == 0;
            rc = enqueue_step(c, fwd, (k + 1) & 1, st);  // candidate relative to sel: see advance()
        }
        cudaError_t e = cudaStreamEndCapture(c->stream, &gph);
        if (rc) return rc;
        CUDA_TRY(e);
        CUDA_TRY(cudaGraphInstantiate(&c->graph[start], gph, 0));
        cudaGraphDestroy(gph);
    }
    c->graph_kernels = (c->launches - before) / 2;  // our kernels per graph launch
    c->launches = before;                          // captured, not launched
    c->graph_len = len;
    return SWE_OK;
}

}  // namespace

// ======================================================================= API

EXPORT const char* swe_cuda_version(void) { return "swe-b200 1.0 (sm_100a, ABI 1)"; }

EXPORT int swe_cuda_nccl_unique_id(void* out, swe_status* st) {
    std::string err;
    if (!g_nccl.load(err)) return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
    ncclUniqueId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
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
    if (grid->ny < ex.nranks)
        return set_status(st, SWE_ERR_CONFIG, -1, -1, 0,
                          "partition_scanlines: %d workers need at least as many rows, grid has %d", ex.nranks,
                          grid->ny);
    auto bands = partition_scanlines(grid->ny, ex.nranks);
    if (ex.nranks > 1)
        for (auto& b : bands)
            if (b.second - b.first < 4)
                return set_status(st, SWE_ERR_CONFIG, -1, -1, 0,
                                  "executor: decomposed bands need at least 4 rows; %d workers on %d rows "
                                  "leaves a band with %d",
                                  ex.nranks, grid->ny, b.second - b.first);
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
    c->j0 = bands[ex.rank].first;
    c->nloc = bands[ex.rank].second - bands[ex.rank].first;
    const int out_w = SWE_TILE_W(c->R);
    c->ntiles = (grid->nx + out_w - 1) / out_w;
    c->pitch = ((c->ntiles * out_w + 2 * c->R + 32) + 31) / 32 * 32;
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
    }
    CUDA_TRY(cudaEventCreate(&c->ev0));
    CUDA_TRY(cudaEventCreate(&c->ev1));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(cudaMalloc(&c->d_buf[k], c->buf_doubles * sizeof(double)));
        fill_benign_kernel<<<148 * 8, 256, 0, c->stream>>>(c->d_buf[k], rows * 3, c->pitch);
        CUDA_TRY(cudaGetLastError());
    }
    const size_t zrows = rows;
    CUDA_TRY(cudaMalloc(&c->d_zw, zrows * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->d_ze, zrows * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->d_zs, grid->nx * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->d_zn, grid->nx * sizeof(double)));
    CUDA_TRY(cudaMalloc(&c->d_zp, static_cast<size_t>(c->nloc + 2 * c->R + 2) * grid->nx * sizeof(double)));
    CUDA_TRY(cudaMemsetAsync(c->d_zw, 0, zrows * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_ze, 0, zrows * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_zs, 0, grid->nx * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_zn, 0, grid->nx * sizeof(double), c->stream));
    CUDA_TRY(cudaMalloc(&c->d_scan, SCAN_N * sizeof(unsigned long long)));
    CUDA_TRY(cudaMalloc(&c->d_flags, 4 * sizeof(unsigned)));
    CUDA_TRY(cudaMalloc(&c->d_stats, 4 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(c->d_stats, 0, 4 * sizeof(unsigned long long), c->stream));
    CUDA_TRY(cudaMalloc(&c->d_ctl, sizeof(SweCtl)));
    CUDA_TRY(cudaMallocHost(&c->h_ctl, sizeof(SweCtl)));
    std::memset(c->h_ctl, 0, sizeof(SweCtl));
    CUDA_TRY(cudaMemcpyAsync(c->d_ctl, c->h_ctl, sizeof(SweCtl), cudaMemcpyHostToDevice, c->stream));

    if (ex.nranks > 1) {
        if (!exec->nccl_id)
            return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: nranks > 1 requires nccl_id");
        CUDA_TRY(cudaMalloc(&c->d_xr, 16 * sizeof(unsigned long long)));
        if (ex.flags & SWE_EXEC_LOCAL_GROUP) {
            if (ex.nranks > kMaxLocalRanks)
                return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: a local group holds at most %d ranks",
                                  kMaxLocalRanks);
            auto* t = new LocalTransport();
            c->tr = t;
            t->key.assign(static_cast<const char*>(exec->nccl_id), SWE_NCCL_ID_BYTES);
            t->rank = ex.rank;
            std::lock_guard<std::mutex> lk(g_groups_m);
            LocalGroup*& g = g_groups[t->key];
            if (!g) {
                g = new LocalGroup();
                g->n = ex.nranks;
            }
            if (g->n != ex.nranks)
                return set_status(st, SWE_ERR_CONFIG, -1, -1, 0, "exec: local group size mismatch");
            ++g->refs;
            t->grp = g;
            CUDA_TRY(cudaEventCreateWithFlags(&g->ready[ex.rank], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&g->done[ex.rank], cudaEventDisableTiming));
        } else {
            std::string err;
            if (!g_nccl.load(err)) return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
            auto* t = new NcclTransport();
            c->tr = t;
            ncclUniqueId id;
            std::memcpy(&id, exec->nccl_id, sizeof id);
            NCCL_TRY(g_nccl.CommInitRank(&t->comm, ex.nranks, id, ex.rank));
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
            if (!encode_rows(&p.tmap_state[k], c->d_buf[k], c->pitch, static_cast<long long>(rows) * 3, 3 * swe_row_group(c->exact), err))
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
    p.ntiles = c->ntiles;
    p.finalize = ex.nranks > 1 ? 0 : 1;
    p.nranks = ex.nranks;
    p.dx = grid->dx;
    p.dy = grid->dy;
    p.g = phys->g;
    p.half_g = 0.5 * phys->g;
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
    cudaFree(c->d_xr);
    for (auto& b : c->d_buf)
        if (b) cudaFree(b);
    cudaFree(c->d_slope);
    cudaFree(c->d_zw);
    cudaFree(c->d_zp);
    cudaFree(c->d_ze);
    cudaFree(c->d_zs);
    cudaFree(c->d_zn);
    cudaFree(c->d_scan);
    cudaFree(c->d_flags);
    cudaFree(c->d_stats);
    cudaFree(c->d_qflag);
    cudaFree(c->d_elig);
    cudaFree(c->d_iflat);
    cudaFree(c->d_active);
    cudaFree(c->d_ctl);
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->stream_edge) cudaStreamDestroy(c->stream_edge);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

namespace {

// Guided chunking: the first ~80 % of a launch's rows go out in `chunk`-row
// items, the rest in quarter-size items, so the dynamic queue ends with short
// items and the last warps finish together.  SWE_GUIDED=0 keeps uniform chunks.
void guided_chunks(StepParams& p, int rows) {
    const char* env = std::getenv("SWE_GUIDED");
    if (env && env[0] == '0') return;
    const int c1 = p.chunk, c2 = std::max(8, c1 / 4);
    if (c1 < 32 || rows < 8 * c1) return;
    const int big = (rows * 4 / 5) / c1;
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
    if (!c->d_slope) CUDA_TRY(cudaMalloc(&c->d_slope, static_cast<size_t>(nloc + 2 * R) * 2 * P * sizeof(double)));
    CUDA_TRY(cudaMemsetAsync(c->d_slope, 0, static_cast<size_t>(nloc + 2 * R) * 2 * P * sizeof(double), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_flags, 0, 4 * sizeof(unsigned), c->stream));
    slopes_kernel<<<148 * 4, 256, 0, c->stream>>>(d_zp, c->d_slope, P, R, nx, nloc, c->j0, c->g.ny,
                                                   2.0 * c->g.dx, 2.0 * c->g.dy, c->d_flags);
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
                             err))
                return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        if (!encode_rows(&c->prm.tmap_slope, c->d_slope, P, static_cast<long long>(nloc + 2 * R) * 2, 2 * G, err))
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0, "%s", err.c_str());
        if (!encode_rows(&c->prm.tmap_slopex, c->d_slope, P, static_cast<long long>(nloc + 2 * R), G, err, 32, 2 * P))
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
    // persistent grid: every resident warp is a worker; small grids keep at
    // least 4 rows per worker so the 2R warm-up rows stay amortised
    const long long units = static_cast<long long>(c->ntiles) * nloc;
    const long long want = std::max<long long>(1, units / (4 * SWE_STEP_WPB));
    long long ncta = std::min<long long>(static_cast<long long>(c->occ) * nsm, want);
    // every worker must span at most 7 tiles (MAXSEG = 8 segments)
    ncta = std::max<long long>(ncta, (c->ntiles + 7 * SWE_STEP_WPB - 1) / (7 * SWE_STEP_WPB));
    c->ncta = static_cast<int>(ncta);
    c->prm.ncta = c->ncta;
    // dynamic work items: ~16 per worker, 16..128 rows each
    {
        const long long workers = ncta * SWE_STEP_WPB;
        long long ch = units / std::max<long long>(1, workers * 16);
        if (ch >= 16) {
            ch = std::min<long long>(128, ch);
        } else {
            // small grids are latency-bound: the shortest items (>= 4 rows) that
            // still give every worker at most one item (512^2: 28 -> 20 us/step)
            ch = std::max<long long>(4, std::min<long long>(16, (units + workers - 1) / workers));
        }
        // early exit: finer items (32 rows) so the active band is balanced
        // across workers and skipped at a finer grain
        if (c->early && c->flat) ch = 32;
        ch = std::min<long long>(ch, nloc);
        c->prm.chunk = static_cast<int>(ch);
        c->prm.nchunks = static_cast<int>((nloc + ch - 1) / ch);
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
            cudaFree(c->d_qflag);
            cudaFree(c->d_elig);
            cudaFree(c->d_iflat);
            cudaFree(c->d_active);
            c->d_qflag = nullptr;
            c->d_elig = c->d_iflat = nullptr;
            c->d_active = nullptr;
            CUDA_TRY(cudaMalloc(&c->d_active, static_cast<size_t>(nitems) * sizeof(unsigned)));
            CUDA_TRY(cudaMalloc(&c->d_qflag, 2 * static_cast<size_t>(nitems) * sizeof(unsigned long long)));
            CUDA_TRY(cudaMalloc(&c->d_elig, nitems));
            CUDA_TRY(cudaMalloc(&c->d_iflat, nitems));
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
    c->overlap = c->ex.nranks > 1 && !(c->early && c->flat) && nloc >= 2 * kEdge + 16;
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
        double* dst = c->d_buf[0] + (static_cast<size_t>(R) * 3 + f) * P + R;
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
    rc = run_scan(c, 0, sc, st);
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
        const double* src = c->d_buf[c->sel] + (static_cast<size_t>(R) * 3 + f) * P + R;
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
    rc = enqueue_step(c, fwd, c->sel ^ 1, st);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    rc = read_ctl(c, st);
    if (rc) return rc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    c->timing.steps += 1;
    c->timing.step_seconds += ms * 1e-3;
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
    double core = std::numeric_limits<double>::infinity();
    if (sc[SCAN_MINR]) {
        const unsigned long long b = ~sc[SCAN_MINR];
        std::memcpy(&core, &b, 8);
    }
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
    int rc = run_scan(c, c->sel, sc, st);
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
    h.done = !(c->t < t_end) || c->t >= t_mark;
    h.status = 0;
    h.finish = 0;
    std::memset(h.red, 0, sizeof h.red);
    int rc = write_ctl(c, st);
    if (rc) return rc;
    const bool use_graph = !(c->ex.flags & SWE_EXEC_NO_GRAPH) && (!c->tr || c->tr->capturable());
    const int chunk = 64;
    uint64_t launched = 0;
    unsigned long long committed_before = 0;
    int rc_final = SWE_OK;
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    while (true) {
        if (h.done) break;
        if (max_steps && launched >= max_steps) break;
        const uint64_t left = max_steps ? max_steps - launched : UINT64_MAX;
        const uint64_t parity = h.step_index;  // next step's parity
        uint64_t n;
        if (use_graph && left >= static_cast<uint64_t>(chunk)) {
            if (c->graph_len != chunk) {
                rc = build_graphs(c, chunk, st);
                if (rc) return rc;
            }
            // graph candidates assume sel = 0 at the chunk start; for sel = 1
            // the strip halo sends target the other buffer, so strips fall
            // back to plain launches in that case.
            if (c->ex.nranks > 1 && h.sel != 0) {
                for (int k = 0; k < chunk; ++k) {
                    rc = enqueue_step(c, ((parity + k) % 2) == 0, (h.sel + k + 1) & 1, st);
                    if (rc) return rc;
                }
            } else {
                CUDA_TRY(cudaGraphLaunch(c->graph[parity % 2], c->stream));
                c->launches += c->graph_kernels;
            }
            n = chunk;
        } else {
            n = std::min<uint64_t>(left, static_cast<uint64_t>(chunk));
            for (uint64_t k = 0; k < n; ++k) {
                rc = enqueue_step(c, ((parity + k) % 2) == 0, (h.sel + k + 1) & 1, st);
                if (rc) return rc;
            }
        }
        (void)n;
        rc = read_ctl(c, st);
        if (rc) return rc;
        // keep the host mirror of the committed selector/time in sync
        c->sel = h.sel;
        c->t = h.t;
        if (h.status != SWE_OK) {
            const unsigned long long steps_ok = h.steps_done;
            rc = resolve(c, st);
            c->sel = h.sel;
            c->t = h.t;
            if (rc) {
                rc_final = rc;
                (void)steps_ok;
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
EXPORT uint64_t swe_cuda_launch_count(const swe_ctx* c) { return c ? c->launches : 0; }
