// swe_runtime.h — internal interfaces of the host runtime behind
// include/swe_cuda.h: the context (swe_capi.cu), the auxiliary kernels
// (swe_aux.cu) and the row-strip transports (swe_transport.cu).  Not part of
// the public C-ABI.
#pragma once

#include <cstdarg>
#include <cstddef>
#include <cstring>
#include <map>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "swe_device.cuh"
#include "swe_launch.h"

namespace swe_rt {
struct Transport;
}

// ---------------------------------------------------------------- context
struct swe_ctx {
    swe_grid g{};
    swe_physics ph{};
    swe_policy pol{};
    swe_boundary_set bnd{};
    swe_exec ex{};
    int R = 1, nloc = 0, j0 = 0, pitch = 0, ntiles = 0;
    int halo_x = 1;  // committed rows exchanged with each strip neighbour (R; test hook may shrink it)
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
    bool multi_ok = false;  // small grid: advance() runs many steps per launch (swe_multi_kernel)
    bool graph_failed = false;  // a step-graph capture failed: advance() launches plainly from then on
    int ncta_multi = 0;
    int multi_chunk = 0, multi_nchunks = 0, occ_multi = 0;  // item rows of multi-step launches (one item per warp)
    // CUDA graphs of `len` consecutive steps, keyed by (len, parity of the
    // first step, committed selector at the start -- strips only: the halo
    // send/recv addresses depend on it); built on first use
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        unsigned long long kernels = 0;  // our kernels per launch of this graph
    };
    std::map<int, Graph> graphs;
    swe_rt::Transport* tr = nullptr;  // row-strip collectives (NCCL or local group); null for one rank
    unsigned long long* d_xr = nullptr;  // local-group allreduce scratch
    // strips: halo exchange overlapped with the interior (edge + interior launches)
    bool overlap = false;
    bool p2p = false;  // strips: fused halo push into the neighbours' buffers (no send/recv per step)
    StepParams prm_edge{}, prm_int{};
    int ncta_edge = 0;
    cudaStream_t stream_edge = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // strips, step() only: timing events around the halo send/recv and the
    // allreduce (recorded when c->time_exchange is set, never under capture)
    cudaEvent_t ev_x[4] = {nullptr, nullptr, nullptr, nullptr};
    bool time_exchange = false;
    unsigned long long launches = 0;
    swe_timing timing{};
    double tz_x = 0, tz_y = 0;
    int always_diag = 0;
};

namespace swe_rt {

// ---------------------------------------------------------------- status (swe_capi.cu)
int set_status(swe_status* st, int code, int i, int j, double t, const char* fmt, ...);
int ok_status(swe_status* st);

#define CUDA_TRY(x)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return set_status(st, SWE_ERR_RUNTIME, -1, -1, 0.0, "CUDA error %s at %s:%d",        \
                              cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)


// ---------------------------------------------------------------- auxiliary kernels (swe_aux.cu)
struct BcSet {
    SweBC bc[4];  // N, S, E, W
};

// Scan words (max-combined, like the step reduction).
enum { SCAN_BAD = 0, SCAN_MINR = 1, SCAN_GUARD = 2, SCAN_DRY = 3, SCAN_MAXSX = 4, SCAN_MAXSY = 5, SCAN_N = 6 };

constexpr int kMaxLocalRanks = 16;  // ranks of a local strip group
struct RedPtrs {
    const unsigned long long* p[kMaxLocalRanks];
};

__global__ void fill_benign_kernel(double* buf, size_t rows3, int P);
__global__ void ghost_fill_rows_kernel(double* b, int P, int R, int nx, int nloc, int j0, int ny,
                                       SweBC w, SweBC e, SweBC s, SweBC n, const double* z_w,
                                       const double* z_e, const double* z_s, const double* z_n,
                                       double h_min);
__global__ void slopes_kernel(const double* zp, double* slope, int P, int R, int nx, int nloc,
                              int j0, int ny, double two_dx, double two_dy, double scale, unsigned* flags);
__global__ void item_flat_kernel(const double* slope, int P, int R, int nx, int nloc, int TW, int chunk,
                                 int ntiles, int nitems, unsigned char* flat);
__global__ void item_elig_kernel(const unsigned char* flat, int nx, int nloc, int TW, int chunk, int ntiles,
                                 int nchunks, int R, unsigned char* elig, unsigned long long* count);
__global__ void edge_z_kernel(const double* zp, int R, int nx, int nloc, double* zw, double* ze);
__global__ void clamp_kernel(const double* zp, int R, int nx, int nloc, int own_s, int own_n, BcSet b,
                             double h_min, unsigned* flag);
__global__ void initial_kernel(swe_initial ic, double dx, int nx, int nloc, int P, int R, double* buf, double* zp);
__global__ void scan_kernel(const double* b, int P, int R, int nx, int nloc, int j0, double g,
                            double dx, double dy, double h_min, int cfl, unsigned long long* out);
__global__ void dry_scan_kernel(const double* b, int P, int R, int nx, int ny, int nloc, int j0, double dt,
                                double dx, double dy, int fwd, int exact, BcSet bs, const double* z_w,
                                const double* z_e, const double* z_s, const double* z_n, double h_min,
                                unsigned long long* out);
__global__ void digest_kernel(const double* b, int P, int R, int nx, int nloc, int j0, unsigned long long* out);
__global__ void selftest_div_kernel(const double* a, const double* b, size_t n, int exact, double* out);
__global__ void max_reduce_kernel(RedPtrs in, int nranks, int n, unsigned long long* out);

// ---------------------------------------------------------------- device allocations (swe_capi.cu)
// cudaMalloc / cudaFree, with guard bands in SWE_CHECKED builds
cudaError_t dev_alloc(void** p, size_t bytes);
void dev_free(void* p);

// ---------------------------------------------------------------- TMA descriptors (swe_capi.cu)
// 2D map over field_rows rows of P doubles at row_stride doubles (P if 0); box
// box_cols x box_rows
bool encode_rows(CUtensorMap* map, double* base, int P, long long field_rows, int box_rows, std::string& err,
                 int box_cols = 32, int row_stride = 0);

// ---------------------------------------------------------------- strip transport (swe_transport.cu)
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
    // The strip neighbours' two state buffers as device pointers this rank's
    // kernels may store to (NVLink peer memory through CUDA IPC or in-process
    // peer access; the same device for the local group), for the fused halo
    // push.  Collective over the group; leaves nulls when unavailable.
    virtual int peer_buffers(swe_ctx* c, double* dn[2], double* up[2], int* nloc_dn, swe_status* st) = 0;
};

// The transport of a context with nranks > 1: NCCL between GPUs, or the local
// group (SWE_EXEC_LOCAL_GROUP) keyed by the nccl_id bytes.  Sets c->tr.
int create_transport(swe_ctx* c, const swe_exec& ex, const void* nccl_id, swe_status* st);
// ncclGetUniqueId through the dlopen'ed NCCL
int nccl_unique_id(void* out, swe_status* st);

}  // namespace swe_rt
