/*
 * swe_cuda.h — C-ABI of libswe_cuda.so, the B200 (sm_100a) executor for the
 * per-time-step MacCormack predictor-corrector path of the 2D shallow-water
 * solver (arXiv 1309.1230 reference, /root/reference/proj).
 *
 * The reference has no FFI layer: its operator boundary for this path is the
 * C++ class swe::Stepper (proj/include/swe/executor.hpp:726-1116), selected by
 * ExecutorKind (executor.hpp:27-67).  Every entry point below replaces one
 * member (or free function) of that interface; the file:line of the member it
 * replaces is given beside each declaration.  A header-only C++ shim that
 * re-exposes the Stepper signatures and rethrows the reference's exception
 * types lives in include/swe_cuda.hpp.
 *
 * Conventions
 *  - Plain pointers and sizes only; no CUDA or torch types cross the boundary.
 *  - Host field arrays follow the FieldSet contract (grid.hpp:136-164):
 *    nx*ny doubles, row-major, x fastest, index = j*nx + i, no ghost cells.
 *  - Every call returns an swe_code and, when `st` is non-NULL, fills it.
 *    Codes 0/2/3/4/5 are the reference's ExitCode values (errors.hpp:9-15);
 *    6 is new (CUDA / NCCL runtime failure).
 *  - On any error the committed state is unchanged (executor.hpp:715-724).
 *  - One host thread per context.
 */
#ifndef SWE_CUDA_H
#define SWE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWE_CUDA_ABI_VERSION 1

/* errors.hpp:9-15 (ExitCode) + SWE_ERR_RUNTIME for device/collective failures */
typedef enum swe_code {
    SWE_OK = 0,
    SWE_ERR_CONFIG = 2,        /* ConfigError        errors.hpp:19-22 */
    SWE_ERR_INSTABILITY = 3,   /* InstabilityError   errors.hpp:27-40 */
    SWE_ERR_STEP_COLLAPSE = 4, /* StepCollapseError  errors.hpp:44-55 */
    SWE_ERR_IO = 5,            /* IoError            errors.hpp:58-61 */
    SWE_ERR_RUNTIME = 6        /* CUDA / NCCL failure (new) */
} swe_code;

/* Error detail.  For SWE_ERR_INSTABILITY: i, j (global cell, -1 when the
 * reference reports none) and t (InstabilityError::cell_i/cell_j/sim_time);
 * h/qx/qy carry the guard values when the stability guard fired.
 * For SWE_ERR_STEP_COLLAPSE: dt and t (StepCollapseError::dt/sim_time). */
typedef struct swe_status {
    int32_t code;
    int32_t i, j;
    double t;
    double dt;
    double h, qx, qy;
    char msg[256];
} swe_status;

/* GridSpec (grid.hpp:21-43) */
typedef struct swe_grid {
    int32_t nx, ny;
    double dx, dy;
} swe_grid;

/* PhysicsParams (scheme.hpp:14-20) */
typedef struct swe_physics {
    double g;          /* default 9.81 */
    double manning_n;  /* 0 = frictionless */
    double nu_art;     /* [0, 0.5); 0 = no smoothing sub-pass */
} swe_physics;

/* StabilityPolicy (timestep.hpp:17-24) */
typedef struct swe_policy {
    double cfl;     /* (0, 1], default 0.9 */
    double dt_max;  /* default +inf */
    double dt_min;  /* default 1e-9 */
    double h_min;   /* default 1e-6 */
} swe_policy;

/* BoundaryKind::Type (grid.hpp:133-149) */
typedef enum swe_bc_type {
    SWE_BC_WALL = 0,
    SWE_BC_TRANSMISSIVE = 1,
    SWE_BC_INFLOW = 2,
    SWE_BC_FIXED_ETA = 3
} swe_bc_type;

typedef struct swe_boundary {
    int32_t type;   /* swe_bc_type */
    double q_n;     /* inflow_discharge */
    double h_in;    /* inflow_discharge (validated only, grid.hpp:177-193) */
    double eta_out; /* fixed_elevation */
} swe_boundary;

/* BoundarySet (grid.hpp:152-175); field order matches the reference. */
typedef struct swe_boundary_set {
    swe_boundary north, south, east, west;
} swe_boundary_set;

/* Executor options (replaces ExecutorKind, executor.hpp:27-67, with the
 * `cuda` strategy SURVEY.md §8(b) proposes). */
enum {
    SWE_EXEC_EXACT = 1u << 0,   /* IEEE expression trees, no FMA contraction:
                                   bit-identical to the reference (the
                                   -fmad=false comparison mode) */
    SWE_EXEC_NO_GRAPH = 1u << 1, /* advance(): plain launches, no CUDA graph */
    SWE_EXEC_EARLY_EXIT = 1u << 2, /* skip work items whose 3x3 item
                                      neighbourhood is a flat bed at rest
                                      (bit-exact: such items are fixed points
                                      of the step) */
    SWE_EXEC_LOCAL_GROUP = 1u << 3 /* nranks > 1 without NCCL: the ranks are
                                      contexts of this process on one device,
                                      driven by one host thread each; nccl_id
                                      points to SWE_NCCL_ID_BYTES naming the
                                      group.  Collectives are CUDA-event-ordered
                                      copies (test transport for the strip
                                      path on a single GPU; no CUDA graphs) */
};

typedef struct swe_exec {
    int32_t device;      /* CUDA ordinal (per rank) */
    uint32_t flags;      /* SWE_EXEC_* */
    int32_t rank;        /* row-strip rank, 0 for one GPU */
    int32_t nranks;      /* row strips, 1 for one GPU */
    const void* nccl_id; /* ncclUniqueId bytes (SWE_NCCL_ID_BYTES) when nranks > 1 */
} swe_exec;

#define SWE_NCCL_ID_BYTES 128

/* StepResult (executor.hpp:228-232) */
typedef struct swe_step_result {
    double dt_used;
    double dt_next;         /* raw CFL dt, no end-time clamp */
    int32_t guard_warnings; /* fixed-elevation ghost clamps this step */
} swe_step_result;

/* InitialCondition (scenarios.hpp:26-42) restricted to the kinds without
 * transcendental functions; values of `kind` follow InitialCondition::Kind. */
enum {
    SWE_IC_FLAT_POOL = 0,     /* h = depth */
    SWE_IC_CHANNEL_SLOPE = 2, /* z = slope*dx*(nx-1-i), h = depth - z */
    SWE_IC_DAM_BREAK = 4      /* h = (i+0.5)*dx < split_x ? h_left : h_right */
};
typedef struct swe_initial {
    int32_t kind;
    double depth, slope, split_x, h_left, h_right;
} swe_initial;

/* RunReport subset + resume record (run.hpp:21-66, 101-179) */
typedef struct swe_run_result {
    uint64_t steps;        /* steps committed by this call */
    uint64_t step_index;   /* parity origin for the next call (resume record) */
    double t_final;
    double dt_next;        /* raw CFL dt from the final committed state */
    int32_t guard_warnings;
} swe_run_result;

/* StepAccounting (executor.hpp:218-222), per step of this rank:
 * halo values received from the strip neighbours, and the predictor /
 * corrector rows the row-chunked march recomputes at work-item boundaries
 * (in full-row units). */
typedef struct swe_accounting {
    int64_t halo_values_exchanged;
    int32_t redundant_star_rows;
    int32_t redundant_corrector_rows;
} swe_accounting;

/* Early-exit accounting since the last load (SWE_EXEC_EARLY_EXIT). */
typedef struct swe_activity {
    uint64_t cells_per_step;  /* interior cells of this rank */
    uint64_t items_per_step;  /* work items (32-column window x row chunk) */
    uint64_t eligible_items;  /* interior items on a locally flat bed */
    uint64_t skipped_cells;   /* cells of skipped items, summed over launches */
} swe_activity;

/* StepTimings-style device counters (executor.hpp:153-172), CUDA-event based */
typedef struct swe_timing {
    uint64_t steps;
    double step_seconds;      /* sum of device time of step launches (K1-K6 + smoothing run fused) */
    /* strips, swe_cuda_step only (device events; advance() runs under CUDA
     * graphs and does not split its time): the halo send/recv, overlapped
     * with the interior rows, and the reduction-word allreduce */
    uint64_t exchange_steps;
    double exchange_seconds;
    double allreduce_seconds;
} swe_timing;

typedef struct swe_ctx swe_ctx;

/* ---- lifecycle ------------------------------------------------------- */

/* Stepper::Stepper (executor.hpp:728-761): validates physics, policy,
 * boundaries and strip partition; allocates device buffers.  For nranks > 1
 * the grid is split into row strips with partition_scanlines semantics
 * (executor.hpp:189-208). */
int swe_cuda_create(const swe_grid* grid, const swe_physics* phys, const swe_policy* pol,
                    const swe_boundary_set* bnd, const swe_exec* exec, swe_ctx** out,
                    swe_status* st);

/* Stepper::~Stepper */
void swe_cuda_destroy(swe_ctx* ctx);

/* Stepper::load (executor.hpp:764-780): z/h/qx/qy are this rank's rows
 * [row_begin, row_end) (the whole grid on one GPU), nx per row.  The bed
 * becomes the run's bed; slopes are computed on the device. */
int swe_cuda_load(swe_ctx* ctx, const double* z, const double* h, const double* qx,
                  const double* qy, double t, swe_status* st);

/* build_initial_state (scenarios.hpp:95-171) + Stepper::load, generated on
 * the device for this rank's rows (no host arrays; a 32768^2 state would need
 * 32 GB of host memory).  Bit-identical to the reference's state; fails with
 * SWE_ERR_CONFIG for drops/vortex (std::exp) and when the stability guard
 * rejects the state, like the reference. */
int swe_cuda_load_initial(swe_ctx* ctx, const swe_initial* ic, double t, swe_status* st);

/* Stepper::state (executor.hpp:783-797): copies this rank's rows out.
 * Any of z/h/qx/qy may be NULL to skip that field. */
int swe_cuda_state(swe_ctx* ctx, double* z, double* h, double* qx, double* qy, double* t,
                   swe_status* st);

/* Stepper::step (executor.hpp:812-841).  t_after = NaN commits t + dt. */
int swe_cuda_step(swe_ctx* ctx, double dt, uint64_t step_index, double t_after,
                  swe_step_result* res, swe_status* st);

/* compute_dt (timestep.hpp:128-179) on the committed device state,
 * including the end-time clamp. */
int swe_cuda_compute_dt(swe_ctx* ctx, double t_end, double* dt, swe_status* st);

/* stability_guard (timestep.hpp:112-115) on the committed device state:
 * SWE_OK or SWE_ERR_INSTABILITY with the row-major first offender. */
int swe_cuda_guard(swe_ctx* ctx, swe_status* st);

/* The run_from time loop (run.hpp:149-163), device resident: landing clamp,
 * step parity and dt hand-off stay on the device; up to max_steps steps
 * (0 = until t_end) are captured in CUDA graphs of `chunk` launches and the
 * host syncs once per chunk.  dt_first = NaN computes the first dt from the
 * state (run.hpp:125-130).  On error the last committed state is kept and
 * res->steps counts the committed steps. */
int swe_cuda_advance(swe_ctx* ctx, double t_end, uint64_t step_index0, double dt_first,
                     uint64_t max_steps, swe_run_result* res, swe_status* st);

/* swe_cuda_advance that also stops after the first committed step with
 * t >= t_mark (run_from's snapshot cadence, run.hpp:159-163): the caller
 * writes the snapshot and calls again with the returned step_index/dt_next.
 * Stepping decisions are the same as advance's, so the committed states are
 * identical with or without marks.  t_mark = +inf is swe_cuda_advance. */
int swe_cuda_advance_marked(swe_ctx* ctx, double t_end, double t_mark, uint64_t step_index0, double dt_first,
                            uint64_t max_steps, swe_run_result* res, swe_status* st);

/* ---- accessors (executor.hpp:799-805) -------------------------------- */
double swe_cuda_time(const swe_ctx* ctx);
int32_t swe_cuda_guard_warnings(const swe_ctx* ctx);
int swe_cuda_timing(const swe_ctx* ctx, swe_timing* out);
/* Stepper::accounting (executor.hpp:804) */
int swe_cuda_accounting(const swe_ctx* ctx, swe_accounting* out);
/* Early-exit counters (all zero skips when SWE_EXEC_EARLY_EXIT is off). */
int swe_cuda_activity(swe_ctx* ctx, swe_activity* out);
/* Rows owned by this rank: [*row_begin, *row_end). */
void swe_cuda_rows(const swe_ctx* ctx, int32_t* row_begin, int32_t* row_end);
/* Committed-halo radius in rows (1 without smoothing, 2 with). */
int32_t swe_cuda_halo_rows(const swe_ctx* ctx);
/* Order-independent 64-bit digest of this rank's committed h, qx, qy bit
 * patterns: the sum (mod 2^64) over owned cells of a splitmix64 mix of the
 * three bit patterns and the global cell index j*nx + i.  The digest of the
 * whole grid is the sum of the ranks' digests, so a strip run and a
 * one-domain run can be compared bit for bit without copying the state to the
 * host (no reference counterpart; a checksum for size-independent parity). */
int swe_cuda_state_digest(swe_ctx* ctx, uint64_t* digest, swe_status* st);

/* ---- multi-GPU plumbing ---------------------------------------------- */
/* The rows [*row_begin, *row_end) that swe_cuda_create gives `rank` of
 * `nranks` strips: the reference's partition_scanlines (executor.hpp:189-208;
 * contiguous bands, sizes differ by <= 1, larger first) with the decomposed
 * executor's >= 4-row band rule; the same errors as create.  Host only (no
 * CUDA call), so the strip protocol can be checked without a GPU. */
int swe_cuda_strip_rows(int32_t ny, int32_t nranks, int32_t rank, int32_t* row_begin, int32_t* row_end,
                        swe_status* st);
/* ncclGetUniqueId into out[SWE_NCCL_ID_BYTES] (rank 0 broadcasts it). */
int swe_cuda_nccl_unique_id(void* out, swe_status* st);

/* ---- diagnostics ----------------------------------------------------- */
/* SWE_CHECKED builds only (tools/checked_run.sh): counts corrupted bytes in
 * the guard bands around every live device allocation of the library; the
 * product build returns SWE_ERR_CONFIG. */
int swe_cuda_debug_guard_check(uint64_t* corrupted_bytes, uint64_t* allocations, swe_status* st);
/* Runs the step kernel's shared-reciprocal division on device arrays copied
 * from the host: out[k] = a[k] / b[k] as the step computes it (exact = 1:
 * SWE_EXEC_EXACT arithmetic with ptxas's per-division acceptance test; 2: the
 * exact step's per-state range test with a[k] as the momentum; 0: the
 * fast-mode quotient).  Used by the parity tests to prove the exact paths
 * equal IEEE division. */
int swe_cuda_selftest_div(const double* a, const double* b, size_t n, int exact, double* out,
                          swe_status* st);

/* ---- misc ------------------------------------------------------------ */
const char* swe_cuda_version(void);
/* Number of this library's kernel launches issued for steps since create:
 * step kernels plus, where used, the early-exit schedule kernel and the strip
 * finalize kernel (bench evidence). */
uint64_t swe_cuda_launch_count(const swe_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* SWE_CUDA_H */
