// swe_types.h — structures shared by the host runtime (swe_capi.cu) and the
// step kernels.  Not part of the public C-ABI (include/swe_cuda.h).
#pragma once

#include <cstdint>

#include <cuda.h>

#include "../../include/swe_cuda.h"

enum { SWE_EDGE_N = 0, SWE_EDGE_S = 1, SWE_EDGE_E = 2, SWE_EDGE_W = 3 };

// Padded rows: cell i of a row sits at column i + SWE_XO.  SWE_XO is even (and
// >= R = 1, 2) so that every window's first output column, tile * TW + SWE_XO,
// is 16-byte aligned: TMA tensor stores must start on a 16-byte-aligned inner
// coordinate (tools/tma_store_probe.cu).
#define SWE_XO 2
// TMA load box of a window (32 lanes, lane 0 at column tile*TW - R + SWE_XO):
// with R = 1 lane 0 sits at an odd column, so the box starts one column
// earlier and is 34 wide (16-byte-aligned start, 272-byte rows); with R = 2 it
// starts at lane 0 and is 32 wide.
constexpr int swe_box_off(int R) { return (SWE_XO - R) & 1; }
constexpr int swe_box_w(int R) { return 32 + 2 * swe_box_off(R); }

struct SweBC {
    int type;  // swe_bc_type
    double q_n;
    double eta_out;
};

// Reduction words, all combined with unsigned max (atomicMax on the device,
// ncclMax across ranks).  Error indices are stored complemented (~idx) so that
// max selects the row-major FIRST offender; 0 means "none".
enum {
    RED_SX = 0,   // bits of max sx = |qx/h| + sqrt(g h)   (non-negative doubles order like u64)
    RED_SY = 1,   // bits of max sy
    RED_E4 = 2,   // ~ first corrector cell consuming a dry U*, found in an edge window or row
                  //   (executor.hpp:429-436)
    RED_E5 = 3,   // 1: the guard screen failed somewhere (executor.hpp:543-556); the first
                  //   offender is found by the exact scan (scan_kernel)
    RED_E2 = 4,   // committed depth below h_min seen by the predictor (scheme.hpp:35-39)
    RED_DIAG = 5, // K6 needs the exact per-cell scan (dx/sx underflow/overflow possible)
    RED_DRY = 6,  // 1: an interior U* was dry; the first consumer is found by dry_scan_kernel
    RED_N = 8
};

// Device control block: the committed-state bookkeeping of swe::Stepper
// (executor.hpp:1106-1115) plus the run_from loop scalars (run.hpp:149-163),
// kept on the device so a CUDA graph of step launches needs no host sync.
struct __align__(16) SweCtl {
    double t;                     // committed time
    double dt_raw;                // raw CFL dt for the next step
    double t_end;                 // advance(): landing target
    double t_mark;                // advance(): also stop once t >= t_mark (snapshot cadence; +inf = off)
    double dt_req;                // step(): dt from the host
    double tcommit_req;           // step(): committed time from the host
    double dt_used, t_commit, dt_next;  // results of the last launch
    double err_dt;                // StepCollapseError::dt
    double err_t;                 // InstabilityError/StepCollapseError sim time
    double max_sx, max_sy;        // CFL maxima of the last launch (diagnosis)
    unsigned long long step_index;  // parity of the next step
    unsigned long long steps_done;  // committed steps since the counter was reset
    int sel;                      // committed buffer (0/1)
    int done;                     // 1 => further launches are no-ops
    int mode;                     // 0 host step, 1 advance
    int status;                   // swe_code of the last launch, 7 = needs host diagnosis
    int err_kind;                 // 2/4/5/6: which plan kernel raised
    int err_i, err_j;
    unsigned int finish;          // CTA arrival counter for the last-block finalize
    unsigned int work[2];         // dynamic work-item counters (slot per concurrent step launch)
    unsigned int nactive;         // early exit: length of the step's active item list
    unsigned long long red[RED_N];
    int diag_flags;               // status 7: 1 = guard screen failed, 2 = interior dry U*
    // multi-step launches (swe_multi_kernel, small grids): per-step work
    // counters and reduction words, triple-buffered by step, and the grid
    // barrier's arrival counter / generation
    unsigned int mwork[3];
    unsigned int bar_count, bar_gen;
    unsigned int pad_[3];
    unsigned long long mred[3][RED_N];
};

#define SWE_STATUS_DIAG 7

// Kernel parameters (passed by value as a __grid_constant__).
struct StepParams {
    // 2D TMA descriptors: state buffer k viewed as [3*(nloc+2R) field rows][P]
    // (box 32 x 3 = h, qx, qy of one row); slopes as [2*(nloc+2R)][P] (box 32 x 2)
    CUtensorMap tmap_state[2];
    CUtensorMap tmap_slope;
    CUtensorMap tmap_slopex;  // the dz/dx rows only (row stride 2P; box 32 x G)
    // TMA-store epilogue: state buffer k as [3*(nloc+2R) field rows][R + nx]
    // (columns past the domain clipped), box TW x 3G (one row group)
    CUtensorMap tmap_out[2];
    double* buf[2];        // committed/candidate state, row-interleaved SoA
    const double* slope;   // dzdx/dzdy rows, same layout; nullptr for a flat bed
    const double* z_w;     // bed z at i=0 per local row
    const double* z_e;     // bed z at i=nx-1 per local row
    const double* z_s;     // bed z at global row 0 per column
    const double* z_n;     // bed z at global row ny-1 per column
    SweCtl* ctl;
    // early exit (SWE_EXEC_EARLY_EXIT): per-buffer quiet flags of the work
    // items (depth bits H of an all-(H, +0, +0) item, else 0), static
    // eligibility (interior item, flat bed over its 3x3 neighbourhood), and
    // counters {skipped cells}
    unsigned long long* qflag[2];
    const unsigned char* elig;
    unsigned* active;      // active item list (schedule kernel -> step kernel)
    // fused halo push (strips): the neighbours' state buffers (peer memory);
    // the epilogue stores its R edge rows straight into their halo rows
    double* peer_dn[2];    // rank - 1 (its rows nloc_dn .. nloc_dn+R-1 take our rows 0 .. R-1)
    double* peer_up[2];    // rank + 1 (its rows -R .. -1 take our rows nloc-R .. nloc-1)
    int p2p, nloc_dn;
    unsigned long long* stats;
    int early;
    int nx, ny;            // global grid
    int nloc, j0;          // rows owned by this rank: global [j0, j0+nloc)
    int pitch;             // doubles per field row (P)
    long long buf_doubles; // doubles per state buffer (SWE_CHECKED bounds)
    int ntiles;            // x tiles
    int ncta;              // CTAs launched
    int chunk;             // rows per dynamic work item
    int nchunks;           // row chunks per tile (items = ntiles * nchunks)
    // rows this launch covers: [row_lo, row_hi), chunk rc starting at
    // row_lo + rc*chunk (+ row_gap for rc > 0); wslot selects the work counter.
    // One launch per step: [0, nloc), gap 0, slot 0.  Strips with overlap:
    // an edge launch (the R-deep bands whose rows the neighbours need) and an
    // interior launch on two streams.
    int row_lo, row_hi, row_gap, wslot;
    // guided chunking: row chunks rc >= tier_rc hold chunk2 rows (short items
    // at the end of the dynamic queue trim the tail); tier_rc = nchunks = uniform
    int tier_rc, chunk2;
    int finalize;          // 1: last CTA finalizes (one rank); 0: host-side allreduce + finalize kernel
    int nranks;
    double dx, dy, g, half_g, neg_g, gnn, h_min, nu;
    double sqrt_g;         // fast-mode CFL speed sqrt(g) * h^(1/2)
    double cfl, dt_max, dt_min;
    double tz_x, tz_y;     // K6 diagnosis triggers (dx/sx would round to 0)
    int always_diag;       // pathological parameters: diagnose every step
    SweBC bc[4];           // N, S, E, W
};
