/*
 * swe_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded restatement of the reference's naive executor
 * (the parity oracle for libswe_cuda.so).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library, and only as the
 * checker or the timed CPU baseline — never as the product path.
 *
 * Parity pinned: tests/test_oracle_golden.py checks this restatement
 * byte-for-byte against (a) the golden SWS1 fixtures in tests/golden/
 * produced by the reference itself (oracle/_ref, built from
 * /root/reference/proj/include by oracle/Makefile, script
 * tests/golden/make_golden.py) and (b) the sha256 digests recorded in
 * SURVEY.md §8(c).
 *
 * Build: -O2 -ffp-contract=off (the reference's own flag,
 * proj/CMakeLists.txt:12-14), never -ffast-math.  Every expression keeps the
 * reference's evaluation order; citations are file:line under
 * /root/reference/proj/include/swe/.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/swe_cuda.h"

#define EXPORT __attribute__((visibility("default")))

typedef struct { double h, qx, qy; } cv; /* CellVec grid.hpp:197-215 */

static cv cv_add(cv a, cv b) { cv r = {a.h + b.h, a.qx + b.qx, a.qy + b.qy}; return r; }
static cv cv_sub(cv a, cv b) { cv r = {a.h - b.h, a.qx - b.qx, a.qy - b.qy}; return r; }
static cv cv_scale(double s, cv a) { cv r = {s * a.h, s * a.qx, s * a.qy}; return r; }
/* std::min(a, b) == (b < a) ? b : a  (executor.hpp:569, timestep.hpp:302) */
static double std_min(double a, double b) { return (b < a) ? b : a; }

enum { E_N = 0, E_S = 1, E_E = 2, E_W = 3 };

typedef struct swo_ctx {
    swe_grid g;
    swe_physics p;
    swe_policy pol;
    swe_boundary_set b;
    int nx, ny, W; /* W = nx + 2: buffer width with ghosts */
    double *z, *dzdx, *dzdy;
    double *cur[3], *star[3], *next[3], *aux[3]; /* (nx+2)*(ny+2), origin (-1,-1) */
    double t;
    int loaded;
    int warnings_total;
    /* error channel: set by the first throwing site */
    int err;
    swe_status st;
} swo_ctx;

static size_t at(const swo_ctx* c, int i, int j) { return (size_t)(j + 1) * c->W + (size_t)(i + 1); }
static cv get(const swo_ctx* c, double* const* s, int i, int j) {
    size_t k = at(c, i, j); cv r = {s[0][k], s[1][k], s[2][k]}; return r;
}
static void put(const swo_ctx* c, double** s, int i, int j, cv u) {
    size_t k = at(c, i, j); s[0][k] = u.h; s[1][k] = u.qx; s[2][k] = u.qy;
}
static const swe_boundary* bnd(const swo_ctx* c, int e) {
    switch (e) { case E_N: return &c->b.north; case E_S: return &c->b.south; case E_E: return &c->b.east; default: return &c->b.west; }
}

static void fail(swo_ctx* c, int code, int i, int j, double t, const char* msg) {
    if (c->err) return;
    c->err = code;
    memset(&c->st, 0, sizeof c->st);
    c->st.code = code; c->st.i = i; c->st.j = j; c->st.t = t;
    snprintf(c->st.msg, sizeof c->st.msg, "%s", msg);
}

/* scheme.hpp:35-39 require_wet: generic InstabilityError(-1,-1,0) */
static void require_wet(swo_ctx* c, cv u) {
    if (!(u.h >= c->pol.h_min)) fail(c, SWE_ERR_INSTABILITY, -1, -1, 0.0, "depth below dry threshold");
}
/* scheme.hpp:42-45 */
static cv flux_x(swo_ctx* c, cv u) {
    require_wet(c, u);
    cv r = {u.qx, u.qx * u.qx / u.h + 0.5 * c->p.g * u.h * u.h, u.qx * u.qy / u.h};
    return r;
}
/* scheme.hpp:48-51 */
static cv flux_y(swo_ctx* c, cv u) {
    require_wet(c, u);
    cv r = {u.qy, u.qx * u.qy / u.h, u.qy * u.qy / u.h + 0.5 * c->p.g * u.h * u.h};
    return r;
}
/* scheme.hpp:54-63 */
static cv source(swo_ctx* c, cv u, double dzdx, double dzdy) {
    require_wet(c, u);
    double fr = 0.0;
    if (c->p.manning_n > 0.0) {
        const double speed = sqrt(u.qx * u.qx + u.qy * u.qy) / u.h;
        fr = c->p.g * c->p.manning_n * c->p.manning_n * speed / pow(u.h, 4.0 / 3.0);
    }
    cv r = {0.0, -c->p.g * u.h * dzdx - fr * u.qx, -c->p.g * u.h * dzdy - fr * u.qy};
    return r;
}
/* scheme.hpp:100-113 */
static cv predictor_cell(swo_ctx* c, cv self, cv nbx, cv nby, double dzdx, double dzdy, double dt, int fwd) {
    const cv fs = flux_x(c, self), fn = flux_x(c, nbx), gs = flux_y(c, self), gn = flux_y(c, nby);
    const cv df = fwd ? cv_sub(fn, fs) : cv_sub(fs, fn);
    const cv dg = fwd ? cv_sub(gn, gs) : cv_sub(gs, gn);
    const cv flux_sum = cv_add(cv_scale(dt / c->g.dx, df), cv_scale(dt / c->g.dy, dg));
    const cv src = source(c, self, dzdx, dzdy);
    return cv_add(cv_sub(self, flux_sum), cv_scale(dt, src));
}
/* scheme.hpp:153-161 */
static cv iface_x(swo_ctx* c, cv a, cv b) { return cv_scale(0.5, cv_add(flux_x(c, a), flux_x(c, b))); }
static cv iface_y(swo_ctx* c, cv a, cv b) { return cv_scale(0.5, cv_add(flux_y(c, a), flux_y(c, b))); }
/* scheme.hpp:167-176 */
static cv wall_x(swo_ctx* c, cv a, cv b) { cv r = {0.0, 0.5 * (flux_x(c, a).qx + flux_x(c, b).qx), 0.0}; return r; }
static cv wall_y(swo_ctx* c, cv a, cv b) { cv r = {0.0, 0.0, 0.5 * (flux_y(c, a).qy + flux_y(c, b).qy)}; return r; }
/* scheme.hpp:185-191 */
static cv corrector_update(swo_ctx* c, cv old, cv hw, cv he, cv hs, cv hn, cv src_sum, double dt) {
    const cv flux_sum = cv_add(cv_scale(dt / c->g.dx, cv_sub(he, hw)), cv_scale(dt / c->g.dy, cv_sub(hn, hs)));
    return cv_add(cv_sub(old, flux_sum), cv_scale(0.5 * dt, src_sum));
}
/* scheme.hpp:197-204 */
static cv smooth_cell(cv self, cv e, cv w, cv n, cv s, double nu) {
    if (nu == 0.0) return self;
    const cv lap = cv_add(cv_add(cv_sub(e, self), cv_sub(w, self)), cv_add(cv_sub(n, self), cv_sub(s, self)));
    return cv_add(self, cv_scale(nu, lap));
}

/* executor.hpp:333-341 pump_state */
static cv pump_state(int e, const swe_boundary* bk, cv in) {
    cv r;
    switch (e) {
        case E_W: r.h = in.h; r.qx = bk->q_n; r.qy = 0.0; break;
        case E_E: r.h = in.h; r.qx = -bk->q_n; r.qy = 0.0; break;
        case E_S: r.h = in.h; r.qx = 0.0; r.qy = bk->q_n; break;
        default: r.h = in.h; r.qx = 0.0; r.qy = -bk->q_n; break;
    }
    return r;
}
/* grid.hpp:242-265 ghost_value + executor.hpp:343-349 edge_ghost */
static cv edge_ghost(int e, const swe_boundary* bk, cv in, double z_in, double h_min, int* clamped) {
    cv r = in;
    switch (bk->type) {
        case SWE_BC_WALL:
            if (e == E_E || e == E_W) r.qx = -in.qx; else r.qy = -in.qy;
            return r;
        case SWE_BC_TRANSMISSIVE: return r;
        case SWE_BC_INFLOW: return pump_state(e, bk, in);
        default: {
            double hg = bk->eta_out - z_in;
            if (hg < h_min) { hg = h_min; if (clamped) *clamped = 1; }
            r.h = hg;
            return r;
        }
    }
}

/* executor.hpp:384-408 fill_ghosts */
static int fill_ghosts(swo_ctx* c, double** s) {
    int clamped = 0;
    const int nx = c->nx, ny = c->ny;
    for (int j = 0; j < ny; ++j) {
        put(c, s, -1, j, edge_ghost(E_W, &c->b.west, get(c, s, 0, j), c->z[(size_t)j * nx], c->pol.h_min, &clamped));
        put(c, s, nx, j, edge_ghost(E_E, &c->b.east, get(c, s, nx - 1, j), c->z[(size_t)j * nx + nx - 1], c->pol.h_min, &clamped));
    }
    for (int i = 0; i < nx; ++i)
        put(c, s, i, -1, edge_ghost(E_S, &c->b.south, get(c, s, i, 0), c->z[i], c->pol.h_min, &clamped));
    for (int i = 0; i < nx; ++i)
        put(c, s, i, ny, edge_ghost(E_N, &c->b.north, get(c, s, i, ny - 1), c->z[(size_t)(ny - 1) * nx + i], c->pol.h_min, &clamped));
    return clamped ? 1 : 0;
}

/* executor.hpp:429-436 require_wet_at */
static void require_wet_at(swo_ctx* c, cv u, int i, int j, double t) {
    if (!(u.h >= c->pol.h_min) && !c->err) {
        char m[200];
        snprintf(m, sizeof m, "predicted depth %f below dry threshold at cell (%d, %d)", u.h, i, j);
        fail(c, SWE_ERR_INSTABILITY, i, j, t, m);
        c->st.h = u.h;
    }
}

/* executor.hpp:451-519 corrector_at */
static cv corrector_at(swo_ctx* c, int i, int j, double dt, int fwd, double t_now) {
    const int nx = c->nx, ny = c->ny;
    const cv old = get(c, c->cur, i, j), ss = get(c, c->star, i, j);
    require_wet_at(c, ss, i, j, t_now);
    cv hw, he, hs, hn;
    const swe_boundary *bw = &c->b.west, *be = &c->b.east, *bs = &c->b.south, *bn = &c->b.north;
    if (i == 0 && bw->type == SWE_BC_WALL) hw = wall_x(c, old, ss);
    else if (i == 0 && bw->type == SWE_BC_INFLOW) hw = iface_x(c, pump_state(E_W, bw, old), pump_state(E_W, bw, ss));
    else {
        const cv cw = fwd ? old : get(c, c->cur, i - 1, j);
        const cv sw = fwd ? get(c, c->star, i - 1, j) : ss;
        require_wet_at(c, sw, i, j, t_now);
        hw = iface_x(c, cw, sw);
    }
    if (i == nx - 1 && be->type == SWE_BC_WALL) he = wall_x(c, old, ss);
    else if (i == nx - 1 && be->type == SWE_BC_INFLOW) he = iface_x(c, pump_state(E_E, be, old), pump_state(E_E, be, ss));
    else {
        const cv ce = fwd ? get(c, c->cur, i + 1, j) : old;
        const cv se = fwd ? ss : get(c, c->star, i + 1, j);
        require_wet_at(c, se, i, j, t_now);
        he = iface_x(c, ce, se);
    }
    if (j == 0 && bs->type == SWE_BC_WALL) hs = wall_y(c, old, ss);
    else if (j == 0 && bs->type == SWE_BC_INFLOW) hs = iface_y(c, pump_state(E_S, bs, old), pump_state(E_S, bs, ss));
    else {
        const cv cs = fwd ? old : get(c, c->cur, i, j - 1);
        const cv sst = fwd ? get(c, c->star, i, j - 1) : ss;
        require_wet_at(c, sst, i, j, t_now);
        hs = iface_y(c, cs, sst);
    }
    if (j == ny - 1 && bn->type == SWE_BC_WALL) hn = wall_y(c, old, ss);
    else if (j == ny - 1 && bn->type == SWE_BC_INFLOW) hn = iface_y(c, pump_state(E_N, bn, old), pump_state(E_N, bn, ss));
    else {
        const cv cn = fwd ? get(c, c->cur, i, j + 1) : old;
        const cv sn = fwd ? ss : get(c, c->star, i, j + 1);
        require_wet_at(c, sn, i, j, t_now);
        hn = iface_y(c, cn, sn);
    }
    const size_t k = (size_t)j * nx + i;
    const cv src_sum = cv_add(source(c, old, c->dzdx[k], c->dzdy[k]), source(c, ss, c->dzdx[k], c->dzdy[k]));
    return corrector_update(c, old, hw, he, hs, hn, src_sum, dt);
}

/* executor.hpp:351-376 make_domain_ctx slopes */
static void make_slopes(swo_ctx* c) {
    const int nx = c->nx, ny = c->ny;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const int iw = i - 1 > 0 ? i - 1 : 0, ie = i + 1 < nx - 1 ? i + 1 : nx - 1;
            const int js = j - 1 > 0 ? j - 1 : 0, jn = j + 1 < ny - 1 ? j + 1 : ny - 1;
            const size_t k = (size_t)j * nx + i;
            c->dzdx[k] = (c->z[(size_t)j * nx + ie] - c->z[(size_t)j * nx + iw]) / (2.0 * c->g.dx);
            c->dzdy[k] = (c->z[(size_t)jn * nx + i] - c->z[(size_t)js * nx + i]) / (2.0 * c->g.dy);
        }
}

static int is_finite(double x) { return isfinite(x); }

/* executor.hpp:1091-1104 finish_dt */
static double finish_dt(swo_ctx* c, double core, long long bad, double t_commit) {
    if (bad >= 0) {
        fail(c, SWE_ERR_INSTABILITY, (int)(bad % c->nx), (int)(bad / c->nx), t_commit,
             "non-finite wave speed in dt reduction");
        return 0.0;
    }
    const double dt_raw = std_min(c->pol.cfl * core, c->pol.dt_max);
    if (dt_raw < c->pol.dt_min) {
        char m[200];
        snprintf(m, sizeof m, "next step size %f collapsed below dt_min %f", dt_raw, c->pol.dt_min);
        fail(c, SWE_ERR_STEP_COLLAPSE, -1, -1, t_commit, m);
        c->st.dt = dt_raw;
    }
    return dt_raw;
}

/* executor.hpp:560-580 min_dt_rows_buf (also timestep.hpp:83-105) */
static double min_dt_buf(swo_ctx* c, double* const* s, long long* bad) {
    double m = INFINITY;
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            const cv u = get(c, s, i, j);
            const double cc = sqrt(c->p.g * u.h);
            const double sx = fabs(u.qx / u.h) + cc;
            const double sy = fabs(u.qy / u.h) + cc;
            const double r = std_min(c->g.dx / sx, c->g.dy / sy);
            if (!(r > 0.0) || !is_finite(r)) {
                if (*bad < 0) *bad = (long long)j * c->nx + i;
                continue;
            }
            if (r < m) m = r;
        }
    return m;
}

static void guard_msg(swo_ctx* c, const char* prefix, int i, int j, cv u, double t) {
    char m[256];
    snprintf(m, sizeof m, "%scell (%d, %d) at t=%f: h=%f qx=%f qy=%f", prefix, i, j, t, u.h, u.qx, u.qy);
    fail(c, SWE_ERR_INSTABILITY, i, j, t, m);
    c->st.h = u.h; c->st.qx = u.qx; c->st.qy = u.qy;
}

/* executor.hpp:543-556 guard_rows_buf */
static int guard_buf(swo_ctx* c, double* const* s, double t, const char* prefix) {
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            const cv u = get(c, s, i, j);
            const int ok = is_finite(u.h) && is_finite(u.qx) && is_finite(u.qy) && u.h >= c->pol.h_min;
            if (!ok) { guard_msg(c, prefix, i, j, u, t); return 1; }
        }
    return 0;
}

static void set_status(swo_ctx* c, swe_status* st) {
    if (st) { if (c->err) *st = c->st; else memset(st, 0, sizeof *st); }
}

/* ---------------------------------------------------------------------- */

EXPORT swo_ctx* swo_create(const swe_grid* g, const swe_physics* p, const swe_policy* pol,
                           const swe_boundary_set* b) {
    swo_ctx* c = (swo_ctx*)calloc(1, sizeof *c);
    c->g = *g; c->p = *p; c->pol = *pol; c->b = *b;
    c->nx = g->nx; c->ny = g->ny; c->W = g->nx + 2;
    const size_t n = (size_t)g->nx * g->ny, nb = (size_t)(g->nx + 2) * (g->ny + 2);
    c->z = calloc(n, 8); c->dzdx = calloc(n, 8); c->dzdy = calloc(n, 8);
    for (int f = 0; f < 3; ++f) {
        c->cur[f] = calloc(nb, 8); c->star[f] = calloc(nb, 8); c->next[f] = calloc(nb, 8);
        c->aux[f] = calloc(nb, 8);
    }
    return c;
}

EXPORT void swo_destroy(swo_ctx* c) {
    if (!c) return;
    free(c->z); free(c->dzdx); free(c->dzdy);
    for (int f = 0; f < 3; ++f) { free(c->cur[f]); free(c->star[f]); free(c->next[f]); free(c->aux[f]); }
    free(c);
}

/* executor.hpp:764-780 */
EXPORT void swo_load(swo_ctx* c, const double* z, const double* h, const double* qx, const double* qy, double t) {
    const int nx = c->nx, ny = c->ny;
    memcpy(c->z, z, (size_t)nx * ny * 8);
    make_slopes(c);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)j * nx + i;
            cv u = {h[k], qx[k], qy[k]};
            put(c, c->cur, i, j, u);
        }
    c->t = t;
    c->loaded = 1;
}

/* executor.hpp:783-797 */
EXPORT void swo_state(swo_ctx* c, double* h, double* qx, double* qy, double* t) {
    const int nx = c->nx, ny = c->ny;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)j * nx + i;
            const cv u = get(c, c->cur, i, j);
            if (h) h[k] = u.h;
            if (qx) qx[k] = u.qx;
            if (qy) qy[k] = u.qy;
        }
    if (t) *t = c->t;
}

EXPORT double swo_time(swo_ctx* c) { return c->t; }
EXPORT int swo_guard_warnings(swo_ctx* c) { return c->warnings_total; }

/* executor.hpp:812-911 step + step_single (naive strategy) */
EXPORT int swo_step(swo_ctx* c, double dt, uint64_t step_index, double t_after, double* dt_next,
                    int* warnings, swe_status* st) {
    c->err = 0;
    if (!c->loaded) { fail(c, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::step: no state loaded"); set_status(c, st); return c->err; }
    if (!(dt > 0.0) || !is_finite(dt)) { fail(c, SWE_ERR_CONFIG, -1, -1, 0, "Stepper::step: dt must be positive and finite"); set_status(c, st); return c->err; }
    const double t_commit = is_finite(t_after) ? t_after : c->t + dt;
    const int fwd = (step_index % 2) == 0;
    const int nx = c->nx, ny = c->ny;
    const int smoothing = c->p.nu_art > 0.0;
    int warn = 0;
    double** cand = smoothing ? c->aux : c->next;

    /* K1 */
    warn += fill_ghosts(c, c->cur);
    /* K2 */
    const int di = fwd ? 1 : -1;
    for (int j = 0; j < ny && !c->err; ++j)
        for (int i = 0; i < nx && !c->err; ++i) {
            const size_t k = (size_t)j * nx + i;
            put(c, c->star, i, j, predictor_cell(c, get(c, c->cur, i, j), get(c, c->cur, i + di, j),
                                                 get(c, c->cur, i, j + di), c->dzdx[k], c->dzdy[k], dt, fwd));
        }
    if (c->err) { set_status(c, st); return c->err; }
    /* K3 */
    warn += fill_ghosts(c, c->star);
    /* K4 */
    for (int j = 0; j < ny && !c->err; ++j)
        for (int i = 0; i < nx && !c->err; ++i) put(c, c->next, i, j, corrector_at(c, i, j, dt, fwd, t_commit));
    if (c->err) { set_status(c, st); return c->err; }
    if (smoothing) {
        warn += fill_ghosts(c, c->next);
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                put(c, c->aux, i, j, smooth_cell(get(c, c->next, i, j), get(c, c->next, i + 1, j), get(c, c->next, i - 1, j),
                                                 get(c, c->next, i, j + 1), get(c, c->next, i, j - 1), c->p.nu_art));
    }
    /* K5 */
    if (guard_buf(c, cand, t_commit, "instability: ")) { set_status(c, st); return c->err; }
    /* K6 */
    long long bad = -1;
    const double core = min_dt_buf(c, cand, &bad);
    const double dtn = finish_dt(c, core, bad, t_commit);
    if (c->err) { set_status(c, st); return c->err; }
    /* commit (executor.hpp:836-840) */
    for (int f = 0; f < 3; ++f) { double* tmp = c->cur[f]; c->cur[f] = cand[f]; cand[f] = tmp; }
    c->t = t_commit;
    c->warnings_total += warn;
    if (dt_next) *dt_next = dtn;
    if (warnings) *warnings = warn;
    set_status(c, st);
    return SWE_OK;
}

/* timestep.hpp:128-179 compute_dt on the committed state (serial band) */
EXPORT int swo_compute_dt(swo_ctx* c, double t_end, double* dt, swe_status* st) {
    c->err = 0;
    long long bad = -1;
    const double core = min_dt_buf(c, c->cur, &bad);
    if (bad >= 0) {
        fail(c, SWE_ERR_INSTABILITY, (int)(bad % c->nx), (int)(bad / c->nx), c->t, "compute_dt: non-finite wave speed");
        set_status(c, st);
        return c->err;
    }
    const double dt_raw = std_min(c->pol.cfl * core, c->pol.dt_max);
    if (dt_raw < c->pol.dt_min) {
        char m[200];
        snprintf(m, sizeof m, "compute_dt: step size %f collapsed below dt_min %f", dt_raw, c->pol.dt_min);
        fail(c, SWE_ERR_STEP_COLLAPSE, -1, -1, c->t, m);
        c->st.dt = dt_raw;
        set_status(c, st);
        return c->err;
    }
    *dt = std_min(dt_raw, t_end - c->t);
    set_status(c, st);
    return SWE_OK;
}

/* timestep.hpp:112-115 stability_guard on the committed state */
EXPORT int swo_guard(swo_ctx* c, swe_status* st) {
    c->err = 0;
    fill_ghosts(c, c->cur); /* harmless; ghosts are not scanned */
    guard_buf(c, c->cur, c->t, "");
    set_status(c, st);
    return c->err;
}

/* run.hpp:101-179 run_from hot loop (no snapshots) */
EXPORT int swo_advance(swo_ctx* c, double t_end, uint64_t step_index0, double dt_first, uint64_t max_steps,
                       swe_run_result* res, swe_status* st) {
    memset(res, 0, sizeof *res);
    uint64_t step_index = step_index0;
    double t = c->t;
    double dt_raw;
    if (is_finite(dt_first)) dt_raw = dt_first;
    else if (t < t_end) {
        int rc = swo_compute_dt(c, INFINITY, &dt_raw, st);
        if (rc) return rc;
    } else dt_raw = 0.0;
    while (t < t_end && (max_steps == 0 || res->steps < max_steps)) {
        const double remaining = t_end - t;
        const int landing = dt_raw >= remaining;
        const double dt = landing ? remaining : dt_raw;
        const double t_after = landing ? t_end : t + dt;
        double dtn; int w;
        int rc = swo_step(c, dt, step_index, t_after, &dtn, &w, st);
        if (rc) { res->step_index = step_index; res->t_final = c->t; res->dt_next = dt_raw; return rc; }
        ++step_index; ++res->steps;
        res->guard_warnings += w;
        t = c->t;
        dt_raw = dtn;
    }
    res->step_index = step_index;
    res->t_final = t;
    res->dt_next = dt_raw;
    if (st) memset(st, 0, sizeof *st);
    return SWE_OK;
}

/* ---- initial conditions (scenarios.hpp:95-171), test fixtures only ---- */

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) ? -1 : (y < x) ? 1 : 0;
}

/* kind: 0 flat_pool, 1 drops, 2 channel_slope, 3 vortex, 4 dam_break.
 * drops: ndrops x {cx, cy, radius, amplitude}. */
EXPORT void swo_build_initial(const swe_grid* g, int kind, double depth, const double* drops, int ndrops,
                              double slope, double center_x, double center_y, double v_peak, double core_radius,
                              double split_x, double h_left, double h_right,
                              double* z, double* h, double* qx, double* qy) {
    const int nx = g->nx, ny = g->ny;
    const size_t n = (size_t)nx * ny;
    memset(z, 0, n * 8); memset(h, 0, n * 8); memset(qx, 0, n * 8); memset(qy, 0, n * 8);
    double contrib[64];
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)j * nx + i;
            switch (kind) {
                case 0: h[k] = depth; break;
                case 1: {
                    for (int d = 0; d < ndrops; ++d) {
                        const double cx = drops[4 * d], cy = drops[4 * d + 1], r = drops[4 * d + 2], a = drops[4 * d + 3];
                        const double di = i - cx, dj = j - cy;
                        contrib[d] = a * exp(-(di * di + dj * dj) / (r * r));
                    }
                    qsort(contrib, (size_t)ndrops, sizeof(double), cmp_double);
                    double bump = 0.0;
                    for (int d = 0; d < ndrops; ++d) bump += contrib[d];
                    h[k] = depth + bump;
                    break;
                }
                case 2: {
                    const double zz = slope * g->dx * (double)(nx - 1 - i);
                    z[k] = zz; h[k] = depth - zz;
                    break;
                }
                case 3: {
                    const double di = i - center_x, dj = j - center_y;
                    const double r2 = (di * di + dj * dj) / (core_radius * core_radius);
                    const double shape = v_peak * exp(0.5 * (1.0 - r2)) / core_radius;
                    h[k] = depth; qx[k] = depth * (-shape * dj); qy[k] = depth * (shape * di);
                    break;
                }
                default: {
                    const double x = (i + 0.5) * g->dx;
                    h[k] = (x < split_x) ? h_left : h_right;
                    break;
                }
            }
        }
}
