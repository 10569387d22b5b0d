// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference solver
// (swe::Stepper, swe::compute_dt, swe::build_initial_state, swe::snapshot_bytes
// from /root/reference/proj/include/swe/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libswe_ref.so.  No reference source is
// copied into this repository; this file only calls the reference's public API.
//
// Used (a) to generate/validate golden fixtures (tests/golden/make_golden.py),
// (b) to pin the C restatement oracle/swe_oracle.c, and (c) as the timed CPU
// baseline (bench.py --impl reference, cpu_baseline.kind = "reference").
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>

#include "swe/executor.hpp"
#include "swe/io.hpp"
#include "swe/run.hpp"
#include "swe/scenarios.hpp"
#include "swe/timestep.hpp"

#include "../include/swe_cuda.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

swe::BoundaryKind to_bk(const swe_boundary& b) {
    switch (b.type) {
        case SWE_BC_WALL: return swe::BoundaryKind::wall();
        case SWE_BC_TRANSMISSIVE: return swe::BoundaryKind::transmissive();
        case SWE_BC_INFLOW: return swe::BoundaryKind::inflow(b.q_n, b.h_in);
        default: return swe::BoundaryKind::fixed_eta(b.eta_out);
    }
}

swe::BoundarySet to_bs(const swe_boundary_set& b) {
    return {to_bk(b.north), to_bk(b.south), to_bk(b.east), to_bk(b.west)};
}

// kind: 0 naive, 1 tiled(tile), 2 decomposed(workers, naive inner), 3 decomposed(workers, tiled inner)
swe::ExecutorKind to_kind(int kind, int workers, int tile) {
    switch (kind) {
        case 1: return swe::ExecutorKind::tiled(tile);
        case 2: return swe::ExecutorKind::decomposed(workers);
        case 3: return swe::ExecutorKind::decomposed(workers, swe::ExecutorKind::Inner::tiled, tile);
        default: return swe::ExecutorKind::naive();
    }
}

void fill_status(swe_status* st, int code, const std::exception* e) {
    if (!st) return;
    std::memset(st, 0, sizeof *st);
    st->code = code;
    st->i = -1;
    st->j = -1;
    if (e) std::snprintf(st->msg, sizeof st->msg, "%s", e->what());
    if (auto* ie = dynamic_cast<const swe::InstabilityError*>(e)) {
        st->i = ie->cell_i();
        st->j = ie->cell_j();
        st->t = ie->sim_time();
    } else if (auto* sc = dynamic_cast<const swe::StepCollapseError*>(e)) {
        st->dt = sc->dt();
        st->t = sc->sim_time();
    }
}

int code_of(const std::exception& e) { return static_cast<int>(swe::exit_code_for(e)); }

struct Ref {
    swe::GridSpec spec;
    swe::PhysicsParams phys;
    swe::StabilityPolicy pol;
    swe::BoundarySet bs;
    swe::Stepper stepper;
    Ref(const swe::GridSpec& s, const swe::PhysicsParams& p, const swe::StabilityPolicy& po,
        const swe::BoundarySet& b, const swe::ExecutorKind& k)
        : spec(s), phys(p), pol(po), bs(b), stepper(s, p, po, b, k) {}
};

}  // namespace

EXPORT void* swr_create(const swe_grid* g, const swe_physics* p, const swe_policy* pol,
                        const swe_boundary_set* b, int kind, int workers, int tile, swe_status* st) {
    try {
        swe::GridSpec spec(g->nx, g->ny, g->dx, g->dy);
        swe::PhysicsParams phys{p->g, p->manning_n, p->nu_art};
        swe::StabilityPolicy po{pol->cfl, pol->dt_max, pol->dt_min, pol->h_min};
        auto* r = new Ref(spec, phys, po, to_bs(*b), to_kind(kind, workers, tile));
        fill_status(st, 0, nullptr);
        return r;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return nullptr;
    }
}

EXPORT void swr_destroy(void* h) { delete static_cast<Ref*>(h); }

EXPORT int swr_load(void* hnd, const double* z, const double* h, const double* qx,
                    const double* qy, double t, swe_status* st) {
    auto* r = static_cast<Ref*>(hnd);
    try {
        swe::FieldSet fs(r->spec);
        const std::size_t n = r->spec.cell_count();
        std::memcpy(fs.z.data(), z, n * 8);
        std::memcpy(fs.h.data(), h, n * 8);
        std::memcpy(fs.qx.data(), qx, n * 8);
        std::memcpy(fs.qy.data(), qy, n * 8);
        fs.t = t;
        r->stepper.load(fs);
        fill_status(st, 0, nullptr);
        return 0;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return code_of(e);
    }
}

EXPORT void swr_state(void* hnd, double* h, double* qx, double* qy, double* t) {
    auto* r = static_cast<Ref*>(hnd);
    const swe::FieldSet fs = r->stepper.state();
    const std::size_t n = r->spec.cell_count();
    if (h) std::memcpy(h, fs.h.data(), n * 8);
    if (qx) std::memcpy(qx, fs.qx.data(), n * 8);
    if (qy) std::memcpy(qy, fs.qy.data(), n * 8);
    if (t) *t = fs.t;
}

EXPORT int swr_step(void* hnd, double dt, std::uint64_t step_index, double t_after,
                    double* dt_next, int* warnings, swe_status* st) {
    auto* r = static_cast<Ref*>(hnd);
    try {
        const swe::StepResult res = r->stepper.step(dt, step_index, t_after);
        if (dt_next) *dt_next = res.dt_next;
        if (warnings) *warnings = res.guard_warnings;
        fill_status(st, 0, nullptr);
        return 0;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return code_of(e);
    }
}

EXPORT double swr_time(void* hnd) { return static_cast<Ref*>(hnd)->stepper.time(); }

EXPORT int swr_compute_dt(void* hnd, double t_end, int workers, double* dt, swe_status* st) {
    auto* r = static_cast<Ref*>(hnd);
    try {
        *dt = swe::compute_dt(r->stepper.state(), r->pol, r->phys, t_end, workers);
        fill_status(st, 0, nullptr);
        return 0;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return code_of(e);
    }
}

EXPORT int swr_guard(void* hnd, swe_status* st) {
    auto* r = static_cast<Ref*>(hnd);
    const swe::GuardReport g = swe::stability_guard(r->stepper.state(), r->pol);
    if (g.pass) {
        fill_status(st, 0, nullptr);
        return 0;
    }
    swe::InstabilityError e("instability: " + g.describe(), g.i, g.j, g.t);
    fill_status(st, 3, &e);
    if (st) {
        st->h = g.h;
        st->qx = g.qx;
        st->qy = g.qy;
    }
    return 3;
}

EXPORT int swr_guard_warnings(void* hnd) { return static_cast<Ref*>(hnd)->stepper.guard_warnings(); }

// Scenario presets (scenarios.hpp:187-329): fills grid/physics/policy/bounds and the
// initial state for gen_<name>(n).  Arrays must hold nx*ny doubles; pass nullptr
// first to query the grid only.
EXPORT int swr_scenario(const char* name, int n, swe_grid* g, swe_physics* p, swe_policy* pol,
                        swe_boundary_set* b, double* t_end, double* z, double* h, double* qx,
                        double* qy, swe_status* st) {
    try {
        const swe::ScenarioConfig sc = swe::scenario_by_name(name, n);
        g->nx = sc.grid.nx;
        g->ny = sc.grid.ny;
        g->dx = sc.grid.dx;
        g->dy = sc.grid.dy;
        p->g = sc.physics.g;
        p->manning_n = sc.physics.manning_n;
        p->nu_art = sc.physics.nu_art;
        pol->cfl = sc.policy.cfl;
        pol->dt_max = sc.policy.dt_max;
        pol->dt_min = sc.policy.dt_min;
        pol->h_min = sc.policy.h_min;
        auto conv = [](const swe::BoundaryKind& k) {
            swe_boundary o{};
            o.type = static_cast<int>(k.type);
            o.q_n = k.q_n;
            o.h_in = k.h_in;
            o.eta_out = k.eta_out;
            return o;
        };
        b->north = conv(sc.boundaries.north);
        b->south = conv(sc.boundaries.south);
        b->east = conv(sc.boundaries.east);
        b->west = conv(sc.boundaries.west);
        *t_end = sc.t_end;
        if (h) {
            const swe::FieldSet fs = swe::build_initial_state(sc);
            const std::size_t cells = sc.grid.cell_count();
            std::memcpy(z, fs.z.data(), cells * 8);
            std::memcpy(h, fs.h.data(), cells * 8);
            std::memcpy(qx, fs.qx.data(), cells * 8);
            std::memcpy(qy, fs.qy.data(), cells * 8);
        }
        fill_status(st, 0, nullptr);
        return 0;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return code_of(e);
    }
}

// SWS1 bytes of (spec, t, z, h, qx, qy) via the reference writer (io.hpp:109-139).
// Returns the byte count; writes into out when out_cap is large enough.
EXPORT long long swr_snapshot_bytes(const swe_grid* g, double t, double gravity, const double* z,
                                    const double* h, const double* qx, const double* qy,
                                    char* out, long long out_cap) {
    swe::FieldSet fs(swe::GridSpec(g->nx, g->ny, g->dx, g->dy));
    const std::size_t n = fs.spec.cell_count();
    std::memcpy(fs.z.data(), z, n * 8);
    std::memcpy(fs.h.data(), h, n * 8);
    std::memcpy(fs.qx.data(), qx, n * 8);
    std::memcpy(fs.qy.data(), qy, n * 8);
    fs.t = t;
    const std::string bytes = swe::snapshot_bytes(fs, gravity);
    if (out && out_cap >= static_cast<long long>(bytes.size())) {
        std::memcpy(out, bytes.data(), bytes.size());
    }
    return static_cast<long long>(bytes.size());
}

// The reference's `run` subcommand body (tools/swe_main.cpp cmd_run): parse the
// config text, integrate to t_end writing SWS1 snapshots and the run report
// into out_dir (run.hpp:101-179).  The parity target of the C++ CLI.
EXPORT int swr_run_config(const char* text, const char* out_dir, double snapshot_every, swe_status* st) {
    try {
        swe::ScenarioConfig sc = swe::parse_config(text);
        sc.out_dir = out_dir;
        if (snapshot_every >= 0.0) sc.snapshot_every = snapshot_every;
        swe::run(sc, true);
        if (st) std::memset(st, 0, sizeof *st);
        return 0;
    } catch (const std::exception& e) {
        fill_status(st, code_of(e), &e);
        return code_of(e);
    }
}
