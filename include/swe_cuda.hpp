// swe_cuda.hpp — header-only C++ shim over the libswe_cuda.so C-ABI that
// re-exposes the reference's swe::Stepper interface
// (/root/reference/proj/include/swe/executor.hpp:726-1116) and rethrows the
// reference's exception types (errors.hpp:17-61).  Tests can template over
// swe::Stepper and swe_b200::Stepper because the member signatures match.
//
//   swe_b200::Stepper st(spec, phys, pol, bounds, swe_b200::ExecutorKind::cuda());
//   st.load(fs);
//   swe_b200::StepResult r = st.step(dt, step_index);      // executor.hpp:812
//   swe_b200::FieldSet out = st.state();                   // executor.hpp:783
#pragma once

#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "swe_cuda.h"

namespace swe_b200 {

// ---- errors.hpp:9-61 ----------------------------------------------------
class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class InstabilityError : public std::runtime_error {
public:
    InstabilityError(const std::string& m, int i, int j, double t) : std::runtime_error(m), i_(i), j_(j), t_(t) {}
    int cell_i() const { return i_; }
    int cell_j() const { return j_; }
    double sim_time() const { return t_; }

private:
    int i_, j_;
    double t_;
};
class StepCollapseError : public std::runtime_error {
public:
    StepCollapseError(const std::string& m, double dt, double t) : std::runtime_error(m), dt_(dt), t_(t) {}
    double dt() const { return dt_; }
    double sim_time() const { return t_; }

private:
    double dt_, t_;
};
class IoError : public std::runtime_error {
public:
    explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void throw_status(const swe_status& st) {
    const std::string m(st.msg);
    switch (st.code) {
        case SWE_ERR_CONFIG: throw ConfigError(m);
        case SWE_ERR_INSTABILITY: throw InstabilityError(m, st.i, st.j, st.t);
        case SWE_ERR_STEP_COLLAPSE: throw StepCollapseError(m, st.dt, st.t);
        case SWE_ERR_IO: throw IoError(m);
        default: throw DeviceError(m);
    }
}

// ---- grid.hpp / scheme.hpp / timestep.hpp value types ---------------------
struct GridSpec {
    int nx = 0, ny = 0;
    double dx = 1.0, dy = 1.0;
    GridSpec() = default;
    GridSpec(int nx_, int ny_, double dx_, double dy_) : nx(nx_), ny(ny_), dx(dx_), dy(dy_) {
        if (nx < 3 || ny < 3) throw ConfigError("GridSpec: nx and ny must be at least 3");
        if (!(dx > 0.0) || !(dy > 0.0) || !std::isfinite(dx) || !std::isfinite(dy))
            throw ConfigError("GridSpec: dx and dy must be positive and finite");
    }
    std::size_t cell_count() const { return static_cast<std::size_t>(nx) * static_cast<std::size_t>(ny); }
    bool operator==(const GridSpec&) const = default;
};

struct PhysicsParams {
    double g = 9.81, manning_n = 0.0, nu_art = 0.0;
};

struct StabilityPolicy {
    double cfl = 0.9;
    double dt_max = std::numeric_limits<double>::infinity();
    double dt_min = 1e-9;
    double h_min = 1e-6;
};

struct BoundaryKind {
    enum class Type { reflective_wall, transmissive, inflow_discharge, fixed_elevation };
    Type type = Type::reflective_wall;
    double q_n = 0.0, h_in = 0.0, eta_out = 0.0;
    static BoundaryKind wall() { return {}; }
    static BoundaryKind transmissive() { return {Type::transmissive, 0.0, 0.0, 0.0}; }
    static BoundaryKind inflow(double q, double h) { return {Type::inflow_discharge, q, h, 0.0}; }
    static BoundaryKind fixed_eta(double e) { return {Type::fixed_elevation, 0.0, 0.0, e}; }
};

struct BoundarySet {
    BoundaryKind north, south, east, west;
    static BoundarySet all(BoundaryKind b) { return {b, b, b, b}; }
};

struct FieldSet {
    GridSpec spec;
    std::vector<double> z, h, qx, qy;
    double t = 0.0;
    FieldSet() = default;
    explicit FieldSet(const GridSpec& s)
        : spec(s), z(s.cell_count(), 0.0), h(s.cell_count(), 0.0), qx(s.cell_count(), 0.0),
          qy(s.cell_count(), 0.0) {}
};

struct StepResult {
    double dt_used = 0.0;
    double dt_next = 0.0;
    int guard_warnings = 0;
};

struct RunResult {
    unsigned long long steps = 0, step_index = 0;
    double t_final = 0.0, dt_next = 0.0;
    int guard_warnings = 0;
};

// The new `cuda` strategy of ExecutorKind (executor.hpp:27-67).
struct ExecutorKind {
    int device = 0;
    bool exact = true;  // -fmad=false expression trees: bit-identical to the reference
    bool graph = true;
    bool early_exit = false;  // skip quiet items on a flat bed (bit-exact)
    bool local_group = false; // strips as contexts of one process on one device (SWE_EXEC_LOCAL_GROUP)
    int rank = 0, nranks = 1;
    const void* nccl_id = nullptr;
    static ExecutorKind cuda(int device = 0, bool exact = true) {
        ExecutorKind k;
        k.device = device;
        k.exact = exact;
        return k;
    }
    std::string name() const {
        return std::string("cuda") + (nranks > 1 ? ":" + std::to_string(nranks) : std::string()) +
               (exact ? "" : ":fast") + (early_exit ? ":early" : "");
    }
};

// StepTimings (executor.hpp:153-172): the six plan kernels run fused in one
// launch, so their device time is reported as fused_seconds.
struct StepTimings {
    double kernel_seconds[6] = {0, 0, 0, 0, 0, 0};
    double smooth_seconds = 0.0, exchange_seconds = 0.0, fused_seconds = 0.0;
    unsigned long long steps = 0;
    double total() const {
        double s = smooth_seconds + exchange_seconds + fused_seconds;
        for (double k : kernel_seconds) s += k;
        return s;
    }
};
struct StepAccounting {  // executor.hpp:218-222
    long long halo_values_exchanged = 0;
    int redundant_star_rows = 0;
    int redundant_corrector_rows = 0;
};
// StepPlan (executor.hpp:134-148): K1..K6 (+ smoothing), all in one launch here
inline std::vector<std::string> step_plan(bool smoothing) {
    std::vector<std::string> k = {"k1_ghost_committed", "k2_predictor", "k3_ghost_star", "k4_corrector"};
    if (smoothing) k.push_back("smooth");
    k.push_back("k5_guard");
    k.push_back("k6_dt_reduce");
    return k;
}

// ---- swe::Stepper ----------------------------------------------------------
class Stepper {
public:
    Stepper(const GridSpec& spec, const PhysicsParams& phys, const StabilityPolicy& pol, const BoundarySet& b,
            const ExecutorKind& kind = ExecutorKind::cuda())
        : spec_(spec), kind_(kind), nu_art_(phys.nu_art) {
        const swe_grid g{spec.nx, spec.ny, spec.dx, spec.dy};
        const swe_physics p{phys.g, phys.manning_n, phys.nu_art};
        const swe_policy po{pol.cfl, pol.dt_max, pol.dt_min, pol.h_min};
        const swe_boundary_set bs{conv(b.north), conv(b.south), conv(b.east), conv(b.west)};
        swe_exec ex{};
        ex.device = kind.device;
        ex.flags = (kind.exact ? SWE_EXEC_EXACT : 0u) | (kind.graph ? 0u : SWE_EXEC_NO_GRAPH) |
                   (kind.early_exit ? SWE_EXEC_EARLY_EXIT : 0u) | (kind.local_group ? SWE_EXEC_LOCAL_GROUP : 0u);
        ex.rank = kind.rank;
        ex.nranks = kind.nranks;
        ex.nccl_id = kind.nccl_id;
        swe_status st{};
        if (swe_cuda_create(&g, &p, &po, &bs, &ex, &ctx_, &st) != SWE_OK) {
            if (ctx_) swe_cuda_destroy(ctx_);
            ctx_ = nullptr;
            throw_status(st);
        }
        swe_cuda_rows(ctx_, &row_begin_, &row_end_);
    }
    ~Stepper() {
        if (ctx_) swe_cuda_destroy(ctx_);
    }
    Stepper(const Stepper&) = delete;
    Stepper& operator=(const Stepper&) = delete;

    // executor.hpp:764-780 (this rank's rows on a strip)
    void load(const FieldSet& fs) {
        if (!(fs.spec == spec_)) throw ConfigError("Stepper::load: grid mismatch");
        const std::size_t off = static_cast<std::size_t>(row_begin_) * spec_.nx;
        swe_status st{};
        if (swe_cuda_load(ctx_, fs.z.data() + off, fs.h.data() + off, fs.qx.data() + off, fs.qy.data() + off, fs.t,
                          &st) != SWE_OK)
            throw_status(st);
        z_ = fs.z;
    }

    // build_initial_state (scenarios.hpp:95-171) + load, generated on the device
    // (flat_pool / channel_slope / dam_break; SWE_IC_* kinds)
    void load_initial(const swe_initial& ic, double t = 0.0) {
        swe_status st{};
        if (swe_cuda_load_initial(ctx_, &ic, t, &st) != SWE_OK) throw_status(st);
        z_.assign(static_cast<std::size_t>(spec_.nx) * spec_.ny, 0.0);
        const std::size_t off = static_cast<std::size_t>(row_begin_) * spec_.nx;
        if (swe_cuda_state(ctx_, z_.data() + off, nullptr, nullptr, nullptr, nullptr, &st) != SWE_OK)
            throw_status(st);
    }

    // executor.hpp:783-797
    FieldSet state() const {
        FieldSet fs(spec_);
        fs.z = z_;
        const std::size_t off = static_cast<std::size_t>(row_begin_) * spec_.nx;
        swe_status st{};
        if (swe_cuda_state(ctx_, nullptr, fs.h.data() + off, fs.qx.data() + off, fs.qy.data() + off, &fs.t, &st) !=
            SWE_OK)
            throw_status(st);
        return fs;
    }

    double time() const { return swe_cuda_time(ctx_); }
    // executor.hpp:801-804
    const ExecutorKind& kind() const { return kind_; }
    std::vector<std::string> plan() const { return step_plan(nu_art_ > 0.0); }
    StepTimings timings() const {
        swe_timing t{};
        swe_cuda_timing(ctx_, &t);
        StepTimings o;
        o.fused_seconds = t.step_seconds;
        o.steps = t.steps;
        return o;
    }
    StepAccounting accounting() const {
        swe_accounting a{};
        swe_cuda_accounting(ctx_, &a);
        return {a.halo_values_exchanged, a.redundant_star_rows, a.redundant_corrector_rows};
    }
    int guard_warnings() const { return swe_cuda_guard_warnings(ctx_); }

    // executor.hpp:812-841
    StepResult step(double dt, unsigned long long step_index,
                    double t_after = std::numeric_limits<double>::quiet_NaN()) {
        swe_step_result r{};
        swe_status st{};
        if (swe_cuda_step(ctx_, dt, step_index, t_after, &r, &st) != SWE_OK) throw_status(st);
        return {r.dt_used, r.dt_next, r.guard_warnings};
    }

    // compute_dt (timestep.hpp:128-179) on the committed state
    double compute_dt(double t_end) const {
        double dt = 0.0;
        swe_status st{};
        if (swe_cuda_compute_dt(ctx_, t_end, &dt, &st) != SWE_OK) throw_status(st);
        return dt;
    }

    // The run_from loop (run.hpp:149-163), device resident.
    RunResult advance(double t_end, unsigned long long step_index0 = 0,
                      double dt_first = std::numeric_limits<double>::quiet_NaN(), unsigned long long max_steps = 0) {
        swe_run_result r{};
        swe_status st{};
        const int rc = swe_cuda_advance(ctx_, t_end, step_index0, dt_first, max_steps, &r, &st);
        last_ = {r.steps, r.step_index, r.t_final, r.dt_next, r.guard_warnings};
        if (rc != SWE_OK) throw_status(st);
        return last_;
    }
    // advance() that also stops after the first committed step with t >= t_mark
    // (run_from's snapshot cadence, run.hpp:159-163)
    RunResult advance_marked(double t_end, double t_mark, unsigned long long step_index0, double dt_first,
                             unsigned long long max_steps = 0) {
        swe_run_result r{};
        swe_status st{};
        const int rc = swe_cuda_advance_marked(ctx_, t_end, t_mark, step_index0, dt_first, max_steps, &r, &st);
        last_ = {r.steps, r.step_index, r.t_final, r.dt_next, r.guard_warnings};
        if (rc != SWE_OK) throw_status(st);
        return last_;
    }
    // stability_guard (timestep.hpp:112-115) on the committed state
    void guard() const {
        swe_status st{};
        if (swe_cuda_guard(ctx_, &st) != SWE_OK) throw_status(st);
    }
    int row_begin() const { return row_begin_; }
    int row_end() const { return row_end_; }
    const RunResult& last_run() const { return last_; }
    swe_ctx* handle() const { return ctx_; }

private:
    static swe_boundary conv(const BoundaryKind& b) {
        swe_boundary o{};
        o.type = static_cast<int32_t>(b.type);
        o.q_n = b.q_n;
        o.h_in = b.h_in;
        o.eta_out = b.eta_out;
        return o;
    }
    GridSpec spec_;
    ExecutorKind kind_;
    double nu_art_ = 0.0;
    swe_ctx* ctx_ = nullptr;
    int32_t row_begin_ = 0, row_end_ = 0;
    std::vector<double> z_;
    RunResult last_{};
};

}  // namespace swe_b200
