// shim_test.cpp — exercises include/swe_cuda.hpp (the C++ Stepper shim) on a
// GPU: step()/advance() equivalence, landing on t_end, error mapping and
// failure atomicity, mirroring test_executor.cpp / test_run.cpp cases.
// Built by __graft_entry__.build(); run by tests/test_gpu_parity.py.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/swe_cuda.hpp"

using namespace swe_b200;

static int failures = 0;
#define CHECK(c)                                                               \
    do {                                                                       \
        if (!(c)) {                                                            \
            std::printf("CHECK failed: %s (%s:%d)\n", #c, __FILE__, __LINE__); \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static FieldSet dam(int n, double hl, double hr) {
    FieldSet fs(GridSpec(n, n, 1.0, 1.0));
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) fs.h[static_cast<std::size_t>(j) * n + i] = ((i + 0.5) < 0.5 * n) ? hl : hr;
    return fs;
}

int main() {
    StabilityPolicy pol;
    pol.cfl = 0.45;
    const PhysicsParams phys;
    const BoundarySet walls = BoundarySet::all(BoundaryKind::wall());
    const FieldSet ic = dam(96, 1.0, 0.5);

    // step() loop == advance() (device-resident run_from), bit for bit
    Stepper a(ic.spec, phys, pol, walls), b(ic.spec, phys, pol, walls);
    a.load(ic);
    b.load(ic);
    double dt = a.compute_dt(1e18);
    for (int k = 0; k < 37; ++k) dt = a.step(dt, static_cast<unsigned long long>(k)).dt_next;
    const RunResult r = b.advance(1e18, 0, std::numeric_limits<double>::quiet_NaN(), 37);
    CHECK(r.steps == 37);
    CHECK(r.step_index == 37);
    CHECK(r.dt_next == dt);
    const FieldSet sa = a.state(), sb = b.state();
    CHECK(sa.t == sb.t);
    CHECK(std::memcmp(sa.h.data(), sb.h.data(), sa.h.size() * 8) == 0);
    CHECK(std::memcmp(sa.qx.data(), sb.qx.data(), sa.qx.size() * 8) == 0);

    // landing exactly on t_end (run.hpp:150-153, test_run.cpp:29-46)
    Stepper c(ic.spec, phys, pol, walls);
    c.load(ic);
    const RunResult rc = c.advance(3.0);
    CHECK(rc.t_final == 3.0);
    CHECK(c.time() == 3.0);

    // dt must be positive and finite (executor.hpp:817-819)
    bool threw = false;
    try {
        a.step(-1.0, 0);
    } catch (const ConfigError&) {
        threw = true;
    }
    CHECK(threw);

    // engineered dry shelf: InstabilityError with a cell and t > 0, committed
    // state unchanged (test_executor.cpp:349-375)
    FieldSet shelf(GridSpec(48, 3, 1.0, 1.0));
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 48; ++i) shelf.h[static_cast<std::size_t>(j) * 48 + i] = ((i + 0.5) < 24.0) ? 1.0 : 1e-4;
    BoundarySet chan = walls;
    chan.north = BoundaryKind::transmissive();
    chan.south = BoundaryKind::transmissive();
    Stepper s(shelf.spec, phys, pol, chan);
    s.load(shelf);
    double d = s.compute_dt(1e9);
    bool failed = false;
    for (int k = 0; k < 200 && !failed; ++k) {
        const FieldSet before = s.state();
        try {
            d = s.step(d, static_cast<unsigned long long>(k)).dt_next;
        } catch (const InstabilityError& e) {
            failed = true;
            CHECK(e.cell_i() >= 0);
            CHECK(e.cell_j() >= 0);
            CHECK(e.sim_time() > 0.0);
            const FieldSet after = s.state();
            CHECK(std::memcmp(before.h.data(), after.h.data(), before.h.size() * 8) == 0);
            CHECK(before.t == after.t);
        }
    }
    CHECK(failed);

    std::printf("%s: %d failures\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
