// swe_cuda_cli.cpp — the reference's command-line driver (proj/tools/swe_main.cpp)
// for the B200 executor: `run` integrates a scenario config to its end time
// writing SWS1 snapshots and the run report (run.hpp:101-179), `bench` times
// executors on five-drops grids and writes the bench CSV (bench.hpp:33-108).
//
// Host code in C++ over the C-ABI (include/swe_cuda.hpp).  The config grammar
// is the reference's (io.hpp:363-486) with the `cuda` executor added:
//
//   [executor]
//   kind = cuda            # naive | tiled | decomposed are accepted too: their
//   ranks = 4              # results are bit-identical to naive by contract, so
//   mode = fast            # they run as exact `cuda` (executor.hpp:913-1084)
//   early_exit = 1
//
//   --executor cuda[:N][:fast|:exact][:early][:local]
//
// N > 1 runs N row strips, one host thread and one GPU each (devices
// 0..N-1) over NCCL; `:local` keeps all strips on device 0 and exchanges
// through the local-group transport instead (single-GPU testing).
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <iterator>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "../../include/swe_cuda.hpp"

namespace {

using namespace swe_b200;

// ------------------------------------------------------------------ scenario
struct Drop {
    double cx = 0.0, cy = 0.0, radius = 1.0, amplitude = 0.0;
};

// InitialCondition (scenarios.hpp:17-42); kind follows InitialCondition::Kind
enum { IC_FLAT = 0, IC_DROPS = 1, IC_CHANNEL = 2, IC_VORTEX = 3, IC_DAM = 4 };
struct Initial {
    int kind = IC_FLAT;
    double depth = 1.0;
    std::vector<Drop> drops;
    double slope = 0.0, center_x = 0.0, center_y = 0.0, v_peak = 0.0, core_radius = 1.0;
    double split_x = 0.0, h_left = 1.0, h_right = 1.0;
};

struct Exec {
    int ranks = 1;
    bool exact = true, early = false, local = false;
    std::string name() const {
        std::string s = "cuda";
        if (ranks > 1) s += ":" + std::to_string(ranks);
        if (!exact) s += ":fast";
        if (early) s += ":early";
        if (local) s += ":local";
        return s;
    }
};

struct Scenario {  // ScenarioConfig (scenarios.hpp:57-70)
    std::string name = "unnamed";
    int nx = 65, ny = 65;
    double dx = 1.0, dy = 1.0;
    PhysicsParams phys;
    StabilityPolicy pol;
    Exec exec;
    BoundarySet bnd = BoundarySet::all(BoundaryKind::wall());
    double t_end = 1.0, snapshot_every = 0.0;
    Initial ic;
    std::string out_dir = "out";
};

[[noreturn]] void fail_line(int line, const std::string& msg) {
    throw ConfigError("config line " + std::to_string(line) + ": " + msg);
}

std::string strip(const std::string& s) {
    const auto a = s.find_first_not_of(" \t\r");
    if (a == std::string::npos) return {};
    return s.substr(a, s.find_last_not_of(" \t\r") - a + 1);
}

double num(const std::string& v, int line) {
    const std::string t = strip(v);
    char* end = nullptr;
    const double d = std::strtod(t.c_str(), &end);
    if (t.empty() || *end != '\0') fail_line(line, "expected a number, got '" + v + "'");
    return d;
}

long integer(const std::string& v, int line) {
    const std::string t = strip(v);
    char* end = nullptr;
    const long n = std::strtol(t.c_str(), &end, 10);
    if (t.empty() || *end != '\0') fail_line(line, "expected an integer, got '" + v + "'");
    return n;
}

std::vector<std::string> words(const std::string& s) {
    std::vector<std::string> out;
    std::istringstream in(s);
    for (std::string w; in >> w;) out.push_back(w);
    return out;
}

BoundaryKind boundary(const std::string& v, int line) {
    const auto w = words(v);
    if (w.empty()) fail_line(line, "empty boundary value");
    const std::size_t want = w[0] == "inflow" ? 3 : w[0] == "fixed_eta" ? 2 : 1;
    if (w[0] != "wall" && w[0] != "transmissive" && w[0] != "inflow" && w[0] != "fixed_eta")
        fail_line(line, "unknown boundary kind '" + w[0] + "'");
    if (w.size() != want) fail_line(line, "wrong parameter count for boundary '" + w[0] + "'");
    if (w[0] == "wall") return BoundaryKind::wall();
    if (w[0] == "transmissive") return BoundaryKind::transmissive();
    if (w[0] == "inflow") return BoundaryKind::inflow(num(w[1], line), num(w[2], line));
    return BoundaryKind::fixed_eta(num(w[1], line));
}

// `cuda[:N][:fast|:exact][:early][:local]`, or a CPU strategy of the reference
Exec parse_exec_spec(const std::string& spec) {
    std::vector<std::string> parts;
    std::istringstream in(spec);
    for (std::string p; std::getline(in, p, ':');) parts.push_back(p);
    if (parts.empty()) throw ConfigError("--executor: empty value");
    Exec e;
    if (parts[0] == "naive" || parts[0] == "tiled" || parts[0] == "decomposed") return e;  // bit-identical to naive
    if (parts[0] != "cuda") throw ConfigError("--executor: unknown strategy '" + parts[0] + "'");
    for (std::size_t k = 1; k < parts.size(); ++k) {
        const std::string& p = parts[k];
        if (p == "fast") e.exact = false;
        else if (p == "exact") e.exact = true;
        else if (p == "early") e.early = true;
        else if (p == "local") e.local = true;
        else if (!p.empty() && std::all_of(p.begin(), p.end(), ::isdigit) && k == 1) e.ranks = std::stoi(p);
        else throw ConfigError("--executor: bad cuda option '" + p + "'");
    }
    if (e.ranks < 1) throw ConfigError("--executor: cuda needs at least one rank");
    return e;
}

// parse_config (io.hpp:363-486) + the cuda executor keys
Scenario parse_config(const std::string& text) {
    Scenario sc;
    std::istringstream in(text);
    std::string raw, section;
    int line = 0;
    const char* sections[] = {"grid", "physics", "policy", "executor", "boundaries", "initial", "run"};
    while (std::getline(in, raw)) {
        ++line;
        const std::string l = strip(raw.substr(0, raw.find('#')));
        if (l.empty()) continue;
        if (l.front() == '[') {
            if (l.back() != ']') fail_line(line, "malformed section header");
            section = strip(l.substr(1, l.size() - 2));
            if (std::none_of(std::begin(sections), std::end(sections), [&](const char* s) { return section == s; }))
                fail_line(line, "unknown section '" + section + "'");
            continue;
        }
        const auto eq = l.find('=');
        if (eq == std::string::npos) fail_line(line, "expected 'key = value'");
        const std::string key = strip(l.substr(0, eq)), val = strip(l.substr(eq + 1));
        if (section.empty()) fail_line(line, "key '" + key + "' outside any section");
        auto unknown = [&] { fail_line(line, "unknown key '" + key + "' in [" + section + "]"); };
        if (section == "grid") {
            if (key == "nx") sc.nx = static_cast<int>(integer(val, line));
            else if (key == "ny") sc.ny = static_cast<int>(integer(val, line));
            else if (key == "dx") sc.dx = num(val, line);
            else if (key == "dy") sc.dy = num(val, line);
            else unknown();
        } else if (section == "physics") {
            if (key == "g") sc.phys.g = num(val, line);
            else if (key == "manning_n") sc.phys.manning_n = num(val, line);
            else if (key == "nu_art") {
                sc.phys.nu_art = num(val, line);
                if (!(sc.phys.nu_art >= 0.0 && sc.phys.nu_art < 0.5)) fail_line(line, "nu_art must lie in [0, 0.5)");
            } else unknown();
        } else if (section == "policy") {
            if (key == "cfl") {
                sc.pol.cfl = num(val, line);
                if (!(sc.pol.cfl > 0.0 && sc.pol.cfl <= 1.0)) fail_line(line, "cfl must lie in (0, 1]");
            } else if (key == "dt_max") sc.pol.dt_max = num(val, line);
            else if (key == "dt_min") sc.pol.dt_min = num(val, line);
            else if (key == "h_min") sc.pol.h_min = num(val, line);
            else unknown();
        } else if (section == "executor") {
            if (key == "kind") {
                if (val == "cuda" || val == "naive" || val == "tiled" || val == "decomposed") {
                    if (val != "cuda") sc.exec = Exec{};
                } else fail_line(line, "unknown executor kind '" + val + "'");
            } else if (key == "tile" || key == "workers" || key == "inner") {
                (void)val;  // CPU strategy parameters: no effect on the results, kept for compatibility
            } else if (key == "ranks") sc.exec.ranks = static_cast<int>(integer(val, line));
            else if (key == "mode") {
                if (val == "exact") sc.exec.exact = true;
                else if (val == "fast") sc.exec.exact = false;
                else fail_line(line, "mode must be exact or fast");
            } else if (key == "early_exit") sc.exec.early = integer(val, line) != 0;
            else unknown();
        } else if (section == "boundaries") {
            if (key == "north") sc.bnd.north = boundary(val, line);
            else if (key == "south") sc.bnd.south = boundary(val, line);
            else if (key == "east") sc.bnd.east = boundary(val, line);
            else if (key == "west") sc.bnd.west = boundary(val, line);
            else unknown();
        } else if (section == "initial") {
            if (key == "kind") {
                const char* kinds[] = {"flat_pool", "drops", "channel_slope", "vortex", "dam_break"};
                const auto it = std::find_if(std::begin(kinds), std::end(kinds), [&](const char* k) { return val == k; });
                if (it == std::end(kinds)) fail_line(line, "unknown initial kind '" + val + "'");
                sc.ic.kind = static_cast<int>(it - std::begin(kinds));
            } else if (key == "depth") sc.ic.depth = num(val, line);
            else if (key == "drop") {
                const auto w = words(val);
                if (w.size() != 4) fail_line(line, "drop needs: drop CX CY RADIUS AMPLITUDE");
                sc.ic.drops.push_back({num(w[0], line), num(w[1], line), num(w[2], line), num(w[3], line)});
            } else if (key == "slope") sc.ic.slope = num(val, line);
            else if (key == "center_x") sc.ic.center_x = num(val, line);
            else if (key == "center_y") sc.ic.center_y = num(val, line);
            else if (key == "v_peak") sc.ic.v_peak = num(val, line);
            else if (key == "core_radius") sc.ic.core_radius = num(val, line);
            else if (key == "split_x") sc.ic.split_x = num(val, line);
            else if (key == "h_left") sc.ic.h_left = num(val, line);
            else if (key == "h_right") sc.ic.h_right = num(val, line);
            else unknown();
        } else {  // run
            if (key == "name") sc.name = val;
            else if (key == "t_end") sc.t_end = num(val, line);
            else if (key == "snapshot_every") sc.snapshot_every = num(val, line);
            else if (key == "out_dir") sc.out_dir = val;
            else unknown();
        }
    }
    GridSpec(sc.nx, sc.ny, sc.dx, sc.dy);  // validates
    if (!(sc.t_end >= 0.0) || !std::isfinite(sc.t_end)) throw ConfigError("scenario: t_end must be >= 0 and finite");
    if (!(sc.snapshot_every >= 0.0)) throw ConfigError("scenario: snapshot_every must be >= 0");
    return sc;
}

// build_initial_state (scenarios.hpp:95-171) on the host, for the kinds that
// use std::exp (drops, vortex); built with -ffp-contract=off like the reference.
FieldSet host_initial(const Scenario& sc) {
    FieldSet fs(GridSpec(sc.nx, sc.ny, sc.dx, sc.dy));
    const Initial& ic = sc.ic;
    std::vector<double> c(ic.drops.size());
    for (int j = 0; j < sc.ny; ++j)
        for (int i = 0; i < sc.nx; ++i) {
            const std::size_t k = static_cast<std::size_t>(j) * sc.nx + i;
            if (ic.kind == IC_DROPS) {
                for (std::size_t d = 0; d < ic.drops.size(); ++d) {
                    const Drop& dr = ic.drops[d];
                    const double di = i - dr.cx, dj = j - dr.cy;
                    c[d] = dr.amplitude * std::exp(-(di * di + dj * dj) / (dr.radius * dr.radius));
                }
                std::sort(c.begin(), c.end());  // value-sorted sum: mirror-symmetric layouts stay symmetric
                double bump = 0.0;
                for (double v : c) bump += v;
                fs.h[k] = ic.depth + bump;
            } else {  // vortex
                const double di = i - ic.center_x, dj = j - ic.center_y;
                const double r2 = (di * di + dj * dj) / (ic.core_radius * ic.core_radius);
                const double shape = ic.v_peak * std::exp(0.5 * (1.0 - r2)) / ic.core_radius;
                fs.h[k] = ic.depth;
                fs.qx[k] = ic.depth * (-shape * dj);
                fs.qy[k] = ic.depth * (shape * di);
            }
        }
    return fs;
}

// ------------------------------------------------------------------ SWS1 (io.hpp:22-160)
void put(std::string& o, const void* p, std::size_t n) { o.append(static_cast<const char*>(p), n); }  // little endian host

void write_snapshot(const FieldSet& fs, const std::string& path, double g, double dt_next,
                    unsigned long long step_index) {
    std::string o;
    const std::size_t n = fs.spec.cell_count();
    o.reserve(56 + 32 * n + 24);
    o += "SWS1";
    const uint32_t hdr[3] = {1u, static_cast<uint32_t>(fs.spec.nx), static_cast<uint32_t>(fs.spec.ny)};
    put(o, hdr, sizeof hdr);
    const double f[5] = {fs.spec.dx, fs.spec.dy, fs.t, g, 0.0};
    put(o, f, sizeof f);
    for (const auto* a : {&fs.z, &fs.h, &fs.qx, &fs.qy}) put(o, a->data(), n * 8);
    const double sidx = static_cast<double>(step_index);
    for (auto [tag, v] : {std::pair<uint32_t, double>{1u, dt_next}, {2u, sidx}}) {
        put(o, &tag, 4);
        put(o, &v, 8);
    }
    std::ofstream out(path, std::ios::binary);
    if (!out || !out.write(o.data(), static_cast<std::streamsize>(o.size())))
        throw IoError("cannot write snapshot '" + path + "'");
}

// read_snapshot (io.hpp:142-241): header, four blocks, trailing resume records
struct Resume {
    FieldSet fs;
    bool has_dt = false, has_idx = false;
    double dt_next = 0.0;
    unsigned long long step_index = 0;
};

Resume read_snapshot(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open snapshot '" + path + "'");
    const std::string b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (b.size() < 56) throw IoError("snapshot: truncated header");
    if (b.compare(0, 4, "SWS1") != 0) throw IoError("snapshot: bad magic");
    uint32_t hdr[3];
    double hf[5];
    std::memcpy(hdr, b.data() + 4, sizeof hdr);
    std::memcpy(hf, b.data() + 16, sizeof hf);
    if (hdr[0] != 1u) throw IoError("snapshot: unsupported version");
    const std::size_t n = static_cast<std::size_t>(hdr[1]) * hdr[2];
    if (b.size() < 56 + 32 * n) throw IoError("snapshot: truncated payload");
    Resume r;
    r.fs = FieldSet(GridSpec(static_cast<int>(hdr[1]), static_cast<int>(hdr[2]), hf[0], hf[1]));
    r.fs.t = hf[2];
    std::vector<double>* blocks[4] = {&r.fs.z, &r.fs.h, &r.fs.qx, &r.fs.qy};
    for (int k = 0; k < 4; ++k) std::memcpy(blocks[k]->data(), b.data() + 56 + 8 * n * k, 8 * n);
    for (std::size_t off = 56 + 32 * n; off < b.size(); off += 12) {
        if (b.size() - off < 12) throw IoError("snapshot: truncated trailing record");
        uint32_t tag;
        double v;
        std::memcpy(&tag, b.data() + off, 4);
        std::memcpy(&v, b.data() + off + 4, 8);
        if (tag == 1u) r.has_dt = true, r.dt_next = v;
        if (tag == 2u) r.has_idx = true, r.step_index = static_cast<unsigned long long>(v);
    }
    return r;
}

std::string short_double(double d) {  // shortest round-tripping form (io.hpp fmt_double_short)
    char b[40];
    for (int p = 15; p <= 17; ++p) {
        std::snprintf(b, sizeof b, "%.*g", p, d);
        if (std::strtod(b, nullptr) == d) break;
    }
    return b;
}

// ------------------------------------------------------------------ run (run.hpp:101-179)
struct Report {
    std::string scenario, executor;
    std::size_t cells = 0;
    unsigned long long steps = 0;
    double t_final = 0.0, wall = 0.0, device_step_seconds = 0.0;
    long long halo_values = 0;
    int redundant_star_rows = 0, redundant_corrector_rows = 0;
    int snapshots = 0, clamp_warnings = 0;
    std::vector<std::string> paths;
    std::string text() const {
        std::ostringstream os;
        const double cps = (wall > 0.0 && steps) ? static_cast<double>(cells) * static_cast<double>(steps) / wall : 0.0;
        os << "scenario: " << scenario << "\nexecutor: " << executor << "\ncells: " << cells << "\nsteps: " << steps
           << "\nt_final: " << short_double(t_final) << "\nwall_seconds: " << short_double(wall)
           << "\ncells_per_second: " << short_double(cps) << "\n";
        // the six plan kernels (+ smoothing) run fused in one launch per step: there
        // is no per-kernel split to report, only the fused step's device time
        os << "plan_kernels: fused (k1_ghost_committed k2_predictor k3_ghost_star k4_corrector smooth k5_guard "
              "k6_dt_reduce in one launch per step)\n";
        os << "fused_step_seconds: " << short_double(device_step_seconds)
           << "\nhalo_exchange: " << (halo_values ? "NCCL send/recv of the R edge rows, overlapped with the interior rows"
                                                   : "none (one rank)")
           << "\nhalo_values_exchanged_per_step: " << halo_values
           << "\nredundant_predictor_rows_per_step: " << redundant_star_rows
           << "\nredundant_corrector_rows_per_step: " << redundant_corrector_rows << "\nsnapshots_written: " << snapshots
           << "\n";
        if (clamp_warnings > 0)
            os << "warning: fixed-elevation boundary clamped ghost depth to h_min (" << clamp_warnings << " fills)\n";
        return os.str();
    }
};

std::string snapshot_path(const Scenario& sc, int ordinal, bool final) {
    char b[16];
    std::snprintf(b, sizeof b, "%06d", ordinal);
    return sc.out_dir + "/" + sc.name + (final ? std::string("_final") : "_" + std::string(b)) + ".sws";
}

// run / run_from (run.hpp:101-179): from the scenario's initial state, or from
// a snapshot with its resume records (step parity and raw dt travel with it)
Report run_scenario(const Scenario& sc, bool write, const Resume* resume = nullptr) {
    const Exec& ex = sc.exec;
    const int nr = ex.ranks;
    const GridSpec spec(sc.nx, sc.ny, sc.dx, sc.dy);
    if (write) std::filesystem::create_directories(sc.out_dir);
    if (resume && (resume->fs.spec.nx != sc.nx || resume->fs.spec.ny != sc.ny))
        throw ConfigError("resume: snapshot grid does not match the config");
    const bool device_ic = !resume && (sc.ic.kind == IC_FLAT || sc.ic.kind == IC_CHANNEL || sc.ic.kind == IC_DAM);
    FieldSet host = resume ? resume->fs : device_ic ? FieldSet() : host_initial(sc);
    FieldSet shared(spec);  // gathered committed state for snapshots
    Report rep;
    rep.scenario = sc.name;
    rep.executor = ex.name();
    rep.cells = spec.cell_count();
    std::vector<unsigned char> id(SWE_NCCL_ID_BYTES, 0);
    if (nr > 1) {
        if (ex.local) {
            std::snprintf(reinterpret_cast<char*>(id.data()), id.size(), "swe-cli-%d-%lld", static_cast<int>(getpid()),
                          static_cast<long long>(std::chrono::steady_clock::now().time_since_epoch().count()));
        } else {
            swe_status st{};
            if (swe_cuda_nccl_unique_id(id.data(), &st) != SWE_OK) throw_status(st);
        }
    }
    std::barrier sync(nr);
    std::atomic<bool> snap_failed{false};
    std::mutex m;
    std::exception_ptr err;
    const auto wall0 = std::chrono::steady_clock::now();
    auto rank_main = [&](int r) {
        try {
            ExecutorKind k;
            k.device = (nr > 1 && !ex.local) ? r : 0;
            k.exact = ex.exact;
            k.early_exit = ex.early;
            k.local_group = ex.local;
            k.rank = r;
            k.nranks = nr;
            k.nccl_id = nr > 1 ? id.data() : nullptr;
            Stepper st(spec, sc.phys, sc.pol, sc.bnd, k);
            const int r0 = st.row_begin(), r1 = st.row_end();
            if (device_ic) {
                swe_initial ic{sc.ic.kind, sc.ic.depth, sc.ic.slope, sc.ic.split_x, sc.ic.h_left, sc.ic.h_right};
                st.load_initial(ic, 0.0);
            } else {
                st.load(host);
                if (!resume) {
                    try {  // build_initial_state's own guard (scenarios.hpp:165-169)
                        st.guard();
                    } catch (const InstabilityError& e) {
                        throw ConfigError(std::string("initial state fails the stability guard: ") + e.what());
                    }
                }
            }
            st.guard();  // run_from's precondition (run.hpp:106-109)
            unsigned long long sidx = resume && resume->has_idx ? resume->step_index : 0, steps = 0;
            double t = resume ? resume->fs.t : 0.0;
            double dt_raw = resume && resume->has_dt ? resume->dt_next : std::numeric_limits<double>::quiet_NaN();
            const double se = sc.snapshot_every;
            double mark = se > 0.0 ? (std::floor(t / se) + 1.0) * se : std::numeric_limits<double>::infinity();
            int ordinal = 0;
            auto snap = [&](double dt_next, bool final) {
                const FieldSet s = st.state();
                const std::size_t a = static_cast<std::size_t>(r0) * sc.nx, b = static_cast<std::size_t>(r1) * sc.nx;
                std::copy(s.h.begin() + a, s.h.begin() + b, shared.h.begin() + a);
                std::copy(s.qx.begin() + a, s.qx.begin() + b, shared.qx.begin() + a);
                std::copy(s.qy.begin() + a, s.qy.begin() + b, shared.qy.begin() + a);
                std::copy(s.z.begin() + a, s.z.begin() + b, shared.z.begin() + a);
                sync.arrive_and_wait();
                if (r == 0) {
                    try {
                        shared.t = s.t;
                        const std::string p = snapshot_path(sc, ordinal, final);
                        if (write) write_snapshot(shared, p, sc.phys.g, dt_next, sidx);
                        rep.paths.push_back(p);
                        rep.snapshots = ordinal + 1;
                    } catch (...) {
                        // every rank leaves the loop together: the others would
                        // otherwise enter collectives rank 0 never joins
                        std::lock_guard<std::mutex> lk(m);
                        if (!err) err = std::current_exception();
                        snap_failed.store(true);
                    }
                }
                ++ordinal;
                sync.arrive_and_wait();
                if (snap_failed.load()) throw DeviceError("run: snapshot write failed on rank 0");
            };
            while (t < sc.t_end) {
                const RunResult res = st.advance_marked(sc.t_end, mark, sidx, dt_raw);
                sidx = res.step_index;
                dt_raw = res.dt_next;
                t = res.t_final;
                steps += res.steps;
                if (res.steps == 0 && t < sc.t_end)
                    throw DeviceError("run: the device loop committed no step before t_end");
                if (se > 0.0 && t >= mark && t < sc.t_end) {
                    snap(dt_raw, false);
                    mark = (std::floor(t / se) + 1.0) * se;
                }
            }
            if (r == 0) {
                rep.steps = steps;
                rep.t_final = t;
                rep.clamp_warnings = st.guard_warnings();
                swe_timing tm{};
                swe_cuda_timing(st.handle(), &tm);
                rep.device_step_seconds = tm.step_seconds;
                rep.redundant_star_rows = st.accounting().redundant_star_rows;
                rep.redundant_corrector_rows = st.accounting().redundant_corrector_rows;
            }
            {  // StepAccounting summed over ranks, like the reference's decomposed bands
                std::lock_guard<std::mutex> lk(m);
                rep.halo_values += st.accounting().halo_values_exchanged;
            }
            if (!std::isfinite(dt_raw)) dt_raw = 0.0;
            snap(dt_raw, true);
        } catch (...) {
            std::lock_guard<std::mutex> lk(m);
            if (!err) err = std::current_exception();
            sync.arrive_and_drop();
        }
    };
    if (nr == 1) {
        rank_main(0);
    } else {
        std::vector<std::thread> th;
        for (int r = 0; r < nr; ++r) th.emplace_back(rank_main, r);
        for (auto& t : th) t.join();
    }
    if (err) std::rethrow_exception(err);
    rep.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    if (write) {
        std::ofstream f(sc.out_dir + "/" + sc.name + "_report.txt");
        f << rep.text();
    }
    return rep;
}

// ------------------------------------------------------------------ bench (bench.hpp:33-108)
Scenario five_drops(int n) {  // gen_five_drops (scenarios.hpp:186-208)
    if (n < 33) throw ConfigError("bench: sizes must be >= 33");
    Scenario sc;
    sc.name = n == 1024 ? "five-drops-big" : "five-drops";
    sc.nx = sc.ny = n;
    sc.pol.cfl = 0.45;
    sc.t_end = 100.0;
    sc.ic.kind = IC_DROPS;
    sc.ic.depth = 1.0;
    const double c = (n - 1) / 2.0, d = n / 4.0, r0 = n / 20.0;
    sc.ic.drops = {{c, c, r0, 0.3}, {c - d, c - d, r0, 0.3}, {c - d, c + d, r0, 0.3}, {c + d, c - d, r0, 0.3},
                   {c + d, c + d, r0, 0.3}};
    return sc;
}

int cmd_bench(const std::string& sizes, int steps, const std::string& execs, int reps, const std::string& csv) {
    if (steps < 1 || reps < 1) throw ConfigError("bench: steps and reps must be >= 1");
    std::vector<int> ns;
    {
        std::istringstream in(sizes);
        for (std::string t; std::getline(in, t, ',');) ns.push_back(std::stoi(t));
    }
    std::vector<Exec> ks;
    {
        std::istringstream in(execs);
        for (std::string t; std::getline(in, t, ',');) ks.push_back(parse_exec_spec(t));
    }
    std::ostringstream table, rows;
    char line[200];
    std::snprintf(line, sizeof line, "%8s  %-20s %8s %6s  %14s  %14s\n", "size", "executor", "steps", "reps", "sec/step",
                  "cells/s");
    table << line;
    rows << "size,executor,steps,reps,median_sec_per_step,cells_per_second\n";
    for (int n : ns) {
        const Scenario sc = five_drops(n);
        const FieldSet ic = host_initial(sc);
        for (const Exec& e : ks) {
            if (e.ranks != 1) throw ConfigError("bench: one rank per measurement");
            std::vector<double> per;
            for (int rep = 0; rep < reps; ++rep) {
                ExecutorKind k;
                k.exact = e.exact;
                k.early_exit = e.early;
                Stepper st(ic.spec, sc.phys, sc.pol, sc.bnd, k);
                st.load(ic);
                double dt = st.compute_dt(std::numeric_limits<double>::infinity());
                dt = st.step(dt, 0).dt_next;  // warm-up, excluded
                const auto t0 = std::chrono::steady_clock::now();
                for (int s = 1; s <= steps; ++s) dt = st.step(dt, static_cast<unsigned long long>(s)).dt_next;
                per.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / steps);
            }
            std::sort(per.begin(), per.end());
            const double med = per[per.size() / 2];
            const double cps = static_cast<double>(ic.spec.cell_count()) / med;
            std::snprintf(line, sizeof line, "%4dx%-4d %-20s %8d %6d  %14.6e  %14.6e\n", n, n, e.name().c_str(), steps,
                          reps, med, cps);
            table << line;
            char a[40], b[40];
            std::snprintf(a, sizeof a, "%.17g", med);
            std::snprintf(b, sizeof b, "%.17g", cps);
            rows << n << ',' << e.name() << ',' << steps << ',' << reps << ',' << a << ',' << b << '\n';
        }
    }
    std::cout << table.str();
    std::ofstream f(csv);
    if (!f) throw IoError("cannot open '" + csv + "' for the bench CSV");
    f << rows.str();
    std::cout << "csv: " << csv << "\n";
    return 0;
}

// ------------------------------------------------------------------ main
int exit_code(const std::exception& e, const char** kind) {
    if (dynamic_cast<const ConfigError*>(&e)) return *kind = "config", 2;
    if (dynamic_cast<const InstabilityError*>(&e)) return *kind = "instability", 3;
    if (dynamic_cast<const StepCollapseError*>(&e)) return *kind = "step-collapse", 4;
    if (dynamic_cast<const IoError*>(&e)) return *kind = "io", 5;
    if (dynamic_cast<const DeviceError*>(&e)) return *kind = "device", 6;
    return *kind = "error", 1;
}

std::string slurp(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw IoError("cannot open config file '" + path + "'");
    std::ostringstream s;
    s << f.rdbuf();
    return s.str();
}

void usage() {
    std::cerr << "usage: swe_cuda run --config FILE [--set section.key=value]... [--executor SPEC] [--out DIR]\n"
                 "                    [--snapshot-every S] [--resume SNAPSHOT.sws] [--quiet]\n"
                 "       swe_cuda bench [--sizes 256,512] [--steps 50] [--executors cuda,cuda:fast] [--reps 3]\n"
                 "                      [--csv bench.csv]\n"
                 "SPEC: cuda[:N][:fast|:exact][:early][:local] (naive|tiled|decomposed run as exact cuda)\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    std::vector<std::string> a(argv + 2, argv + argc);
    auto opt = [&](std::size_t& k) -> std::string {
        if (k + 1 >= a.size()) throw ConfigError("option " + a[k] + " needs a value");
        return a[++k];
    };
    try {
        if (cmd == "run") {
            std::string config, exec, out, resume_path;
            std::vector<std::string> sets;
            double se = -1.0;
            bool quiet = false;
            for (std::size_t k = 0; k < a.size(); ++k) {
                if (a[k] == "--config") config = opt(k);
                else if (a[k] == "--set") sets.push_back(opt(k));
                else if (a[k] == "--executor") exec = opt(k);
                else if (a[k] == "--out") out = opt(k);
                else if (a[k] == "--snapshot-every") se = std::stod(opt(k));
                else if (a[k] == "--quiet") quiet = true;
                else if (a[k] == "--resume") resume_path = opt(k);
                else throw ConfigError("unknown option '" + a[k] + "'");
            }
            if (config.empty()) throw ConfigError("run: --config is required");
            std::string text = slurp(config);
            Scenario sc = parse_config(text);
            for (const std::string& s : sets) {  // apply_override (io.hpp:559-572): reparse with the key appended
                const auto eq = s.find('='), dot = s.find('.');
                if (eq == std::string::npos || dot == std::string::npos || dot > eq)
                    throw ConfigError("--set expects section.key=value, got '" + s + "'");
                text += "\n[" + s.substr(0, dot) + "]\n" + s.substr(dot + 1, eq - dot - 1) + " = " + s.substr(eq + 1) + "\n";
                sc = parse_config(text);
            }
            if (!exec.empty()) sc.exec = parse_exec_spec(exec);
            if (!out.empty()) sc.out_dir = out;
            if (se >= 0.0) sc.snapshot_every = se;
            Resume res;
            if (!resume_path.empty()) res = read_snapshot(resume_path);
            const Report r = run_scenario(sc, true, resume_path.empty() ? nullptr : &res);
            if (!quiet) std::cout << r.text() << "final_snapshot: " << r.paths.back() << "\n";
            return 0;
        }
        if (cmd == "bench") {
            std::string sizes = "256,512", execs = "cuda,cuda:fast", csv = "bench.csv";
            int steps = 50, reps = 3;
            for (std::size_t k = 0; k < a.size(); ++k) {
                if (a[k] == "--sizes") sizes = opt(k);
                else if (a[k] == "--steps") steps = std::stoi(opt(k));
                else if (a[k] == "--executors") execs = opt(k);
                else if (a[k] == "--reps") reps = std::stoi(opt(k));
                else if (a[k] == "--csv") csv = opt(k);
                else throw ConfigError("unknown option '" + a[k] + "'");
            }
            return cmd_bench(sizes, steps, execs, reps, csv);
        }
        usage();
        return 2;
    } catch (const std::exception& e) {
        const char* kind = "error";
        const int code = exit_code(e, &kind);
        std::cerr << "swe_cuda: error [" << kind << "]: " << e.what() << "\n";
        return code;
    }
}
