// oracle/_ref driver: links the UNMODIFIED reference library sources
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile against the
// Eigen storage shim in oracle/shim) and exposes its public API as a small
// command-line tool. TEST INFRASTRUCTURE ONLY: used to generate the golden
// fixtures under tests/golden/ and as the CPU "reference" arm of bench.py.
// Nothing in the product links or calls this.
//
// Every code path below goes through the reference's public entry points:
//   load_config / build_model / build_spec / build_options   (config.hpp:55-70)
//   window_extents / memory_estimate / build_matrix / RowKernel (abstraction.hpp:70-125)
//   build_target_hit / mask_absorbing                          (abstraction.hpp:117-121)
//   synthesize / bellman_step                                  (synthesis.hpp:46-66)
//   write_results / write_matrix                               (io.hpp:13-23)
//   parallel_for / resolve_threads                             (parallel.hpp:13-51)
//   read_results / simulate / empirical_rate / write_trajectory_csv (io.hpp:14, sim.hpp:42-50)
#include "gridmdp/config.hpp"
#include "gridmdp/io.hpp"
#include "gridmdp/parallel.hpp"
#include "gridmdp/sim.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

using namespace gridmdp;

namespace {

struct Args {
    std::string cmd, config, out, vnext, results, x0, dist_mode = "random", traj;
    long long runs = -1, seed = -1;
    std::string custom_pdf, custom_lb, custom_ub; // NoiseSpec::custom over the config's model
    int threads = -1, time_steps = -1;
    std::string mode;
    long long row_begin = -1, row_end = -1;
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

Config effective(const Args& a) {
    Config cfg = load_config(a.config);
    if (a.threads >= 0) cfg.threads = a.threads;
    if (a.runs >= 0) cfg.runs = static_cast<int>(a.runs);
    if (a.seed >= 0) cfg.seed = static_cast<std::uint64_t>(a.seed);
    if (!a.mode.empty()) cfg.mode = a.mode;
    if (a.time_steps >= 0) cfg.time_steps = a.time_steps;
    return cfg;
}

void write_raw(const std::string& path, const void* p, std::size_t bytes) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoError("cannot open '" + path + "'");
    os.write(static_cast<const char*>(p), static_cast<std::streamsize>(bytes));
}

std::vector<double> read_f64(const std::string& path) {
    std::ifstream is(path, std::ios::binary | std::ios::ate);
    if (!is) throw IoError("cannot open '" + path + "'");
    const auto n = static_cast<std::size_t>(is.tellg());
    std::vector<double> v(n / 8);
    is.seekg(0);
    is.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n));
    return v;
}

void print_sizes(const SystemModel& m) {
    std::cout << "states: " << m.n_states() << "\n";
    std::cout << "inputs: " << m.n_inputs() << "\n";
    std::cout << "disturbances: " << m.n_disturbances() << "\n";
    std::cout << "state_input_pairs: " << m.n_states() * m.n_inputs() << "\n";
    std::cout << "rows: " << m.n_rows() << "\n";
    const IndexVec w = window_extents(m);
    Index width = 1;
    std::cout << "window:";
    for (Index e : w) {
        width *= e;
        std::cout << " " << e;
    }
    std::cout << "\n";
    std::cout << "row_width: " << width << "\n";
    std::cout << "memory_estimate_bytes: " << memory_estimate(m) << "\n";
}

std::vector<double> braced(const std::string& s) {
    std::vector<double> v;
    std::string inner = s.substr(1, s.size() - 2);
    std::size_t pos = 0;
    while (pos <= inner.size()) {
        const std::size_t comma = inner.find(',', pos);
        v.push_back(std::stod(comma == std::string::npos ? inner.substr(pos) : inner.substr(pos, comma - pos)));
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return v;
}

// The config's model, or -- with --custom-pdf -- the same grids and dynamics with
// NoiseSpec::custom (noise.cpp:75-85) whose pdf callback evaluates the reference's
// own expression language (parse_expression / eval, expr.hpp:66-74) over xi.
SystemModel model_of(const Config& cfg, const Args& a) {
    SystemModel m = build_model(cfg);
    if (a.custom_pdf.empty()) return m;
    const int n = m.state_dim();
    const Expr e = parse_expression(a.custom_pdf, Dims{n, 0, 0}, cfg.constants);
    CustomDensity cd;
    cd.pdf = [e](const Vector& xi) { return eval(e, xi.data(), nullptr, nullptr); };
    const std::vector<double> lo = braced(a.custom_lb), hi = braced(a.custom_ub);
    Vector l(n), h(n);
    for (int d = 0; d < n; ++d) {
        l[d] = lo[static_cast<std::size_t>(d)];
        h[d] = hi[static_cast<std::size_t>(d)];
    }
    cd.support = Box(l, h);
    return make_model(m.state, m.input, m.disturbance, m.dynamics,
                      NoiseSpec::custom(cd, m.noise.gamma(), m.noise.mode()));
}

int run(const Args& a) {
    const Config cfg = effective(a);
    const SystemModel m = model_of(cfg, a);
    if (a.cmd == "estimate") {
        print_sizes(m);
        return 0;
    }
    if (a.cmd == "matrix") { // unmasked build, like `gridmdp abstract --dump-matrix`
        const TransitionMatrix tm = build_matrix(m, cfg.threads);
        write_matrix(tm, a.out);
        return 0;
    }
    if (a.cmd == "prism") { // export_prism (io.cpp:289-317), like `gridmdp export-prism`
        const TransitionMatrix tm = build_matrix(m, cfg.threads);
        export_prism(tm, a.out);
        return 0;
    }
    if (a.cmd == "masked-matrix") { // masked as synthesize_with_matrix does
        const Spec spec = build_spec(cfg);
        TransitionMatrix tm = build_matrix(m, cfg.threads);
        mask_absorbing(tm, spec, cfg.threads);
        write_matrix(tm, a.out);
        return 0;
    }
    if (a.cmd == "target-hit") {
        const Spec spec = build_spec(cfg);
        const TargetHitVector t0 = build_target_hit(m, spec, cfg.threads);
        write_raw(a.out, t0.data(), static_cast<std::size_t>(t0.size()) * 8);
        return 0;
    }
    if (a.cmd == "synthesize") {
        const Spec spec = build_spec(cfg);
        const SynthesisOptions opts = build_options(cfg);
        const double t0 = now_s();
        const SynthesisResult res = synthesize(m, spec, opts);
        std::cout << "time_synthesize_s: " << now_s() - t0 << "\n";
        write_results(res, a.out);
        return 0;
    }
    if (a.cmd == "step") { // one bellman_step with an arbitrary v_next
        const Spec spec = build_spec(cfg);
        const std::vector<double> vn = read_f64(a.vnext);
        Eigen::VectorXd v_next(m.n_states());
        std::memcpy(v_next.data(), vn.data(), static_cast<std::size_t>(m.n_states()) * 8);
        Eigen::VectorXd v_out;
        std::vector<std::uint32_t> pol(static_cast<std::size_t>(m.n_states()));
        std::vector<std::uint32_t> wst(static_cast<std::size_t>(m.n_states()));
        const double t0 = now_s();
        if (cfg.mode == "matrix") {
            TransitionMatrix tm = build_matrix(m, cfg.threads);
            TargetHitVector th;
            if (spec.is_reach()) {
                mask_absorbing(tm, spec, cfg.threads);
                th = build_target_hit(m, spec, cfg.threads);
            }
            bellman_step(m, spec, &tm, spec.is_reach() ? &th : nullptr, v_next, v_out, pol.data(),
                         wst.data(), cfg.threads);
        } else {
            bellman_step(m, spec, nullptr, nullptr, v_next, v_out, pol.data(), wst.data(),
                         cfg.threads);
        }
        std::cout << "time_step_s: " << now_s() - t0 << "\n";
        write_raw(a.out + ".v", v_out.data(), static_cast<std::size_t>(v_out.size()) * 8);
        write_raw(a.out + ".pol", pol.data(), pol.size() * 4);
        write_raw(a.out + ".wst", wst.data(), wst.size() * 4);
        return 0;
    }
    if (a.cmd == "time-rows") {
        // CPU baseline sample: RowKernel::compute + fill_row (the body of
        // build_matrix, abstraction.cpp:211-223) over rows [row_begin,row_end)
        // with the reference's own parallel_for and thread resolution.
        const Index rb = a.row_begin, re = a.row_end;
        const int threads = resolve_threads(cfg.threads);
        const Index n_u = m.n_inputs(), n_w = m.n_disturbances();
        double checksum = 0.0;
        std::vector<double> partial(static_cast<std::size_t>(threads), 0.0);
        const double t0 = now_s();
        parallel_for(re - rb, threads, [&](Index b, Index e) {
            RowKernel k(m);
            std::vector<double> row(static_cast<std::size_t>(k.row_width()));
            double s = 0.0;
            for (Index r = rb + b; r < rb + e; ++r) {
                const Index iw = r % n_w, p = r / n_w;
                k.compute(p / n_u, p % n_u, iw);
                k.fill_row(row.data());
                s += row[0] + static_cast<double>(k.origin_flat());
            }
            partial[static_cast<std::size_t>(b * threads / (re - rb))] += s;
        });
        const double dt = now_s() - t0;
        for (double s : partial) checksum += s;
        const IndexVec w = window_extents(m);
        Index R = 1;
        for (Index e : w) R *= e;
        std::printf("rows %lld R %lld threads %d seconds %.6f checksum %.17g\n",
                    static_cast<long long>(re - rb), static_cast<long long>(R), threads, dt,
                    checksum);
        return 0;
    }
    if (a.cmd == "simulate") { // as `gridmdp simulate` (tools/gridmdp_main.cpp:119-140)
        const SynthesisResult res = read_results(a.results);
        std::vector<double> x;
        {
            std::string inner = a.x0.substr(1, a.x0.size() - 2);
            std::size_t pos = 0;
            while (pos <= inner.size()) {
                const std::size_t comma = inner.find(',', pos);
                x.push_back(std::stod(comma == std::string::npos ? inner.substr(pos) : inner.substr(pos, comma - pos)));
                if (comma == std::string::npos) break;
                pos = comma + 1;
            }
        }
        Vector x0(static_cast<Eigen::Index>(x.size()));
        for (std::size_t i = 0; i < x.size(); ++i) x0[static_cast<Eigen::Index>(i)] = x[i];
        const DisturbanceMode dm = a.dist_mode == "worst-case" ? DisturbanceMode::worst_case : DisturbanceMode::random;
        const double t0 = now_s();
        const TrajectoryBatch batch = simulate(m, res.spec, res, x0, cfg.runs, cfg.seed, dm, cfg.threads);
        const double dt = now_s() - t0;
        std::size_t steps = 0;
        for (const Trajectory& t : batch.runs) steps += static_cast<std::size_t>(t.steps());
        std::cout << "runs: " << batch.runs.size() << "\n";
        std::cout << "empirical_rate: " << empirical_rate(batch) << "\n";
        std::printf("satisfied: %zu\nsteps_total: %zu\ntime_simulate_s: %.6f\n",
                    static_cast<std::size_t>(empirical_rate(batch) * batch.runs.size() + 0.5), steps, dt);
        if (!a.traj.empty()) write_trajectory_csv(batch, a.traj);
        return 0;
    }
    throw ConfigError("unknown command '" + a.cmd + "'");
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr,
                     "usage: gridmdp_ref {estimate|matrix|masked-matrix|target-hit|synthesize|step|"
                     "time-rows|simulate} -c CFG [-o OUT] [--mode M] [--threads N] [--time-steps T] "
                     "[--vnext F] [--rows B E] [--results R --x0 {..} --runs N --seed S --dist-mode D --traj F]\n");
        return 1;
    }
    Args a;
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw ConfigError("missing value for " + k);
            return argv[++i];
        };
        try {
            if (k == "-c") a.config = next();
            else if (k == "-o") a.out = next();
            else if (k == "--mode") a.mode = next();
            else if (k == "--threads") a.threads = std::stoi(next());
            else if (k == "--time-steps") a.time_steps = std::stoi(next());
            else if (k == "--vnext") a.vnext = next();
            else if (k == "--results") a.results = next();
            else if (k == "--x0") a.x0 = next();
            else if (k == "--dist-mode") a.dist_mode = next();
            else if (k == "--traj") a.traj = next();
            else if (k == "--runs") a.runs = std::stoll(next());
            else if (k == "--custom-pdf") a.custom_pdf = next();
            else if (k == "--custom-lb") a.custom_lb = next();
            else if (k == "--custom-ub") a.custom_ub = next();
            else if (k == "--seed") a.seed = std::stoll(next());
            else if (k == "--rows") {
                a.row_begin = std::stoll(next());
                a.row_end = std::stoll(next());
            } else {
                std::fprintf(stderr, "unknown flag %s\n", k.c_str());
                return 1;
            }
        } catch (const std::exception& e) {
            std::fprintf(stderr, "error: %s\n", e.what());
            return 1;
        }
    }
    try {
        return run(a);
    } catch (const ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const MemoryError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const DomainError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 5;
    } catch (const std::out_of_range& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 4;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
