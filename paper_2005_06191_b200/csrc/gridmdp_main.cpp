// `gridmdp` CLI of the B200 engine: the reference's verbs, flags, key: value
// report lines and exit codes (tools/gridmdp_main.cpp:16-227), driving the
// C ABI of libgridmdp_b200.so. New options are CLI-only (`--device`, `--gpus`,
// `--devices`, `--exchange`, `--transport`), so the
// shared .cfg files stay valid for the reference parser (config.cpp:165-167).
#include "gridmdp_b200.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <string>
#include <thread>
#include <vector>

namespace {

struct Args {
    std::string verb, config, mode, output, dump, results, x0, dist_mode = "random", traj;
    long long threads = -1, mem_budget = -1, seed = -1, runs = -1, time_steps = -1;
    int device = 0;
    // multi-GPU synthesis (CLI only): --gpus N (devices 0..N-1) or --devices a,b,..
    std::vector<int> devices;
    int exchange = GM_XCHG_AUTO, transport = GM_XPORT_NCCL;
};

// HBM bandwidth the roofline_frac line divides by: the measured copy bandwidth of a
// B200 (MEASURED_PEAKS.json hbm_gbs), GM_HBM_PEAK_GBS overrides it.
double hbm_peak_gbs() {
    const char* e = std::getenv("GM_HBM_PEAK_GBS");
    return e ? std::atof(e) : 6545.0;
}

double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int exit_code(const gm_status& st) {
    switch (st.code) {
        case GM_ERR_CONFIG: return 2;
        case GM_ERR_MEMORY: return 3;
        case GM_ERR_DOMAIN: return 4;
        case GM_ERR_RANGE: return 4;
        case GM_ERR_IO: return 5;
        default: return 1;
    }
}

int fail(const gm_status& st) {
    std::cerr << "error: " << st.msg << "\n";
    return exit_code(st);
}

int resolve_threads(int t) {
    if (t > 0) return t;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 0 ? static_cast<int>(hw) : 1;
}

void print_sizes(const gm_sizes& s) {
    std::cout << "states: " << s.n_states << "\n";
    std::cout << "inputs: " << s.n_inputs << "\n";
    std::cout << "disturbances: " << s.n_disturbances << "\n";
    std::cout << "state_input_pairs: " << s.n_states * s.n_inputs << "\n";
    if (s.size_overflow) { // MemoryError from checked_mul (common.hpp:67-71) -> exit 3
        std::cout.flush();
        std::cerr << "error: memory_estimate: size arithmetic overflows 64 bits\n";
        std::exit(3);
    }
    std::cout << "rows: " << s.rows << "\n";
    std::cout << "row_width: " << s.row_width << "\n";
    std::cout << "memory_estimate_bytes: " << s.memory_estimate << "\n";
}

int load(const Args& a, gm_model** m, gm_sizes* sz) {
    gm_overrides ov;
    ov.threads = static_cast<int32_t>(a.threads);
    ov.time_steps = static_cast<int32_t>(a.time_steps);
    ov.mem_budget = a.mem_budget;
    ov.seed = a.seed;
    ov.runs = static_cast<int32_t>(a.runs);
    ov.mode = a.mode.empty() ? nullptr : a.mode.c_str();
    ov.output = a.output.empty() ? nullptr : a.output.c_str();
    gm_status st;
    if (gm_model_load(a.config.c_str(), &ov, m, &st) != GM_OK) return fail(st);
    if (gm_model_sizes(*m, sz, &st) != GM_OK) return fail(st);
    return 0;
}

int cmd_estimate(const Args& a) {
    gm_model* m = nullptr;
    gm_sizes sz;
    if (int rc = load(a, &m, &sz)) return rc;
    print_sizes(sz);
    gm_model_free(m);
    return 0;
}

int cmd_abstract(const Args& a) {
    gm_model* m = nullptr;
    gm_sizes sz;
    if (int rc = load(a, &m, &sz)) return rc;
    print_sizes(sz);
    gm_status st;
    if (sz.mem_budget != 0 && sz.memory_estimate > static_cast<uint64_t>(sz.mem_budget)) {
        std::cerr << "error: matrix needs " << sz.memory_estimate << " bytes but the budget is " << sz.mem_budget
                  << "; use ofa mode\n";
        return 3;
    }
    // device 0 is the default; selecting it eagerly would turn the reference's validation
    // errors (spec, budget) into device errors on hosts without a GPU
    if (a.device != 0 && gm_set_device(a.device, &st) != GM_OK) return fail(st);
    const auto t0 = std::chrono::steady_clock::now();
    gm_matrix* tm = nullptr;
    if (gm_build_matrix(m, 0, sz.rows, &tm, &st) != GM_OK) return fail(st);
    std::cout << "time_abstract_s: " << since(t0) << "\n";
    std::cout << "probs_per_s: " << static_cast<double>(sz.rows) * static_cast<double>(sz.row_width) / since(t0)
              << "\n";
    if (!a.dump.empty()) {
        if (gm_matrix_write(tm, m, a.dump.c_str(), &st) != GM_OK) return fail(st);
        std::cout << "matrix_dump: " << a.dump << "\n";
    }
    gm_matrix_free(tm);
    gm_model_free(m);
    return 0;
}

int cmd_synthesize(const Args& a) {
    gm_model* m = nullptr;
    gm_sizes sz;
    if (int rc = load(a, &m, &sz)) return rc;
    print_sizes(sz);
    std::cout << "mode: " << (sz.mode == GM_MODE_OFA ? "ofa" : "matrix") << "\n";
    std::cout << "threads: " << resolve_threads(sz.threads) << "\n";
    std::cout << "time_steps: " << sz.horizon << "\n";
    gm_status st;
    // device 0 is the default; selecting it eagerly would turn the reference's validation
    // errors (spec, budget) into device errors on hosts without a GPU
    if (a.device != 0 && gm_set_device(a.device, &st) != GM_OK) return fail(st);
    const auto t0 = std::chrono::steady_clock::now();
    gm_result* r = nullptr;
    double build_ms = 0.0, sweep_ms = 0.0;
    int gpus = 1;
    if (!a.devices.empty()) { // one process, one host thread + stream per device
        gm_multi_stats ms;
        gpus = static_cast<int>(a.devices.size());
        if (gm_synthesize_multi(m, gpus, a.devices.data(), a.exchange, a.transport, &r, &ms, &st) != GM_OK)
            return fail(st);
        build_ms = ms.build_ms;
        sweep_ms = ms.sweep_ms;
        std::cout << "time_synthesize_s: " << since(t0) << "\n";
        if (gpus > 1)
            std::cout << "v_exchange: " << (ms.exchange_used == GM_XCHG_HALO ? "halo" : "allgather") << " "
                      << (ms.transport_used == GM_XPORT_NCCL ? "nccl" : ms.transport_used == GM_XPORT_STORE ? "store" : "peer") << " ("
                      << (ms.exchange_used == GM_XCHG_HALO ? ms.halo_states : ms.allgather_states)
                      << " states per step)\n";
    } else {
        if (gm_synthesize(m, &r, &st) != GM_OK) return fail(st);
        std::cout << "time_synthesize_s: " << since(t0) << "\n";
        gm_model_last_times(m, &build_ms, &sweep_ms, &st);
    }
    // engine report lines (device time, CUDA events): stage (i), stage (ii), and the
    // sweep against the HBM roofline (8 bytes per term T*V: the bytes matrix mode
    // streams, the HBM-equivalent in OFA mode; SURVEY.md 8 d)
    const double terms = static_cast<double>(sz.rows) * static_cast<double>(sz.row_width) * sz.horizon;
    std::cout << "gpus: " << gpus << "\n";
    std::cout << "time_build_s: " << build_ms / 1e3 << "\n";
    std::cout << "time_sweep_s: " << sweep_ms / 1e3 << "\n";
    if (sweep_ms > 0) {
        std::cout << "sweep_terms_per_s: " << terms / (sweep_ms / 1e3) << "\n";
        std::cout << "roofline_frac: " << terms * 8 / (sweep_ms / 1e3) / 1e9 / (hbm_peak_gbs() * gpus) << "\n";
    }
    if (sz.mode == GM_MODE_MATRIX && build_ms > 0)
        std::cout << "probs_per_s: " << static_cast<double>(sz.rows) * static_cast<double>(sz.row_width) / (build_ms / 1e3)
                  << "\n";
    // output path: exec.output / -o, default results.bin (gridmdp_main.cpp:113)
    std::string out = gm_model_output_path(m);
    if (out.empty()) out = "results.bin";
    if (gm_result_write(r, out.c_str(), &st) != GM_OK) return fail(st);
    std::cout << "output: " << out << "\n";
    gm_result_free(r);
    gm_model_free(m);
    return 0;
}

int cmd_export_prism(const Args& a) {
    // tools/gridmdp_main.cpp:142-152
    gm_model* m = nullptr;
    gm_sizes sz;
    if (int rc = load(a, &m, &sz)) return rc;
    const std::string out = gm_model_output_path(m);
    gm_status st;
    if (out.empty()) {
        std::cerr << "error: export-prism needs --output or exec.output\n";
        return 2;
    }
    if (sz.mem_budget != 0 && sz.memory_estimate > static_cast<uint64_t>(sz.mem_budget)) {
        std::cerr << "error: matrix exceeds the configured budget; export needs matrix mode\n";
        return 3;
    }
    if (a.device != 0 && gm_set_device(a.device, &st) != GM_OK) return fail(st);
    gm_matrix* tm = nullptr;
    if (gm_build_matrix(m, 0, sz.rows, &tm, &st) != GM_OK) return fail(st);
    if (gm_matrix_write_prism(tm, m, out.c_str(), &st) != GM_OK) return fail(st);
    std::cout << "output: " << out << "\n";
    gm_matrix_free(tm);
    gm_model_free(m);
    return 0;
}

// parse_point (tools/gridmdp_main.cpp:56-71)
bool parse_point(const std::string& s, std::vector<double>& out, int& rc) {
    if (s.size() < 2 || s.front() != '{' || s.back() != '}') {
        std::cerr << "error: --x0 expects a braced vector like {0, 0}\n";
        rc = 2;
        return false;
    }
    const std::string inner = s.substr(1, s.size() - 2);
    size_t pos = 0;
    try {
        while (pos <= inner.size()) {
            const size_t comma = inner.find(',', pos);
            const std::string item = comma == std::string::npos ? inner.substr(pos) : inner.substr(pos, comma - pos);
            out.push_back(std::stod(item));
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
    } catch (const std::exception& e) { // std::invalid_argument / out_of_range from stod
        std::cerr << "error: " << e.what() << "\n";
        rc = dynamic_cast<const std::out_of_range*>(&e) ? 4 : 1;
        return false;
    }
    return true;
}

int cmd_simulate(const Args& a) {
    // tools/gridmdp_main.cpp:119-140: closed-loop Monte Carlo under a stored result
    gm_model* m = nullptr;
    gm_sizes sz;
    if (int rc = load(a, &m, &sz)) return rc;
    const std::string rp = a.results.empty() ? std::string(gm_model_output_path(m)) : a.results;
    if (rp.empty()) {
        std::cerr << "error: simulate needs --results or exec.output in the config\n";
        return 2;
    }
    gm_status st;
    gm_result* res = nullptr;
    if (gm_result_read(rp.c_str(), &res, &st) != GM_OK) return fail(st);
    std::vector<double> x0;
    int rc = 0;
    if (!parse_point(a.x0, x0, rc)) return rc;
    int32_t runs = 0;
    uint64_t seed = 0;
    if (gm_model_sim_defaults(m, &runs, &seed, &st) != GM_OK) return fail(st);
    if (a.device != 0 && gm_set_device(a.device, &st) != GM_OK) return fail(st);
    gm_sim* sim = nullptr;
    if (gm_simulate(m, res, x0.data(), static_cast<int32_t>(x0.size()), runs, seed, a.dist_mode == "worst-case",
                    a.traj.empty() ? 0 : 1, &sim, &st) != GM_OK)
        return fail(st);
    int32_t n = 0;
    int64_t ok = 0;
    double rate = 0.0, v = 0.0;
    if (gm_sim_summary(sim, &n, &ok, &rate, &st) != GM_OK) return fail(st);
    std::cout << "runs: " << n << "\n";
    std::cout << "empirical_rate: " << rate << "\n";
    if (gm_result_value_at(res, x0.data(), static_cast<int32_t>(x0.size()), 0, &v, &st) != GM_OK) return fail(st);
    std::cout << "value_at_x0: " << v << "\n";
    if (!a.traj.empty()) {
        if (gm_sim_write_csv(sim, a.traj.c_str(), &st) != GM_OK) return fail(st);
        std::cout << "trajectories: " << a.traj << "\n";
    }
    gm_sim_free(sim);
    gm_result_free(res);
    gm_model_free(m);
    return 0;
}

int not_in_engine(const std::string& verb) {
    std::cerr << "error: '" << verb
              << "' is outside the B200 engine's hot path (MDP construction + synthesis); use the reference CLI\n";
    return 1;
}

void usage() {
    std::cout << "finite MDP abstraction and max-min controller synthesis on uniform grids (B200 engine)\n"
                 "usage: gridmdp {estimate-mem|abstract|synthesize|simulate|export-prism} -c CFG [options]\n"
                 "  --threads N --mem-budget B --seed S --runs R --time-steps T -o PATH\n"
                 "  abstract: --dump-matrix PATH     synthesize: --mode matrix|ofa\n"
                 "  GPU (CLI only): --device N\n"
                 "  synthesize on several GPUs: --gpus N | --devices a,b,.. [--exchange auto|halo|allgather]\n"
                 "                              [--transport nccl|peer]\n";
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        std::cerr << "A subcommand is required\n";
        return 106;
    }
    Args a;
    a.verb = argv[1];
    if (a.verb == "-h" || a.verb == "--help") {
        usage();
        return 0;
    }
    static const std::map<std::string, int> verbs = {
        {"estimate-mem", 0}, {"abstract", 1}, {"synthesize", 2}, {"simulate", 3}, {"export-prism", 4}};
    if (!verbs.count(a.verb)) {
        std::cerr << "The following argument was not expected: " << a.verb << "\n";
        return 109;
    }
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i], v;
        const auto eq = k.find('=');
        bool has_inline = k.rfind("--", 0) == 0 && eq != std::string::npos;
        if (has_inline) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        }
        auto val = [&]() -> std::string {
            if (has_inline) return v;
            if (i + 1 >= argc) {
                std::cerr << k << " requires an argument\n";
                std::exit(107);
            }
            return argv[++i];
        };
        auto num = [&](long long& dst) {
            const std::string s = val();
            char* end = nullptr;
            dst = std::strtoll(s.c_str(), &end, 10);
            if (s.empty() || *end) {
                std::cerr << "Could not convert: " << k << " = " << s << "\n";
                std::exit(105);
            }
        };
        if (k == "-h" || k == "--help") {
            usage();
            return 0;
        } else if (k == "-c" || k == "--config") a.config = val();
        else if (k == "--threads") num(a.threads);
        else if (k == "--mem-budget") num(a.mem_budget);
        else if (k == "--seed") num(a.seed);
        else if (k == "--runs") num(a.runs);
        else if (k == "--time-steps") num(a.time_steps);
        else if (k == "-o" || k == "--output") a.output = val();
        else if (k == "--device") {
            long long d = 0;
            num(d);
            a.device = static_cast<int>(d);
        } else if (k == "--gpus" && a.verb == "synthesize") {
            long long n = 0;
            num(n);
            if (n < 1) {
                std::cerr << "--gpus: " << n << " not >= 1\n";
                return 105;
            }
            a.devices.clear();
            for (int d = 0; d < n; ++d) a.devices.push_back(d);
        } else if (k == "--devices" && a.verb == "synthesize") {
            const std::string s = val();
            a.devices.clear();
            size_t pos = 0;
            while (pos <= s.size()) {
                const size_t c = s.find(',', pos);
                const std::string item = s.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
                char* end = nullptr;
                const long d = std::strtol(item.c_str(), &end, 10);
                if (item.empty() || *end || d < 0) {
                    std::cerr << "Could not convert: --devices = " << s << "\n";
                    return 105;
                }
                a.devices.push_back(static_cast<int>(d));
                if (c == std::string::npos) break;
                pos = c + 1;
            }
        } else if (k == "--exchange" && a.verb == "synthesize") {
            const std::string e = val();
            if (e == "auto") a.exchange = GM_XCHG_AUTO;
            else if (e == "halo") a.exchange = GM_XCHG_HALO;
            else if (e == "allgather") a.exchange = GM_XCHG_ALLGATHER;
            else {
                std::cerr << "--exchange: " << e << " not in {auto,halo,allgather}\n";
                return 105;
            }
        } else if (k == "--transport" && a.verb == "synthesize") {
            const std::string t = val();
            if (t == "nccl") a.transport = GM_XPORT_NCCL;
            else if (t == "peer") a.transport = GM_XPORT_PEER;
            else if (t == "store") a.transport = GM_XPORT_STORE;
            else {
                std::cerr << "--transport: " << t << " not in {nccl,peer,store}\n";
                return 105;
            }
        } else if (k == "--dump-matrix" && a.verb == "abstract") a.dump = val();
        else if (k == "--mode" && a.verb == "synthesize") {
            a.mode = val();
            if (a.mode != "matrix" && a.mode != "ofa") {
                std::cerr << "--mode: " << a.mode << " not in {matrix,ofa}\n";
                return 105;
            }
        } else if (a.verb == "simulate" && k == "--results") a.results = val();
        else if (a.verb == "simulate" && k == "--x0") a.x0 = val();
        else if (a.verb == "simulate" && k == "--traj") a.traj = val();
        else if (a.verb == "simulate" && k == "--dist-mode") {
            a.dist_mode = val();
            if (a.dist_mode != "random" && a.dist_mode != "worst-case") {
                std::cerr << "--dist-mode: " << a.dist_mode << " not in {random,worst-case}\n";
                return 105;
            }
        } else {
            std::cerr << "The following argument was not expected: " << k << "\n";
            return 109;
        }
    }
    if (a.config.empty()) {
        std::cerr << "--config is required\n";
        return 106;
    }
    switch (verbs.at(a.verb)) {
        case 0: return cmd_estimate(a);
        case 1: return cmd_abstract(a);
        case 2: return cmd_synthesize(a);
        case 3:
            if (a.x0.empty()) {
                std::cerr << "--x0 is required\n";
                return 106;
            }
            return cmd_simulate(a);
        case 4: return cmd_export_prism(a);
        default: return not_in_engine(a.verb);
    }
}
