// gridmdp_b200_adapter.cpp — the reference's hot-path entry points, with their exact
// signatures, implemented on the B200 engine's C ABI (include/gridmdp_b200.h).
//
// A maintainer of the reference (/root/reference/proj) drops this translation unit
// into the library in place of the bodies it replaces:
//   build_matrix          include/gridmdp/abstraction.hpp:112   (src/abstraction.cpp:197-225)
//   build_target_hit      include/gridmdp/abstraction.hpp:117   (src/abstraction.cpp:246-271)
//   synthesize            include/gridmdp/synthesis.hpp:46-47   (src/synthesis.cpp:214-228)
//   synthesize_with_matrix include/gridmdp/synthesis.hpp:51-53  (src/synthesis.cpp:199-212)
//   bellman_step          include/gridmdp/synthesis.hpp:58-61   (src/synthesis.cpp:147-161)
// Everything else (config, expressions, grids, noise, spec, io, sim, mask_absorbing)
// stays the reference's. The model crosses the boundary as the reference holds it
// in memory — grids, the dynamics' expression node pools, the noise parameters,
// the spec and the options (gm_model_create) — so no configuration text is needed.
// SynthesisResult is filled as run_backward does (src/synthesis.cpp:170-188):
// grids, spec, gamma and mode from the inputs, tables from the engine.
//
// integration/Makefile links it against the reference's own objects with these
// five definitions weakened (objcopy), which is exactly the drop-in: every caller
// of the reference API (here oracle/ref_driver.cpp) runs on the GPU unchanged.
#include "gridmdp/abstraction.hpp"
#include "gridmdp/synthesis.hpp"

#include "gridmdp_b200.h"

#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace gridmdp {

namespace {

[[noreturn]] void rethrow(const gm_status& st) {
    // gm_code -> the reference's exception taxonomy (common.hpp:16-41)
    switch (st.code) {
        case GM_ERR_CONFIG: throw ConfigError(st.msg);
        case GM_ERR_MEMORY: throw MemoryError(st.msg);
        case GM_ERR_DOMAIN: throw DomainError(st.msg);
        case GM_ERR_IO: throw IoError(st.msg);
        case GM_ERR_RANGE: throw std::out_of_range(st.msg);
        default: throw std::runtime_error(st.msg);
    }
}

void ok(gm_code rc, const gm_status& st) {
    if (rc != GM_OK) rethrow(st);
}

std::vector<double> vec(const Vector& v) { return std::vector<double>(v.data(), v.data() + v.size()); }

// The reference's in-memory model as a gm_model_desc (storage owned here).
struct Described {
    std::vector<std::vector<double>> arrays;
    std::vector<std::vector<gm_expr_node>> pools;
    std::vector<gm_expr_desc> dyn;
    gm_model_desc d{};

    const double* keep(const Vector& v) {
        arrays.push_back(vec(v));
        return arrays.back().data();
    }
    gm_grid_desc grid(const UniformGrid& g) {
        if (g.dim() == 0) return gm_grid_desc{0, nullptr, nullptr, nullptr};
        return gm_grid_desc{g.dim(), keep(g.lb()), keep(g.ub()), keep(g.eta())};
    }
    gm_expr_desc expr(const Expr& e) {
        std::vector<gm_expr_node> pool;
        for (const Expr::Node& n : e.nodes()) { // expr.hpp:36-52, same Op numbering
            gm_expr_node x{};
            x.op = static_cast<int32_t>(n.op);
            x.var_class = static_cast<int32_t>(n.var_class);
            x.var_index = n.var_index;
            for (int k = 0; k < 3; ++k) x.kid[k] = n.kid[k];
            x.value = n.value;
            pool.push_back(x);
        }
        pools.push_back(std::move(pool));
        return gm_expr_desc{pools.back().data(), static_cast<int32_t>(pools.back().size()), e.root()};
    }

    Described(const SystemModel& m, const Spec& spec, const SynthesisOptions& opts) {
        arrays.reserve(32);
        pools.reserve(m.dynamics.size());
        d.state = grid(m.state);
        d.input = grid(m.input);
        d.disturbance = grid(m.disturbance);
        for (const Expr& e : m.dynamics) dyn.push_back(expr(e));
        d.dynamics = dyn.data();
        d.n_dynamics = static_cast<int32_t>(dyn.size());
        const NoiseSpec& ns = m.noise;
        if (ns.family() == NoiseFamily::custom) // a C++ callback cannot cross the C ABI
            throw ConfigError("B200 engine: custom densities are given as expressions (noise.pdf)");
        d.noise_family = static_cast<int32_t>(ns.family()); // noise.hpp:12, same numbering
        d.noise_mode = ns.mode() == NoiseMode::multiplicative ? 1 : 0;
        d.gamma = ns.gamma();
        d.noise_dim = ns.dim();
        d.param1 = keep(ns.param1());
        d.param2 = ns.param2().size() ? keep(ns.param2()) : nullptr;
        d.spec_kind = static_cast<int32_t>(spec.kind); // spec.hpp:12, same numbering
        d.horizon = spec.horizon;
        if (spec.target.dim()) {
            d.target_lo = keep(spec.target.lo);
            d.target_hi = keep(spec.target.hi);
        }
        if (spec.avoid.dim()) {
            d.avoid_lo = keep(spec.avoid.lo);
            d.avoid_hi = keep(spec.avoid.hi);
        }
        d.mode = opts.mode == SynthesisMode::ofa ? GM_MODE_OFA : GM_MODE_MATRIX;
        d.threads = opts.threads;
        d.mem_budget = opts.memory_budget;
    }
};

struct ModelHandle {
    gm_model* h = nullptr;
    ModelHandle(const SystemModel& m, const Spec& spec, const SynthesisOptions& opts) {
        Described D(m, spec, opts);
        gm_status st;
        ok(gm_model_create(&D.d, &h, &st), st);
    }
    ~ModelHandle() { gm_model_free(h); }
};

struct MatrixHandle {
    gm_matrix* h = nullptr;
    ~MatrixHandle() { gm_matrix_free(h); }
};

struct ResultHandle {
    gm_result* h = nullptr;
    ~ResultHandle() { gm_result_free(h); }
};

SynthesisResult to_result(const SystemModel& m, const Spec& spec, gm_result* r) {
    // run_backward's result fields (src/synthesis.cpp:170-188)
    SynthesisResult res;
    res.state_grid = m.state;
    res.input_grid = m.input;
    res.disturbance_grid = m.disturbance;
    res.spec = spec;
    res.gamma = m.noise.gamma();
    gm_status st;
    int64_t n_x = 0;
    int32_t T = 0, has_abs = 0, mode = 0;
    ok(gm_result_shape(r, &n_x, &T, &has_abs, &mode, &st), st);
    res.mode = mode == GM_MODE_OFA ? SynthesisMode::ofa : SynthesisMode::matrix;
    res.values.resize(n_x, T + 1); // column-major, as the engine's tables
    res.policy.resize(n_x, T);
    res.worst_dist.resize(n_x, T);
    res.absorbing.assign(has_abs ? static_cast<std::size_t>(n_x) : 0, 0);
    ok(gm_result_copy(r, res.values.data(), res.policy.data(), res.worst_dist.data(),
                      has_abs ? res.absorbing.data() : nullptr, &st),
       st);
    return res;
}

// The engine's device copy of a host TransitionMatrix (abstraction.hpp:22-65).
void upload(const ModelHandle& mh, const TransitionMatrix& tm, MatrixHandle& out) {
    gm_status st;
    ok(gm_matrix_upload(mh.h, 0, tm.rows(), tm.origins().data(), tm.payload().data(), &out.h, &st), st);
}

} // namespace

TransitionMatrix build_matrix(const SystemModel& m, int threads) {
    SynthesisOptions opts;
    opts.threads = threads;
    const ModelHandle mh(m, Spec{}, opts);
    gm_status st;
    gm_sizes sz;
    ok(gm_model_sizes(mh.h, &sz, &st), st);
    MatrixHandle dm;
    ok(gm_build_matrix(mh.h, 0, sz.rows, &dm.h, &st), st);
    TransitionMatrix tm; // friend of TransitionMatrix (abstraction.hpp:50)
    tm.state_ = m.state;
    tm.n_inputs_ = m.n_inputs();
    tm.n_dist_ = m.n_disturbances();
    tm.rows_ = sz.rows;
    tm.row_width_ = sz.row_width;
    tm.extents_.assign(sz.extents, sz.extents + sz.n_dim);
    tm.origins_.resize(sz.rows);
    tm.probs_.resize(sz.rows * sz.row_width);
    ok(gm_matrix_copy_rows(dm.h, 0, sz.rows, tm.origins_.data(), tm.probs_.data(), &st), st);
    return tm;
}

TargetHitVector build_target_hit(const SystemModel& m, const Spec& spec, int threads) {
    SynthesisOptions opts;
    opts.threads = threads;
    const ModelHandle mh(m, spec, opts);
    TargetHitVector t0x(m.n_rows());
    gm_status st;
    ok(gm_build_target_hit(mh.h, 0, m.n_rows(), t0x.data(), &st), st);
    return t0x;
}

// Devices of this process for synthesize: GRIDMDP_B200_DEVICES="0,1,2,3" (the reference's
// SynthesisOptions has no device field; the variable keeps its signature unchanged).
std::vector<int32_t> adapter_devices() {
    std::vector<int32_t> out;
    const char* e = std::getenv("GRIDMDP_B200_DEVICES");
    if (!e || !*e) return out;
    std::string s(e);
    size_t pos = 0;
    while (pos <= s.size()) {
        const size_t c = s.find(',', pos);
        out.push_back(static_cast<int32_t>(std::stoi(s.substr(pos, c == std::string::npos ? std::string::npos : c - pos))));
        if (c == std::string::npos) break;
        pos = c + 1;
    }
    return out;
}

SynthesisResult synthesize(const SystemModel& m, const Spec& spec, const SynthesisOptions& opts) {
    const ModelHandle mh(m, spec, opts);
    ResultHandle r;
    gm_status st;
    const std::vector<int32_t> dev = adapter_devices();
    if (dev.size() > 1) { // state shards over the listed GPUs, V exchanged by NCCL (parallel.hpp:23-51's role)
        const char* tp = std::getenv("GRIDMDP_B200_TRANSPORT");
        const int32_t transport = tp && std::string(tp) == "peer"    ? GM_XPORT_PEER
                                 : tp && std::string(tp) == "store" ? GM_XPORT_STORE
                                                                    : GM_XPORT_NCCL;
        ok(gm_synthesize_multi(mh.h, static_cast<int32_t>(dev.size()), dev.data(), GM_XCHG_AUTO, transport, &r.h,
                               nullptr, &st),
           st);
    } else {
        if (dev.size() == 1) ok(gm_set_device(dev[0], &st), st);
        ok(gm_synthesize(mh.h, &r.h, &st), st); // budget check, build, mask, T0x, backward
    }
    return to_result(m, spec, r.h);
}

SynthesisResult synthesize_with_matrix(const SystemModel& m, TransitionMatrix& tm, const TargetHitVector* t0x,
                                       const Spec& spec, const SynthesisOptions& opts) {
    const ModelHandle mh(m, spec, opts);
    MatrixHandle dm;
    upload(mh, tm, dm);
    ResultHandle r;
    gm_status st;
    ok(gm_synthesize_with_matrix(mh.h, dm.h, t0x ? t0x->data() : nullptr, &r.h, &st), st);
    if (spec.is_reach()) // the reference masks the caller's kernel in place (synthesis.cpp:205)
        ok(gm_matrix_copy_rows(dm.h, 0, tm.rows(), nullptr, tm.payload().data(), &st), st);
    return to_result(m, spec, r.h);
}

void bellman_step(const SystemModel& m, const Spec& spec, const TransitionMatrix* tm, const TargetHitVector* t0x,
                  const Eigen::VectorXd& v_next, Eigen::VectorXd& v_out, std::uint32_t* policy_out,
                  std::uint32_t* wstar_out, int threads) {
    SynthesisOptions opts;
    opts.threads = threads;
    opts.mode = tm ? SynthesisMode::matrix : SynthesisMode::ofa;
    const ModelHandle mh(m, spec, opts);
    MatrixHandle dm;
    if (tm) upload(mh, *tm, dm);
    v_out.resize(m.n_states());
    gm_status st;
    ok(gm_bellman_step(mh.h, dm.h, t0x ? t0x->data() : nullptr, v_next.data(), v_out.data(), policy_out, wstar_out,
                       &st),
       st);
}

} // namespace gridmdp
