// Host-side front end of the B200 engine: the reference's config-driven model
// description (config, expression language, grids, noise sizing, spec) restated
// in C++ so the drop-in keeps its exact grammar, sizes and error texts, plus the
// device descriptor (GmDev) and the dynamics bytecode the kernels interpret.
#pragma once

#include "gm_device.h"

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace gmh {

// --- error taxonomy (reference common.hpp:16-41) --------------------------
struct ConfigErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseErr : ConfigErr { using ConfigErr::ConfigErr; };
struct DomainErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct MemoryErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaErr : std::runtime_error { using std::runtime_error::runtime_error; };

uint64_t mul_checked(uint64_t a, uint64_t b, const char* what);

// --- uniform grids (reference grid.hpp:16-46, grid.cpp:12-45) -------------
struct Grid {
    std::vector<double> lb, ub, eta;
    std::vector<int64_t> count, stride;
    int64_t total = 1;
    int dim() const { return static_cast<int>(lb.size()); }
    double rep(int d, int64_t j) const { return lb[d] + static_cast<double>(j) * eta[d]; }
};
Grid grid_from(const std::vector<double>& lb, const std::vector<double>& ub,
               const std::vector<double>& eta);
std::vector<double> grid_point(const Grid& g, int64_t flat); // index_to_point (throws out_of_range)
int64_t grid_index(const Grid& g, const std::vector<double>& x); // point_to_index

// --- expression language (reference expr.hpp:30-61, expr.cpp:13-501) ------
enum class XOp : uint8_t {
    add, sub, mul, div, pow, lt, le, gt, ge, eq, ne, neg,
    sin, cos, tan, asin, acos, atan, exp, ln, sqrt, abs, min, max, ite,
    literal, variable
};
struct XNode {
    XOp op = XOp::literal;
    double value = 0.0;
    uint8_t vclass = 0; // 0 state, 1 input, 2 disturbance
    int vindex = 0;
    int32_t kid[3] = {-1, -1, -1};
};
struct Expr {
    std::vector<XNode> nodes;
    int32_t root = -1;
    int n = 0, m = 0, p = 0;
};
Expr parse_expr_text(const std::string& text, int n, int m, int p,
                     const std::map<std::string, double>& constants);
double eval_expr(const Expr& e, const double* x, const double* u, const double* w);
std::string expr_to_string(const Expr& e, int32_t node);

// --- noise (reference noise.hpp, noise.cpp:22-200) --------------------------
struct Noise {
    int family = GM_NORMAL;
    int mult = 0;
    double gamma = 0.0;
    std::vector<double> p1, p2; // custom: support lower / upper corner
    Expr pdf;                   // custom: joint density over xi (state variables x_i)
    int dim() const { return static_cast<int>(p1.size()); }
};
std::optional<std::vector<double>> cut_radius(const Noise& ns);

// --- spec (reference spec.hpp, spec.cpp) ----------------------------------
struct BoxV {
    std::vector<double> lo, hi;
    int dim() const { return static_cast<int>(lo.size()); }
    bool empty() const;
    bool contains(const std::vector<double>& x) const;
};
struct SpecV {
    int kind = GM_SPEC_SAFETY;
    int horizon = 1;
    BoxV target, avoid;
    bool reach() const { return kind != GM_SPEC_SAFETY; }
};
void check_spec(const SpecV& s, const Grid& g);

// --- config (reference config.hpp:22-47, config.cpp:68-237) ---------------
struct GridCfg { int dim = 0; std::vector<double> lb, ub, eta; };
struct BoxCfg { std::vector<double> lb, ub; };
struct Cfg {
    GridCfg states, inputs;
    std::optional<GridCfg> dist;
    std::vector<std::string> dynamics;
    std::map<std::string, double> constants;
    std::string noise_type = "normal";
    int noise_mult = 0;
    double gamma = 0.0;
    std::vector<double> sigma, a, b, rate, alpha, beta;
    std::string pdf;                       // noise.type = custom (engine extension)
    std::vector<double> support_lb, support_ub;
    std::string spec_type;
    int time_steps = 0;
    std::optional<BoxCfg> target, avoid;
    int threads = 0;
    std::string mode = "matrix";
    uint64_t mem_budget = 0;
    uint64_t seed = 0;
    int runs = 100;
    std::string output;
};
Cfg parse_cfg_text(const std::string& text, const std::string& name);
Cfg load_cfg_file(const std::string& path);

// --- the model ---------------------------------------------------------------
struct Program {
    std::vector<GmIns> code;
    std::vector<double> lits;
    std::vector<int32_t> entry; // n+1 offsets into code
    int nregs = 1;
};

struct Model {
    Cfg cfg;
    Grid X, U, W;
    std::vector<Expr> dyn;
    Noise noise;
    SpecV spec;
    int mode = GM_MODE_MATRIX_;
    int threads = 0;
    uint64_t mem_budget = 0;

    std::vector<int64_t> extents;    // window_extents
    int64_t R = 1;                   // row width
    std::optional<std::vector<double>> radius;
    Program prog;

    int64_t n_x() const { return X.total; }
    int64_t n_u() const { return U.total; }
    int64_t n_w() const { return W.total; }
    int64_t rows() const; // checked
    uint64_t memory_estimate() const;
    void refresh(); // recompute extents / program after construction
    GmDev device_descriptor() const;
    // host re-evaluation of one row's dynamics (RowKernel::compute); throws the
    // reference's DomainError text on failure
    void row_image(int64_t row, std::vector<double>& mu) const;
};

Model build_model_from_cfg(const Cfg& cfg);
// make_model (model.cpp:15-29) from already-built parts, e.g. the reference's own
// SystemModel / Spec / SynthesisOptions handed over the C ABI (gm_model_create)
Model build_model_from_parts(const Grid& X, const Grid& U, const Grid& W, std::vector<Expr> dyn, int family,
                             int mult, double gamma, const std::vector<double>& p1, const std::vector<double>& p2,
                             Expr pdf, const SpecV& spec, int mode, int threads, uint64_t mem_budget);
// An expression from a reference node pool (Expr::Node, expr.hpp:36-52), validated.
Expr expr_from_nodes(std::vector<XNode> nodes, int32_t root, int n, int m, int p, const std::string& what);
void finish_model(Model& M);
// save_config (config.cpp:270-310)
std::string save_config_text(const Cfg& c);
SpecV spec_from_cfg(const Cfg& cfg);
int tpr_for_width(int64_t R);
int64_t row_pitch(int64_t R); // row stride of stored matrices (doubles)

std::string fmt_shortest(double v);
std::string fmt_vec(const std::vector<double>& v);

} // namespace gmh
