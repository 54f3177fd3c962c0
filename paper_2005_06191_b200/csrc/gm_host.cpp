// Host front end: config interpreter, expression language, grids, noise sizing,
// spec checks, and the lowering of a model to the device descriptor + bytecode.
//
// Semantics follow the reference exactly (file:line cited per function); the
// code is organised for the GPU engine: expressions are lowered to a register
// bytecode with lazy ite jumps that the kernels interpret, and host evaluation
// exists only to reproduce the reference's DomainError text for the lowest
// failing row that a kernel flags.
#include "gm_host.hpp"

#include <algorithm>
#include <charconv>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <sstream>

namespace gmh {

namespace {
constexpr double kTol = 1e-9; // index tolerance, grid.cpp:10 / abstraction.cpp:10
constexpr double kRoot2 = 1.4142135623730951; // noise.cpp:10
}

uint64_t mul_checked(uint64_t a, uint64_t b, const char* what) {
    // common.hpp:67-71
    if (a != 0 && b > UINT64_MAX / a)
        throw MemoryErr(std::string(what) + ": size arithmetic overflows 64 bits");
    return a * b;
}

std::string fmt_shortest(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

std::string fmt_vec(const std::vector<double>& v) {
    std::string s = "{";
    for (size_t i = 0; i < v.size(); ++i) {
        if (i) s += ", ";
        s += fmt_shortest(v[i]);
    }
    return s + "}";
}

// ===========================================================================
// grids — grid.cpp:12-96
// ===========================================================================

Grid grid_from(const std::vector<double>& lb, const std::vector<double>& ub,
               const std::vector<double>& eta) {
    if (lb.size() != ub.size() || lb.size() != eta.size())
        throw ConfigErr("make_grid: lb/ub/eta dimension mismatch");
    Grid g;
    g.lb = lb;
    g.ub = ub;
    g.eta = eta;
    const size_t d = lb.size();
    g.count.assign(d, 0);
    g.stride.assign(d, 0);
    g.total = 1;
    for (size_t i = 0; i < d; ++i) {
        if (!(eta[i] > 0.0)) {
            std::ostringstream os;
            os << "make_grid: eta[" << i << "] = " << eta[i] << " must be positive";
            throw ConfigErr(os.str());
        }
        if (lb[i] > ub[i]) {
            std::ostringstream os;
            os << "make_grid: lb[" << i << "] = " << lb[i] << " exceeds ub[" << i << "] = " << ub[i];
            throw ConfigErr(os.str());
        }
        const double q = (ub[i] - lb[i]) / eta[i];
        g.count[i] = static_cast<int64_t>(std::floor(q + kTol)) + 1;
        g.total = static_cast<int64_t>(
            mul_checked(static_cast<uint64_t>(g.total), static_cast<uint64_t>(g.count[i]), "make_grid"));
    }
    int64_t s = 1;
    for (size_t i = d; i-- > 0;) {
        g.stride[i] = s;
        s *= g.count[i];
    }
    return g;
}

std::vector<double> grid_point(const Grid& g, int64_t i) {
    if (i < 0 || i >= g.total)
        throw std::out_of_range("index_to_point: flat index " + std::to_string(i) + " out of range");
    std::vector<double> p(g.dim());
    for (int d = 0; d < g.dim(); ++d) {
        const int64_t j = i / g.stride[d];
        i %= g.stride[d];
        p[d] = g.rep(d, j);
    }
    return p;
}

int64_t grid_index(const Grid& g, const std::vector<double>& x) {
    if (static_cast<int>(x.size()) != g.dim())
        throw std::out_of_range("point_to_index: point dimension mismatch");
    int64_t flat = 0;
    for (int d = 0; d < g.dim(); ++d) {
        const double t = (x[d] - g.lb[d]) / g.eta[d];
        if (t < -0.5 - kTol || t > static_cast<double>(g.count[d] - 1) + 0.5 + kTol) {
            std::ostringstream os;
            os << "point_to_index: coordinate " << x[d] << " of axis " << d
               << " lies outside the quantized region";
            throw std::out_of_range(os.str());
        }
        int64_t j = static_cast<int64_t>(std::floor(t + 0.5));
        j = std::clamp<int64_t>(j, 0, g.count[d] - 1);
        flat += j * g.stride[d];
    }
    return flat;
}

// ===========================================================================
// expression language — grammar of expr.cpp:13-25, parser expr.cpp:41-288
// ===========================================================================

namespace {

struct FnDef {
    const char* name;
    XOp op;
    int arity;
};
const FnDef kFns[] = {
    {"sin", XOp::sin, 1},   {"cos", XOp::cos, 1},   {"tan", XOp::tan, 1},  {"asin", XOp::asin, 1},
    {"acos", XOp::acos, 1}, {"atan", XOp::atan, 1}, {"exp", XOp::exp, 1},  {"ln", XOp::ln, 1},
    {"sqrt", XOp::sqrt, 1}, {"abs", XOp::abs, 1},   {"min", XOp::min, 2},  {"max", XOp::max, 2},
    {"ite", XOp::ite, 3},
};

// Recursive-descent reader. Positions are 1-based line:col of the cursor at
// the time of the error (expr.cpp:64-68); nesting deeper than 200 levels of
// cmp/sum/term/unary is rejected (expr.cpp:107,135,147,159).
class Reader {
public:
    Reader(const std::string& t, int n, int m, int p, const std::map<std::string, double>& c)
        : s_(t), n_(n), m_(m), p_(p), consts_(c) {}

    Expr run() {
        Expr e;
        e.n = n_;
        e.m = m_;
        e.p = p_;
        out_ = &e.nodes;
        if (s_.find_first_not_of(" \t\r\n") == std::string::npos) error("empty expression");
        e.root = cmp(0);
        blank();
        if (i_ < s_.size()) error(std::string("unexpected trailing input '") + s_[i_] + "'");
        return e;
    }

private:
    const std::string& s_;
    int n_, m_, p_;
    const std::map<std::string, double>& consts_;
    std::vector<XNode>* out_ = nullptr;
    size_t i_ = 0;
    int line_ = 1, col_ = 1;

    [[noreturn]] void error(const std::string& what) const {
        std::ostringstream os;
        os << "expression error at " << line_ << ":" << col_ << ": " << what;
        throw ParseErr(os.str());
    }
    void step() {
        if (s_[i_] == '\n') {
            ++line_;
            col_ = 1;
        } else {
            ++col_;
        }
        ++i_;
    }
    void blank() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\r' || s_[i_] == '\n'))
            step();
    }
    char look() {
        blank();
        return i_ < s_.size() ? s_[i_] : '\0';
    }
    bool take(char c) {
        if (look() != c) return false;
        step();
        return true;
    }
    bool take2(char a, char b) {
        blank();
        if (i_ + 1 < s_.size() && s_[i_] == a && s_[i_ + 1] == b) {
            step();
            step();
            return true;
        }
        return false;
    }
    int32_t push(const XNode& nd) {
        out_->push_back(nd);
        return static_cast<int32_t>(out_->size() - 1);
    }
    int32_t lit(double v) {
        XNode nd;
        nd.op = XOp::literal;
        nd.value = v;
        return push(nd);
    }
    int32_t bin(XOp op, int32_t a, int32_t b) {
        XNode nd;
        nd.op = op;
        nd.kid[0] = a;
        nd.kid[1] = b;
        return push(nd);
    }

    int32_t cmp(int depth) {
        if (depth > 200) error("expression nested too deeply");
        int32_t lhs = sum(depth + 1);
        for (;;) {
            blank();
            XOp op;
            if (take2('<', '=')) op = XOp::le;
            else if (take2('>', '=')) op = XOp::ge;
            else if (take2('=', '=')) op = XOp::eq;
            else if (take2('!', '=')) op = XOp::ne;
            else if (look() == '<') { step(); op = XOp::lt; }
            else if (look() == '>') { step(); op = XOp::gt; }
            else break;
            lhs = bin(op, lhs, sum(depth + 1));
        }
        return lhs;
    }
    int32_t sum(int depth) {
        if (depth > 200) error("expression nested too deeply");
        int32_t lhs = term(depth + 1);
        for (char c = look(); c == '+' || c == '-'; c = look()) {
            step();
            lhs = bin(c == '+' ? XOp::add : XOp::sub, lhs, term(depth + 1));
        }
        return lhs;
    }
    int32_t term(int depth) {
        if (depth > 200) error("expression nested too deeply");
        int32_t lhs = unary(depth + 1);
        for (char c = look(); c == '*' || c == '/'; c = look()) {
            step();
            lhs = bin(c == '*' ? XOp::mul : XOp::div, lhs, unary(depth + 1));
        }
        return lhs;
    }
    int32_t unary(int depth) {
        if (depth > 200) error("expression nested too deeply");
        if (look() == '-') {
            step();
            const int32_t child = unary(depth + 1);
            XNode& c = (*out_)[static_cast<size_t>(child)];
            if (c.op == XOp::literal) { // negative literals fold (expr.cpp:163-168)
                c.value = -c.value;
                return child;
            }
            XNode nd;
            nd.op = XOp::neg;
            nd.kid[0] = child;
            return push(nd);
        }
        return power(depth + 1);
    }
    int32_t power(int depth) {
        const int32_t base = primary(depth + 1);
        if (look() == '^') { // right-assoc, exponent is a unary (expr.cpp:177-184)
            step();
            return bin(XOp::pow, base, unary(depth + 1));
        }
        return base;
    }
    int32_t primary(int depth) {
        const char c = look();
        if (c == '(') {
            step();
            const int32_t inner = cmp(depth + 1);
            if (!take(')')) error("expected ')'");
            return inner;
        }
        if (c == '.' || (c >= '0' && c <= '9')) return number();
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') return ident(depth);
        if (c == '\0') error("unexpected end of expression");
        error(std::string("unexpected character '") + c + "'");
    }
    int32_t number() {
        blank();
        const size_t start = i_;
        while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '.')) step();
        if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
            const size_t si = i_;
            const int sl = line_, sc = col_;
            step();
            if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) step();
            if (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) {
                while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) step();
            } else {
                i_ = si;
                line_ = sl;
                col_ = sc;
            }
        }
        const std::string tok = s_.substr(start, i_ - start);
        char* end = nullptr;
        const double v = std::strtod(tok.c_str(), &end);
        if (end != tok.c_str() + tok.size()) error("malformed number '" + tok + "'");
        return lit(v);
    }
    int32_t ident(int depth) {
        blank();
        const size_t start = i_;
        while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_')) step();
        const std::string name = s_.substr(start, i_ - start);
        if (look() == '(') {
            for (const FnDef& f : kFns)
                if (name == f.name) return call(f, depth);
            error("unknown function '" + name + "'");
        }
        if (name.size() >= 2 && (name[0] == 'x' || name[0] == 'u' || name[0] == 'w')) {
            bool digits = true;
            for (size_t k = 1; k < name.size(); ++k)
                if (!std::isdigit(static_cast<unsigned char>(name[k]))) { digits = false; break; }
            if (digits) {
                const int idx = std::atoi(name.c_str() + 1);
                int cls, lim;
                const char* what;
                if (name[0] == 'x') { cls = 0; lim = n_; what = "state"; }
                else if (name[0] == 'u') { cls = 1; lim = m_; what = "input"; }
                else { cls = 2; lim = p_; what = "disturbance"; }
                if (idx >= lim) {
                    std::ostringstream os;
                    os << what << " variable " << name << " out of range (dimension " << lim << ")";
                    error(os.str());
                }
                XNode nd;
                nd.op = XOp::variable;
                nd.vclass = static_cast<uint8_t>(cls);
                nd.vindex = idx;
                return push(nd);
            }
        }
        auto it = consts_.find(name);
        if (it != consts_.end()) return lit(it->second);
        error("unknown identifier '" + name + "'");
    }
    int32_t call(const FnDef& f, int depth) {
        take('(');
        int32_t args[3] = {-1, -1, -1};
        for (int k = 0; k < f.arity; ++k) {
            if (k > 0 && !take(',')) error(std::string("expected ',' in call to ") + f.name);
            args[k] = cmp(depth + 1);
        }
        if (!take(')')) error(std::string("expected ')' closing call to ") + f.name);
        XNode nd;
        nd.op = f.op;
        nd.kid[0] = args[0];
        nd.kid[1] = args[1];
        nd.kid[2] = args[2];
        return push(nd);
    }
};

// Precedence-aware printer (expr.cpp:290-398): used for DomainError texts.
int prec_of(XOp op) {
    switch (op) {
        case XOp::lt: case XOp::le: case XOp::gt: case XOp::ge: case XOp::eq: case XOp::ne: return 1;
        case XOp::add: case XOp::sub: return 2;
        case XOp::mul: case XOp::div: return 3;
        case XOp::neg: return 4;
        case XOp::pow: return 5;
        default: return 6;
    }
}
const char* infix_of(XOp op) {
    switch (op) {
        case XOp::add: return " + ";
        case XOp::sub: return " - ";
        case XOp::mul: return "*";
        case XOp::div: return "/";
        case XOp::pow: return "^";
        case XOp::lt: return " < ";
        case XOp::le: return " <= ";
        case XOp::gt: return " > ";
        case XOp::ge: return " >= ";
        case XOp::eq: return " == ";
        case XOp::ne: return " != ";
        default: return "?";
    }
}
const char* fname_of(XOp op) {
    for (const FnDef& f : kFns)
        if (f.op == op) return f.name;
    return "?";
}
void print_rec(const Expr& e, int32_t id, std::string& out, int parent) {
    const XNode& nd = e.nodes[static_cast<size_t>(id)];
    const int pr = prec_of(nd.op);
    switch (nd.op) {
        case XOp::literal: {
            const bool wrap = nd.value < 0.0 || std::signbit(nd.value);
            if (wrap) out += '(';
            out += fmt_shortest(nd.value);
            if (wrap) out += ')';
            return;
        }
        case XOp::variable:
            out += (nd.vclass == 0 ? 'x' : nd.vclass == 1 ? 'u' : 'w');
            out += std::to_string(nd.vindex);
            return;
        case XOp::neg: {
            const bool wrap = pr < parent;
            if (wrap) out += '(';
            out += '-';
            print_rec(e, nd.kid[0], out, pr);
            if (wrap) out += ')';
            return;
        }
        case XOp::sin: case XOp::cos: case XOp::tan: case XOp::asin: case XOp::acos:
        case XOp::atan: case XOp::exp: case XOp::ln: case XOp::sqrt: case XOp::abs:
        case XOp::min: case XOp::max: case XOp::ite:
            out += fname_of(nd.op);
            out += '(';
            print_rec(e, nd.kid[0], out, 0);
            for (int k = 1; k < 3 && nd.kid[k] >= 0; ++k) {
                out += ", ";
                print_rec(e, nd.kid[k], out, 0);
            }
            out += ')';
            return;
        default: {
            const bool wrap = pr < parent;
            if (wrap) out += '(';
            if (nd.op == XOp::pow) {
                print_rec(e, nd.kid[0], out, pr + 1);
                out += infix_of(nd.op);
                print_rec(e, nd.kid[1], out, 4);
            } else {
                print_rec(e, nd.kid[0], out, pr);
                out += infix_of(nd.op);
                print_rec(e, nd.kid[1], out, pr + 1);
            }
            if (wrap) out += ')';
            return;
        }
    }
}

[[noreturn]] void fail_domain(const Expr& e, int32_t id, const char* what) {
    throw DomainErr(std::string(what) + " in subexpression '" + expr_to_string(e, id) + "'");
}

// Host evaluator (expr.cpp:404-480): the authority for DomainError texts.
double eval_rec(const Expr& e, int32_t id, const double* x, const double* u, const double* w) {
    const XNode& nd = e.nodes[static_cast<size_t>(id)];
    auto K = [&](int k) { return eval_rec(e, nd.kid[k], x, u, w); };
    switch (nd.op) {
        case XOp::literal: return nd.value;
        case XOp::variable: return nd.vclass == 0 ? x[nd.vindex] : nd.vclass == 1 ? u[nd.vindex] : w[nd.vindex];
        case XOp::add: { const double a = K(0); return a + K(1); }
        case XOp::sub: { const double a = K(0); return a - K(1); }
        case XOp::mul: { const double a = K(0); return a * K(1); }
        case XOp::div: {
            const double a = K(0), b = K(1);
            if (b == 0.0) fail_domain(e, id, "division by zero");
            return a / b;
        }
        case XOp::pow: {
            const double a = K(0), b = K(1);
            if (a < 0.0 && b != std::floor(b)) fail_domain(e, id, "non-integer power of a negative base");
            if (a == 0.0 && b < 0.0) fail_domain(e, id, "division by zero");
            return std::pow(a, b);
        }
        case XOp::lt: { const double a = K(0); return a < K(1) ? 1.0 : 0.0; }
        case XOp::le: { const double a = K(0); return a <= K(1) ? 1.0 : 0.0; }
        case XOp::gt: { const double a = K(0); return a > K(1) ? 1.0 : 0.0; }
        case XOp::ge: { const double a = K(0); return a >= K(1) ? 1.0 : 0.0; }
        case XOp::eq: { const double a = K(0); return a == K(1) ? 1.0 : 0.0; }
        case XOp::ne: { const double a = K(0); return a != K(1) ? 1.0 : 0.0; }
        case XOp::neg: return -K(0);
        case XOp::sin: return std::sin(K(0));
        case XOp::cos: return std::cos(K(0));
        case XOp::tan: return std::tan(K(0));
        case XOp::asin: {
            const double a = K(0);
            if (a < -1.0 || a > 1.0) fail_domain(e, id, "asin argument outside [-1, 1]");
            return std::asin(a);
        }
        case XOp::acos: {
            const double a = K(0);
            if (a < -1.0 || a > 1.0) fail_domain(e, id, "acos argument outside [-1, 1]");
            return std::acos(a);
        }
        case XOp::atan: return std::atan(K(0));
        case XOp::exp: return std::exp(K(0));
        case XOp::ln: {
            const double a = K(0);
            if (a <= 0.0) fail_domain(e, id, "ln of a non-positive value");
            return std::log(a);
        }
        case XOp::sqrt: {
            const double a = K(0);
            if (a < 0.0) fail_domain(e, id, "sqrt of a negative value");
            return std::sqrt(a);
        }
        case XOp::abs: return std::fabs(K(0));
        case XOp::min: { const double a = K(0), b = K(1); return std::fmin(a, b); }
        case XOp::max: { const double a = K(0), b = K(1); return std::fmax(a, b); }
        case XOp::ite: return K(0) != 0.0 ? K(1) : K(2);
    }
    return 0.0;
}

} // namespace

Expr parse_expr_text(const std::string& text, int n, int m, int p,
                     const std::map<std::string, double>& constants) {
    return Reader(text, n, m, p, constants).run();
}

double eval_expr(const Expr& e, const double* x, const double* u, const double* w) {
    return eval_rec(e, e.root, x, u, w);
}

std::string expr_to_string(const Expr& e, int32_t node) {
    std::string s;
    print_rec(e, node, s, 0);
    return s;
}

// ===========================================================================
// bytecode lowering: tree -> register program (device interpreter input)
// ===========================================================================

namespace {

struct Lowering {
    const Expr& e;
    Program& P;
    int maxreg = 0;

    void emit(uint8_t op, int dst, int a, int b, int32_t arg) {
        if (dst >= GMD_MAXREGS || a >= GMD_MAXREGS || b >= GMD_MAXREGS)
            throw ConfigErr("expression needs more than " + std::to_string(GMD_MAXREGS) +
                            " device evaluation registers");
        maxreg = std::max(maxreg, dst + 1);
        GmIns in;
        in.op = op;
        in.dst = static_cast<uint8_t>(dst);
        in.a = static_cast<uint8_t>(a);
        in.b = static_cast<uint8_t>(b);
        in.arg = arg;
        P.code.push_back(in);
    }
    int32_t lit_index(double v) {
        for (size_t i = 0; i < P.lits.size(); ++i) {
            double q = P.lits[i];
            if (std::memcmp(&q, &v, sizeof v) == 0) return static_cast<int32_t>(i);
        }
        P.lits.push_back(v);
        return static_cast<int32_t>(P.lits.size() - 1);
    }
    // evaluates node `id` into register r, using registers >= r as scratch;
    // operand order left to right as the host evaluator.
    void gen(int32_t id, int r) {
        const XNode& nd = e.nodes[static_cast<size_t>(id)];
        switch (nd.op) {
            case XOp::literal: emit(GI_LIT, r, 0, 0, lit_index(nd.value)); return;
            case XOp::variable:
                emit(nd.vclass == 0 ? GI_LDX : nd.vclass == 1 ? GI_LDU : GI_LDW, r, 0, 0, nd.vindex);
                return;
            case XOp::ite: {
                gen(nd.kid[0], r);
                const size_t jz = P.code.size();
                emit(GI_JZ, r, r, 0, 0);
                gen(nd.kid[1], r);
                const size_t jmp = P.code.size();
                emit(GI_JMP, r, 0, 0, 0);
                P.code[jz].arg = static_cast<int32_t>(P.code.size());
                gen(nd.kid[2], r);
                P.code[jmp].arg = static_cast<int32_t>(P.code.size());
                return;
            }
            default: break;
        }
        uint8_t op;
        int arity = 2;
        switch (nd.op) {
            case XOp::add: op = GI_ADD; break;
            case XOp::sub: op = GI_SUB; break;
            case XOp::mul: op = GI_MUL; break;
            case XOp::div: op = GI_DIV; break;
            case XOp::pow: op = GI_POW; break;
            case XOp::lt: op = GI_LT; break;
            case XOp::le: op = GI_LE; break;
            case XOp::gt: op = GI_GT; break;
            case XOp::ge: op = GI_GE; break;
            case XOp::eq: op = GI_EQ; break;
            case XOp::ne: op = GI_NE; break;
            case XOp::min: op = GI_MIN; break;
            case XOp::max: op = GI_MAX; break;
            case XOp::neg: op = GI_NEG; arity = 1; break;
            case XOp::sin: op = GI_SIN; arity = 1; break;
            case XOp::cos: op = GI_COS; arity = 1; break;
            case XOp::tan: op = GI_TAN; arity = 1; break;
            case XOp::asin: op = GI_ASIN; arity = 1; break;
            case XOp::acos: op = GI_ACOS; arity = 1; break;
            case XOp::atan: op = GI_ATAN; arity = 1; break;
            case XOp::exp: op = GI_EXP; arity = 1; break;
            case XOp::ln: op = GI_LN; arity = 1; break;
            case XOp::sqrt: op = GI_SQRT; arity = 1; break;
            case XOp::abs: op = GI_ABS; arity = 1; break;
            default: throw ConfigErr("internal: unknown expression node");
        }
        gen(nd.kid[0], r);
        if (arity == 2) {
            gen(nd.kid[1], r + 1);
            emit(op, r, r, r + 1, id);
        } else {
            emit(op, r, r, 0, id);
        }
    }
};

} // namespace

// ===========================================================================
// noise sizing — cutting_radius noise.cpp:137-180, parameter checks :22-73
// ===========================================================================

std::optional<std::vector<double>> cut_radius(const Noise& ns) {
    const int n = ns.dim();
    std::vector<double> r(static_cast<size_t>(n), 0.0);
    if (ns.mult) return std::nullopt;
    switch (ns.family) {
        case GM_NORMAL: {
            if (ns.gamma == 0.0) return std::nullopt;
            double log_c = 0.0; // log of 1 / peak density
            for (int j = 0; j < n; ++j) log_c += 0.5 * std::log(2.0 * M_PI * ns.p1[j] * ns.p1[j]);
            const double t = -2.0 * (std::log(ns.gamma) + log_c);
            if (t <= 0.0) return r;
            for (int i = 0; i < n; ++i) r[i] = ns.p1[i] * std::sqrt(t);
            return r;
        }
        case GM_EXPONENTIAL: {
            if (ns.gamma == 0.0) return std::nullopt;
            double log_peak = 0.0;
            for (int j = 0; j < n; ++j) log_peak += std::log(ns.p1[j]);
            const double t = log_peak - std::log(ns.gamma);
            if (t <= 0.0) return r;
            for (int i = 0; i < n; ++i) r[i] = t / ns.p1[i];
            return r;
        }
        case GM_UNIFORM:
            for (int i = 0; i < n; ++i) r[i] = std::max(std::fabs(ns.p1[i]), std::fabs(ns.p2[i]));
            return r;
        case GM_BETA:
            for (int i = 0; i < n; ++i) r[i] = 1.0;
            return r;
        case GM_CUSTOM: // noise.cpp:172-177
            for (int i = 0; i < n; ++i) r[i] = std::max(std::fabs(ns.p1[i]), std::fabs(ns.p2[i]));
            return r;
    }
    return std::nullopt;
}

namespace {
void need(bool ok, const char* msg) {
    if (!ok) throw ConfigErr(msg);
}
Noise make_noise(int family, const std::vector<double>& a, const std::vector<double>& b,
                 double gamma, int mult) {
    need(gamma >= 0.0 && gamma <= 1.0, "noise: cutting threshold gamma must lie in [0, 1]");
    Noise ns;
    ns.family = family;
    ns.mult = mult;
    ns.gamma = gamma;
    ns.p1 = a;
    ns.p2 = b;
    auto all = [](const std::vector<double>& v, auto f) { return std::all_of(v.begin(), v.end(), f); };
    switch (family) {
        case GM_NORMAL:
            need(all(a, [](double s) { return s > 0.0; }), "noise: normal std deviations must be positive");
            break;
        case GM_UNIFORM: {
            need(a.size() == b.size(), "noise: uniform bounds dimension mismatch");
            bool ok = true;
            for (size_t i = 0; i < a.size(); ++i) ok = ok && a[i] < b[i];
            need(ok, "noise: uniform support requires a < b");
            break;
        }
        case GM_EXPONENTIAL:
            need(all(a, [](double s) { return s > 0.0; }), "noise: exponential rates must be positive");
            break;
        case GM_CUSTOM: { // noise.cpp:75-85
            bool nonempty = !a.empty() && a.size() == b.size();
            for (size_t i = 0; nonempty && i < a.size(); ++i) nonempty = a[i] <= b[i];
            need(nonempty, "noise: custom density requires a non-empty support box");
            break;
        }
        case GM_BETA:
            need(a.size() == b.size(), "noise: beta shape dimension mismatch");
            need(all(a, [](double s) { return s > 0.0; }) && all(b, [](double s) { return s > 0.0; }),
                 "noise: beta shapes must be positive");
            break;
    }
    return ns;
}
} // namespace

// ===========================================================================
// spec — spec.hpp:14-28, spec.cpp:41-60
// ===========================================================================

bool BoxV::empty() const {
    if (lo.empty()) return true;
    for (size_t d = 0; d < lo.size(); ++d)
        if (lo[d] > hi[d]) return true;
    return false;
}

bool BoxV::contains(const std::vector<double>& x) const {
    if (x.size() != lo.size()) return false;
    for (size_t d = 0; d < lo.size(); ++d)
        if (!(x[d] >= lo[d])) return false;
    for (size_t d = 0; d < lo.size(); ++d)
        if (!(x[d] <= hi[d])) return false;
    return true;
}

namespace {
void box_within(const BoxV& b, const Grid& g, const char* name) {
    if (b.dim() == 0) return;
    if (b.dim() != g.dim())
        throw ConfigErr(std::string(name) + " box dimension does not match the state grid");
    for (int d = 0; d < g.dim(); ++d) {
        if (b.lo[d] > b.hi[d]) throw ConfigErr(std::string(name) + " box has lb > ub");
        if (b.lo[d] < g.lb[d] || b.hi[d] > g.ub[d])
            throw ConfigErr(std::string(name) + " box must lie within the state box");
    }
}
} // namespace

void check_spec(const SpecV& s, const Grid& g) {
    if (s.horizon < 1) throw ConfigErr("spec: time horizon must be at least 1");
    if (s.reach() && s.target.dim() == 0)
        throw ConfigErr("spec: reachability/reach-avoid requires a target box");
    if (s.kind == GM_SPEC_SAFETY && (s.target.dim() != 0 || s.avoid.dim() != 0))
        throw ConfigErr("spec: safety takes no target/avoid boxes");
    box_within(s.target, g, "target");
    box_within(s.avoid, g, "avoid");
}

// ===========================================================================
// config interpreter — config.cpp:11-237 (same statements, keys, order of
// checks and messages)
// ===========================================================================

namespace {

std::string strip(const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return {};
    const auto e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}

struct Stmt {
    std::string value;
    int line = 0;
    bool used = false;
};

class CfgReader {
public:
    CfgReader(std::istream& in, std::string name) : name_(std::move(name)) {
        std::string raw;
        int ln = 0;
        while (std::getline(in, raw)) {
            ++ln;
            const auto hash = raw.find('#');
            if (hash != std::string::npos) raw.erase(hash);
            const std::string s = strip(raw);
            if (s.empty()) continue;
            if (s.back() != ';') bad(ln, "statement must end with ';'");
            const auto eq = s.find('=');
            if (eq == std::string::npos) bad(ln, "expected 'key = value;'");
            const std::string key = strip(s.substr(0, eq));
            const std::string val = strip(s.substr(eq + 1, s.size() - eq - 2));
            if (key.empty()) bad(ln, "empty key");
            if (st_.count(key)) bad(ln, "duplicate key '" + key + "'");
            st_[key] = Stmt{val, ln, false};
        }
    }

    Cfg read() {
        Cfg c;
        c.states = grid("states");
        c.inputs = grid("inputs");
        if (prefixed("disturbances.")) c.dist = grid("disturbances");
        for (int i = 0; i < c.states.dim; ++i) {
            const std::string k = "dynamics.x" + std::to_string(i);
            const Stmt* s = find(k);
            if (!s) throw ConfigErr(name_ + ": missing mandatory key '" + k + "'");
            c.dynamics.push_back(s->value);
        }
        for (auto& kv : st_) {
            if (kv.first.rfind("constants.", 0) == 0) {
                c.constants[kv.first.substr(10)] = num(kv.second.line, kv.second.value);
                kv.second.used = true;
            }
        }
        c.noise_type = req("noise.type").value;
        if (const Stmt* s = find("noise.mode")) {
            if (s->value == "additive") c.noise_mult = 0;
            else if (s->value == "multiplicative") c.noise_mult = 1;
            else bad(s->line, "noise.mode must be additive or multiplicative");
        }
        if (const Stmt* s = find("noise.cutting_probability")) c.gamma = num(s->line, s->value);
        if (c.noise_type == "normal") {
            c.sigma = vec("noise.sigma");
        } else if (c.noise_type == "uniform") {
            c.a = vec("noise.a");
            c.b = vec("noise.b");
        } else if (c.noise_type == "exponential") {
            c.rate = vec("noise.rate");
        } else if (c.noise_type == "beta") {
            c.alpha = vec("noise.alpha");
            c.beta = vec("noise.beta");
        } else if (c.noise_type == "custom") {
            // engine extension of NoiseSpec::custom (noise.hpp:16-19, noise.cpp:75-85):
            // the joint pdf as an expression over the noise coordinates x0..x{n-1}
            c.pdf = req("noise.pdf").value;
            c.support_lb = vec("noise.support.lb");
            c.support_ub = vec("noise.support.ub");
        } else {
            throw ConfigErr(name_ + ": unknown noise.type '" + c.noise_type + "'");
        }
        c.spec_type = req("spec.type").value;
        c.time_steps = static_cast<int>(integer("spec.time_steps"));
        if (prefixed("target.")) {
            BoxCfg b;
            b.lb = vec("target.lb");
            b.ub = vec("target.ub");
            c.target = b;
        }
        if (prefixed("avoid.")) {
            BoxCfg b;
            b.lb = vec("avoid.lb");
            b.ub = vec("avoid.ub");
            c.avoid = b;
        }
        if (const Stmt* s = find("exec.threads")) c.threads = static_cast<int>(intval(s->line, s->value));
        if (const Stmt* s = find("exec.mode")) {
            if (s->value != "matrix" && s->value != "ofa") bad(s->line, "exec.mode must be matrix or ofa");
            c.mode = s->value;
        }
        if (const Stmt* s = find("exec.mem_budget"))
            c.mem_budget = static_cast<uint64_t>(intval(s->line, s->value));
        if (const Stmt* s = find("exec.seed")) c.seed = static_cast<uint64_t>(intval(s->line, s->value));
        if (const Stmt* s = find("exec.runs")) c.runs = static_cast<int>(intval(s->line, s->value));
        if (const Stmt* s = find("exec.output")) c.output = s->value;
        for (const auto& kv : st_)
            if (!kv.second.used) bad(kv.second.line, "unknown key '" + kv.first + "'");
        validate(c);
        return c;
    }

private:
    std::string name_;
    std::map<std::string, Stmt> st_;

    [[noreturn]] void bad(int line, const std::string& msg) const {
        std::ostringstream os;
        os << name_ << ":" << line << ": " << msg;
        throw ConfigErr(os.str());
    }
    double num(int line, const std::string& tok) const {
        const std::string t = strip(tok);
        char* end = nullptr;
        const double v = std::strtod(t.c_str(), &end);
        if (t.empty() || end != t.c_str() + t.size()) bad(line, "malformed number '" + t + "'");
        return v;
    }
    int64_t intval(int line, const std::string& tok) const {
        const std::string t = strip(tok);
        char* end = nullptr;
        const long long v = std::strtoll(t.c_str(), &end, 10);
        if (t.empty() || end != t.c_str() + t.size()) bad(line, "malformed integer '" + t + "'");
        return v;
    }
    std::vector<double> vecval(int line, const std::string& tok) const {
        const std::string t = strip(tok);
        if (t.size() < 2 || t.front() != '{' || t.back() != '}')
            bad(line, "expected a braced vector {a, b, ...}, got '" + t + "'");
        std::vector<double> out;
        const std::string inner = t.substr(1, t.size() - 2);
        size_t pos = 0;
        for (;;) {
            const size_t comma = inner.find(',', pos);
            out.push_back(num(line, comma == std::string::npos ? inner.substr(pos)
                                                                : inner.substr(pos, comma - pos)));
            if (comma == std::string::npos) break;
            pos = comma + 1;
        }
        return out;
    }
    Stmt* find(const std::string& k) {
        auto it = st_.find(k);
        if (it == st_.end()) return nullptr;
        it->second.used = true;
        return &it->second;
    }
    bool prefixed(const std::string& p) const {
        auto it = st_.lower_bound(p);
        return it != st_.end() && it->first.rfind(p, 0) == 0;
    }
    const Stmt& req(const std::string& k) {
        const Stmt* s = find(k);
        if (!s) throw ConfigErr(name_ + ": missing mandatory key '" + k + "'");
        return *s;
    }
    int64_t integer(const std::string& k) {
        const Stmt& s = req(k);
        return intval(s.line, s.value);
    }
    std::vector<double> vec(const std::string& k) {
        const Stmt& s = req(k);
        return vecval(s.line, s.value);
    }
    GridCfg grid(const std::string& pre) {
        GridCfg g;
        g.dim = static_cast<int>(integer(pre + ".dim"));
        g.lb = vec(pre + ".lb");
        g.ub = vec(pre + ".ub");
        g.eta = vec(pre + ".eta");
        if (g.dim < 0) throw ConfigErr(name_ + ": " + pre + ".dim must be non-negative");
        for (const auto* v : {&g.lb, &g.ub, &g.eta})
            if (static_cast<int>(v->size()) != g.dim)
                throw ConfigErr(name_ + ": " + pre + " vectors must have " + std::to_string(g.dim) +
                                " entries");
        return g;
    }
    void validate(const Cfg& c) const {
        auto per_state = [&](const std::vector<double>& v, const char* key) {
            if (!v.empty() && static_cast<int>(v.size()) != c.states.dim)
                throw ConfigErr(name_ + ": " + key + " must have one entry per state dimension");
        };
        per_state(c.sigma, "noise.sigma");
        per_state(c.a, "noise.a");
        per_state(c.b, "noise.b");
        per_state(c.rate, "noise.rate");
        per_state(c.alpha, "noise.alpha");
        per_state(c.beta, "noise.beta");
        per_state(c.support_lb, "noise.support.lb");
        per_state(c.support_ub, "noise.support.ub");
        auto box = [&](const std::optional<BoxCfg>& b, const char* key) {
            if (b && (static_cast<int>(b->lb.size()) != c.states.dim ||
                      static_cast<int>(b->ub.size()) != c.states.dim))
                throw ConfigErr(name_ + ": " + key + " box must match the state dimension");
        };
        box(c.target, "target");
        box(c.avoid, "avoid");
    }
};

} // namespace

Cfg parse_cfg_text(const std::string& text, const std::string& name) {
    std::istringstream in(text);
    return CfgReader(in, name).read();
}

Cfg load_cfg_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoErr("cannot open config file '" + path + "'");
    return CfgReader(in, path).read();
}

SpecV spec_from_cfg(const Cfg& c) {
    SpecV s;
    if (c.spec_type == "safety") s.kind = GM_SPEC_SAFETY;
    else if (c.spec_type == "reachability") s.kind = GM_SPEC_REACH;
    else if (c.spec_type == "reach-avoid" || c.spec_type == "reach_avoid") s.kind = GM_SPEC_REACH_AVOID;
    else throw ConfigErr("unknown specification kind '" + c.spec_type + "'");
    s.horizon = c.time_steps;
    if (c.target) s.target = BoxV{c.target->lb, c.target->ub};
    if (c.avoid) s.avoid = BoxV{c.avoid->lb, c.avoid->ub};
    return s;
}

// ===========================================================================
// model — config.cpp:318-372, model.cpp:7-31, abstraction.cpp:16-48
// ===========================================================================

int64_t Model::rows() const {
    return static_cast<int64_t>(mul_checked(mul_checked(static_cast<uint64_t>(n_x()),
                                                        static_cast<uint64_t>(n_u()), "rows"),
                                            static_cast<uint64_t>(n_w()), "rows"));
}

uint64_t Model::memory_estimate() const {
    uint64_t width = 1;
    for (int64_t e : extents) width = mul_checked(width, static_cast<uint64_t>(e), "memory_estimate");
    const uint64_t r = static_cast<uint64_t>(rows());
    const uint64_t payload =
        mul_checked(mul_checked(r, width, "memory_estimate"), 8ULL, "memory_estimate");
    const uint64_t origins = mul_checked(r, 8ULL, "memory_estimate");
    if (payload > UINT64_MAX - origins - 4096ULL)
        throw MemoryErr("memory_estimate: size arithmetic overflows 64 bits");
    return payload + origins + 4096ULL;
}

int64_t row_pitch(int64_t R) {
    // stored rows start on the largest power-of-two granule (<= GM_PITCH_GRANULE doubles,
    // default 32 = 256 bytes) that costs at most 1/32 of padding: whole-line loads and stores
    static const char* gr = std::getenv("GM_PITCH_GRANULE");
    const int64_t top = gr ? std::max(1, std::atoi(gr)) : 32;
    for (int64_t g = top; g >= 2; g /= 2) {
        const int64_t p = (R + g - 1) / g * g;
        if ((p - R) * 32 <= R) return p;
    }
    return R;
}

int tpr_for_width(int64_t R) {
    // Threads cooperating on one row's dot product (identical in matrix and
    // OFA mode, so both accumulate in the same order): ~16 terms per thread,
    // power of two in [1, 128].
    int64_t t = R / 16;
    int p = 1;
    while (p * 2 <= t && p < 128) p *= 2;
    return p;
}

void Model::refresh() {
    const int n = X.dim();
    radius = cut_radius(noise);
    extents.assign(static_cast<size_t>(n), 1);
    for (int d = 0; d < n; ++d) {
        if (!radius) {
            extents[d] = X.count[d];
        } else if ((*radius)[d] == 0.0) {
            extents[d] = 1;
        } else {
            const int64_t cap =
                static_cast<int64_t>(std::floor(2.0 * (*radius)[d] / X.eta[d] + 1.0 + kTol)) + 1;
            extents[d] = std::min(X.count[d], cap);
        }
    }
    R = 1;
    for (int64_t e : extents) R = static_cast<int64_t>(mul_checked(static_cast<uint64_t>(R),
                                                                   static_cast<uint64_t>(e), "row width"));
    prog = Program{};
    prog.entry.push_back(0);
    int nregs = 1;
    for (size_t i = 0; i < dyn.size(); ++i) {
        Lowering L{dyn[i], prog};
        try {
            L.gen(dyn[i].root, 0);
        } catch (const ConfigErr& e) {
            throw ConfigErr("dynamics.x" + std::to_string(i) + ": " + e.what());
        }
        nregs = std::max(nregs, L.maxreg);
        prog.entry.push_back(static_cast<int32_t>(prog.code.size()));
    }
    if (noise.family == GM_CUSTOM) { // the pdf as expression n (noise coordinates in x)
        Lowering L{noise.pdf, prog};
        try {
            L.gen(noise.pdf.root, 0);
        } catch (const ConfigErr& e) {
            throw ConfigErr(std::string("noise.pdf: ") + e.what());
        }
        nregs = std::max(nregs, L.maxreg);
        prog.entry.push_back(static_cast<int32_t>(prog.code.size()));
    }
    prog.nregs = nregs;
}

Model build_model_from_cfg(const Cfg& c) {
    Model M;
    M.cfg = c;
    M.X = grid_from(c.states.lb, c.states.ub, c.states.eta);
    M.U = grid_from(c.inputs.lb, c.inputs.ub, c.inputs.eta);
    if (c.dist) M.W = grid_from(c.dist->lb, c.dist->ub, c.dist->eta);
    const int n = c.states.dim, m = c.inputs.dim, p = c.dist ? c.dist->dim : 0;
    for (size_t i = 0; i < c.dynamics.size(); ++i) {
        try {
            M.dyn.push_back(parse_expr_text(c.dynamics[i], n, m, p, c.constants));
        } catch (const ParseErr& e) {
            throw ConfigErr("dynamics.x" + std::to_string(i) + ": " + e.what());
        }
    }
    const double g = c.gamma;
    if (c.noise_type == "normal") M.noise = make_noise(GM_NORMAL, c.sigma, {}, g, c.noise_mult);
    else if (c.noise_type == "uniform") M.noise = make_noise(GM_UNIFORM, c.a, c.b, g, c.noise_mult);
    else if (c.noise_type == "exponential") M.noise = make_noise(GM_EXPONENTIAL, c.rate, {}, g, c.noise_mult);
    else if (c.noise_type == "custom") {
        M.noise = make_noise(GM_CUSTOM, c.support_lb, c.support_ub, g, c.noise_mult);
        try {
            M.noise.pdf = parse_expr_text(c.pdf, n, 0, 0, c.constants);
        } catch (const ParseErr& e) {
            throw ConfigErr(std::string("noise.pdf: ") + e.what());
        }
    } else M.noise = make_noise(GM_BETA, c.alpha, c.beta, g, c.noise_mult);

    M.spec = spec_from_cfg(c);
    M.mode = c.mode == "ofa" ? GM_MODE_OFA_ : GM_MODE_MATRIX_;
    M.threads = c.threads;
    M.mem_budget = c.mem_budget;
    finish_model(M);
    return M;
}

// make_model checks (model.cpp:15-29), then sizes and the dynamics program
void finish_model(Model& M) {
    const int n = M.X.dim(), m = M.U.dim(), p = M.W.dim();
    if (n == 0) throw ConfigErr("model: the state grid must have at least one dimension");
    if (static_cast<int>(M.dyn.size()) != n) {
        std::ostringstream os;
        os << "model: " << M.dyn.size() << " dynamics expressions for a " << n << "-dimensional state";
        throw ConfigErr(os.str());
    }
    if (M.noise.dim() != n) throw ConfigErr("model: noise dimension must equal the state dimension");
    if (n > GMD_MAXD || m > GMD_MAXD || p > GMD_MAXD)
        throw ConfigErr("model: more than " + std::to_string(GMD_MAXD) +
                        " dimensions per grid exceeds the device limit");
    M.refresh();
}

Expr expr_from_nodes(std::vector<XNode> nodes, int32_t root, int n, int m, int p, const std::string& what) {
    // a node pool as the reference's parser / ExprBuilder lays it out (expr.hpp:36-60):
    // children precede their parent, so the tree is acyclic by construction
    const int32_t N = static_cast<int32_t>(nodes.size());
    auto bad = [&](int32_t i, const std::string& why) -> ConfigErr {
        return ConfigErr(what + ": node " + std::to_string(i) + " " + why);
    };
    if (root < 0 || root >= N) throw ConfigErr(what + ": root outside the node pool");
    for (int32_t i = 0; i < N; ++i) {
        const XNode& x = nodes[static_cast<size_t>(i)];
        const int op = static_cast<int>(x.op);
        if (op < 0 || op > static_cast<int>(XOp::variable)) throw bad(i, "has an unknown operator");
        const int arity = x.op == XOp::literal || x.op == XOp::variable ? 0
                          : x.op == XOp::ite                            ? 3
                          : (x.op == XOp::neg || (x.op >= XOp::sin && x.op <= XOp::abs)) ? 1
                                                                                         : 2;
        for (int k = 0; k < 3; ++k) {
            const int32_t c = x.kid[k];
            if (k < arity && (c < 0 || c >= i)) throw bad(i, "has a child outside the preceding nodes");
        }
        if (x.op == XOp::variable) {
            const int lim = x.vclass == 0 ? n : x.vclass == 1 ? m : x.vclass == 2 ? p : -1;
            if (lim < 0 || x.vindex < 0 || x.vindex >= lim) throw bad(i, "names a variable outside the declared dimensions");
        }
    }
    Expr e;
    e.nodes = std::move(nodes);
    e.root = root;
    e.n = n;
    e.m = m;
    e.p = p;
    return e;
}

Model build_model_from_parts(const Grid& X, const Grid& U, const Grid& W, std::vector<Expr> dyn, int family,
                             int mult, double gamma, const std::vector<double>& p1, const std::vector<double>& p2,
                             Expr pdf, const SpecV& spec, int mode, int threads, uint64_t mem_budget) {
    Model M;
    M.X = X;
    M.U = U;
    M.W = W;
    M.dyn = std::move(dyn);
    if (family < GM_NORMAL || family > GM_CUSTOM) throw ConfigErr("noise: unknown family");
    M.noise = make_noise(family, p1, p2, gamma, mult);
    if (family == GM_CUSTOM) M.noise.pdf = std::move(pdf);
    M.spec = spec;
    M.mode = mode == GM_MODE_OFA_ ? GM_MODE_OFA_ : GM_MODE_MATRIX_;
    M.threads = threads;
    M.mem_budget = mem_budget;
    finish_model(M);
    // the Config a save_config of this model writes (config.cpp:270-310): expressions
    // rendered back to text (constants were substituted when the reference parsed them)
    Cfg& c = M.cfg;
    c.states = GridCfg{X.dim(), X.lb, X.ub, X.eta};
    c.inputs = GridCfg{U.dim(), U.lb, U.ub, U.eta};
    if (W.dim() > 0) c.dist = GridCfg{W.dim(), W.lb, W.ub, W.eta};
    for (const Expr& e : M.dyn) c.dynamics.push_back(expr_to_string(e, e.root));
    static const char* names[] = {"normal", "uniform", "exponential", "beta", "custom"};
    c.noise_type = names[family];
    c.noise_mult = mult;
    c.gamma = gamma;
    switch (family) {
        case GM_NORMAL: c.sigma = p1; break;
        case GM_UNIFORM: c.a = p1; c.b = p2; break;
        case GM_EXPONENTIAL: c.rate = p1; break;
        case GM_BETA: c.alpha = p1; c.beta = p2; break;
        default:
            c.support_lb = p1;
            c.support_ub = p2;
            c.pdf = expr_to_string(M.noise.pdf, M.noise.pdf.root);
    }
    c.spec_type = spec.kind == GM_SPEC_SAFETY ? "safety" : spec.kind == GM_SPEC_REACH ? "reachability" : "reach-avoid";
    c.time_steps = spec.horizon;
    if (spec.target.dim()) c.target = BoxCfg{spec.target.lo, spec.target.hi};
    if (spec.avoid.dim()) c.avoid = BoxCfg{spec.avoid.lo, spec.avoid.hi};
    c.mode = M.mode == GM_MODE_OFA_ ? "ofa" : "matrix";
    c.threads = threads;
    c.mem_budget = mem_budget;
    return M;
}

// save_config, config.cpp:270-310 (same key order and number formatting)
std::string save_config_text(const Cfg& c) {
    std::ostringstream os;
    auto grid = [&](const char* prefix, const GridCfg& g) {
        os << prefix << ".dim = " << g.dim << ";\n";
        os << prefix << ".lb = " << fmt_vec(g.lb) << ";\n";
        os << prefix << ".ub = " << fmt_vec(g.ub) << ";\n";
        os << prefix << ".eta = " << fmt_vec(g.eta) << ";\n";
    };
    grid("states", c.states);
    grid("inputs", c.inputs);
    if (c.dist) grid("disturbances", *c.dist);
    for (size_t i = 0; i < c.dynamics.size(); ++i) os << "dynamics.x" << i << " = " << c.dynamics[i] << ";\n";
    for (const auto& [k, v] : c.constants) os << "constants." << k << " = " << fmt_shortest(v) << ";\n";
    os << "noise.type = " << c.noise_type << ";\n";
    os << "noise.mode = " << (c.noise_mult ? "multiplicative" : "additive") << ";\n";
    os << "noise.cutting_probability = " << fmt_shortest(c.gamma) << ";\n";
    if (!c.sigma.empty()) os << "noise.sigma = " << fmt_vec(c.sigma) << ";\n";
    if (!c.a.empty()) os << "noise.a = " << fmt_vec(c.a) << ";\n";
    if (!c.b.empty()) os << "noise.b = " << fmt_vec(c.b) << ";\n";
    if (!c.rate.empty()) os << "noise.rate = " << fmt_vec(c.rate) << ";\n";
    if (!c.alpha.empty()) os << "noise.alpha = " << fmt_vec(c.alpha) << ";\n";
    if (!c.beta.empty()) os << "noise.beta = " << fmt_vec(c.beta) << ";\n";
    if (c.noise_type == "custom") { // engine extension keys (noise.type = custom)
        os << "noise.pdf = " << c.pdf << ";\n";
        os << "noise.support.lb = " << fmt_vec(c.support_lb) << ";\n";
        os << "noise.support.ub = " << fmt_vec(c.support_ub) << ";\n";
    }
    os << "spec.type = " << c.spec_type << ";\n";
    os << "spec.time_steps = " << c.time_steps << ";\n";
    if (c.target) {
        os << "target.lb = " << fmt_vec(c.target->lb) << ";\n";
        os << "target.ub = " << fmt_vec(c.target->ub) << ";\n";
    }
    if (c.avoid) {
        os << "avoid.lb = " << fmt_vec(c.avoid->lb) << ";\n";
        os << "avoid.ub = " << fmt_vec(c.avoid->ub) << ";\n";
    }
    os << "exec.threads = " << c.threads << ";\n";
    os << "exec.mode = " << c.mode << ";\n";
    os << "exec.mem_budget = " << c.mem_budget << ";\n";
    os << "exec.seed = " << c.seed << ";\n";
    os << "exec.runs = " << c.runs << ";\n";
    if (!c.output.empty()) os << "exec.output = " << c.output << ";\n";
    return os.str();
}

namespace {
// Eigen's default row-vector print (values padded to the widest, one space
// apart), used in the "(x=[..], nu=[..], w=[..])" suffix of abstraction.cpp:96-101.
std::string eigen_row(const std::vector<double>& v) {
    size_t width = 0;
    std::vector<std::string> parts;
    for (double d : v) {
        std::ostringstream os;
        os << d;
        parts.push_back(os.str());
        width = std::max(width, parts.back().size());
    }
    std::string s;
    for (size_t i = 0; i < parts.size(); ++i) {
        if (i) s += ' ';
        s += std::string(width - parts[i].size(), ' ') + parts[i];
    }
    return s;
}
} // namespace

void Model::row_image(int64_t row, std::vector<double>& mu) const {
    const int64_t iw = row % n_w();
    const int64_t pr = row / n_w();
    const int64_t ix = pr / n_u(), iu = pr % n_u();
    std::vector<double> x(X.dim()), u(U.dim()), w(W.dim());
    int64_t rem = ix;
    for (int d = 0; d < X.dim(); ++d) { x[d] = X.rep(d, rem / X.stride[d]); rem %= X.stride[d]; }
    rem = iu;
    for (int d = 0; d < U.dim(); ++d) { u[d] = U.rep(d, rem / U.stride[d]); rem %= U.stride[d]; }
    rem = iw;
    for (int d = 0; d < W.dim(); ++d) { w[d] = W.rep(d, rem / W.stride[d]); rem %= W.stride[d]; }
    mu.assign(static_cast<size_t>(X.dim()), 0.0);
    try {
        for (int i = 0; i < X.dim(); ++i) mu[i] = eval_expr(dyn[i], x.data(), u.data(), w.data());
    } catch (const DomainErr& e) {
        throw DomainErr(std::string(e.what()) + " at (x=[" + eigen_row(x) + "], nu=[" + eigen_row(u) +
                        "], w=[" + eigen_row(w) + "])");
    }
}

GmDev Model::device_descriptor() const {
    GmDev D;
    std::memset(&D, 0, sizeof D);
    const int n = X.dim();
    D.n = n;
    D.m = U.dim();
    D.p = W.dim();
    D.family = noise.family;
    D.mult = noise.mult;
    D.cut = !radius ? GM_CUT_NONE : ((*radius).size() > 0 && (*radius)[0] == 0.0 ? GM_CUT_DEGENERATE : GM_CUT_RADIUS);
    D.spec_kind = spec.kind;
    D.has_avoid = spec.avoid.dim() > 0 ? 1 : 0;
    D.tpr = tpr_for_width(R);
    D.n_ins = static_cast<int>(prog.code.size());
    D.n_lits = static_cast<int>(prog.lits.size());
    D.nregs = prog.nregs;
    D.n_x = n_x();
    D.n_u = n_u();
    D.n_w = n_w();
    D.rows = rows();
    D.R = R;
    D.pitch = row_pitch(R);
    for (int d = 0; d < n; ++d) {
        D.xcount[d] = X.count[d];
        D.xstride[d] = X.stride[d];
        D.xlb[d] = X.lb[d];
        D.xeta[d] = X.eta[d];
        D.radius[d] = radius ? (*radius)[d] : 0.0;
        D.s[d] = noise.family == GM_NORMAL ? noise.p1[d] * kRoot2 : noise.p1[d];
        D.inv_s[d] = 1.0 / D.s[d];
        D.p2[d] = noise.p2.empty() ? 0.0 : noise.p2[d];
        D.W[d] = static_cast<int>(extents[d]);
        if (spec.target.dim() == n) { D.tlo[d] = spec.target.lo[d]; D.thi[d] = spec.target.hi[d]; }
        if (spec.avoid.dim() == n) { D.alo[d] = spec.avoid.lo[d]; D.ahi[d] = spec.avoid.hi[d]; }
    }
    for (int d = 0; d < U.dim(); ++d) { D.ustride[d] = U.stride[d]; D.ulb[d] = U.lb[d]; D.ueta[d] = U.eta[d]; }
    for (int d = 0; d < W.dim(); ++d) { D.wstride[d] = W.stride[d]; D.wlb[d] = W.lb[d]; D.weta[d] = W.eta[d]; }
    int off = 0;
    for (int d = 0; d < n; ++d) { D.mass_off[d] = off; off += D.W[d]; }
    D.mass_off[n] = off;
    D.sumW = off;
    if (n == 1) { // virtual leading axis of width 1 and mass 1.0
        D.s_axes = 0;
        D.P_size = 1;
        D.Wm = 1;
        D.Wl = D.W[0];
        D.mm_off = off; // slot sumW of a row's mass buffer holds the virtual 1.0
        D.ml_off = 0;
    } else {
        D.s_axes = n - 2;
        int64_t ps = 1;
        for (int d = 0; d < n - 2; ++d) ps *= D.W[d];
        D.P_size = static_cast<int>(ps);
        D.Wm = D.W[n - 2];
        D.Wl = D.W[n - 1];
        D.mm_off = D.mass_off[n - 2];
        D.ml_off = D.mass_off[n - 1];
    }
    D.n_lines = static_cast<int>(R / D.Wl);
    D.div_Wm = gm_fastdiv(static_cast<uint32_t>(D.Wm));
    D.div_Wl = gm_fastdiv(static_cast<uint32_t>(D.Wl));
    D.div_lines = gm_fastdiv(static_cast<uint32_t>(D.n_lines));
    D.div_P = gm_fastdiv(static_cast<uint32_t>(D.P_size));
    D.div_mw = gm_fastdiv(static_cast<uint32_t>(D.sumW + 1));
    for (int d = 0; d < n; ++d) D.div_W[d] = gm_fastdiv(static_cast<uint32_t>(D.W[d]));
    {
        int64_t st = 1;
        for (int d = D.s_axes - 1; d >= 0; --d) {
            D.Ps[d] = static_cast<int>(st);
            D.div_Ps[d] = gm_fastdiv(static_cast<uint32_t>(st));
            st *= D.W[d];
        }
    }
    D.idx32 = rows() < (int64_t(1) << 31) ? 1 : 0;
    if (D.idx32) {
        D.div_nw = gm_fastdiv(static_cast<uint32_t>(D.n_w));
        D.div_nu = gm_fastdiv(static_cast<uint32_t>(D.n_u));
        for (int d = 0; d < n; ++d) D.div_xs[d] = gm_fastdiv(static_cast<uint32_t>(D.xstride[d]));
        for (int d = 0; d < D.m; ++d) D.div_us[d] = gm_fastdiv(static_cast<uint32_t>(D.ustride[d]));
        for (int d = 0; d < D.p; ++d) D.div_ws[d] = gm_fastdiv(static_cast<uint32_t>(D.wstride[d]));
    }
    for (size_t i = 0; i < prog.entry.size() && i <= GMD_MAXD + 1; ++i) D.entry[i] = prog.entry[i];
    if (noise.family == GM_CUSTOM)
        for (int d = 0; d < n; ++d) {
            D.sup_lo[d] = noise.p1[d];
            D.sup_hi[d] = noise.p2[d];
        }
    return D;
}

} // namespace gmh
