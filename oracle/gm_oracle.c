/*
 * gm_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE;
 * see gm_oracle.h). Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/src). Arithmetic follows the
 * reference's evaluation order exactly; compile without FMA contraction.
 */
#define _GNU_SOURCE
#include "gm_oracle.h"

#include <ctype.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define IDX_TOL 1e-9 /* grid.cpp:10, abstraction.cpp:10 */
#define SQRT2 1.4142135623730951 /* noise.cpp:10 */

/* ------------------------------------------------------------------ grids */

typedef struct {
    int dim;
    double lb[OC_MAXD], ub[OC_MAXD], eta[OC_MAXD];
    int64_t count[OC_MAXD], stride[OC_MAXD], total;
} grid_t;

/* make_grid: grid.cpp:12-45 */
static int grid_make(grid_t* g, int dim, const double* lb, const double* ub, const double* eta) {
    g->dim = dim;
    g->total = 1;
    for (int i = 0; i < dim; ++i) {
        if (!(eta[i] > 0.0) || lb[i] > ub[i]) return 0;
        g->lb[i] = lb[i];
        g->ub[i] = ub[i];
        g->eta[i] = eta[i];
        const double q = (ub[i] - lb[i]) / eta[i];
        g->count[i] = (int64_t)floor(q + IDX_TOL) + 1;
        g->total *= g->count[i];
    }
    for (int i = dim - 1; i >= 0; --i) g->stride[i] = (i == dim - 1) ? 1 : g->stride[i + 1] * g->count[i + 1];
    return 1;
}

/* ------------------------------------------------------------ expressions */

enum { O_ADD, O_SUB, O_MUL, O_DIV, O_POW, O_LT, O_LE, O_GT, O_GE, O_EQ, O_NE, O_NEG, O_SIN, O_COS, O_TAN,
       O_ASIN, O_ACOS, O_ATAN, O_EXP, O_LN, O_SQRT, O_ABS, O_MIN, O_MAX, O_ITE, O_LIT, O_VAR };

typedef struct {
    int op;
    double value;
    int vclass, vindex;
    int kid[3];
} node_t;

typedef struct {
    node_t* nodes;
    int n_nodes, cap, root;
} expr_t;

typedef struct {
    const char* s;
    size_t i;
    expr_t* e;
    int n, m, p;
    int n_const;
    const char* const* cn;
    const double* cv;
    int bad;
} parser_t;

static int px_push(parser_t* P, node_t nd) {
    expr_t* e = P->e;
    if (e->n_nodes == e->cap) {
        e->cap = e->cap ? 2 * e->cap : 64;
        e->nodes = (node_t*)realloc(e->nodes, (size_t)e->cap * sizeof(node_t));
    }
    e->nodes[e->n_nodes] = nd;
    return e->n_nodes++;
}
static node_t mk(int op) {
    node_t n;
    memset(&n, 0, sizeof n);
    n.op = op;
    n.kid[0] = n.kid[1] = n.kid[2] = -1;
    return n;
}
static void ws(parser_t* P) {
    while (P->s[P->i] == ' ' || P->s[P->i] == '\t' || P->s[P->i] == '\r' || P->s[P->i] == '\n') ++P->i;
}
static char pk(parser_t* P) {
    ws(P);
    return P->s[P->i];
}
static int bin(parser_t* P, int op, int a, int b) {
    node_t n = mk(op);
    n.kid[0] = a;
    n.kid[1] = b;
    return px_push(P, n);
}
static int p_cmp(parser_t* P);
static int p_unary(parser_t* P);

/* parse_number / parse_ident / parse_call / parse_primary: expr.cpp:186-287 */
static int p_primary(parser_t* P) {
    const char c = pk(P);
    if (c == '(') {
        ++P->i;
        const int inner = p_cmp(P);
        if (pk(P) != ')') { P->bad = 1; return -1; }
        ++P->i;
        return inner;
    }
    if (c == '.' || isdigit((unsigned char)c)) {
        const size_t st = P->i;
        while (isdigit((unsigned char)P->s[P->i]) || P->s[P->i] == '.') ++P->i;
        if (P->s[P->i] == 'e' || P->s[P->i] == 'E') {
            size_t save = P->i++;
            if (P->s[P->i] == '+' || P->s[P->i] == '-') ++P->i;
            if (isdigit((unsigned char)P->s[P->i])) {
                while (isdigit((unsigned char)P->s[P->i])) ++P->i;
            } else {
                P->i = save;
            }
        }
        char tok[128];
        size_t len = P->i - st;
        if (len >= sizeof tok) { P->bad = 1; return -1; }
        memcpy(tok, P->s + st, len);
        tok[len] = 0;
        char* end;
        node_t n = mk(O_LIT);
        n.value = strtod(tok, &end);
        if (end != tok + len) { P->bad = 1; return -1; }
        return px_push(P, n);
    }
    if (isalpha((unsigned char)c) || c == '_') {
        const size_t st = P->i;
        while (isalnum((unsigned char)P->s[P->i]) || P->s[P->i] == '_') ++P->i;
        char name[128];
        size_t len = P->i - st;
        if (len >= sizeof name) { P->bad = 1; return -1; }
        memcpy(name, P->s + st, len);
        name[len] = 0;
        if (pk(P) == '(') {
            static const struct { const char* nm; int op, ar; } fns[] = {
                {"sin", O_SIN, 1}, {"cos", O_COS, 1}, {"tan", O_TAN, 1}, {"asin", O_ASIN, 1}, {"acos", O_ACOS, 1},
                {"atan", O_ATAN, 1}, {"exp", O_EXP, 1}, {"ln", O_LN, 1}, {"sqrt", O_SQRT, 1}, {"abs", O_ABS, 1},
                {"min", O_MIN, 2}, {"max", O_MAX, 2}, {"ite", O_ITE, 3}};
            for (size_t f = 0; f < sizeof fns / sizeof fns[0]; ++f) {
                if (strcmp(name, fns[f].nm) != 0) continue;
                ++P->i; /* '(' */
                node_t n = mk(fns[f].op);
                for (int a = 0; a < fns[f].ar; ++a) {
                    if (a > 0) {
                        if (pk(P) != ',') { P->bad = 1; return -1; }
                        ++P->i;
                    }
                    n.kid[a] = p_cmp(P);
                }
                if (pk(P) != ')') { P->bad = 1; return -1; }
                ++P->i;
                return px_push(P, n);
            }
            P->bad = 1;
            return -1;
        }
        if (len >= 2 && (name[0] == 'x' || name[0] == 'u' || name[0] == 'w')) {
            int digits = 1;
            for (size_t k = 1; k < len; ++k)
                if (!isdigit((unsigned char)name[k])) digits = 0;
            if (digits) {
                node_t n = mk(O_VAR);
                n.vclass = name[0] == 'x' ? 0 : name[0] == 'u' ? 1 : 2;
                n.vindex = atoi(name + 1);
                const int lim = n.vclass == 0 ? P->n : n.vclass == 1 ? P->m : P->p;
                if (n.vindex >= lim) { P->bad = 1; return -1; }
                return px_push(P, n);
            }
        }
        for (int k = 0; k < P->n_const; ++k) {
            if (strcmp(name, P->cn[k]) == 0) {
                node_t n = mk(O_LIT);
                n.value = P->cv[k];
                return px_push(P, n);
            }
        }
        P->bad = 1;
        return -1;
    }
    P->bad = 1;
    return -1;
}

/* parse_power: expr.cpp:177-184 (right-assoc, exponent is a unary) */
static int p_power(parser_t* P) {
    const int base = p_primary(P);
    if (pk(P) == '^') {
        ++P->i;
        return bin(P, O_POW, base, p_unary(P));
    }
    return base;
}
/* parse_unary: expr.cpp:158-175 (negative literals fold) */
static int p_unary(parser_t* P) {
    if (pk(P) == '-') {
        ++P->i;
        const int child = p_unary(P);
        if (child >= 0 && P->e->nodes[child].op == O_LIT) {
            P->e->nodes[child].value = -P->e->nodes[child].value;
            return child;
        }
        node_t n = mk(O_NEG);
        n.kid[0] = child;
        return px_push(P, n);
    }
    return p_power(P);
}
/* parse_term / parse_sum: expr.cpp:134-156 (left-assoc) */
static int p_term(parser_t* P) {
    int lhs = p_unary(P);
    for (char c = pk(P); c == '*' || c == '/'; c = pk(P)) {
        ++P->i;
        lhs = bin(P, c == '*' ? O_MUL : O_DIV, lhs, p_unary(P));
    }
    return lhs;
}
static int p_sum(parser_t* P) {
    int lhs = p_term(P);
    for (char c = pk(P); c == '+' || c == '-'; c = pk(P)) {
        ++P->i;
        lhs = bin(P, c == '+' ? O_ADD : O_SUB, lhs, p_term(P));
    }
    return lhs;
}
/* parse_expr: expr.cpp:106-122 (comparisons, left-assoc) */
static int p_cmp(parser_t* P) {
    int lhs = p_sum(P);
    for (;;) {
        ws(P);
        const char a = P->s[P->i], b = a ? P->s[P->i + 1] : 0;
        int op;
        if (a == '<' && b == '=') op = O_LE, P->i += 2;
        else if (a == '>' && b == '=') op = O_GE, P->i += 2;
        else if (a == '=' && b == '=') op = O_EQ, P->i += 2;
        else if (a == '!' && b == '=') op = O_NE, P->i += 2;
        else if (a == '<') op = O_LT, P->i += 1;
        else if (a == '>') op = O_GT, P->i += 1;
        else break;
        lhs = bin(P, op, lhs, p_sum(P));
    }
    return lhs;
}

/* eval_node: expr.cpp:404-480. A domain error sets *bad and returns 0. */
static double ev(const expr_t* e, int id, const double* x, const double* u, const double* w, int* bad) {
    const node_t* nd = &e->nodes[id];
    double a, b;
#define K(i) ev(e, nd->kid[i], x, u, w, bad)
    switch (nd->op) {
        case O_LIT: return nd->value;
        case O_VAR: return nd->vclass == 0 ? x[nd->vindex] : nd->vclass == 1 ? u[nd->vindex] : w[nd->vindex];
        case O_ADD: a = K(0); return a + K(1);
        case O_SUB: a = K(0); return a - K(1);
        case O_MUL: a = K(0); return a * K(1);
        case O_DIV:
            a = K(0); b = K(1);
            if (b == 0.0) { *bad = 1; return 0.0; }
            return a / b;
        case O_POW:
            a = K(0); b = K(1);
            if (a < 0.0 && b != floor(b)) { *bad = 1; return 0.0; }
            if (a == 0.0 && b < 0.0) { *bad = 1; return 0.0; }
            return pow(a, b);
        case O_LT: a = K(0); return a < K(1) ? 1.0 : 0.0;
        case O_LE: a = K(0); return a <= K(1) ? 1.0 : 0.0;
        case O_GT: a = K(0); return a > K(1) ? 1.0 : 0.0;
        case O_GE: a = K(0); return a >= K(1) ? 1.0 : 0.0;
        case O_EQ: a = K(0); return a == K(1) ? 1.0 : 0.0;
        case O_NE: a = K(0); return a != K(1) ? 1.0 : 0.0;
        case O_NEG: return -K(0);
        case O_SIN: return sin(K(0));
        case O_COS: return cos(K(0));
        case O_TAN: return tan(K(0));
        case O_ASIN: a = K(0); if (a < -1.0 || a > 1.0) { *bad = 1; return 0.0; } return asin(a);
        case O_ACOS: a = K(0); if (a < -1.0 || a > 1.0) { *bad = 1; return 0.0; } return acos(a);
        case O_ATAN: return atan(K(0));
        case O_EXP: return exp(K(0));
        case O_LN: a = K(0); if (a <= 0.0) { *bad = 1; return 0.0; } return log(a);
        case O_SQRT: a = K(0); if (a < 0.0) { *bad = 1; return 0.0; } return sqrt(a);
        case O_ABS: return fabs(K(0));
        case O_MIN: a = K(0); b = K(1); return fmin(a, b);
        case O_MAX: a = K(0); b = K(1); return fmax(a, b);
        case O_ITE: return K(0) != 0.0 ? K(1) : K(2);
    }
#undef K
    return 0.0;
}

/* ------------------------------------------------------------------ model */

struct oc_model {
    grid_t X, U, W;
    expr_t dyn[OC_MAXD];
    int family, mult;
    double gamma;
    double p1[OC_MAXD], p2[OC_MAXD];
    int has_radius, degenerate;
    double radius[OC_MAXD];
    int64_t ext[OC_MAXD], R, sumW;
    int spec_kind, horizon, has_target, has_avoid;
    double tlo[OC_MAXD], thi[OC_MAXD], alo[OC_MAXD], ahi[OC_MAXD];
    uint8_t* absorb; /* per state, reach kinds */
};

/* cutting_radius: noise.cpp:137-180 */
static void radius_of(oc_model* M) {
    const int n = M->X.dim;
    M->has_radius = 0;
    if (M->mult) return;
    switch (M->family) {
        case 0: {
            if (M->gamma == 0.0) return;
            double log_c = 0.0;
            for (int j = 0; j < n; ++j) log_c += 0.5 * log(2.0 * M_PI * M->p1[j] * M->p1[j]);
            const double t = -2.0 * (log(M->gamma) + log_c);
            M->has_radius = 1;
            for (int i = 0; i < n; ++i) M->radius[i] = t <= 0.0 ? 0.0 : M->p1[i] * sqrt(t);
            return;
        }
        case 2: {
            if (M->gamma == 0.0) return;
            double lp = 0.0;
            for (int j = 0; j < n; ++j) lp += log(M->p1[j]);
            const double t = lp - log(M->gamma);
            M->has_radius = 1;
            for (int i = 0; i < n; ++i) M->radius[i] = t <= 0.0 ? 0.0 : t / M->p1[i];
            return;
        }
        case 1:
            M->has_radius = 1;
            for (int i = 0; i < n; ++i) M->radius[i] = fmax(fabs(M->p1[i]), fabs(M->p2[i]));
            return;
        default:
            M->has_radius = 1;
            for (int i = 0; i < n; ++i) M->radius[i] = 1.0;
            return;
    }
}

static int in_box(int n, const double* p, const double* lo, const double* hi) {
    for (int d = 0; d < n; ++d)
        if (!(p[d] >= lo[d])) return 0;
    for (int d = 0; d < n; ++d)
        if (!(p[d] <= hi[d])) return 0;
    return 1;
}

int oc_model_new(const oc_desc* d, oc_model** out, char* err, int errlen) {
    oc_model* M = (oc_model*)calloc(1, sizeof *M);
    if (!grid_make(&M->X, d->n, d->xlb, d->xub, d->xeta) || !grid_make(&M->U, d->m, d->ulb, d->uub, d->ueta) ||
        !grid_make(&M->W, d->p, d->wlb, d->wub, d->weta)) {
        snprintf(err, (size_t)errlen, "bad grid");
        free(M);
        return 2;
    }
    for (int i = 0; i < d->n; ++i) {
        parser_t P;
        memset(&P, 0, sizeof P);
        P.s = d->dyn[i];
        P.e = &M->dyn[i];
        P.n = d->n;
        P.m = d->m;
        P.p = d->p;
        P.n_const = d->n_const;
        P.cn = d->const_names;
        P.cv = d->const_vals;
        M->dyn[i].root = p_cmp(&P);
        ws(&P);
        if (P.bad || P.s[P.i] != 0 || M->dyn[i].root < 0) {
            snprintf(err, (size_t)errlen, "parse error in dynamics.x%d", i);
            oc_model_free(M);
            return 2;
        }
    }
    M->family = d->family;
    M->mult = d->mult;
    M->gamma = d->gamma;
    for (int i = 0; i < d->n; ++i) {
        M->p1[i] = d->p1[i];
        M->p2[i] = d->p2 ? d->p2[i] : 0.0;
    }
    radius_of(M);
    M->degenerate = M->has_radius && d->n > 0 && M->radius[0] == 0.0; /* abstraction.cpp:69 */
    /* window_extents: abstraction.cpp:16-35 */
    M->R = 1;
    M->sumW = 0;
    for (int k = 0; k < d->n; ++k) {
        int64_t w;
        if (!M->has_radius) w = M->X.count[k];
        else if (M->radius[k] == 0.0) w = 1;
        else {
            const int64_t cap = (int64_t)floor(2.0 * M->radius[k] / M->X.eta[k] + 1.0 + IDX_TOL) + 1;
            w = M->X.count[k] < cap ? M->X.count[k] : cap;
        }
        M->ext[k] = w;
        M->R *= w;
        M->sumW += w;
    }
    M->spec_kind = d->spec_kind;
    M->horizon = d->horizon;
    M->has_target = d->has_target;
    M->has_avoid = d->has_avoid;
    for (int k = 0; k < d->n; ++k) {
        if (d->has_target) { M->tlo[k] = d->tlo[k]; M->thi[k] = d->thi[k]; }
        if (d->has_avoid) { M->alo[k] = d->alo[k]; M->ahi[k] = d->ahi[k]; }
    }
    /* absorbing_states: spec.cpp:51-60 */
    M->absorb = (uint8_t*)calloc((size_t)M->X.total, 1);
    if (M->spec_kind != 0) {
        double p[OC_MAXD];
        for (int64_t i = 0; i < M->X.total; ++i) {
            int64_t rem = i;
            for (int k = 0; k < d->n; ++k) {
                const int64_t j = rem / M->X.stride[k];
                rem %= M->X.stride[k];
                p[k] = M->X.lb[k] + (double)j * M->X.eta[k];
            }
            M->absorb[i] = (uint8_t)((M->has_target && in_box(d->n, p, M->tlo, M->thi)) ||
                                     (M->has_avoid && in_box(d->n, p, M->alo, M->ahi)));
        }
    }
    *out = M;
    return 0;
}

void oc_model_free(oc_model* M) {
    if (!M) return;
    for (int i = 0; i < OC_MAXD; ++i) free(M->dyn[i].nodes);
    free(M->absorb);
    free(M);
}

/* memory_estimate: abstraction.cpp:37-48 (0 on overflow) */
void oc_sizes(const oc_model* M, int64_t* out, uint64_t* mem) {
    out[0] = M->X.total;
    out[1] = M->U.total;
    out[2] = M->W.total;
    out[3] = M->X.total * M->U.total * M->W.total;
    out[4] = M->R;
    for (int k = 0; k < M->X.dim; ++k) out[5 + k] = M->ext[k];
    unsigned __int128 rows = (unsigned __int128)(uint64_t)out[3];
    unsigned __int128 v = rows * (uint64_t)M->R * 8u + rows * 8u + 4096u;
    *mem = (v >> 64) ? 0 : (uint64_t)v;
}

void oc_absorbing(const oc_model* M, uint8_t* f) { memcpy(f, M->absorb, (size_t)M->X.total); }

/* ------------------------------------------------------------- row kernel */

/* inc_beta: noise.cpp:375-403 */
static double inc_beta(double a, double b, double x, int* bad) {
    if (x <= 0.0) return 0.0;
    if (x >= 1.0) return 1.0;
    if (x > (a + 1.0) / (a + b + 2.0)) return 1.0 - inc_beta(b, a, 1.0 - x, bad);
    const double lbeta = lgamma(a) + lgamma(b) - lgamma(a + b);
    const double front = exp(log(x) * a + log1p(-x) * b - lbeta) / a;
    double f = 1.0, c = 1.0, d = 0.0;
    for (int i = 0; i <= 400; ++i) {
        const int m = i / 2;
        double num;
        if (i == 0) num = 1.0;
        else if (i % 2 == 0) num = m * (b - m) * x / ((a + 2.0 * m - 1.0) * (a + 2.0 * m));
        else num = -((a + m) * (a + b + m) * x) / ((a + 2.0 * m) * (a + 2.0 * m + 1.0));
        d = 1.0 + num * d;
        if (fabs(d) < 1e-30) d = 1e-30;
        d = 1.0 / d;
        c = 1.0 + num / c;
        if (fabs(c) < 1e-30) c = 1e-30;
        f *= c * d;
        if (fabs(1.0 - c * d) < 1e-15) {
            const double r = front * (f - 1.0);
            return r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
        }
    }
    *bad = 1;
    return 0.0;
}

/* axis_mass: noise.cpp:92-122 */
static double axis_mass(const oc_model* M, int k, double lo, double hi, int* bad) {
    if (hi <= lo) return 0.0;
    switch (M->family) {
        case 0: {
            const double s = M->p1[k] * SQRT2;
            return 0.5 * (erf(hi / s) - erf(lo / s));
        }
        case 1: {
            const double a = M->p1[k], b = M->p2[k];
            const double ov = (b < hi ? b : hi) - (lo < a ? a : lo);
            return ov > 0.0 ? ov / (b - a) : 0.0;
        }
        case 2: {
            const double l = M->p1[k];
            const double ch = hi <= 0.0 ? 0.0 : -expm1(-l * hi);
            const double cl = lo <= 0.0 ? 0.0 : -expm1(-l * lo);
            return ch - cl;
        }
        default: {
            const double a = M->p1[k], b = M->p2[k];
            const double ch = hi <= 0.0 ? 0.0 : (hi >= 1.0 ? 1.0 : inc_beta(a, b, hi, bad));
            const double cl = lo <= 0.0 ? 0.0 : (lo >= 1.0 ? 1.0 : inc_beta(a, b, lo, bad));
            return ch - cl;
        }
    }
}

/* axis_transformed_mass: noise.cpp:124-131 */
static double tmass(const oc_model* M, int k, double lo, double hi, double mean, double scale, int* bad) {
    if (scale == 0.0) return (mean >= lo && mean <= hi) ? 1.0 : 0.0;
    double a = (lo - mean) / scale, b = (hi - mean) / scale;
    if (scale < 0.0) { const double t = a; a = b; b = t; }
    return axis_mass(M, k, a, b, bad);
}

typedef struct {
    double x[OC_MAXD], u[OC_MAXD], w[OC_MAXD], mu[OC_MAXD];
    int64_t o[OC_MAXD];
    double* mass; /* sumW */
} rowk_t;

/* RowKernel::compute: abstraction.cpp:72-121. Returns 0 on a domain error. */
static int row_compute(const oc_model* M, rowk_t* K, int64_t ix, int64_t iu, int64_t iw) {
    int64_t rem = ix;
    for (int d = 0; d < M->X.dim; ++d) {
        const int64_t j = rem / M->X.stride[d];
        rem %= M->X.stride[d];
        K->x[d] = M->X.lb[d] + (double)j * M->X.eta[d];
    }
    rem = iu;
    for (int d = 0; d < M->U.dim; ++d) {
        const int64_t j = rem / M->U.stride[d];
        rem %= M->U.stride[d];
        K->u[d] = M->U.lb[d] + (double)j * M->U.eta[d];
    }
    rem = iw;
    for (int d = 0; d < M->W.dim; ++d) {
        const int64_t j = rem / M->W.stride[d];
        rem %= M->W.stride[d];
        K->w[d] = M->W.lb[d] + (double)j * M->W.eta[d];
    }
    int bad = 0;
    for (int i = 0; i < M->X.dim; ++i) {
        K->mu[i] = ev(&M->dyn[i], M->dyn[i].root, K->x, K->u, K->w, &bad);
        if (bad) return 0;
    }
    for (int d = 0; d < M->X.dim; ++d) {
        const int64_t W = M->ext[d];
        int64_t o;
        if (!M->has_radius) o = 0;
        else if (M->degenerate) o = (int64_t)floor((K->mu[d] - M->X.lb[d]) / M->X.eta[d] + 0.5);
        else o = (int64_t)ceil((K->mu[d] - M->radius[d] - 0.5 * M->X.eta[d] - M->X.lb[d]) / M->X.eta[d] - IDX_TOL);
        if (o < 0) o = 0;
        if (o > M->X.count[d] - W) o = M->X.count[d] - W;
        K->o[d] = o;
    }
    return 1;
}

/* fill_axis_masses: abstraction.cpp:130-146 */
static int row_masses(const oc_model* M, rowk_t* K) {
    int bad = 0, off = 0;
    for (int d = 0; d < M->X.dim; ++d) {
        const double scale = M->mult ? K->x[d] : 1.0;
        const double half = 0.5 * M->X.eta[d];
        for (int64_t t = 0; t < M->ext[d]; ++t) {
            const double rep = M->X.lb[d] + (double)(K->o[d] + t) * M->X.eta[d];
            K->mass[off + t] = tmass(M, d, rep - half, rep + half, K->mu[d], scale, &bad);
        }
        off += (int)M->ext[d];
    }
    return !bad;
}

/* fill_product: abstraction.cpp:150-159 (same association: prefix acc carried) */
static double* fill_product(const oc_model* M, const double* mass, int d, double acc, double* out) {
    int off = 0;
    for (int e = 0; e < d; ++e) off += (int)M->ext[e];
    const double* md = mass + off;
    if (d == M->X.dim - 1) {
        for (int64_t t = 0; t < M->ext[d]; ++t) *out++ = acc * md[t];
        return out;
    }
    for (int64_t t = 0; t < M->ext[d]; ++t) out = fill_product(M, mass, d + 1, acc * md[t], out);
    return out;
}

/* box_mass via cell_probability_impl: noise.cpp:223-258 */
static double box_mass(const oc_model* M, const rowk_t* K, int* bad) {
    double p = 1.0;
    for (int d = 0; d < M->X.dim; ++d) {
        p *= tmass(M, d, M->tlo[d], M->thi[d], K->mu[d], M->mult ? K->x[d] : 1.0, bad);
        if (p == 0.0) break;
    }
    return p < 1.0 ? (0.0 < p ? p : 0.0) : 1.0;
}

/* ------------------------------------------------------------- threading */

typedef struct {
    int64_t begin, end;
    void* ctx;
    void (*fn)(void* ctx, int64_t b, int64_t e, int64_t* bad_row);
    int64_t bad_row;
} job_t;

static void* job_run(void* a) {
    job_t* j = (job_t*)a;
    j->fn(j->ctx, j->begin, j->end, &j->bad_row);
    return NULL;
}

/* parallel_for: parallel.hpp:23-51 (static contiguous chunks; first error by chunk order) */
static int64_t par_for(int64_t n, int threads, void* ctx, void (*fn)(void*, int64_t, int64_t, int64_t*)) {
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    if (n <= 0) return -1;
    if (threads > n) threads = (int)n;
    job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const int64_t chunk = (n + threads - 1) / threads;
    int used = 0;
    for (int t = 0; t < threads; ++t) {
        const int64_t b = (int64_t)t * chunk, e = b + chunk < n ? b + chunk : n;
        if (b >= e) break;
        jobs[t] = (job_t){b, e, ctx, fn, -1};
        if (threads == 1) job_run(&jobs[t]);
        else pthread_create(&th[t], NULL, job_run, &jobs[t]);
        ++used;
    }
    int64_t bad = -1;
    for (int t = 0; t < used; ++t) {
        if (threads > 1) pthread_join(th[t], NULL);
        if (bad < 0 && jobs[t].bad_row >= 0) bad = jobs[t].bad_row;
    }
    free(jobs);
    free(th);
    return bad;
}

/* --------------------------------------------------------------- builders */

typedef struct {
    oc_model* M;
    int64_t r0;
    int64_t* origins;
    double* probs;
    double* t0x;
} build_ctx;

/* build_matrix body: abstraction.cpp:209-223 (rows here, pairs there: same order) */
static void build_job(void* c, int64_t b, int64_t e, int64_t* bad) {
    build_ctx* C = (build_ctx*)c;
    const oc_model* M = C->M;
    rowk_t K;
    K.mass = (double*)malloc((size_t)(M->sumW > 0 ? M->sumW : 1) * sizeof(double));
    const int64_t nu = M->U.total, nw = M->W.total;
    for (int64_t k = b; k < e; ++k) {
        const int64_t row = C->r0 + k, iw = row % nw, p = row / nw;
        if (!row_compute(M, &K, p / nu, p % nu, iw) || !row_masses(M, &K)) { *bad = row; break; }
        int64_t flat = 0;
        for (int d = 0; d < M->X.dim; ++d) flat += K.o[d] * M->X.stride[d];
        C->origins[k] = flat;
        fill_product(M, K.mass, 0, 1.0, C->probs + k * M->R);
    }
    free(K.mass);
}

static void fail_row(const oc_model* M, int64_t row, char* err, int errlen) {
    snprintf(err, (size_t)errlen, "domain error at row %lld", (long long)row);
    (void)M;
}

int oc_build_matrix(oc_model* M, int64_t r0, int64_t r1, int64_t* origins, double* probs, int threads, char* err,
                    int errlen) {
    build_ctx C = {M, r0, origins, probs, NULL};
    const int64_t bad = par_for(r1 - r0, threads, &C, build_job);
    if (bad >= 0) { fail_row(M, bad, err, errlen); return 4; }
    return 0;
}

/* build_target_hit body: abstraction.cpp:255-269 */
static void t0x_job(void* c, int64_t b, int64_t e, int64_t* bad) {
    build_ctx* C = (build_ctx*)c;
    const oc_model* M = C->M;
    rowk_t K;
    K.mass = NULL;
    const int64_t nu = M->U.total, nw = M->W.total;
    for (int64_t k = b; k < e; ++k) {
        const int64_t row = C->r0 + k, iw = row % nw, p = row / nw, ix = p / nu;
        if (M->absorb[ix]) { C->t0x[k] = 0.0; continue; }
        int bd = 0;
        if (!row_compute(M, &K, ix, p % nu, iw)) { *bad = row; break; }
        C->t0x[k] = M->has_target ? box_mass(M, &K, &bd) : 0.0;
        if (bd) { *bad = row; break; }
    }
}

int oc_target_hit(oc_model* M, int64_t r0, int64_t r1, double* t0x, int threads, char* err, int errlen) {
    build_ctx C = {M, r0, NULL, NULL, t0x};
    const int64_t bad = par_for(r1 - r0, threads, &C, t0x_job);
    if (bad >= 0) { fail_row(M, bad, err, errlen); return 4; }
    return 0;
}

/* mask_absorbing: abstraction.cpp:273-344 (zero iff post rep in T, or in A) */
void oc_mask(const oc_model* M, int64_t rows, const int64_t* origins, double* probs) {
    if (M->spec_kind == 0) return;
    const int n = M->X.dim;
    for (int64_t r = 0; r < rows; ++r) {
        int64_t o[OC_MAXD], rem = origins[r];
        for (int d = 0; d < n; ++d) { o[d] = rem / M->X.stride[d]; rem %= M->X.stride[d]; }
        for (int64_t t = 0; t < M->R; ++t) {
            int64_t tt = t;
            int zt = 1, za = M->has_avoid;
            for (int d = n - 1; d >= 0; --d) {
                const int64_t j = tt % M->ext[d];
                tt /= M->ext[d];
                const double rep = M->X.lb[d] + (double)(o[d] + j) * M->X.eta[d];
                zt = zt && M->has_target && rep >= M->tlo[d] && rep <= M->thi[d];
                za = za && rep >= M->alo[d] && rep <= M->ahi[d];
            }
            if (zt || za) probs[r * M->R + t] = 0.0;
        }
    }
}

/* ---------------------------------------------------------------- synthesis */

/* dot_slab: synthesis.cpp:18-47 (row-major slab order, serial sum, exact zeros kept) */
static double dot_slab(const oc_model* M, const double* row, const int64_t* origin, const double* v,
                       const uint8_t* absorb) {
    const int n = M->X.dim;
    const int64_t wl = M->ext[n - 1];
    int64_t base = 0;
    for (int d = 0; d < n; ++d) base += origin[d] * M->X.stride[d];
    int64_t j[OC_MAXD] = {0};
    double sum = 0.0;
    const double* r = row;
    for (;;) {
        const double* vv = v + base;
        if (absorb) {
            const uint8_t* aa = absorb + base;
            for (int64_t t = 0; t < wl; ++t) sum += aa[t] ? 0.0 : r[t] * vv[t];
        } else {
            for (int64_t t = 0; t < wl; ++t) sum += r[t] * vv[t];
        }
        r += wl;
        int d = n - 2;
        for (; d >= 0; --d) {
            base += M->X.stride[d];
            if (++j[d] < M->ext[d]) break;
            base -= M->ext[d] * M->X.stride[d];
            j[d] = 0;
        }
        if (d < 0) break;
    }
    return sum;
}

typedef struct {
    oc_model* M;
    const double *probs, *t0x, *v;
    const int64_t* origins;
    int64_t r0;
    double* v_in;
} step_ctx;

/* bellman_impl pass 1: synthesis.cpp:75-109 (parallel over (state, input) pairs) */
static void step_job(void* c, int64_t b, int64_t e, int64_t* bad) {
    step_ctx* C = (step_ctx*)c;
    const oc_model* M = C->M;
    const int reach = M->spec_kind != 0;
    const int64_t nu = M->U.total, nw = M->W.total;
    rowk_t K;
    K.mass = (double*)malloc((size_t)(M->sumW > 0 ? M->sumW : 1) * sizeof(double));
    double* rowbuf = C->probs ? NULL : (double*)malloc((size_t)M->R * sizeof(double));
    for (int64_t pl = b; pl < e; ++pl) { /* pl: pair index relative to r0/nw */
        const int64_t p = C->r0 / nw + pl, ix = p / nu, iu = p % nu;
        const int absorbed = reach && M->absorb[ix];
        for (int64_t iw = 0; iw < nw; ++iw) {
            const int64_t rl = pl * nw + iw; /* local row */
            if (absorbed) { C->v_in[rl] = 0.0; continue; }
            double s;
            if (C->probs) {
                int64_t o[OC_MAXD], rem = C->origins[rl];
                for (int d = 0; d < M->X.dim; ++d) { o[d] = rem / M->X.stride[d]; rem %= M->X.stride[d]; }
                s = dot_slab(M, C->probs + rl * M->R, o, C->v, NULL);
                if (reach) s += C->t0x[rl];
            } else {
                int bd = 0;
                if (!row_compute(M, &K, ix, iu, iw) || !row_masses(M, &K)) { *bad = p * nw + iw; goto out; }
                fill_product(M, K.mass, 0, 1.0, rowbuf);
                s = dot_slab(M, rowbuf, K.o, C->v, reach ? M->absorb : NULL);
                if (reach) s += box_mass(M, &K, &bd);
                if (bd) { *bad = p * nw + iw; goto out; }
            }
            C->v_in[rl] = s;
        }
    }
out:
    free(K.mass);
    free(rowbuf);
}

int oc_bellman_step(oc_model* M, const double* probs, const int64_t* origins, const double* t0x, int64_t x0,
                    int64_t x1, const double* v_next, double* v_out, uint32_t* pol, uint32_t* wst, double* v_in_out,
                    int threads, char* err, int errlen) {
    const int64_t nu = M->U.total, nw = M->W.total;
    const int64_t pairs = (x1 - x0) * nu;
    double* v_in = v_in_out ? v_in_out : (double*)malloc((size_t)(pairs * nw > 0 ? pairs * nw : 1) * sizeof(double));
    step_ctx C = {M, probs, t0x, v_next, origins, x0 * nu * nw, v_in};
    const int64_t bad = par_for(pairs, threads, &C, step_job);
    if (bad >= 0) {
        if (!v_in_out) free(v_in);
        fail_row(M, bad, err, errlen);
        return 4;
    }
    /* pass 2: synthesis.cpp:112-142 (min over w strict <, max over u strict >) */
    const int reach = M->spec_kind != 0;
    for (int64_t ix = x0; ix < x1; ++ix) {
        const int64_t xl = ix - x0;
        if (reach && M->absorb[ix]) {
            v_out[xl] = 0.0;
            if (pol) pol[xl] = 0;
            if (wst) wst[xl] = 0;
            continue;
        }
        double best = -INFINITY;
        int64_t bu = 0, bw = 0;
        for (int64_t iu = 0; iu < nu; ++iu) {
            double mn = INFINITY;
            int64_t mw = 0;
            const int64_t base = (xl * nu + iu) * nw;
            for (int64_t iw = 0; iw < nw; ++iw)
                if (v_in[base + iw] < mn) { mn = v_in[base + iw]; mw = iw; }
            if (mn > best) { best = mn; bu = iu; bw = mw; }
        }
        const double q = 0.0 < best ? best : 0.0;
        v_out[xl] = q < 1.0 ? q : 1.0;
        if (pol) pol[xl] = (uint32_t)bu;
        if (wst) wst[xl] = (uint32_t)bw;
    }
    if (!v_in_out) free(v_in);
    return 0;
}

/* synthesize + run_backward: synthesis.cpp:165-228 (matrix mode masks the kernel
 * and builds T0x first, synthesis.cpp:199-212) */
int oc_synthesize(oc_model* M, int matrix_mode, double* values, uint32_t* pol, uint32_t* wst, int threads, char* err,
                  int errlen) {
    const int64_t n_x = M->X.total, rows = n_x * M->U.total * M->W.total;
    const int T = M->horizon;
    const int reach = M->spec_kind != 0;
    double *probs = NULL, *t0x = NULL;
    int64_t* origins = NULL;
    int rc = 0;
    if (matrix_mode) {
        probs = (double*)malloc((size_t)(rows * M->R) * sizeof(double));
        origins = (int64_t*)malloc((size_t)rows * sizeof(int64_t));
        if (!probs || !origins) { snprintf(err, (size_t)errlen, "oracle: out of host memory"); rc = 3; goto done; }
        if ((rc = oc_build_matrix(M, 0, rows, origins, probs, threads, err, errlen))) goto done;
        if (reach) {
            oc_mask(M, rows, origins, probs);
            t0x = (double*)malloc((size_t)rows * sizeof(double));
            if ((rc = oc_target_hit(M, 0, rows, t0x, threads, err, errlen))) goto done;
        }
    }
    for (int64_t i = 0; i < n_x; ++i) values[(size_t)T * (size_t)n_x + (size_t)i] = reach ? 0.0 : 1.0;
    for (int k = T - 1; k >= 0; --k) {
        rc = oc_bellman_step(M, probs, origins, t0x, 0, n_x, values + (size_t)(k + 1) * (size_t)n_x,
                             values + (size_t)k * (size_t)n_x, pol + (size_t)k * (size_t)n_x,
                             wst + (size_t)k * (size_t)n_x, NULL, threads, err, errlen);
        if (rc) goto done;
    }
done:
    free(probs);
    free(origins);
    free(t0x);
    return rc;
}
