// Row-level device code of stage (i) and of the OFA row prologue: decode,
// dynamics, slab origins, cell masses, target-hit masses, and the kernels that
// evaluate the dynamics (k_prologue, k_build_ws). Included by gm_kernels.cu
// (ahead-of-time, dynamics by the bytecode interpreter) and compiled at run time
// by NVRTC with GM_JIT_DYNAMICS (gm_jit.cpp: the config's dynamics as straight-line
// device code, same IEEE operations and libdevice functions, same bits).
#pragma once

#ifdef __CUDACC_RTC__
// prologue options / row flags (gm_kernels.cuh in the ahead-of-time build)
enum : unsigned char { RF_ABSORBED = 1, RF_ERROR = 2 };
enum : int { PF_SKIP_ABSORBED = 1, PF_T0X = 2, PF_MASSES = 4 };
#endif

constexpr int kThreads = 256;

// Grid dimensions of the row code: compile-time constants in the kernels compiled at
// run time for one model (gm_jit.cpp: loops unroll, the per-row x / u / w / mu
// arrays live in registers instead of local memory), the descriptor's otherwise.
#ifdef GM_JIT_NDIM
#define GM_DN(D) GM_JIT_NDIM
#define GM_DM(D) GM_JIT_MDIM
#define GM_DP(D) GM_JIT_PDIM
#else
#define GM_DN(D) ((D).n)
#define GM_DM(D) ((D).m)
#define GM_DP(D) ((D).p)
#endif
constexpr double kIdxTol = 1e-9; // abstraction.cpp:10

// x86-64 cvttsd2si semantics of static_cast<int64_t>(double) in the reference:
// NaN / out-of-range produce INT64_MIN (which the origin clamp maps to 0).
__device__ __forceinline__ long long to_i64_x86(double v) {
    if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return (long long)0x8000000000000000ULL;
    return static_cast<long long>(v);
}

// std::min / std::max argument order semantics (b < a ? b : a), NaN-exact
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__device__ void decode_row(const GmDev& D, long long row, long long& ix, double* x, double* u,
                           double* w) {
    if (D.idx32) { // same integers by multiply-shift division
        const int r32 = static_cast<int>(row);
        const int pr = D.div_nw.div(r32), iw = r32 - pr * static_cast<int>(D.n_w);
        const int x32 = D.div_nu.div(pr), iu = pr - x32 * static_cast<int>(D.n_u);
        ix = x32;
        int rem = x32;
        for (int d = 0; d < GM_DN(D); ++d) {
            const int j = D.div_xs[d].div(rem);
            rem -= j * static_cast<int>(D.xstride[d]);
            x[d] = D.xlb[d] + static_cast<double>(j) * D.xeta[d];
        }
        rem = iu;
        for (int d = 0; d < GM_DM(D); ++d) {
            const int j = D.div_us[d].div(rem);
            rem -= j * static_cast<int>(D.ustride[d]);
            u[d] = D.ulb[d] + static_cast<double>(j) * D.ueta[d];
        }
        rem = iw;
        for (int d = 0; d < GM_DP(D); ++d) {
            const int j = D.div_ws[d].div(rem);
            rem -= j * static_cast<int>(D.wstride[d]);
            w[d] = D.wlb[d] + static_cast<double>(j) * D.weta[d];
        }
        return;
    }
    const long long iw = row % D.n_w;
    const long long pr = row / D.n_w;
    const long long iu = pr % D.n_u;
    ix = pr / D.n_u;
    long long rem = ix;
    for (int d = 0; d < GM_DN(D); ++d) {
        const long long j = rem / D.xstride[d];
        rem -= j * D.xstride[d];
        x[d] = D.xlb[d] + static_cast<double>(j) * D.xeta[d];
    }
    rem = iu;
    for (int d = 0; d < GM_DM(D); ++d) {
        const long long j = rem / D.ustride[d];
        rem -= j * D.ustride[d];
        u[d] = D.ulb[d] + static_cast<double>(j) * D.ueta[d];
    }
    rem = iw;
    for (int d = 0; d < GM_DP(D); ++d) {
        const long long j = rem / D.wstride[d];
        rem -= j * D.wstride[d];
        w[d] = D.wlb[d] + static_cast<double>(j) * D.weta[d];
    }
}

#ifdef GM_JIT_DYNAMICS
// the config's dynamics compiled to straight-line code (gm_jit.cpp: gm_dyn_jit)
__device__ __forceinline__ bool run_dynamics(const GmDev&, const GmIns*, const double*, const double* x,
                                             const double* u, const double* w, double* mu) {
    return gm_dyn_jit(x, u, w, mu);
}
#else
// Dynamics bytecode interpreter (semantics of expr.cpp:404-480: IEEE double,
// comparisons 1/0, lazy ite, domain errors). Returns false on a domain error.
// One expression of the program (pc range entry[e]..entry[e+1]) into `out`;
// false on a domain error.
__device__ bool run_expr(const GmDev& D, const GmIns* __restrict__ prog, const double* __restrict__ lits, int e,
                         const double* x, const double* u, const double* w, double& out) {
    double r[GMD_MAXREGS];
    int pc = D.entry[e];
    const int end = D.entry[e + 1];
    while (pc < end) {
        const GmIns I = prog[pc++];
        const double a = r[I.a];
        const double b = r[I.b];
        double v;
        switch (I.op) {
            case GI_LIT: v = lits[I.arg]; break;
            case GI_LDX: v = x[I.arg]; break;
            case GI_LDU: v = u[I.arg]; break;
            case GI_LDW: v = w[I.arg]; break;
            case GI_ADD: v = a + b; break;
            case GI_SUB: v = a - b; break;
            case GI_MUL: v = a * b; break;
            case GI_DIV:
                if (b == 0.0) return false;
                v = a / b;
                break;
            case GI_POW:
                if (a < 0.0 && b != floor(b)) return false;
                if (a == 0.0 && b < 0.0) return false;
                v = (b == 2.0) ? a * a : pow(a, b);
                break;
            case GI_LT: v = a < b ? 1.0 : 0.0; break;
            case GI_LE: v = a <= b ? 1.0 : 0.0; break;
            case GI_GT: v = a > b ? 1.0 : 0.0; break;
            case GI_GE: v = a >= b ? 1.0 : 0.0; break;
            case GI_EQ: v = a == b ? 1.0 : 0.0; break;
            case GI_NE: v = a != b ? 1.0 : 0.0; break;
            case GI_NEG: v = -a; break;
            case GI_SIN: v = sin(a); break;
            case GI_COS: v = cos(a); break;
            case GI_TAN: v = tan(a); break;
            case GI_ASIN:
                if (a < -1.0 || a > 1.0) return false;
                v = asin(a);
                break;
            case GI_ACOS:
                if (a < -1.0 || a > 1.0) return false;
                v = acos(a);
                break;
            case GI_ATAN: v = atan(a); break;
            case GI_EXP: v = exp(a); break;
            case GI_LN:
                if (a <= 0.0) return false;
                v = log(a);
                break;
            case GI_SQRT:
                if (a < 0.0) return false;
                v = sqrt(a);
                break;
            case GI_ABS: v = fabs(a); break;
            case GI_MIN: v = fmin(a, b); break;
            case GI_MAX: v = fmax(a, b); break;
            case GI_JZ:
                if (a == 0.0) pc = I.arg;
                continue;
            case GI_JMP:
                pc = I.arg;
                continue;
            default: return false;
        }
        r[I.dst] = v;
    }
    out = r[0];
    return true;
}

__device__ bool run_dynamics(const GmDev& D, const GmIns* __restrict__ prog,
                             const double* __restrict__ lits, const double* x, const double* u,
                             const double* w, double* mu) {
    for (int i = 0; i < D.n; ++i)
        if (!run_expr(D, prog, lits, i, x, u, w, mu[i])) return false;
    return true;
}
#endif

// Regularized incomplete beta, Lentz continued fraction (noise.cpp:375-403);
// the reference's reflection recursion is unrolled into a loop.
__device__ double inc_beta(double a, double b, double x, bool& ok) {
    int refl = 0;
    double res;
    for (;;) {
        if (x <= 0.0) { res = 0.0; break; }
        if (x >= 1.0) { res = 1.0; break; }
        if (x > (a + 1.0) / (a + b + 2.0) && refl < 64) {
            const double t = a;
            a = b;
            b = t;
            x = 1.0 - x;
            ++refl;
            continue;
        }
        const double lbeta = lgamma(a) + lgamma(b) - lgamma(a + b);
        const double front = exp(log(x) * a + log1p(-x) * b - lbeta) / a;
        double f = 1.0, c = 1.0, d = 0.0;
        bool conv = false;
        for (int i = 0; i <= 400; ++i) {
            const int m = i / 2;
            double num;
            if (i == 0) num = 1.0;
            else if (i % 2 == 0)
                num = m * (b - m) * x / ((a + 2.0 * m - 1.0) * (a + 2.0 * m));
            else
                num = -((a + m) * (a + b + m) * x) / ((a + 2.0 * m) * (a + 2.0 * m + 1.0));
            d = 1.0 + num * d;
            if (fabs(d) < 1e-30) d = 1e-30;
            d = 1.0 / d;
            c = 1.0 + num / c;
            if (fabs(c) < 1e-30) c = 1e-30;
            f *= c * d;
            if (fabs(1.0 - c * d) < 1e-15) {
                res = smin(1.0, smax(0.0, front * (f - 1.0)));
                conv = true;
                break;
            }
        }
        if (!conv) { ok = false; res = 0.0; }
        break;
    }
    for (int i = 0; i < refl; ++i) res = 1.0 - res;
    return res;
}

// axis_mass (noise.cpp:92-122)
__device__ double axis_mass(const GmDev& D, int d, double lo, double hi, bool& ok) {
    if (hi <= lo) return 0.0;
    switch (D.family) {
        case GM_NORMAL: {
            const double is = D.inv_s[d];
            return 0.5 * (erf(hi * is) - erf(lo * is));
        }
        case GM_UNIFORM: {
            const double a = D.s[d], b = D.p2[d];
            const double ov = smin(hi, b) - smax(lo, a);
            return ov > 0.0 ? ov / (b - a) : 0.0;
        }
        case GM_EXPONENTIAL: {
            const double l = D.s[d];
            const double ch = hi <= 0.0 ? 0.0 : -expm1(-l * hi);
            const double cl = lo <= 0.0 ? 0.0 : -expm1(-l * lo);
            return ch - cl;
        }
        default: { // beta
            const double a = D.s[d], b = D.p2[d];
            const double ch = hi <= 0.0 ? 0.0 : (hi >= 1.0 ? 1.0 : inc_beta(a, b, hi, ok));
            const double cl = lo <= 0.0 ? 0.0 : (lo >= 1.0 ? 1.0 : inc_beta(a, b, lo, ok));
            return ch - cl;
        }
    }
}

// axis_transformed_mass (noise.cpp:124-131)
__device__ __forceinline__ double tmass(const GmDev& D, int d, double lo, double hi, double mean,
                                        double scale, bool& ok) {
    if (scale == 0.0) return (mean >= lo && mean <= hi) ? 1.0 : 0.0;
    double a = scale == 1.0 ? lo - mean : (lo - mean) / scale; // x / 1.0 == x exactly
    double b = scale == 1.0 ? hi - mean : (hi - mean) / scale;
    if (scale < 0.0) {
        const double t = a;
        a = b;
        b = t;
    }
    return axis_mass(D, d, a, b, ok);
}

// Per-boundary CDF term of axis_mass (noise.cpp:92-122): erf(x/s) for the normal,
// the exponential / beta CDFs; axis_mass(lo, hi) = combine(F(hi), F(lo)).
__device__ __forceinline__ double axis_F(const GmDev& D, int d, double x, bool& ok) {
    switch (D.family) {
        case GM_NORMAL: return erf(x * D.inv_s[d]);
        case GM_EXPONENTIAL: return x <= 0.0 ? 0.0 : -expm1(-D.s[d] * x);
        default: return x <= 0.0 ? 0.0 : (x >= 1.0 ? 1.0 : inc_beta(D.s[d], D.p2[d], x, ok));
    }
}

__device__ __forceinline__ bool same_bits(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}

// fill_axis_masses for one axis (abstraction.cpp:130-146): the W cell masses of
// axis d, each exactly axis_transformed_mass(d, rep-η/2, rep+η/2, μ, scale)
// (noise.cpp:124-131). Adjacent cells share a boundary: when the transformed
// boundary of cell t+1 is bitwise equal to the one of cell t, the reference
// evaluates the same CDF argument twice; the value is reused instead, so the
// masses are bit-identical while erf/expm1/inc_beta calls drop from 2W to W+1.
__device__ void axis_masses(const GmDev& D, int d, long long o, double mu, double scale, double* out, int stride,
                            bool& ok) {
    const double eta = D.xeta[d], half = 0.5 * D.xeta[d], lb = D.xlb[d];
    double cx0 = 0.0, cF0 = 0.0, cx1 = 0.0, cF1 = 0.0;
    bool h0 = false, h1 = false;
    for (int t = 0; t < D.W[d]; ++t) {
        const double rep = lb + static_cast<double>(o + t) * eta;
        const double lo = rep - half, hi = rep + half;
        double m;
        if (scale == 0.0) {
            m = (mu >= lo && mu <= hi) ? 1.0 : 0.0;
        } else {
            double a = scale == 1.0 ? lo - mu : (lo - mu) / scale; // x / 1.0 == x exactly
            double b = scale == 1.0 ? hi - mu : (hi - mu) / scale;
            if (scale < 0.0) {
                const double tmp = a;
                a = b;
                b = tmp;
            }
            if (b <= a) {
                m = 0.0;
            } else if (D.family == GM_UNIFORM) {
                const double ua = D.s[d], ub = D.p2[d];
                const double ov = smin(b, ub) - smax(a, ua);
                m = ov > 0.0 ? ov / (ub - ua) : 0.0;
            } else {
                const double Fa = (h0 && same_bits(a, cx0)) ? cF0 : (h1 && same_bits(a, cx1)) ? cF1 : axis_F(D, d, a, ok);
                const double Fb = (h0 && same_bits(b, cx0)) ? cF0 : (h1 && same_bits(b, cx1)) ? cF1 : axis_F(D, d, b, ok);
                m = D.family == GM_NORMAL ? 0.5 * (Fb - Fa) : Fb - Fa;
                cx0 = a; cF0 = Fa; h0 = true;
                cx1 = b; cF1 = Fb; h1 = true;
            }
        }
        out[static_cast<long long>(t) * stride] = m;
    }
}

// slab origin along one axis (abstraction.cpp:103-120)
__device__ __forceinline__ long long slab_origin(const GmDev& D, int d, double mu) {
    long long o;
    if (D.cut == GM_CUT_NONE) {
        o = 0;
    } else if (D.cut == GM_CUT_DEGENERATE) {
        const double t = (mu - D.xlb[d]) / D.xeta[d];
        o = to_i64_x86(floor(t + 0.5));
    } else {
        const double t = (mu - D.radius[d] - 0.5 * D.xeta[d] - D.xlb[d]) / D.xeta[d];
        o = to_i64_x86(ceil(t - kIdxTol));
    }
    if (o < 0) o = 0;
    if (o > D.xcount[d] - D.W[d]) o = D.xcount[d] - D.W[d];
    return o;
}

__device__ __forceinline__ bool in_box(const GmDev& D, const double* p, const double* lo,
                                       const double* hi) {
    for (int d = 0; d < GM_DN(D); ++d)
        if (!(p[d] >= lo[d])) return false;
    for (int d = 0; d < GM_DN(D); ++d)
        if (!(p[d] <= hi[d])) return false;
    return true;
}

__device__ __forceinline__ void record_error(unsigned long long* err, long long row) {
    atomicMin(err, static_cast<unsigned long long>(row));
}

// Flat offset of a slab's last post-state from its origin (the gathers of a row read
// V[origin .. origin + span]); the checked build asserts every row's slab is in V.
__device__ __forceinline__ long long slab_span(const GmDev& D) {
    long long s = 0;
    for (int d = 0; d < GM_DN(D); ++d) s += static_cast<long long>(D.W[d] - 1) * D.xstride[d];
    return s;
}
#define GM_CHECK_SLAB(D, o) GM_CHECK((o) >= 0 && (o) + slab_span(D) < (D).n_x)

extern __shared__ __align__(16) double g_sm[];

// Prefix product of entry a of the P table (fill_product's recursion carried as
// acc, abstraction.cpp:150-159): acc = ((1 * m0[j0]) * m1[j1]) * ... in axis
// order, with (j0, j1, ...) decoded from a first axis first.
__device__ __forceinline__ double prefix_product(const GmDev& D, const double* m, int a) {
    double acc = 1.0;
    int rem = a;
    for (int d = 0; d < D.s_axes; ++d) {
        const int j = D.div_Ps[d].div(rem);
        rem -= j * D.Ps[d];
        acc *= m[D.mass_off[d] + j];
    }
    return acc;
}

#if !defined(__CUDACC_RTC__) || defined(GM_JIT_PROLOGUE)
// One thread per row: image, origin, per-axis masses (SoA, pitch nrows), T0x.
__global__ void __launch_bounds__(kThreads) k_prologue(GmDev D, long long row0, long long nrows, int flags,
                                                      long long* __restrict__ origin_out,
                                                      double* __restrict__ t0x_out,
                                                      uint8_t* __restrict__ rowflag_out,
                                                      double* __restrict__ mass_out,
                                                      unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GmIns* sprog = reinterpret_cast<GmIns*>(smem_raw);
    double* slits = reinterpret_cast<double*>(smem_raw + ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16);
    for (int i = threadIdx.x; i < D.n_ins; i += blockDim.x) sprog[i] = D.prog[i];
    for (int i = threadIdx.x; i < D.n_lits; i += blockDim.x) slits[i] = D.lits[i];
    __syncthreads();

    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= nrows) return;
    const long long row = row0 + i;
    double x[GMD_MAXD], u[GMD_MAXD], w[GMD_MAXD], mu[GMD_MAXD];
    long long ix;
    decode_row(D, row, ix, x, u, w);
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const bool absorbed = reach && D.absorb != nullptr && D.absorb[ix];
    uint8_t fl = absorbed ? RF_ABSORBED : 0;
    if (absorbed && (flags & PF_SKIP_ABSORBED)) {
        if (t0x_out) t0x_out[i] = 0.0;
        if (rowflag_out) rowflag_out[i] = fl;
        return;
    }
    if (!run_dynamics(D, sprog, slits, x, u, w, mu)) {
        record_error(err, row);
        if (rowflag_out) rowflag_out[i] = fl | RF_ERROR;
        return;
    }
    long long org[GMD_MAXD];
    long long flat = 0;
    for (int d = 0; d < GM_DN(D); ++d) {
        org[d] = slab_origin(D, d, mu[d]);
        flat += org[d] * D.xstride[d];
    }
    GM_CHECK_SLAB(D, flat);
    if (origin_out) origin_out[i] = flat;
    bool ok = true;
    if (flags & PF_MASSES) { // per-cell form: keeps this kernel at 64 registers (axis_masses: 80)
        for (int d = 0; d < GM_DN(D); ++d) {
            const double scale = D.mult ? x[d] : 1.0;
            const double half = 0.5 * D.xeta[d];
            double* md = mass_out + static_cast<long long>(D.mass_off[d]) * nrows + i;
            for (int t = 0; t < D.W[d]; ++t) {
                const double rep = D.xlb[d] + static_cast<double>(org[d] + t) * D.xeta[d];
                md[static_cast<long long>(t) * nrows] = tmass(D, d, rep - half, rep + half, mu[d], scale, ok);
            }
        }
    }
    if ((flags & PF_T0X) && t0x_out) {
        double p = 0.0;
        if (!absorbed) { // cell_probability_impl (noise.cpp:251-257) over the target box
            p = 1.0;
            for (int d = 0; d < GM_DN(D); ++d) {
                const double scale = D.mult ? x[d] : 1.0;
                p *= tmass(D, d, D.tlo[d], D.thi[d], mu[d], scale, ok);
                if (p == 0.0) break;
            }
            p = smin(1.0, smax(0.0, p));
        }
        t0x_out[i] = p;
    }
    if (!ok) {
        record_error(err, row);
        fl |= RF_ERROR;
    }
    if (rowflag_out) rowflag_out[i] = fl;
}
#endif

// Lane-stride walk over a row: lane l of a group of tpr visits t = l, l+tpr, ...
// as (L, k) = (slab line, last-axis offset), plus (a, j) for TAB_P.
struct Walk {
    int L, k, a, j;
    int qL, qk, qa, qj, Wl, Wm;
    __device__ __forceinline__ void init(const GmDev& D, int lane, int tpr) {
        Wl = D.Wl;
        Wm = D.Wm;
        L = D.div_Wl.div(lane);
        k = lane - L * Wl;
        a = D.div_Wm.div(L);
        j = L - a * Wm;
        qL = D.div_Wl.div(tpr);
        qk = tpr - qL * Wl;
        qa = D.div_Wm.div(qL);
        qj = qL - qa * Wm;
    }
    template <bool AJ>
    __device__ __forceinline__ void next() {
        k += qk;
        const int c = k >= Wl;
        k -= c ? Wl : 0;
        L += qL + c;
        if (AJ) {
            j += qj + c;
            const int c2 = j >= Wm;
            j -= c2 ? Wm : 0;
            a += qa + c2;
        }
    }
};

// ---------------------------------------------------------------------------
// Stage (i), fused and warp-specialised. The row prologue (decode, dynamics
// bytecode, slab origin, target-hit mass: one thread per row, a long serial
// chain) of batch k+1 runs on the `npw` producer warps while the consumer
// warps build batch k (cell masses, prefix tables); then every warp, producers
// included once their prologue is done, claims rows of batch k to expand.
// Barriers: 0 = whole CTA (batch boundary), 1 = consumer warps, 2 = "tables of
// batch k ready" (consumers arrive, producers wait).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct ProBuf { // one batch's prologue results in shared memory (row stride n = state dim)
    double* mu;  // [rb][n]
    double* x;   // [rb][n]
    double* ok;  // [rb]
    int* org;    // [rb][n]
    int n;
};

__device__ __forceinline__ int pro_doubles(int rb, int n) { return 2 * rb * n + rb + (rb * n + 1) / 2; }

__device__ __forceinline__ ProBuf pro_buf(int base, int rb, int n) {
    ProBuf p;
    p.mu = g_sm + base;
    p.x = p.mu + rb * n;
    p.ok = p.x + rb * n;
    p.org = reinterpret_cast<int*>(p.ok + rb);
    p.n = n;
    return p;
}

// RowKernel::compute (abstraction.cpp:72-121) + box_mass (:187-191) for rows
// b0 + [ti, ti+nt, ...) of a batch
__device__ __forceinline__ void build_prologue(const GmDev& D, const GmIns* sprog, const double* slits,
                                               long long row0, long long nrows, long long b0, int rb, int ti,
                                               int nt, const ProBuf& pb, long long* __restrict__ origin_out,
                                               double* __restrict__ t0x_out, unsigned long long* err) {
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    for (int i = ti; i < rb; i += nt) {
        const long long r = b0 + i;
        double ok = 0.0;
        if (r < nrows) {
            double x[GMD_MAXD], u[GMD_MAXD], w[GMD_MAXD], mu[GMD_MAXD];
            long long ix;
            decode_row(D, row0 + r, ix, x, u, w);
            if (run_dynamics(D, sprog, slits, x, u, w, mu)) {
                ok = 1.0;
                long long flat = 0;
                for (int d = 0; d < GM_DN(D); ++d) {
                    const long long o = slab_origin(D, d, mu[d]);
                    pb.org[i * pb.n + d] = static_cast<int>(o);
                    flat += o * D.xstride[d];
                    pb.mu[i * pb.n + d] = mu[d];
                    pb.x[i * pb.n + d] = x[d];
                }
                GM_CHECK_SLAB(D, flat);
                GM_CHECK(r < nrows && i < rb);
                origin_out[r] = flat;
                if (D.origin_host) D.origin_host[r] = flat;
                if (t0x_out) {
                    const bool absorbed = reach && D.absorb != nullptr && D.absorb[ix];
                    double p = 0.0;
                    bool bok = true;
                    if (!absorbed) {
                        p = 1.0;
                        for (int d = 0; d < GM_DN(D); ++d) {
                            p *= tmass(D, d, D.tlo[d], D.thi[d], mu[d], D.mult ? x[d] : 1.0, bok);
                            if (p == 0.0) break;
                        }
                        p = smin(1.0, smax(0.0, p));
                    }
                    if (!bok) record_error(err, row0 + r);
                    t0x_out[r] = p;
                    if (D.t0x_host) D.t0x_host[r] = p;
                }
            } else {
                record_error(err, row0 + r);
            }
        }
        pb.ok[i] = ok;
    }
}

// Three-role pipeline over batches j = blockIdx.x + i*gridDim.x of rb rows.
// Iteration i: producer warps run the row prologue of batch i+2 (-> pro[(i+2)&1]),
// consumer warps turn batch i+1's prologue into cell masses and the prefix table
// P (-> tab[(i+1)&1]), filler warps expand batch i from tab[i&1] (per row: line
// prefixes Q[L] = P[a]*mm[j] into a per-warp scratch, then lane-strided
// evict-first stores of Q[L]*ml[k] through the element table ET); producers and
// consumers join the fill when their own work is done. One CTA barrier per
// iteration. The fill streams continuously: ~8 storing warps per SM saturate
// HBM writes for this row pattern (scripts/store_probe.cu).
// QS = per-warp Q scratch + element table (n_lines and W_last small enough);
// otherwise rows are expanded by the incremental slab walk, q = P[a]*mm[j] per term.
#ifdef GM_FILL_WL
// ld.shared.f64 at a register address plus an immediate offset (one LDS, no address math)
template <int OFF>
__device__ __forceinline__ double lds_imm(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(OFF));
    return v;
}
// The lane's elements t = lane + 32 i of one row, i = 0 .. ceil(pitch/32) - 1, unrolled
// at compile time: element i = s + PER*b is Q[L(s) + DL*b] * ml[k(s)], one LDS, one
// DMUL, one evict-first STG with immediate offsets; elements past R (row padding)
// store +0.0, lanes past the pitch (a pitch that is not a multiple of 32) none.
// s = i mod PER < GM_FILL_NS = min(PER, number of chunks) register slots.
template <int I>
struct FillRow {
    static __device__ __forceinline__ void run(const unsigned* fq, const double* mv, double* o, int lane) {
        constexpr int PER = GM_FILL_PER, S = I % PER, B = I / PER;
        constexpr int OFF = 8 * (32 * PER / GM_FILL_WL) * B;
        static_assert(S < GM_FILL_NS, "register slot");
        if constexpr (32 * I + 31 < GM_FILL_R) {
            __stcs(o + 32 * I, lds_imm<OFF>(fq[S]) * mv[S]);
        } else if constexpr (32 * I + 31 < GM_FILL_PITCH) {
            const double q = lane + 32 * I < GM_FILL_R ? lds_imm<OFF>(fq[S]) : 0.0;
            __stcs(o + 32 * I, q * mv[S]);
        } else {
            const double q = lane + 32 * I < GM_FILL_R ? lds_imm<OFF>(fq[S]) : 0.0;
            if (lane + 32 * I < GM_FILL_PITCH) __stcs(o + 32 * I, q * mv[S]);
        }
        if constexpr (I + 1 < (GM_FILL_PITCH + 31) / 32) FillRow<I + 1>::run(fq, mv, o, lane);
    }
};
#endif

#if !defined(__CUDACC_RTC__) || defined(GM_JIT_BUILD)
template <bool QS, int MINB = 3>
__global__ void __launch_bounds__(kThreads, MINB) k_build_ws(GmDev D, long long row0, long long nrows, int rb,
                                                      int npw, int ncw, int opts,
                                                      long long* __restrict__ origin_out,
                                                      double* __restrict__ t0x_out, double* __restrict__ probs,
                                                      unsigned long long* err) {
    const int mw = D.sumW + 1;
    const int R = static_cast<int>(D.R);
    const int nl = D.n_lines;
    const int tsz = rb * (mw + D.P_size), psz = pro_doubles(rb, D.n);
    const int offT = 0, offPro = offT + 2 * tsz, offQs = offPro + 2 * psz;
    const int offProg = offQs + (QS ? (kThreads / 32) * (nl + 1) : 0); // per-warp Q[nl] + a zero slot
    GmIns* sprog = reinterpret_cast<GmIns*>(g_sm + offProg);
    double* slits = g_sm + offProg + D.n_ins;
    int* claim = reinterpret_cast<int*>(slits + D.n_lits); // fill-row counters by batch parity
    int* ET = claim + 2;
    // the launcher's shared-memory size covers the whole layout
    GM_CHECK(static_cast<unsigned>(reinterpret_cast<const char*>(ET + (QS ? D.pitch : 0)) -
                                   reinterpret_cast<const char*>(g_sm)) <= gm_dyn_smem_bytes());
    GM_CHECK(npw * 32 + ncw * 32 <= kThreads);
    for (int c = threadIdx.x; c < D.n_ins; c += blockDim.x) sprog[c] = D.prog[c];
    for (int c = threadIdx.x; c < D.n_lits; c += blockDim.x) slits[c] = D.lits[c];
    if (threadIdx.x < 2) claim[threadIdx.x] = 0;
    if (QS) {
        // entries past R (row padding) point at the warp's zero slot Q[nl]: 0 * ml[0] = +0.0
        for (int t = threadIdx.x; t < D.pitch; t += blockDim.x) {
            const int L = D.div_Wl.div(t < R ? t : 0);
            ET[t] = t < R ? (L * 8) | ((t - L * D.Wl) * 8) << 16 : nl * 8;
            GM_CHECK((ET[t] & 0xffff) <= nl * 8 && (ET[t] >> 16) < D.Wl * 8 && nl * 8 < 0x10000);
        }
        if (threadIdx.x < kThreads / 32) g_sm[offQs + threadIdx.x * (nl + 1) + nl] = 0.0;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef GM_FILL_WL
    // Row shape fixed at run-time compilation (NVRTC, gm_jit.cpp shape_defines): the
    // lane -> element map does not depend on the row, so each lane's Q-scratch index
    // and last-axis cell of its first PER elements are kernel-lifetime registers;
    // element i = s + PER*b of the lane reads Q[fq[s] + DL*b] * ml[fm[s]]
    // (32*PER is a multiple of Wl, so the cell repeats with period PER).
    constexpr int F_WL = GM_FILL_WL, F_WM = GM_FILL_WM, F_NL = GM_FILL_NL, F_PER = GM_FILL_PER;
    constexpr int F_R = GM_FILL_R, F_NQ = (F_NL + 31) / 32, F_NS = GM_FILL_NS;
    unsigned fq[F_NS]; // shared-window byte addresses of Q[L(s)] in this warp's scratch
    {
        const unsigned sm0 = static_cast<unsigned>(__cvta_generic_to_shared(g_sm));
#pragma unroll
        for (int s = 0; s < F_NS; ++s)
            fq[s] = sm0 + 8u * static_cast<unsigned>(offQs + warp * (F_NL + 1) + (lane + 32 * s) / F_WL);
        // every Q element a lane reads (t < R) lies in its warp's scratch
        GM_CHECK(D.Wl == F_WL && D.Wm == F_WM && D.n_lines == F_NL && D.R == F_R && D.pitch == GM_FILL_PITCH);
        for (int t = lane; t < F_R; t += 32) GM_CHECK(t / F_WL < F_NL);
    }
#endif
    const int np = npw * 32, nc = ncw * 32;
    const int role = warp < npw ? 0 : (warp < npw + ncw ? 1 : 2); // producer, consumer, filler
    const int ct = threadIdx.x - np;
    Walk wk0;
    wk0.init(D, lane, 32);
    auto first_row = [&](long long j) { return (static_cast<long long>(blockIdx.x) + j * gridDim.x) * rb; };
#ifdef GM_DIAG
    // opts bit 4: cycle totals of one thread per role (CTA 0; GM_DIAG builds only: the
    // counters cost registers in the shipped kernel)
    const bool prof = (opts & 16) && blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == np ||
                                                         threadIdx.x == np + nc);
    long long tp[3] = {0, 0, 0}, tl = clock64();
#define GM_TP(k)                          \
    if (prof) {                           \
        const long long n_ = clock64();   \
        tp[k] += n_ - tl;                 \
        tl = n_;                          \
    }
#else
#define GM_TP(k)
#endif
    __syncthreads();
    if (role == 0 && first_row(0) < nrows)
        build_prologue(D, sprog, slits, row0, nrows, first_row(0), rb, threadIdx.x, np, pro_buf(offPro, rb, D.n),
                       origin_out, t0x_out, err);
    __syncthreads();
    for (long long i = -1; first_row(i < 0 ? 0 : i) < nrows; ++i) {
        if (threadIdx.x == 0 && i >= 0) claim[(i + 1) & 1] = 0; // used by the next iteration only
        if (role == 0) {
            const long long bn = first_row(i + 2);
            if (bn < nrows)
                build_prologue(D, sprog, slits, row0, nrows, bn, rb, threadIdx.x, np,
                               pro_buf(offPro + static_cast<int>((i + 2) & 1) * psz, rb, D.n), origin_out, t0x_out, err);
        } else if (role == 1) {
            const long long bn = first_row(i + 1);
            if (bn < nrows) {
                const ProBuf cur = pro_buf(offPro + static_cast<int>((i + 1) & 1) * psz, rb, D.n);
                double* tb = g_sm + offT + static_cast<int>((i + 1) & 1) * tsz;
                // fill_axis_masses (abstraction.cpp:130-146): thread per (row, axis). (Evaluating
                // each distinct (origin, mu, scale) once per batch and copying the repeats cut
                // the instructions 4 % but lengthened the consumers' critical path: C2b build
                // 20 -> 28 ms; the W+1 serial CDF calls of one item set the pipeline's pace.)
                for (int c = ct; c < rb * D.n; c += nc) {
                    const int d = c / rb, r = c - d * rb;
                    if (cur.ok[r] != 0.0) {
                        bool ok = true;
                        axis_masses(D, d, cur.org[r * cur.n + d], cur.mu[r * cur.n + d],
                                    D.mult ? cur.x[r * cur.n + d] : 1.0, tb + r * mw + D.mass_off[d], 1, ok);
                        if (!ok) record_error(err, row0 + bn + r);
                    } else {
                        for (int t = 0; t < D.W[d]; ++t) tb[r * mw + D.mass_off[d] + t] = 1.0;
                    }
                }
                for (int r = ct; r < rb; r += nc) tb[r * mw + D.sumW] = 1.0; // virtual-axis slot
                named_sync(1, nc);
                // prefix products over the leading axes (abstraction.cpp:150-159 association)
                double* P = tb + rb * mw;
                for (int c = ct; c < rb * D.P_size; c += nc) {
                    const int r = D.div_P.div(c), a = c - r * D.P_size;
                    P[c] = prefix_product(D, tb + r * mw, a);
                }
            }
        }
        GM_TP(0)
        if (i >= 0) {
            // fill_product (abstraction.cpp:150-159) of batch i: warps claim rows
            const long long b0 = first_row(i);
            const double* tb = g_sm + offT + static_cast<int>(i & 1) * tsz;
            const double* P = tb + rb * mw;
            double* Qs = g_sm + offQs + warp * (nl + 1);
            for (;;) {
                int r = 0;
                if (lane == 0) r = atomicAdd(&claim[i & 1], 1);
                r = __shfl_sync(0xffffffffu, r, 0);
                const long long row = b0 + r;
                if (r >= rb || row >= nrows) break;
                GM_CHECK(r >= 0 && row >= 0);
                const double* m = tb + r * mw;
                const double* Pr = P + r * D.P_size;
                double* out = probs + row * D.pitch;
                const int pitch = static_cast<int>(D.pitch); // rows end in zero padding up to the pitch
#ifdef GM_DIAG
                if (opts & 96) { // timing diagnostics (GM_DIAG builds only): 32 = constant stores, 64 = no stores
                    if (opts & 32)
                        for (int t = lane; t < pitch; t += 32) __stcs(out + t, 0.0);
                    continue;
                }
#endif
                if (QS) {
#ifdef GM_FILL_WL
                    // line prefixes Q[L] = P[a] * mm[j] (abstraction.cpp:150-159 association)
#pragma unroll
                    for (int c = 0; c < F_NQ; ++c) {
                        const int L = lane + 32 * c; // constant divisors: multiply-shift
                        if (F_NL % 32 == 0 || L < F_NL) Qs[L] = Pr[L / F_WM] * m[D.mm_off + L % F_WM];
                    }
                    __syncwarp();
                    double mv[F_NS];
#pragma unroll
                    for (int s2 = 0; s2 < F_NS; ++s2) mv[s2] = m[D.ml_off + (lane + 32 * s2) % F_WL];
                    FillRow<0>::run(fq, mv, out + lane, lane);
                    __syncwarp();
#else
                    for (int L = lane; L < nl; L += 32) {
                        const int a = D.div_Wm.div(L), j = L - a * D.Wm;
                        Qs[L] = Pr[a] * m[D.mm_off + j];
                    }
                    __syncwarp();
                    const char* qb = reinterpret_cast<const char*>(Qs);
                    const char* mb = reinterpret_cast<const char*>(m + D.ml_off);
                    const int* e = ET + lane;
                    double* o = out + lane;
                    const int n_it = (pitch - lane + 31) >> 5;
#pragma unroll 4
                    for (int k = 0; k < n_it; ++k, e += 32, o += 32) {
                        const int ev = *e;
                        __stcs(o, *reinterpret_cast<const double*>(qb + (ev & 0xffff)) *
                                      *reinterpret_cast<const double*>(mb + (ev >> 16)));
                    }
                    __syncwarp();
#endif
                } else {
                    Walk wk = wk0;
#pragma unroll 4
                    for (int t = lane; t < R; t += 32) {
                        __stcs(out + t, (Pr[wk.a] * m[D.mm_off + wk.j]) * m[D.ml_off + wk.k]);
                        wk.template next<true>();
                    }
                    for (int t = R + lane; t < pitch; t += 32) __stcs(out + t, 0.0);
                }
            }
        }
        GM_TP(1)
        __syncthreads();
        GM_TP(2)
    }
#undef GM_TP
#ifdef GM_DIAG
    if (prof)
        printf("k_build_ws %s: rb %d npw %d ncw %d cycles: own work %lld, fill %lld, barrier %lld\n",
               role == 0 ? "producer" : (role == 1 ? "consumer" : "filler"), rb, npw, ncw, tp[0], tp[1], tp[2]);
#endif
}
#endif
