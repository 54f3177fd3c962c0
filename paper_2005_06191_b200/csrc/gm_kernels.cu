// sm_100a kernels of the B200 AMYTISS engine.
//
// Stage (i)  MDP construction:  prologue (per-row image, slab origin, per-axis
//            CDF masses, target-hit mass) -> expand (outer product, coalesced
//            stores of the fixed-width slab rows).
// Stage (ii) Bellman synthesis: expect_matrix (stream stored rows, gather V)
//            or prologue -> expect_ofa (recompute rows in shared memory, gather
//            V), then maxmin (min over disturbances, max over inputs).
//
// Compiled with --fmad=false: every index/representative/mass expression is
// rounded exactly like the reference's unfused mul+add (abstraction.cpp:78,
// 113-115, 139-143), so origins and slab extents are bit-exact; the dot
// product uses explicit fma() and one fixed lane order shared by the matrix
// and on-the-fly kernels, so both modes produce identical bits.
#include "gm_kernels.cuh"

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace gmk {

namespace {

constexpr int kThreads = 256;
constexpr double kIdxTol = 1e-9; // abstraction.cpp:10

inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline int grid_for(long long work, int per_block) {
    long long b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > (1LL << 30)) b = (1LL << 30);
    return static_cast<int>(b);
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

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
    const long long iw = row % D.n_w;
    const long long pr = row / D.n_w;
    const long long iu = pr % D.n_u;
    ix = pr / D.n_u;
    long long rem = ix;
    for (int d = 0; d < D.n; ++d) {
        const long long j = rem / D.xstride[d];
        rem -= j * D.xstride[d];
        x[d] = D.xlb[d] + static_cast<double>(j) * D.xeta[d];
    }
    rem = iu;
    for (int d = 0; d < D.m; ++d) {
        const long long j = rem / D.ustride[d];
        rem -= j * D.ustride[d];
        u[d] = D.ulb[d] + static_cast<double>(j) * D.ueta[d];
    }
    rem = iw;
    for (int d = 0; d < D.p; ++d) {
        const long long j = rem / D.wstride[d];
        rem -= j * D.wstride[d];
        w[d] = D.wlb[d] + static_cast<double>(j) * D.weta[d];
    }
}

// Dynamics bytecode interpreter (semantics of expr.cpp:404-480: IEEE double,
// comparisons 1/0, lazy ite, domain errors). Returns false on a domain error.
__device__ bool run_dynamics(const GmDev& D, const GmIns* __restrict__ prog,
                             const double* __restrict__ lits, const double* x, const double* u,
                             const double* w, double* mu) {
    double r[GMD_MAXREGS];
    for (int i = 0; i < D.n; ++i) {
        int pc = D.entry[i];
        const int end = D.entry[i + 1];
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
        mu[i] = r[0];
    }
    return true;
}

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
            const double s = D.s[d];
            return 0.5 * (erf(hi / s) - erf(lo / s));
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
    double a = (lo - mean) / scale;
    double b = (hi - mean) / scale;
    if (scale < 0.0) {
        const double t = a;
        a = b;
        b = t;
    }
    return axis_mass(D, d, a, b, ok);
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
    for (int d = 0; d < D.n; ++d)
        if (!(p[d] >= lo[d])) return false;
    for (int d = 0; d < D.n; ++d)
        if (!(p[d] <= hi[d])) return false;
    return true;
}

__device__ __forceinline__ void record_error(unsigned long long* err, long long row) {
    atomicMin(err, static_cast<unsigned long long>(row));
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

__global__ void k_absorb(GmDev D, uint8_t* flags) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= D.n_x) return;
    double p[GMD_MAXD];
    long long rem = i;
    for (int d = 0; d < D.n; ++d) {
        const long long j = rem / D.xstride[d];
        rem -= j * D.xstride[d];
        p[d] = D.xlb[d] + static_cast<double>(j) * D.xeta[d];
    }
    bool a = false;
    if (D.spec_kind != GM_SPEC_SAFETY) {
        a = in_box(D, p, D.tlo, D.thi) || (D.has_avoid && in_box(D, p, D.alo, D.ahi));
    }
    flags[i] = a ? 1 : 0;
}

__global__ void k_zero_absorbing(GmDev D, double* v) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= D.n_x) return;
    if (D.absorb[i]) v[i] = 0.0;
}

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
    for (int d = 0; d < D.n; ++d) {
        org[d] = slab_origin(D, d, mu[d]);
        flat += org[d] * D.xstride[d];
    }
    if (origin_out) origin_out[i] = flat;
    bool ok = true;
    if (flags & PF_MASSES) {
        for (int d = 0; d < D.n; ++d) {
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
            for (int d = 0; d < D.n; ++d) {
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

// Shared-memory layout of a batch of rows for expand / expect_ofa.
struct BatchSmem {
    double* mass;   // [rb][sumW+1]  (slot sumW = 1.0: virtual axis)
    double* P;      // [rb][P_size]  prefix products over the leading axes
    double* red;    // [kThreads/32] cross-warp partial sums
    int* lines;     // [n_lines] (when staged)
};

__device__ __forceinline__ BatchSmem carve(const GmDev& D, int rb, int table_in_smem) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BatchSmem S;
    double* p = reinterpret_cast<double*>(smem_raw);
    S.mass = p;
    p += static_cast<long long>(rb) * (D.sumW + 1);
    S.P = p;
    p += static_cast<long long>(rb) * D.P_size;
    S.red = p;
    p += kThreads / 32;
    S.lines = table_in_smem ? reinterpret_cast<int*>(p) : const_cast<int*>(D.line_off);
    return S;
}

// Loads masses of rows [b0, b0+rb) and builds their prefix tables P (the
// prefix product 1.0*m0[j0]*m1[j1]*... over axes 0..n-3, abstraction.cpp:157).
__device__ __forceinline__ void stage_rows(const GmDev& D, const BatchSmem& S, const double* __restrict__ mass,
                                           long long nrows, long long b0, int rb) {
    const int mw = D.sumW + 1;
    for (int c = threadIdx.x; c < rb * mw; c += blockDim.x) {
        const int i = c % rb, q = c / rb; // consecutive threads -> consecutive rows (coalesced SoA)
        double v = 1.0;
        if (q < D.sumW && b0 + i < nrows) v = mass[static_cast<long long>(q) * nrows + b0 + i];
        S.mass[i * mw + q] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < rb * D.P_size; c += blockDim.x) {
        const int i = c / D.P_size, a = c % D.P_size;
        const double* mrow = S.mass + i * mw;
        // decode a over W[0..s_axes) row-major, multiply in axis order
        int rem = a;
        int div = D.P_size;
        double acc = 1.0;
        for (int d = 0; d < D.s_axes; ++d) {
            div /= D.W[d];
            const int j = rem / div;
            rem -= j * div;
            acc *= mrow[D.mass_off[d] + j];
        }
        S.P[i * D.P_size + a] = acc;
    }
}

__device__ __forceinline__ void stage_table(const GmDev& D, const BatchSmem& S, int table_in_smem) {
    if (!table_in_smem) return;
    for (int c = threadIdx.x; c < D.n_lines; c += blockDim.x) S.lines[c] = D.line_off[c];
}

// Lane-stride walk over the slab: lane l of a row group visits t = l, l+tpr, ...
// tracking (a, j, k) = (prefix index, second-to-last axis, last axis).
struct Walk {
    int a, j, k;
    int qa, qj, qk;
    int Wm, Wl;
    __device__ __forceinline__ void init(const GmDev& D, int lane, int tpr) {
        Wm = D.Wm;
        Wl = D.Wl;
        const int B2 = Wm * Wl;
        a = lane / B2;
        int r = lane - a * B2;
        j = r / Wl;
        k = r - j * Wl;
        qa = tpr / B2;
        r = tpr - qa * B2;
        qj = r / Wl;
        qk = r - qj * Wl;
    }
    __device__ __forceinline__ void next() {
        k += qk;
        int c = k >= Wl;
        k -= c ? Wl : 0;
        j += qj + c;
        c = j >= Wm;
        j -= c ? Wm : 0;
        a += qa + c;
    }
    __device__ __forceinline__ int line() const { return a * Wm + j; }
};

// Sum over the tpr lanes of a row group (fixed butterfly; then warps in order).
__device__ __forceinline__ double group_reduce(double s, int tpr, const BatchSmem& S, int group_lane0_tid) {
    const int wl = tpr < 32 ? tpr : 32;
    for (int off = wl >> 1; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (tpr > 32) {
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) S.red[warp] = s;
        __syncthreads();
        if (threadIdx.x == group_lane0_tid) {
            const int w0 = group_lane0_tid >> 5, nw = tpr >> 5;
            double t = S.red[w0];
            for (int q = 1; q < nw; ++q) t += S.red[w0 + q];
            s = t;
        }
        __syncthreads();
    }
    return s;
}

// Stage (i) expansion: a warp writes one row's R products per pass, lane-strided
// (coalesced 256-byte stores).
__global__ void __launch_bounds__(kThreads) k_expand(GmDev D, long long nrows, int rb, int table_in_smem,
                                                    const double* __restrict__ mass,
                                                    double* __restrict__ probs) {
    const BatchSmem S = carve(D, rb, 0);
    (void)table_in_smem;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int mw = D.sumW + 1;
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        stage_rows(D, S, mass, nrows, b0, rb);
        __syncthreads();
        for (int i = warp; i < rb; i += nwarps) {
            const long long row = b0 + i;
            if (row >= nrows) break;
            const double* Pr = S.P + i * D.P_size;
            const double* mm = S.mass + i * mw + D.mm_off;
            const double* ml = S.mass + i * mw + D.ml_off;
            double* out = probs + row * D.R;
            Walk wk;
            wk.init(D, lane, 32);
            for (long long t = lane; t < D.R; t += 32) {
                out[t] = (Pr[wk.a] * mm[wk.j]) * ml[wk.k];
                wk.next();
            }
        }
    }
}

// Stage (ii), on the fly: row groups of tpr threads recompute each row from the
// staged masses and dot it with V (synthesis.cpp:100-104 + dot_slab :18-47).
__global__ void __launch_bounds__(kThreads) k_expect_ofa(GmDev D, long long nrows, int rb, int table_in_smem,
                                                        const double* __restrict__ mass,
                                                        const long long* __restrict__ origin,
                                                        const double* __restrict__ t0x,
                                                        const uint8_t* __restrict__ rowflag,
                                                        const double* __restrict__ V,
                                                        double* __restrict__ v_in) {
    const BatchSmem S = carve(D, rb, table_in_smem);
    stage_table(D, S, table_in_smem);
    const int tpr = D.tpr;
    const int groups = kThreads / tpr;
    const int g = threadIdx.x / tpr, lane = threadIdx.x % tpr;
    const int mw = D.sumW + 1;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const int iters = (rb + groups - 1) / groups;
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        stage_rows(D, S, mass, nrows, b0, rb);
        __syncthreads();
        for (int it = 0; it < iters; ++it) {
            const int i = g + it * groups;
            const long long row = b0 + i;
            const bool valid = i < rb && row < nrows;
            const uint8_t fl = valid ? rowflag[row] : RF_ABSORBED;
            double s = 0.0;
            if (!(fl & (RF_ABSORBED | RF_ERROR))) {
                const double* Pr = S.P + i * D.P_size;
                const double* mm = S.mass + i * mw + D.mm_off;
                const double* ml = S.mass + i * mw + D.ml_off;
                const double* vb = V + origin[row];
                const int* lines = S.lines;
                Walk wk;
                wk.init(D, lane, tpr);
#pragma unroll 4
                for (long long t = lane; t < D.R; t += tpr) {
                    const double p = (Pr[wk.a] * mm[wk.j]) * ml[wk.k];
                    const double v = __ldg(vb + lines[wk.line()] + wk.k);
                    s = fma(p, v, s);
                    wk.next();
                }
            }
            s = group_reduce(s, tpr, S, g * tpr);
            if (valid && lane == 0) {
                double r = 0.0;
                if (!(fl & (RF_ABSORBED | RF_ERROR))) r = reach ? s + t0x[row] : s;
                v_in[row] = r;
            }
        }
    }
}

// Stage (ii), stored matrix: row groups stream each row (evict-first loads)
// and gather V at the row's origin (synthesis.cpp:95-99).
__global__ void __launch_bounds__(kThreads) k_expect_matrix(GmDev D, long long row0, long long r_lo,
                                                           long long r_hi, int table_in_smem,
                                                           const double* __restrict__ probs,
                                                           const long long* __restrict__ origins,
                                                           const double* __restrict__ t0x,
                                                           const double* __restrict__ V,
                                                           double* __restrict__ v_in) {
    const BatchSmem S = carve(D, 0, table_in_smem);
    stage_table(D, S, table_in_smem);
    __syncthreads();
    const int tpr = D.tpr;
    const int groups = kThreads / tpr;
    const int g = threadIdx.x / tpr, lane = threadIdx.x % tpr;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const long long nrows = r_hi - r_lo;
    const long long total_groups = static_cast<long long>(gridDim.x) * groups;
    const long long iters = (nrows + total_groups - 1) / total_groups;
    for (long long it = 0; it < iters; ++it) {
        const long long rl = (it * gridDim.x + blockIdx.x) * groups + g; // local row
        const bool valid = rl < nrows;
        const long long r = r_lo + rl; // row inside the matrix
        bool skip = !valid;
        long long ix = 0;
        if (valid) {
            ix = (row0 + r) / (D.n_u * D.n_w);
            skip = reach && D.absorb != nullptr && D.absorb[ix];
        }
        double s = 0.0;
        if (!skip) {
            const double* pr = probs + r * D.R;
            const double* vb = V + origins[r];
            const int* lines = S.lines;
            Walk wk;
            wk.init(D, lane, tpr);
#pragma unroll 4
            for (long long t = lane; t < D.R; t += tpr) {
                const double p = __ldcs(pr + t);
                const double v = __ldg(vb + lines[wk.line()] + wk.k);
                s = fma(p, v, s);
                wk.next();
            }
        }
        s = group_reduce(s, tpr, S, g * tpr);
        if (valid && lane == 0) v_in[rl] = skip ? 0.0 : (reach ? s + t0x[r] : s);
    }
}

// min over w (strict <, ascending), then max over u (strict >, ascending):
// lowest-index ties (synthesis.cpp:112-142). L lanes per state.
template <int L>
__global__ void __launch_bounds__(kThreads) k_maxmin(GmDev D, long long x0, long long nx,
                                                    const double* __restrict__ v_in,
                                                    double* __restrict__ v_out,
                                                    uint32_t* __restrict__ pol,
                                                    uint32_t* __restrict__ wst) {
    const long long gt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long xi = gt / L;
    const int lane = static_cast<int>(gt % L);
    const bool valid = xi < nx;
    const long long ix = x0 + xi;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const bool absorbed = valid && reach && D.absorb != nullptr && D.absorb[ix];
    double best = -INFINITY;
    long long bu = 0, bw = 0;
    if (valid && !absorbed) {
        const double* base = v_in + xi * D.n_u * D.n_w;
        for (long long iu = lane; iu < D.n_u; iu += L) {
            double mn = INFINITY;
            long long mw = 0;
            const double* q = base + iu * D.n_w;
            for (long long iw = 0; iw < D.n_w; ++iw) {
                const double v = q[iw];
                if (v < mn) {
                    mn = v;
                    mw = iw;
                }
            }
            if (mn > best) {
                best = mn;
                bu = iu;
                bw = mw;
            }
        }
    }
    if (L > 1) {
        for (int off = L >> 1; off >= 1; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const long long ou = __shfl_xor_sync(0xffffffffu, bu, off);
            const long long ow = __shfl_xor_sync(0xffffffffu, bw, off);
            if (ob > best || (ob == best && ou < bu)) {
                best = ob;
                bu = ou;
                bw = ow;
            }
        }
    }
    if (!valid || lane != 0) return;
    if (absorbed) {
        v_out[xi] = 0.0;
        if (pol) pol[xi] = 0;
        if (wst) wst[xi] = 0;
        return;
    }
    v_out[xi] = smin(1.0, smax(0.0, best));
    if (pol) pol[xi] = static_cast<uint32_t>(bu);
    if (wst) wst[xi] = static_cast<uint32_t>(bw);
}

// mask_absorbing: zero stored entries whose post representative lies in T or
// in A, per-axis membership (abstraction.cpp:273-344).
__global__ void k_mask(GmDev D, long long r_lo, long long nrows, double* probs,
                       const long long* __restrict__ origins, const uint8_t* __restrict__ inT,
                       const uint8_t* __restrict__ inA, const long long* __restrict__ axis_off) {
    const long long total = nrows * D.R;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long rl = e / D.R;
        long long t = e - rl * D.R;
        long long rem = origins[r_lo + rl];
        long long o[GMD_MAXD];
        for (int d = 0; d < D.n; ++d) {
            o[d] = rem / D.xstride[d];
            rem -= o[d] * D.xstride[d];
        }
        bool zt = true, za = inA != nullptr;
        for (int d = D.n - 1; d >= 0; --d) {
            const long long j = t % D.W[d];
            t /= D.W[d];
            const long long c = axis_off[d] + o[d] + j;
            zt = zt && inT[c];
            if (inA) za = za && inA[c];
        }
        if (zt || za) probs[(r_lo + rl) * D.R + (e - rl * D.R)] = 0.0;
    }
}

} // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

BatchPlan plan_batches(const GmDev& D, bool ofa) {
    BatchPlan b;
    b.tpr = ofa ? D.tpr : 32;
    b.groups = kThreads / b.tpr;
    const size_t per_row = static_cast<size_t>(D.sumW + 1 + D.P_size) * sizeof(double);
    const size_t fixed = (kThreads / 32) * sizeof(double);
    const size_t table = static_cast<size_t>(D.n_lines) * sizeof(int);
    const size_t soft = 48 * 1024, hard = 200 * 1024;
    // rows per batch: aim for >= 2 rows per group so each CTA has work while
    // staging, within a soft budget that allows several CTAs per SM.
    size_t budget = soft;
    b.table_in_smem = ofa && (fixed + table + per_row * b.groups <= soft) ? 1 : 0;
    size_t avail = budget - fixed - (b.table_in_smem ? table : 0);
    long long rb = per_row ? static_cast<long long>(avail / per_row) : kThreads;
    if (rb < b.groups) {
        budget = hard;
        avail = budget - fixed - (b.table_in_smem ? table : 0);
        rb = static_cast<long long>(avail / per_row);
    }
    if (rb < 1) throw std::runtime_error("row too wide for the device batch layout (" +
                                         std::to_string(per_row) + " bytes of shared memory per row)");
    rb = std::min<long long>(rb, kThreads);
    if (rb >= b.groups) rb -= rb % b.groups;
    b.rb = static_cast<int>(rb);
    b.smem = fixed + per_row * static_cast<size_t>(b.rb) + (b.table_in_smem ? table : 0);
    return b;
}

void absorb_flags(const GmDev& D, uint8_t* d_flags, cudaStream_t s) {
    k_absorb<<<grid_for(D.n_x, kThreads), kThreads, 0, s>>>(D, d_flags);
    check_launch("absorb_flags");
}

void zero_absorbing(const GmDev& D, double* d_v, cudaStream_t s) {
    if (D.spec_kind == GM_SPEC_SAFETY || !D.absorb) return;
    k_zero_absorbing<<<grid_for(D.n_x, kThreads), kThreads, 0, s>>>(D, d_v);
    check_launch("zero_absorbing");
}

void prologue(const GmDev& D, long long row0, long long nrows, int flags, long long* origin_out,
              double* t0x_out, uint8_t* rowflag_out, double* mass_out,
              unsigned long long* d_err_row, cudaStream_t s) {
    if (nrows <= 0) return;
    const size_t smem = ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16 + D.n_lits * sizeof(double);
    if (smem > 48 * 1024) {
        static bool set = false;
        if (!set) {
            cudaFuncSetAttribute(k_prologue, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            set = true;
        }
    }
    k_prologue<<<grid_for(nrows, kThreads), kThreads, smem, s>>>(D, row0, nrows, flags, origin_out, t0x_out,
                                                                rowflag_out, mass_out, d_err_row);
    check_launch("prologue");
}

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <class K>
static int resident_grid(K kernel, size_t smem, long long batches) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    long long g = static_cast<long long>(per_sm) * num_sms();
    if (g > batches) g = batches;
    return static_cast<int>(std::max<long long>(g, 1));
}

void expand(const GmDev& D, long long nrows, const double* mass, double* probs_out, cudaStream_t s) {
    if (nrows <= 0) return;
    BatchPlan b = plan_batches(D, false);
    b.smem -= b.table_in_smem ? static_cast<size_t>(D.n_lines) * sizeof(int) : 0;
    if (b.smem > 48 * 1024) cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b.smem);
    const long long batches = (nrows + b.rb - 1) / b.rb;
    k_expand<<<resident_grid(k_expand, b.smem, batches), kThreads, b.smem, s>>>(D, nrows, b.rb, 0, mass, probs_out);
    check_launch("expand");
}

void expect_ofa(const GmDev& D, long long nrows, const double* mass, const long long* origin,
                const double* t0x, const uint8_t* rowflag, const double* V, double* v_in,
                cudaStream_t s) {
    if (nrows <= 0) return;
    const BatchPlan b = plan_batches(D, true);
    if (b.smem > 48 * 1024)
        cudaFuncSetAttribute(k_expect_ofa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b.smem);
    const long long batches = (nrows + b.rb - 1) / b.rb;
    k_expect_ofa<<<resident_grid(k_expect_ofa, b.smem, batches), kThreads, b.smem, s>>>(
        D, nrows, b.rb, b.table_in_smem, mass, origin, t0x, rowflag, V, v_in);
    check_launch("expect_ofa");
}

void expect_matrix(const GmDev& D, long long row0, long long r_lo, long long r_hi,
                   const double* probs, const long long* origins, const double* t0x,
                   const double* V, double* v_in, cudaStream_t s) {
    if (r_hi <= r_lo) return;
    const size_t table = static_cast<size_t>(D.n_lines) * sizeof(int);
    const int in_smem = table <= 32 * 1024 ? 1 : 0;
    const size_t smem = (kThreads / 32) * sizeof(double) + (in_smem ? table : 0);
    const int groups = kThreads / D.tpr;
    const long long blocks_needed = (r_hi - r_lo + groups - 1) / groups;
    k_expect_matrix<<<resident_grid(k_expect_matrix, smem, blocks_needed), kThreads, smem, s>>>(
        D, row0, r_lo, r_hi, in_smem, probs, origins, t0x, V, v_in);
    check_launch("expect_matrix");
}

void maxmin(const GmDev& D, long long x0, long long nx, const double* v_in, double* v_out,
            uint32_t* pol, uint32_t* wst, cudaStream_t s) {
    if (nx <= 0) return;
    const long long nuw = D.n_u * D.n_w;
    if (nuw <= 8) {
        k_maxmin<1><<<grid_for(nx, kThreads), kThreads, 0, s>>>(D, x0, nx, v_in, v_out, pol, wst);
    } else {
        k_maxmin<32><<<grid_for(nx * 32, kThreads), kThreads, 0, s>>>(D, x0, nx, v_in, v_out, pol, wst);
    }
    check_launch("maxmin");
}

void mask(const GmDev& D, long long r_lo, long long nrows, double* probs, const long long* origins,
          const uint8_t* inT, const uint8_t* inA, const long long* axis_off, cudaStream_t s) {
    if (nrows <= 0) return;
    const long long total = nrows * D.R;
    int blocks = grid_for(total, kThreads);
    blocks = std::min(blocks, num_sms() * 8);
    k_mask<<<blocks, kThreads, 0, s>>>(D, r_lo, nrows, probs, origins, inT, inA, axis_off);
    check_launch("mask");
}

} // namespace gmk
