// OFA consumer device code (stage ii, on the fly: synthesis.cpp:100-104 + dot_slab
// :18-47) and the shared-memory row batches it shares with the single-role build.
// Included by gm_kernels.cu (ahead-of-time kernels) and compiled at run time by
// NVRTC with GM_OFA_SHAPE (gm_jit.cpp): the consumer specialised to one model's
// row shape (k_expect_ofa_shape), same terms, same fma order, same bits.
#pragma once

// ---------------------------------------------------------------------------
// Row batches in shared memory (expand / expect_ofa)
//
// A row's probabilities factor as p(L, k) = Q[L] * ml[k] with L the slab line
// (all axes but the last), Q[L] = P[a] * mm[j] the line prefix, P[a] the prefix
// product over the leading axes (1.0*m0[j0]*m1[j1]*..., abstraction.cpp:150-159)
// and ml the last axis' masses. Q is staged per row when it fits (TAB_Q);
// otherwise P is staged and Q[L] is formed per term (TAB_P). Both give the
// same bits: the rounding sequence is identical.
//
// Shared memory is one double array addressed by integer offsets (so every
// access compiles to LDS with a register offset):
//   [0, rb*mw)            per-axis masses, slot sumW of each row = 1.0
//   [offP, +rb*P_size)    prefix products over the leading axes
//   [offQ, +rb*n_lines)   line prefixes (TAB_Q)
//   [offR, +8)            cross-warp partial sums
//   ints after that       slab line offsets (when staged)
// ---------------------------------------------------------------------------

enum { TAB_Q = 0, TAB_P = 1 };

struct Layout {
    int mw, offP, offQ, offR, offL; // offL in ints
    __device__ __forceinline__ Layout(const GmDev& D, int rb, int tab) {
        mw = D.sumW + 1;
        offP = rb * mw;
        offQ = offP + rb * D.P_size;
        offR = offQ + (tab == TAB_Q ? rb * D.n_lines : 0);
        offL = 2 * (offR + kThreads / 32);
    }
};

__device__ __forceinline__ const int* sm_ints() { return reinterpret_cast<const int*>(g_sm); }

// Builds the prefix tables P (and Q) from the staged masses of rb rows.
__device__ __forceinline__ void stage_tables(const GmDev& D, const Layout& Y, int rb, int tab) {
    const int mw = Y.mw;
    if (D.s_axes == 0) {
        for (int i = threadIdx.x; i < rb; i += blockDim.x) g_sm[Y.offP + i] = 1.0;
    } else {
        // one item per (row, run of the last prefix axis): the prefix over the other
        // axes once, then W_last products -- the association of prefix_product
        const int last = D.s_axes - 1, wl = D.W[last];
        const int nb = D.P_size / wl;
        for (int c = threadIdx.x; c < rb * nb; c += blockDim.x) {
            const int i = c / nb, b = c - i * nb;
            const double* m = g_sm + i * mw;
            double acc = 1.0;
            int rem = b * wl;
            for (int d = 0; d < last; ++d) {
                const int j = D.div_Ps[d].div(rem);
                rem -= j * D.Ps[d];
                acc *= m[D.mass_off[d] + j];
            }
            double* P = g_sm + Y.offP + i * D.P_size + b * wl;
            const double* ml = m + D.mass_off[last];
            for (int j = 0; j < wl; ++j) P[j] = acc * ml[j];
        }
    }
    if (tab == TAB_Q) {
        __syncthreads();
        const int nl = D.n_lines;
        if (nl <= static_cast<int>(blockDim.x)) {
            // Q[L] = P[a] * mm[j], L = a*Wm + j: each thread owns one line L of rows
            // ri, ri+rp, ... (rp = rows per pass), so (a, j) are fixed per thread
            const int rp = D.div_lines.div(blockDim.x);
            const int ri = D.div_lines.div(threadIdx.x), L = threadIdx.x - ri * nl;
            if (ri < rp) {
                const int a = D.div_Wm.div(L), j = L - a * D.Wm;
                for (int i = ri; i < rb; i += rp)
                    g_sm[Y.offQ + i * nl + L] = g_sm[Y.offP + i * D.P_size + a] * g_sm[i * mw + D.mm_off + j];
            }
            return;
        }
        // wide rows: one item per (row, prefix entry a): its Wm lines Q[a*Wm + j]
        for (int c = threadIdx.x; c < rb * D.P_size; c += blockDim.x) {
            const int i = D.div_P.div(c), a = c - i * D.P_size;
            const double pa = g_sm[Y.offP + c];
            const double* mm = g_sm + i * mw + D.mm_off;
            double* q = g_sm + Y.offQ + i * D.n_lines + a * D.Wm;
            for (int j = 0; j < D.Wm; ++j) q[j] = pa * mm[j];
        }
    }
}

// Loads the masses of rows [b0, b0+rb) (SoA, pitch nrows) and builds P (and Q).
__device__ __forceinline__ void stage_rows(const GmDev& D, const Layout& Y, const double* __restrict__ mass,
                                           long long nrows, long long b0, int rb, GmFastDiv div_rb, int tab) {
    const int mw = Y.mw;
    // all threads load in parallel; consecutive threads -> consecutive rows of a plane
    for (int c = threadIdx.x; c < rb * mw; c += blockDim.x) {
        const int q = div_rb.div(c), i = c - q * rb;
        double v = 1.0;
        if (q < D.sumW && b0 + i < nrows) v = mass[static_cast<long long>(q) * nrows + b0 + i];
        g_sm[i * mw + q] = v;
    }
    __syncthreads();
    stage_tables(D, Y, rb, tab);
}

// Sum over the tpr lanes of a row group: fixed xor butterfly inside the warp,
// then the group's warps in increasing order. Identical in every kernel.
__device__ __forceinline__ double group_reduce(double s, int tpr, int offR, int group_lane0_tid) {
    const int wl = tpr < 32 ? tpr : 32;
    for (int off = wl >> 1; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (tpr > 32) { // per-group named barrier: groups of a CTA do not wait for each other
        const int warp = threadIdx.x >> 5;
        const int bar = 1 + group_lane0_tid / tpr;
        if ((threadIdx.x & 31) == 0) g_sm[offR + warp] = s;
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(tpr) : "memory");
        if (threadIdx.x == group_lane0_tid) {
            const int w0 = group_lane0_tid >> 5, nw = tpr >> 5;
            double t = g_sm[offR + w0];
            for (int q = 1; q < nw; ++q) t += g_sm[offR + w0 + q];
            s = t;
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(tpr) : "memory");
    }
    return s;
}

// V gather at vb[off]: one mad.wide.s32 per access (keeps the 64-bit row base
// in registers instead of re-extending origin + offset per term).
__device__ __forceinline__ double ldg_at(const double* vb, int off) {
    const double* a;
    asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(a) : "r"(off), "l"(vb));
    return __ldg(a);
}

// One row's dot product in the canonical order: lane-strided terms accumulated
// with fma in increasing t (padding slots contribute fma(0,0,s) == s).
// MODE 0: stored row; MODE 1: recompute from Q; MODE 2: recompute from P.
// Term sources: stored row `prow` (global); Q row at g_sm[qo]; P row at g_sm[po];
// masses mm at g_sm[mmo], ml at g_sm[mlo]; line table `lines` (smem ints or global).
// LS: line offsets from the global table (0), from the table staged in shared
// memory (1), or (MODE 2 only) from a shared table of the leading-prefix offsets
// plus j * (stride of the middle axis) (2): line_off[a*Wm + j] == pre[a] + j*sM.
template <int MODE, int U, int LS>
__device__ __forceinline__ double row_dot(const GmDev& D, int lane, int tpr, const double* __restrict__ prow,
                                          int qo, int po, int mmo, int mlo, const double* __restrict__ vb,
                                          const int* __restrict__ gl, int lo, int sM = 0) {
    static_assert(LS != 2 || MODE == 2, "prefix offset table needs the (a, j, k) walk");
    const int R = static_cast<int>(D.R);
    const int n_it = lane < R ? (R - lane + tpr - 1) / tpr : 0;
    Walk w;
    w.init(D, lane, tpr);
    const double* pp = prow + lane;
    int pi = qo + lane; // MODE 3: stored row staged in shared memory at g_sm[qo]
    const int* si = sm_ints();
    double s = 0.0;
    auto term = [&](double& p, double& v) {
        if (MODE == 0) p = __ldcs(pp);
        else if (MODE == 1) p = g_sm[qo + w.L] * g_sm[mlo + w.k];
        else if (MODE == 2) p = (g_sm[po + w.a] * g_sm[mmo + w.j]) * g_sm[mlo + w.k];
        else p = g_sm[pi];
        const int off = (LS == 2 ? si[lo + w.a] + w.j * sM : (LS == 1 ? si[lo + w.L] : __ldg(gl + w.L))) + w.k;
        v = ldg_at(vb, off);
        pp += tpr;
        pi += tpr;
        w.template next<MODE == 2>();
    };
    const int n_full = n_it - n_it % U;
    for (int b = 0; b < n_full; b += U) {
        double p[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) term(p[u], v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
    }
    const int rem = n_it - n_full;
    if (rem) {
        double p[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = 0.0;
            v[u] = 0.0;
            if (u < rem) term(p[u], v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
    }
    return s;
}

// OFA row dot with the last-axis cell hoisted out of the term loop (same terms,
// same fma order as row_dot<MODE, U, LS>): a lane's last-axis cell advances by
// tpr mod Wl per term, so it is periodic with period Wl / gcd(tpr mod Wl, Wl);
// when U is a multiple of that period, slot u of every U-term block always sees
// the same cell k_u. ml[k_u], k_u and the carry into the line index after slot u
// are loaded once per row into registers: one shared load and the k walk less
// per term (the kernel is bound by the L1/shared pipe).
template <int MODE, int U, int LS>
__device__ __forceinline__ double row_dot_pk(const GmDev& D, int lane, int tpr, int qo, int po, int mmo, int mlo,
                                             const double* __restrict__ vb, const int* __restrict__ gl, int lo,
                                             int sM) {
    static_assert(MODE == 1 || MODE == 2, "recomputed rows only");
    static_assert(LS != 2 || MODE == 2, "prefix offset table needs the (a, j, k) walk");
    const int R = static_cast<int>(D.R);
    const int n_it = lane < R ? (R - lane + tpr - 1) / tpr : 0;
    Walk w;
    w.init(D, lane, tpr);
    double ml[U];
    int kk[U], cc[U];
    {
        int k = w.k;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            kk[u] = k;
            ml[u] = g_sm[mlo + k];
            k += w.qk;
            cc[u] = k >= w.Wl;
            k -= cc[u] ? w.Wl : 0;
        }
    }
    const int* si = sm_ints();
    double s = 0.0;
    auto term = [&](int u, double& p, double& v) {
        const double lead = MODE == 1 ? g_sm[qo + w.L] : g_sm[po + w.a] * g_sm[mmo + w.j];
        p = lead * ml[u];
        const int off = (LS == 2 ? si[lo + w.a] + w.j * sM : (LS == 1 ? si[lo + w.L] : __ldg(gl + w.L))) + kk[u];
        v = ldg_at(vb, off);
        w.L += w.qL + cc[u];
        if (MODE == 2) {
            w.j += w.qj + cc[u];
            const int c2 = w.j >= w.Wm;
            w.j -= c2 ? w.Wm : 0;
            w.a += w.qa + c2;
        }
    };
    // software-pipelined by one block: the U gathers of block b+1 are issued
    // before the fma chain of block b (ptxas otherwise places each gather right
    // before its fma at some U: one load in flight)
    const int n_full = n_it - n_it % U;
    double pc[U], vc[U];
    if (n_full > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) term(u, pc[u], vc[u]);
    }
    for (int b = U; b < n_full; b += U) {
        double pn[U], vn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) term(u, pn[u], vn[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(pc[u], vc[u], s);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pc[u] = pn[u];
            vc[u] = vn[u];
        }
    }
    if (n_full > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(pc[u], vc[u], s);
    }
    const int rem = n_it - n_full;
    if (rem) {
        double p[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = 0.0;
            v[u] = 0.0;
            if (u < rem) term(u, p[u], v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
    }
    return s;
}

// Stage (ii), on the fly (synthesis.cpp:100-104 + dot_slab :18-47): row groups
// of tpr threads recompute each row from the staged masses and dot it with V.
template <int TAB, int LS, int U, bool PK>
__device__ __forceinline__ void expect_ofa_body(GmDev D, long long nrows, int rb, GmFastDiv div_rb,
                                                        const double* __restrict__ mass,
                                                        const long long* __restrict__ origin,
                                                        const double* __restrict__ t0x,
                                                        const uint8_t* __restrict__ rowflag,
                                                        const double* __restrict__ V,
                                                        double* __restrict__ v_in) {
    const Layout Y(D, rb, TAB);
    GM_CHECK(static_cast<unsigned>(8 * Y.offR + 8 * (kThreads / 32)) <= gm_dyn_smem_bytes());
    GM_CHECK(LS != 1 || static_cast<unsigned>(4 * (Y.offL + D.n_lines)) <= gm_dyn_smem_bytes());
    GM_CHECK(LS != 2 || static_cast<unsigned>(4 * (Y.offL + D.P_size)) <= gm_dyn_smem_bytes());
    if (LS == 1) {
        int* si = reinterpret_cast<int*>(g_sm);
        for (int c = threadIdx.x; c < D.n_lines; c += blockDim.x) si[Y.offL + c] = D.line_off[c];
    } else if (LS == 2) { // offsets of the leading prefixes a (j = 0 lines)
        int* si = reinterpret_cast<int*>(g_sm);
        for (int c = threadIdx.x; c < D.P_size; c += blockDim.x) si[Y.offL + c] = D.line_off[c * D.Wm];
    }
    const int sM = (LS == 2 && D.Wm > 1) ? D.line_off[1] - D.line_off[0] : 0;
    const int tpr = D.tpr;
    const int groups = kThreads / tpr;
    const int g = threadIdx.x / tpr, lane = threadIdx.x - g * tpr;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const int iters = (rb + groups - 1) / groups;
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        stage_rows(D, Y, mass, nrows, b0, rb, div_rb, TAB);
        __syncthreads();
        for (int it = 0; it < iters; ++it) {
            const int i = g + it * groups;
            const long long row = b0 + i;
            const bool valid = i < rb && row < nrows;
            const uint8_t fl = valid ? rowflag[row] : RF_ABSORBED;
            double s = 0.0;
            if (!(fl & (RF_ABSORBED | RF_ERROR))) {
                GM_CHECK_SLAB(D, origin[row]);
                if (PK)
                    s = row_dot_pk<TAB == TAB_Q ? 1 : 2, U, LS>(D, lane, tpr, Y.offQ + i * D.n_lines,
                                                                Y.offP + i * D.P_size, i * Y.mw + D.mm_off,
                                                                i * Y.mw + D.ml_off, V + origin[row], D.line_off,
                                                                Y.offL, sM);
                else
                    s = row_dot<TAB == TAB_Q ? 1 : 2, U, LS>(D, lane, tpr, nullptr, Y.offQ + i * D.n_lines,
                                                             Y.offP + i * D.P_size, i * Y.mw + D.mm_off,
                                                             i * Y.mw + D.ml_off, V + origin[row], D.line_off, Y.offL,
                                                             sM);
            }
            s = group_reduce(s, tpr, Y.offR, g * tpr);
            if (valid && lane == 0) {
                double r = 0.0;
                if (!(fl & (RF_ABSORBED | RF_ERROR))) r = reach ? s + t0x[row] : s;
                v_in[row] = r;
            }
        }
    }
}

// separate entry points: the pipelined hoisted-cell body gets a 2-CTA register cap
// (128: no spills; the 3-CTA cap of 80 spilled 36-240 B and measured 3-7% slower
// on C4 / C4' / bmw7_mid, scripts/r02_pk_minb.sh), the plain body keeps the
// compiler's own choice (48 registers)
template <int TAB, int LS, int U = 4>
__global__ void __launch_bounds__(kThreads) k_expect_ofa(GmDev D, long long nrows, int rb, GmFastDiv div_rb,
                                                        const double* __restrict__ mass,
                                                        const long long* __restrict__ origin,
                                                        const double* __restrict__ t0x,
                                                        const uint8_t* __restrict__ rowflag,
                                                        const double* __restrict__ V,
                                                        double* __restrict__ v_in) {
    expect_ofa_body<TAB, LS, U, false>(D, nrows, rb, div_rb, mass, origin, t0x, rowflag, V, v_in);
}
#ifndef GM_OFA_PK_MINB
#define GM_OFA_PK_MINB 2
#endif
template <int TAB, int LS, int U>
__global__ void __launch_bounds__(kThreads, GM_OFA_PK_MINB) k_expect_ofa_pk(GmDev D, long long nrows, int rb, GmFastDiv div_rb,
                                                              const double* __restrict__ mass,
                                                              const long long* __restrict__ origin,
                                                              const double* __restrict__ t0x,
                                                              const uint8_t* __restrict__ rowflag,
                                                              const double* __restrict__ V,
                                                              double* __restrict__ v_in) {
    expect_ofa_body<TAB, LS, U, true>(D, nrows, rb, div_rb, mass, origin, t0x, rowflag, V, v_in);
}


#ifdef GM_OFA_SHAPE
// ---------------------------------------------------------------------------
// The OFA consumer compiled at run time for one model's row shape (NVRTC,
// gm_jit.cpp ofa_shape_defines): tpr, W_last, R, n_lines and the period PER of
// a lane's last-axis cell (tpr*PER ≡ 0 mod W_last) are constants. Lane ℓ's term
// i = S + PER*B is t = ℓ + tpr*i: line L(S) + DL*B, cell k(S), DL = tpr*PER/W_last.
// So the lane's line-table and Q addresses are registers plus compile-time
// offsets, its PER last-axis masses are registers per row, and its V bases
// (origin + k(S)) are PER pointers per row: one term is LDS (Q), LDS (line
// offset), IMAD.WIDE, LDG (V), DMUL (Q*ml, the stored product), DFMA, in
// increasing t — row_dot<1, U, 1>'s terms in row_dot's order, the same bits.
// ---------------------------------------------------------------------------
template <int OFF>
__device__ __forceinline__ double ofa_lds_f64(unsigned addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ int ofa_lds_s32(unsigned addr) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFF));
    return v;
}

constexpr int kOfaTpr = GM_OFA_TPR, kOfaWl = GM_OFA_WL, kOfaR = GM_OFA_R, kOfaNl = GM_OFA_NL, kOfaPer = GM_OFA_PER;
constexpr int kOfaDl = kOfaTpr * kOfaPer / kOfaWl;
constexpr int kOfaNit = (kOfaR + kOfaTpr - 1) / kOfaTpr;

template <int I>
struct OfaDot {
    static __device__ __forceinline__ double run(double s, const unsigned* qa, const unsigned* la, const double* ml,
                                                 const double* const* vb, int lane) {
        constexpr int S = I % kOfaPer, B = I / kOfaPer;
        if constexpr ((I + 1) * kOfaTpr <= kOfaR) { // every lane has term I
            const double p = ofa_lds_f64<8 * kOfaDl * B>(qa[S]) * ml[S];
            s = fma(p, ldg_at(vb[S], ofa_lds_s32<4 * kOfaDl * B>(la[S])), s);
        } else if (lane + I * kOfaTpr < kOfaR) {
            const double p = ofa_lds_f64<8 * kOfaDl * B>(qa[S]) * ml[S];
            s = fma(p, ldg_at(vb[S], ofa_lds_s32<4 * kOfaDl * B>(la[S])), s);
        }
        if constexpr (I + 1 < kOfaNit) return OfaDot<I + 1>::run(s, qa, la, ml, vb, lane);
        return s;
    }
};

// Two rows per lane group in flight (GM_OFA_ROWS 2): two independent fma chains, each
// in its row's canonical order, sharing the line-offset loads.
template <int I>
struct OfaDot2 {
    static __device__ __forceinline__ void run(double& sA, double& sB, const unsigned* qA, const unsigned* qB,
                                               const unsigned* la, const double* mA, const double* mB,
                                               const double* const* vA, const double* const* vB, int lane) {
        constexpr int S = I % kOfaPer, B = I / kOfaPer;
        if ((I + 1) * kOfaTpr <= kOfaR || lane + I * kOfaTpr < kOfaR) {
            const int off = ofa_lds_s32<4 * kOfaDl * B>(la[S]);
            const double pA = ofa_lds_f64<8 * kOfaDl * B>(qA[S]) * mA[S];
            const double pB = ofa_lds_f64<8 * kOfaDl * B>(qB[S]) * mB[S];
            const double va = ldg_at(vA[S], off), vb = ldg_at(vB[S], off);
            sA = fma(pA, va, sA);
            sB = fma(pB, vb, sB);
        }
        if constexpr (I + 1 < kOfaNit) OfaDot2<I + 1>::run(sA, sB, qA, qB, la, mA, mB, vA, vB, lane);
    }
};

#ifndef GM_OFA_ROWS
#define GM_OFA_ROWS 1
#endif

extern "C" __global__ void __launch_bounds__(kThreads) k_expect_ofa_shape(GmDev D, long long nrows, int rb,
                                                                        GmFastDiv div_rb,
                                                                        const double* __restrict__ mass,
                                                                        const long long* __restrict__ origin,
                                                                        const double* __restrict__ t0x,
                                                                        const uint8_t* __restrict__ rowflag,
                                                                        const double* __restrict__ V,
                                                                        double* __restrict__ v_in) {
    const Layout Y(D, rb, TAB_Q);
    GM_CHECK(D.tpr == kOfaTpr && D.Wl == kOfaWl && D.R == kOfaR && D.n_lines == kOfaNl);
    GM_CHECK(static_cast<unsigned>(4 * (Y.offL + kOfaNl)) <= gm_dyn_smem_bytes());
    int* si = reinterpret_cast<int*>(g_sm);
    for (int c = threadIdx.x; c < kOfaNl; c += blockDim.x) si[Y.offL + c] = D.line_off[c];
    constexpr int groups = kThreads / kOfaTpr;
    const int g = threadIdx.x / kOfaTpr, lane = threadIdx.x - g * kOfaTpr;
    const unsigned sm0 = static_cast<unsigned>(__cvta_generic_to_shared(g_sm));
    int Ls[kOfaPer], ks[kOfaPer];
    unsigned la[kOfaPer];
#pragma unroll
    for (int S = 0; S < kOfaPer; ++S) {
        const int t = lane + kOfaTpr * S;
        Ls[S] = t / kOfaWl;
        ks[S] = t - Ls[S] * kOfaWl;
        la[S] = sm0 + 4u * static_cast<unsigned>(Y.offL + Ls[S]);
    }
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const int iters = (rb + groups - 1) / groups;
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        stage_rows(D, Y, mass, nrows, b0, rb, div_rb, TAB_Q);
        __syncthreads();
#if GM_OFA_ROWS == 2
        for (int it = 0; it < (rb + 2 * groups - 1) / (2 * groups); ++it) {
            const int iA = g + 2 * it * groups, iB = iA + groups;
            const long long rA = b0 + iA, rB = b0 + iB;
            const bool validA = iA < rb && rA < nrows, validB = iB < rb && rB < nrows;
            const uint8_t fA = validA ? rowflag[rA] : RF_ABSORBED, fB = validB ? rowflag[rB] : RF_ABSORBED;
            const bool liveA = !(fA & (RF_ABSORBED | RF_ERROR)), liveB = !(fB & (RF_ABSORBED | RF_ERROR));
            double sA = 0.0, sB = 0.0;
            if (liveA || liveB) {
                // a row without terms borrows the other row's operands (its sum is discarded)
                const int jA = liveA ? iA : iB, jB = liveB ? iB : iA;
                const long long oA = origin[b0 + jA], oB = origin[b0 + jB];
                GM_CHECK_SLAB(D, oA);
                GM_CHECK_SLAB(D, oB);
                unsigned qA[kOfaPer], qB[kOfaPer];
                double mA[kOfaPer], mB[kOfaPer];
                const double *vA[kOfaPer], *vB[kOfaPer];
#pragma unroll
                for (int S = 0; S < kOfaPer; ++S) {
                    qA[S] = sm0 + 8u * static_cast<unsigned>(Y.offQ + jA * kOfaNl + Ls[S]);
                    qB[S] = sm0 + 8u * static_cast<unsigned>(Y.offQ + jB * kOfaNl + Ls[S]);
                    mA[S] = g_sm[jA * Y.mw + D.ml_off + ks[S]];
                    mB[S] = g_sm[jB * Y.mw + D.ml_off + ks[S]];
                    vA[S] = V + oA + ks[S];
                    vB[S] = V + oB + ks[S];
                }
                OfaDot2<0>::run(sA, sB, qA, qB, la, mA, mB, vA, vB, lane);
            }
            sA = group_reduce(sA, kOfaTpr, Y.offR, g * kOfaTpr);
            sB = group_reduce(sB, kOfaTpr, Y.offR, g * kOfaTpr);
            if (lane == 0) {
                if (validA) v_in[rA] = liveA ? (reach ? sA + t0x[rA] : sA) : 0.0;
                if (validB) v_in[rB] = liveB ? (reach ? sB + t0x[rB] : sB) : 0.0;
            }
        }
        continue;
#endif
        for (int it = 0; it < iters; ++it) {
            const int i = g + it * groups;
            const long long row = b0 + i;
            const bool valid = i < rb && row < nrows;
            const uint8_t fl = valid ? rowflag[row] : RF_ABSORBED;
            double s = 0.0;
            if (!(fl & (RF_ABSORBED | RF_ERROR))) {
                GM_CHECK_SLAB(D, origin[row]);
                const int qo = Y.offQ + i * kOfaNl, mlo = i * Y.mw + D.ml_off;
                const double* vrow = V + origin[row];
                unsigned qa[kOfaPer];
                double ml[kOfaPer];
                const double* vb[kOfaPer];
#pragma unroll
                for (int S = 0; S < kOfaPer; ++S) {
                    qa[S] = sm0 + 8u * static_cast<unsigned>(qo + Ls[S]);
                    ml[S] = g_sm[mlo + ks[S]];
                    vb[S] = vrow + ks[S];
                }
                s = OfaDot<0>::run(0.0, qa, la, ml, vb, lane);
            }
            s = group_reduce(s, kOfaTpr, Y.offR, g * kOfaTpr);
            if (valid && lane == 0) {
                double r = 0.0;
                if (!(fl & (RF_ABSORBED | RF_ERROR))) r = reach ? s + t0x[row] : s;
                v_in[row] = r;
            }
        }
    }
}

// The same consumer with each row's line prefix and the line's V offset packed in one
// 16-byte shared-memory entry (Q[L] as f64, line_off[L] as s32): one LDS.128 per term
// instead of an LDS.64 and an LDS.32. Shared layout in doubles: masses [rb][mw] | P
// [rb][P_size] | QO [rb][n_lines][2] | group partials [8].
template <int OFF>
__device__ __forceinline__ void ofa_lds_qo(unsigned addr, double& q, int& off) {
    unsigned long long a, b;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2+%3];" : "=l"(a), "=l"(b) : "r"(addr), "n"(OFF));
    q = __longlong_as_double(static_cast<long long>(a));
    off = static_cast<int>(b);
}

template <int I>
struct OfaDotQO {
    static __device__ __forceinline__ double run(double s, const unsigned* qa, const double* ml,
                                                 const double* const* vb, int lane) {
        constexpr int S = I % kOfaPer, B = I / kOfaPer;
        if ((I + 1) * kOfaTpr <= kOfaR || lane + I * kOfaTpr < kOfaR) {
            double q;
            int off;
            ofa_lds_qo<16 * kOfaDl * B>(qa[S], q, off);
            s = fma(q * ml[S], ldg_at(vb[S], off), s);
        }
        if constexpr (I + 1 < kOfaNit) return OfaDotQO<I + 1>::run(s, qa, ml, vb, lane);
        return s;
    }
};

extern "C" __global__ void __launch_bounds__(kThreads) k_expect_ofa_packed(GmDev D, long long nrows, int rb,
                                                                         GmFastDiv div_rb,
                                                                         const double* __restrict__ mass,
                                                                         const long long* __restrict__ origin,
                                                                         const double* __restrict__ t0x,
                                                                         const uint8_t* __restrict__ rowflag,
                                                                         const double* __restrict__ V,
                                                                         double* __restrict__ v_in) {
    const Layout Y(D, rb, TAB_P); // masses and P as the P-table consumers lay them out
    const int offQO = (Y.offQ + 1) & ~1, offR = offQO + 2 * rb * kOfaNl; // 16-byte entries
    GM_CHECK(D.tpr == kOfaTpr && D.Wl == kOfaWl && D.R == kOfaR && D.n_lines == kOfaNl);
    GM_CHECK(static_cast<unsigned>(8 * (offR + kThreads / 32)) <= gm_dyn_smem_bytes());
    constexpr int groups = kThreads / kOfaTpr;
    const int g = threadIdx.x / kOfaTpr, lane = threadIdx.x - g * kOfaTpr;
    const unsigned sm0 = static_cast<unsigned>(__cvta_generic_to_shared(g_sm));
    int Ls[kOfaPer], ks[kOfaPer];
#pragma unroll
    for (int S = 0; S < kOfaPer; ++S) {
        const int t = lane + kOfaTpr * S;
        Ls[S] = t / kOfaWl;
        ks[S] = t - Ls[S] * kOfaWl;
    }
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const int iters = (rb + groups - 1) / groups;
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        stage_rows(D, Y, mass, nrows, b0, rb, div_rb, TAB_P); // masses + P
        __syncthreads();
        // Q[L] = P[a] * mm[j] (stage_tables' product) next to the line's V offset
        for (int c = threadIdx.x; c < rb * kOfaNl; c += blockDim.x) {
            const int i = c / kOfaNl, L = c - i * kOfaNl;
            const int a = D.div_Wm.div(L), j = L - a * D.Wm;
            double* e = g_sm + offQO + 2 * c;
            e[0] = g_sm[Y.offP + i * D.P_size + a] * g_sm[i * Y.mw + D.mm_off + j];
            e[1] = __longlong_as_double(static_cast<long long>(D.line_off[L]));
        }
        __syncthreads();
        for (int it = 0; it < iters; ++it) {
            const int i = g + it * groups;
            const long long row = b0 + i;
            const bool valid = i < rb && row < nrows;
            const uint8_t fl = valid ? rowflag[row] : RF_ABSORBED;
            double s = 0.0;
            if (!(fl & (RF_ABSORBED | RF_ERROR))) {
                GM_CHECK_SLAB(D, origin[row]);
                const int mlo = i * Y.mw + D.ml_off;
                const double* vrow = V + origin[row];
                unsigned qa[kOfaPer];
                double ml[kOfaPer];
                const double* vb[kOfaPer];
#pragma unroll
                for (int S = 0; S < kOfaPer; ++S) {
                    qa[S] = sm0 + 16u * static_cast<unsigned>(offQO / 2 + i * kOfaNl + Ls[S]);
                    ml[S] = g_sm[mlo + ks[S]];
                    vb[S] = vrow + ks[S];
                }
                s = OfaDotQO<0>::run(0.0, qa, ml, vb, lane);
            }
            s = group_reduce(s, kOfaTpr, offR, g * kOfaTpr);
            if (valid && lane == 0) {
                double r = 0.0;
                if (!(fl & (RF_ABSORBED | RF_ERROR))) r = reach ? s + t0x[row] : s;
                v_in[row] = r;
            }
        }
    }
}

// The shape kernel with each lane group owning one row slot and walking its own rows:
// masses, prefix products and line prefixes of a row are staged by the group's tpr
// threads under the group's named barrier, so the groups of a CTA never wait for
// each other (the CTA-wide batch barriers of k_expect_ofa_shape are the kernel's
// largest stall after the gathers). Same tables, same terms, same bits.
extern "C" __global__ void __launch_bounds__(kThreads) k_expect_ofa_group(GmDev D, long long nrows, int rb,
                                                                        GmFastDiv div_rb,
                                                                        const double* __restrict__ mass,
                                                                        const long long* __restrict__ origin,
                                                                        const double* __restrict__ t0x,
                                                                        const uint8_t* __restrict__ rowflag,
                                                                        const double* __restrict__ V,
                                                                        double* __restrict__ v_in) {
    constexpr int groups = kThreads / kOfaTpr;
    const Layout Y(D, groups, TAB_Q); // one row slot per group
    GM_CHECK(D.tpr == kOfaTpr && D.Wl == kOfaWl && D.R == kOfaR && D.n_lines == kOfaNl);
    GM_CHECK(static_cast<unsigned>(4 * (Y.offL + kOfaNl)) <= gm_dyn_smem_bytes());
    int* si = reinterpret_cast<int*>(g_sm);
    for (int c = threadIdx.x; c < kOfaNl; c += blockDim.x) si[Y.offL + c] = D.line_off[c];
    __syncthreads();
    const int g = threadIdx.x / kOfaTpr, lane = threadIdx.x - g * kOfaTpr;
    const int bar = 1 + g; // the group's named barrier (group_reduce uses the same one)
    const unsigned sm0 = static_cast<unsigned>(__cvta_generic_to_shared(g_sm));
    int Ls[kOfaPer], ks[kOfaPer];
    unsigned la[kOfaPer];
#pragma unroll
    for (int S = 0; S < kOfaPer; ++S) {
        const int t = lane + kOfaTpr * S;
        Ls[S] = t / kOfaWl;
        ks[S] = t - Ls[S] * kOfaWl;
        la[S] = sm0 + 4u * static_cast<unsigned>(Y.offL + Ls[S]);
    }
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const int mw = Y.mw;
    double* m = g_sm + g * mw;
    double* P = g_sm + Y.offP + g * D.P_size;
    double* Q = g_sm + Y.offQ + g * kOfaNl;
    for (long long row = static_cast<long long>(blockIdx.x) * groups + g; row < nrows;
         row += static_cast<long long>(gridDim.x) * groups) {
        const uint8_t fl = rowflag[row];
        const bool live = !(fl & (RF_ABSORBED | RF_ERROR));
        double s = 0.0;
        if (live) {
            named_sync(bar, kOfaTpr); // the slot's previous row is done
            for (int q = lane; q < mw; q += kOfaTpr) m[q] = q < D.sumW ? mass[static_cast<long long>(q) * nrows + row] : 1.0;
            named_sync(bar, kOfaTpr);
            // prefix products (stage_tables' association): per run of the last prefix axis
            if (D.s_axes == 0) {
                if (lane == 0) P[0] = 1.0;
            } else {
                const int last = D.s_axes - 1, wl = D.W[last], nb = D.P_size / wl;
                for (int b = lane; b < nb; b += kOfaTpr) {
                    double acc = 1.0;
                    int rem = b * wl;
                    for (int d = 0; d < last; ++d) {
                        const int j = D.div_Ps[d].div(rem);
                        rem -= j * D.Ps[d];
                        acc *= m[D.mass_off[d] + j];
                    }
                    const double* ml = m + D.mass_off[last];
                    for (int j = 0; j < wl; ++j) P[b * wl + j] = acc * ml[j];
                }
            }
            named_sync(bar, kOfaTpr);
            for (int L = lane; L < kOfaNl; L += kOfaTpr) {
                const int a = D.div_Wm.div(L), j = L - a * D.Wm;
                Q[L] = P[a] * m[D.mm_off + j];
            }
            named_sync(bar, kOfaTpr);
            GM_CHECK_SLAB(D, origin[row]);
            const double* vrow = V + origin[row];
            unsigned qa[kOfaPer];
            double ml[kOfaPer];
            const double* vb[kOfaPer];
#pragma unroll
            for (int S = 0; S < kOfaPer; ++S) {
                qa[S] = sm0 + 8u * static_cast<unsigned>(Y.offQ + g * kOfaNl + Ls[S]);
                ml[S] = m[D.ml_off + ks[S]];
                vb[S] = vrow + ks[S];
            }
            s = OfaDot<0>::run(0.0, qa, la, ml, vb, lane);
        }
        s = group_reduce(s, kOfaTpr, Y.offR, g * kOfaTpr);
        if (lane == 0) v_in[row] = live ? (reach ? s + t0x[row] : s) : 0.0;
    }
}
#endif
