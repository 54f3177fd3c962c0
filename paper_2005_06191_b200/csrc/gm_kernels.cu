#include <numeric>
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
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace gmk {

namespace {
std::mutex g_var_mu;
char g_variant[KF_COUNT][96] = {};
void note_variant(int fam, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void note_variant(int fam, const char* fmt, ...) {
    char buf[96];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    std::lock_guard<std::mutex> lk(g_var_mu);
    std::memcpy(g_variant[fam], buf, sizeof buf);
}
} // namespace

const char* last_variant(int family) {
    if (family < 0 || family >= KF_COUNT) return "";
    return g_variant[family];
}


namespace {


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

#include "gm_rowdev.cuh"

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

#include "gm_ofa.cuh"

// Stage (i), fused: each CTA batch evaluates its rows' prologue (image, origin,
// target-hit mass: one thread per row), their per-axis cell masses (one thread
// per row x cell), the prefix tables, then streams the R products of every row
// (warp per row, coalesced evict-first stores). The row prologue of one CTA
// overlaps the store phase of the others on the same SM.
template <int TAB>
__global__ void __launch_bounds__(kThreads, 4) k_build(GmDev D, long long row0, long long nrows, int rb,
                                                   GmFastDiv div_rb,
                                                   long long* __restrict__ origin_out,
                                                   double* __restrict__ t0x_out, double* __restrict__ probs,
                                                   unsigned long long* err) {
    const Layout Y(D, rb, TAB);
    // per-row prologue data and the dynamics program after the batch tables
    const int offMu = Y.offR + kThreads / 32;          // [rb][GMD_MAXD] image
    const int offX = offMu + rb * GMD_MAXD;             // [rb][GMD_MAXD] state (multiplicative scale)
    const int offOk = offX + rb * GMD_MAXD;             // [rb] 1.0 = row ok
    const int offO = offOk + rb;                        // ints: [rb][GMD_MAXD] origin per axis
    const int offProg = offO + (rb * GMD_MAXD + 1) / 2; // GmIns (8 bytes each), then literals
    GmIns* sprog = reinterpret_cast<GmIns*>(g_sm + offProg);
    double* slits = g_sm + offProg + D.n_ins;
    int* sorg = reinterpret_cast<int*>(g_sm + offO);
    for (int c = threadIdx.x; c < D.n_ins; c += blockDim.x) sprog[c] = D.prog[c];
    for (int c = threadIdx.x; c < D.n_lits; c += blockDim.x) slits[c] = D.lits[c];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int mw = Y.mw;
    const int R = static_cast<int>(D.R);
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    Walk wk0;
    wk0.init(D, lane, 32);
    for (long long b0 = static_cast<long long>(blockIdx.x) * rb; b0 < nrows;
         b0 += static_cast<long long>(gridDim.x) * rb) {
        __syncthreads();
        if (threadIdx.x < rb) { // RowKernel::compute (abstraction.cpp:72-121) + box_mass (:187-191)
            const int i = threadIdx.x;
            const long long r = b0 + i;
            double ok = 0.0;
            if (r < nrows) {
                double x[GMD_MAXD], u[GMD_MAXD], w[GMD_MAXD], mu[GMD_MAXD];
                long long ix;
                decode_row(D, row0 + r, ix, x, u, w);
                if (run_dynamics(D, sprog, slits, x, u, w, mu)) {
                    ok = 1.0;
                    long long flat = 0;
                    for (int d = 0; d < D.n; ++d) {
                        const long long o = slab_origin(D, d, mu[d]);
                        sorg[i * GMD_MAXD + d] = static_cast<int>(o);
                        flat += o * D.xstride[d];
                        g_sm[offMu + i * GMD_MAXD + d] = mu[d];
                        g_sm[offX + i * GMD_MAXD + d] = x[d];
                    }
                    origin_out[r] = flat;
                    if (D.origin_host) D.origin_host[r] = flat;
                    if (t0x_out) {
                        const bool absorbed = reach && D.absorb != nullptr && D.absorb[ix];
                        double p = 0.0;
                        bool bok = true;
                        if (!absorbed) {
                            p = 1.0;
                            for (int d = 0; d < D.n; ++d) {
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
            g_sm[offOk + i] = ok;
        }
        __syncthreads();
        // fill_axis_masses (abstraction.cpp:130-146): thread per (row, axis), boundary
        // CDF values shared between adjacent cells when bitwise equal (axis_masses)
        for (int c = threadIdx.x; c < rb * D.n; c += blockDim.x) {
            const int d = c / rb, i = c - d * rb;
            if (g_sm[offOk + i] != 0.0) {
                bool ok = true;
                axis_masses(D, d, sorg[i * GMD_MAXD + d], g_sm[offMu + i * GMD_MAXD + d],
                            D.mult ? g_sm[offX + i * GMD_MAXD + d] : 1.0, g_sm + i * mw + D.mass_off[d], 1, ok);
                if (!ok) record_error(err, row0 + b0 + i);
            } else {
                for (int t = 0; t < D.W[d]; ++t) g_sm[i * mw + D.mass_off[d] + t] = 1.0;
            }
        }
        for (int i = threadIdx.x; i < rb; i += blockDim.x) g_sm[i * mw + D.sumW] = 1.0; // virtual-axis slot
        __syncthreads();
        stage_tables(D, Y, rb, TAB);
        __syncthreads();
        for (int i = warp; i < rb; i += nwarps) { // fill_product (abstraction.cpp:150-159)
            const long long row = b0 + i;
            if (row >= nrows) break;
            const int qo = Y.offQ + i * D.n_lines, po = Y.offP + i * D.P_size;
            const int mmo = i * mw + D.mm_off, mlo = i * mw + D.ml_off;
            double* out = probs + row * D.pitch;
            for (long long t = R + lane; t < D.pitch; t += 32) __stcs(out + t, 0.0); // row padding
            Walk wk = wk0; // the lane's walk is row independent (initialised once per CTA)
#pragma unroll 4
            for (int t = lane; t < R; t += 32) {
                const double p = TAB == TAB_Q ? g_sm[qo + wk.L] * g_sm[mlo + wk.k]
                                              : (g_sm[po + wk.a] * g_sm[mmo + wk.j]) * g_sm[mlo + wk.k];
                __stcs(out + t, p);
                wk.template next<TAB == TAB_P>();
            }
        }
    }
}

// Stage (ii), stored matrix (synthesis.cpp:95-99): row groups stream each row
// (evict-first, 8 loads in flight per lane) and gather V at the row's origin.
template <bool LS>
__global__ void __launch_bounds__(kThreads) k_expect_matrix(GmDev D, long long row0, long long r_lo,
                                                           long long r_hi, const double* __restrict__ probs,
                                                           const long long* __restrict__ origins,
                                                           const double* __restrict__ t0x,
                                                           const double* __restrict__ V,
                                                           double* __restrict__ v_in) {
    const Layout Y(D, 0, TAB_P);
    if (LS) {
        int* si = reinterpret_cast<int*>(g_sm);
        for (int c = threadIdx.x; c < D.n_lines; c += blockDim.x) si[Y.offL + c] = D.line_off[c];
    }
    __syncthreads();
    const int tpr = D.tpr;
    const int groups = kThreads / tpr;
    const int g = threadIdx.x / tpr, lane = threadIdx.x - g * tpr;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const long long nrows = r_hi - r_lo;
    const long long total_groups = static_cast<long long>(gridDim.x) * groups;
    const long long iters = (nrows + total_groups - 1) / total_groups;
    const long long nuw = D.n_u * D.n_w;
    for (long long it = 0; it < iters; ++it) {
        const long long rl = (it * gridDim.x + blockIdx.x) * groups + g; // local row
        const bool valid = rl < nrows;
        const long long r = r_lo + rl; // row inside the matrix
        bool skip = !valid;
        if (valid && reach && D.absorb != nullptr) skip = D.absorb[(row0 + r) / nuw];
        double s = 0.0;
        if (!skip) GM_CHECK_SLAB(D, origins[r]);
        if (!skip)
            s = row_dot<0, 8, LS>(D, lane, tpr, probs + r * D.pitch, 0, 0, 0, 0, V + origins[r], D.line_off, Y.offL);
        s = group_reduce(s, tpr, Y.offR, g * tpr);
        if (valid && lane == 0) v_in[rl] = skip ? 0.0 : (reach ? s + t0x[r] : s);
    }
}

// Stage (ii), stored matrix, element-offset table: the slab walk of a lane is the
// same for every row, so the CTA tabulates E[t] = line_off[L(t)] + k(t) once in
// shared memory and each term costs one LDS + the two loads + one fma (the walk
// kernel above spends ~19 instructions per term). Same canonical per-lane order
// (t = lane, lane+TPR, ...; batches of 8 with zero padding), so the result is
// bitwise that of every other row kernel.
//
// Row schedule (flags bit 1 clear): CTA-interleaved groups of `groups` rows;
// (bit 1 set) each CTA owns one contiguous range of rows, so consecutive states
// (whose slabs overlap) run back to back on one SM and reuse V lines in L1.
// flags bit 0: row / (n_u n_w) fits the 32-bit multiply-shift division.
struct RowSched {
    long long per_cta, iters, stride;
    bool contig;
    __device__ __forceinline__ RowSched(long long nrows, int groups, int flags) {
        contig = flags & 2;
        if (contig) {
            per_cta = ((nrows + gridDim.x - 1) / gridDim.x + groups - 1) / groups * groups;
            iters = per_cta / groups;
        } else {
            const long long total = static_cast<long long>(gridDim.x) * groups;
            per_cta = 0;
            iters = (nrows + total - 1) / total;
        }
    }
    __device__ __forceinline__ long long row(long long it, int groups, int g) const {
        return contig ? blockIdx.x * per_cta + it * groups + g : (it * gridDim.x + blockIdx.x) * groups + g;
    }
};

template <int TPR, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_expect_matrix_et(GmDev D, long long row0, long long r_lo,
                                                              long long r_hi, GmFastDiv div_nuw, int flags,
                                                              const double* __restrict__ probs,
                                                              const long long* __restrict__ origins,
                                                              const double* __restrict__ t0x,
                                                              const double* __restrict__ V,
                                                              double* __restrict__ v_in) {
    constexpr int groups = kThreads / TPR;
    const int R = static_cast<int>(D.R);
    int* E = reinterpret_cast<int*>(g_sm + kThreads / 32); // after the group partials
    for (int t = threadIdx.x; t < R; t += kThreads) {
        const int L = D.div_Wl.div(t);
        E[t] = D.line_off[L] + (t - L * D.Wl);
        GM_CHECK(E[t] >= 0 && E[t] <= slab_span(D));
    }
    __syncthreads();
    const int g = threadIdx.x / TPR, lane = threadIdx.x % TPR;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const long long nrows = r_hi - r_lo;
    const RowSched rs(nrows, groups, flags);
    const long long nuw = D.n_u * D.n_w;
    const int n_it = lane < R ? (R - lane + TPR - 1) / TPR : 0;
    const int n_full = n_it - n_it % U;
    const int rem = n_it - n_full;
    for (long long it = 0; it < rs.iters; ++it) {
        const long long rl = rs.row(it, groups, g);
        const bool valid = rl < nrows;
        const long long r = r_lo + rl;
        bool skip = !valid;
        if (valid && reach && D.absorb != nullptr) {
            const long long row = row0 + r;
            skip = D.absorb[(flags & 1) ? static_cast<long long>(div_nuw.div(static_cast<int>(row))) : row / nuw];
        }
        double s = 0.0;
        if (!skip) {
            GM_CHECK_SLAB(D, origins[r]);
            const double* pr = probs + r * D.pitch + lane;
            const double* vb = V + origins[r];
            const int* e = E + lane;
            for (int b = 0; b < n_full; b += U) {
                double p[U], v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    p[u] = __ldcs(pr + u * TPR);
                    v[u] = ldg_at(vb, e[u * TPR]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
                pr += U * TPR;
                e += U * TPR;
            }
            if (rem) {
                double p[U], v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    p[u] = 0.0;
                    v[u] = 0.0;
                    if (u < rem) {
                        p[u] = __ldcs(pr + u * TPR);
                        v[u] = ldg_at(vb, e[u * TPR]);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
            }
        }
        s = group_reduce(s, TPR, 0, g * TPR);
        if (valid && lane == 0) v_in[rl] = skip ? 0.0 : (reach ? s + t0x[r] : s);
    }
}

// Stage (ii), stored matrix, short rows (TPR <= 4: R < 64). The rows of a warp's
// chunk (32/TPR rows) are contiguous in the matrix, so the warp stages the chunk in
// shared memory with coalesced 8-byte cp.async copies, double-buffered (chunk c+1
// in flight while chunk c is reduced); each row group then reduces its row from
// shared memory exactly as k_expect_matrix_et does (lane-strided fma in increasing
// t, the TPR-lane butterfly): the same bits, without the per-lane strided loads
// of rows 27-32 doubles apart that leave those sweeps at 25-30 % of HBM.
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int TPR, int U>
__global__ void __launch_bounds__(kThreads) k_expect_matrix_small(GmDev D, long long row0, long long r_lo,
                                                                 long long r_hi, int rpc, int chunk_len,
                                                                 const double* __restrict__ probs,
                                                                 const long long* __restrict__ origins,
                                                                 const double* __restrict__ t0x,
                                                                 const double* __restrict__ V,
                                                                 double* __restrict__ v_in) {
    const int RPC = rpc; // rows per warp chunk (<= 32 / TPR: lanes past them idle in the dot)
    const int R = static_cast<int>(D.R);
    const long long pitch = D.pitch;
    int* E = reinterpret_cast<int*>(g_sm);
    const int offB = (R + 1) / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* buf = g_sm + offB + static_cast<long long>(warp) * 2 * chunk_len;
    GM_CHECK(static_cast<unsigned>(8 * (offB + (kThreads / 32) * 2 * chunk_len)) <= gm_dyn_smem_bytes());
    GM_CHECK(chunk_len == RPC * pitch && RPC * TPR <= 32);
    for (int t = threadIdx.x; t < R; t += kThreads) {
        const int L = D.div_Wl.div(t);
        E[t] = D.line_off[L] + (t - L * D.Wl);
        GM_CHECK(E[t] >= 0 && E[t] <= slab_span(D));
    }
    __syncthreads();
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const long long nrows = r_hi - r_lo, nuw = D.n_u * D.n_w;
    const long long nchunks = (nrows + RPC - 1) / RPC;
    const long long wstride = static_cast<long long>(gridDim.x) * (kThreads / 32);
    const int j = lane / TPR, q = lane % TPR; // row of the chunk, lane within the row group
    auto issue = [&](long long c, int b) {
        if (c < nchunks) {
            const long long rc = r_lo + c * RPC;
            const long long len = (nrows - c * RPC < RPC ? nrows - c * RPC : RPC) * pitch;
            const double* src = probs + rc * pitch;
            double* dst = buf + b * chunk_len;
            for (long long e = lane; e < len; e += 32) cp_async8(dst + e, src + e);
        }
        cp_async_commit(); // an empty group keeps the wait counts uniform
    };
    long long c = static_cast<long long>(blockIdx.x) * (kThreads / 32) + warp;
    issue(c, 0);
    for (int b = 0; c < nchunks; c += wstride, b ^= 1) {
        issue(c + wstride, b ^ 1);
        cp_async_wait<1>(); // chunk c has landed
        __syncwarp();
        const long long rl = c * RPC + j; // local row
        const bool valid = j < RPC && rl < nrows;
        const long long r = r_lo + rl;
        bool skip = !valid;
        if (valid && reach && D.absorb != nullptr) skip = D.absorb[(row0 + r) / nuw];
        double s = 0.0;
        if (!skip) {
            GM_CHECK_SLAB(D, origins[r]);
            const double* pr = buf + b * chunk_len + j * pitch;
            const double* vb = V + origins[r];
            // U gathers in flight per lane, then their fmas in increasing t; the last
            // block is predicated (absent terms add fma(0, 0, s) == s)
            int t = q;
            for (; t + (U - 1) * TPR < R; t += U * TPR) {
                double v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = ldg_at(vb, E[t + u * TPR]);
#pragma unroll
                for (int u = 0; u < U; ++u) s = fma(pr[t + u * TPR], v[u], s);
            }
            if (t < R) {
                double v[U], p[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool in = t + u * TPR < R;
                    v[u] = in ? ldg_at(vb, E[t + u * TPR]) : 0.0;
                    p[u] = in ? pr[t + u * TPR] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
            }
        }
        for (int off = TPR >> 1; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (valid && q == 0) v_in[rl] = skip ? 0.0 : (reach ? s + t0x[r] : s);
        __syncwarp(); // the buffer is refilled by the next issue
    }
    cp_async_wait<0>();
}

// One row's lane-strided partial sum of k_expect_matrix_et (canonical order: terms
// t = lane, lane+TPR, ... with fma in increasing t; the zero-padded tail adds +0).
template <int TPR, int U>
__device__ __forceinline__ double et_row_partial(const double* __restrict__ pr, const double* vb, const int* e,
                                                 int n_full, int rem) {
    double s = 0.0;
    for (int b = 0; b < n_full; b += U) {
        double p[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = __ldcs(pr + u * TPR);
            v[u] = ldg_at(vb, e[u * TPR]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
        pr += U * TPR;
        e += U * TPR;
    }
    if (rem) {
        double p[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = 0.0;
            v[u] = 0.0;
            if (u < rem) {
                p[u] = __ldcs(pr + u * TPR);
                v[u] = ldg_at(vb, e[u * TPR]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(p[u], v[u], s);
    }
    return s;
}

// k_expect_matrix_et for TPR = 32 with two consecutive rows per warp: each row's
// partial sums are the one-row kernel's, and one transposed butterfly reduces
// both (level 16 sends the other half's row: lanes 0-15 continue with row A,
// 16-31 with row B, so lane 0 / lane 16 end with exactly the canonical lane-0
// sums of A / B, a + b == b + a in IEEE). Halves the reduction and the per-row
// schedule overhead.
template <int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_expect_matrix_et2(GmDev D, long long row0, long long r_lo,
                                                               long long r_hi, GmFastDiv div_nuw, int flags,
                                                               const double* __restrict__ probs,
                                                               const long long* __restrict__ origins,
                                                               const double* __restrict__ t0x,
                                                               const double* __restrict__ V,
                                                               double* __restrict__ v_in) {
    constexpr int W = kThreads / 32;
    const int R = static_cast<int>(D.R);
    int* E = reinterpret_cast<int*>(g_sm + kThreads / 32);
    for (int t = threadIdx.x; t < R; t += kThreads) {
        const int L = D.div_Wl.div(t);
        E[t] = D.line_off[L] + (t - L * D.Wl);
        GM_CHECK(E[t] >= 0 && E[t] <= slab_span(D));
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const long long nrows = r_hi - r_lo, npairs = (nrows + 1) / 2;
    const long long nuw = D.n_u * D.n_w;
    const int n_it = lane < R ? (R - lane + 31) / 32 : 0;
    const int n_full = n_it - n_it % U, rem = n_it - n_full;
    auto absorbed = [&](long long r) {
        const long long row = row0 + r;
        return D.absorb[(flags & 1) ? static_cast<long long>(div_nuw.div(static_cast<int>(row))) : row / nuw] != 0;
    };
    for (long long pi = static_cast<long long>(blockIdx.x) * W + warp; pi < npairs;
         pi += static_cast<long long>(gridDim.x) * W) {
        const long long rlA = 2 * pi, rlB = rlA + 1;
        const bool hasB = rlB < nrows;
        const long long rA = r_lo + rlA, rB = rA + 1;
        bool skA = false, skB = !hasB;
        if (reach && D.absorb != nullptr) {
            skA = absorbed(rA);
            if (hasB) skB = absorbed(rB);
        }
        if (!skA) GM_CHECK_SLAB(D, origins[rA]);
        if (!skB) GM_CHECK_SLAB(D, origins[rB]);
        const double sA = skA ? 0.0
                              : et_row_partial<32, U>(probs + rA * D.pitch + lane, V + origins[rA], E + lane, n_full, rem);
        const double sB = skB ? 0.0
                              : et_row_partial<32, U>(probs + rB * D.pitch + lane, V + origins[rB], E + lane, n_full, rem);
        const bool hi = lane >= 16;
        double s = (hi ? sB : sA) + __shfl_xor_sync(0xffffffffu, hi ? sA : sB, 16);
        for (int off = 8; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) v_in[rlA] = skA ? 0.0 : (reach ? s + t0x[rA] : s);
        if (lane == 16 && hasB) v_in[rlB] = skB ? 0.0 : (reach ? s + t0x[rB] : s);
    }
}

// Stage (ii), stored matrix, both passes in one kernel for small states (all
// n_u*n_w rows of a state fit one CTA: n_u*n_w*TPR <= 256 threads): each CTA
// copies the rows of `spb` consecutive states (contiguous in the matrix) into
// shared memory with coalesced evict-first loads, every row group reduces its row
// exactly as k_expect_matrix_et (lane-strided fma in increasing t, the TPR-lane
// butterfly), and one thread per state runs pass 2 as k_maxmin does (strict <
// over w, strict > over u, lowest-index ties, clamp): the same bits, one launch
// per step and no v_in round trip (C2a: R = 27, 25 rows per state).
template <int TPR>
__global__ void __launch_bounds__(kThreads) k_step_small(GmDev D, long long x0, long long nx, int spb,
                                                        const double* __restrict__ probs, long long r_base,
                                                        const long long* __restrict__ origins,
                                                        const double* __restrict__ t0x,
                                                        const double* __restrict__ V, double* __restrict__ v_in,
                                                        double* __restrict__ v_out, uint32_t* __restrict__ pol,
                                                        uint32_t* __restrict__ wst) {
    const int R = static_cast<int>(D.R);
    const int nuw = static_cast<int>(D.n_u * D.n_w);
    const long long pitch = D.pitch;
    int* E = reinterpret_cast<int*>(g_sm);
    const int offS = (R + 1) / 2; // doubles after E
    double* stage = g_sm + offS;
    double* vrow = stage + static_cast<long long>(spb) * nuw * pitch;
    GM_CHECK(static_cast<unsigned>(8 * (offS + spb * nuw * pitch + spb * nuw)) <= gm_dyn_smem_bytes());
    for (int t = threadIdx.x; t < R; t += kThreads) {
        const int L = D.div_Wl.div(t);
        E[t] = D.line_off[L] + (t - L * D.Wl);
        GM_CHECK(E[t] >= 0 && E[t] <= slab_span(D));
    }
    const int G = nuw * TPR;
    const int st = threadIdx.x / G, w = threadIdx.x - st * G, j = w / TPR, lane = w - j * TPR;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    for (long long xs = static_cast<long long>(blockIdx.x) * spb; xs < nx;
         xs += static_cast<long long>(gridDim.x) * spb) {
        const int ns = static_cast<int>(nx - xs < spb ? nx - xs : spb);
        const long long rl0 = r_base + xs * nuw; // first matrix row of the chunk
        const long long nd = static_cast<long long>(ns) * nuw * pitch;
        __syncthreads();
        const double* src = probs + rl0 * pitch;
        for (long long c = threadIdx.x; c < nd; c += kThreads) stage[c] = __ldcs(src + c);
        __syncthreads();
        const bool active = st < ns;
        const long long x = x0 + xs + (active ? st : 0);
        const bool skip = !active || (reach && D.absorb != nullptr && D.absorb[x]);
        const long long r = rl0 + static_cast<long long>(active ? st : 0) * nuw + j;
        double s = 0.0;
        if (!skip) {
            GM_CHECK_SLAB(D, origins[r]);
            const double* pr = stage + (static_cast<long long>(st) * nuw + j) * pitch;
            const double* vb = V + origins[r];
            for (int t = lane; t < R; t += TPR) s = fma(pr[t], ldg_at(vb, E[t]), s);
        }
        for (int off = TPR >> 1; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (active && lane == 0) {
            const double vr = skip ? 0.0 : (reach ? s + t0x[r] : s);
            vrow[st * nuw + j] = vr;
            v_in[(xs + st) * nuw + j] = vr; // the step's row values stay readable (gm_copy_row_values)
        }
        __syncthreads();
        if (threadIdx.x < ns) { // pass 2 (synthesis.cpp:112-142), as k_maxmin
            const long long xi = xs + threadIdx.x, xx = x0 + xi;
            if (reach && D.absorb != nullptr && D.absorb[xx]) {
                v_out[xi] = 0.0;
                if (pol) pol[xi] = 0;
                if (wst) wst[xi] = 0;
            } else {
                const double* q = vrow + threadIdx.x * nuw;
                double best = -INFINITY;
                uint32_t bu = 0, bw = 0;
                for (int iu = 0; iu < D.n_u; ++iu) {
                    double mn = INFINITY;
                    uint32_t mw = 0;
                    for (int iw = 0; iw < D.n_w; ++iw) {
                        const double v = q[iu * D.n_w + iw];
                        if (v < mn) {
                            mn = v;
                            mw = static_cast<uint32_t>(iw);
                        }
                    }
                    if (mn > best) {
                        best = mn;
                        bu = static_cast<uint32_t>(iu);
                        bw = mw;
                    }
                }
                v_out[xi] = smin(1.0, smax(0.0, best));
                if (pol) pol[xi] = bu;
                if (wst) wst[xi] = bw;
            }
        }
    }
}

// The pass-2 epilogue's peer stores (GmMirror): the value of absolute state x into
// every other device's value table whose read interval holds x.
__device__ __forceinline__ void mirror_store(const GmMirror& mir, long long x, double v) {
    for (int i = 0; i < mir.n; ++i)
        if (x >= mir.lo[i] && x < mir.hi[i]) mir.dst[i][x] = v;
}

// Stage (ii), stored matrix, the whole step for small states with one warp per
// state (both passes; C2a: 25 rows of 27 entries per state). The warp copies its
// state's rows (contiguous in the matrix) into its shared-memory slot with
// coalesced 8-byte cp.async copies, re-pitched to `ps` (conflict-free row reads);
// row groups of TPR lanes reduce the rows exactly as k_expect_matrix_et (lane-
// strided fma in increasing t, the TPR-lane butterfly) into the slot's row values;
// the copy of the warp's next state is issued, and the warp runs pass 2 over the
// row values as k_maxmin<32> (strict < over w, strict > over u, lowest-index ties,
// clamp). The same bits as expect_matrix + maxmin, one launch per step, no v_in
// round trip (v_in is still written: the step's row values stay readable), and
// no CTA-wide barrier after the offset table.
template <int TPR, int U>
__global__ void __launch_bounds__(kThreads) k_step_warp(GmDev D, long long x0, long long nx, int ps, int wslot,
                                                      const double* __restrict__ probs,
                                                      const long long* __restrict__ origins,
                                                      const double* __restrict__ t0x,
                                                      const double* __restrict__ V, double* __restrict__ v_in,
                                                      double* __restrict__ v_out, uint32_t* __restrict__ pol,
                                                      uint32_t* __restrict__ wst, GmMirror mir) {
    constexpr int RPP = 32 / TPR; // rows per pass of the warp
    const int R = static_cast<int>(D.R), P = static_cast<int>(D.pitch);
    const int nu = static_cast<int>(D.n_u), nw = static_cast<int>(D.n_w), nuw = nu * nw;
    int* E = reinterpret_cast<int*>(g_sm);
    const int offW = (R + 1) / 2; // doubles after E
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* stage = g_sm + offW + static_cast<long long>(warp) * wslot;
    double* vrow = stage + nuw * ps;
    long long* sorg = reinterpret_cast<long long*>(vrow + nuw); // the state's row origins, copied with its rows
    GM_CHECK(static_cast<unsigned>(8 * (offW + (kThreads / 32) * wslot)) <= gm_dyn_smem_bytes());
    GM_CHECK(wslot >= nuw * (ps + 2) && ps >= R);
    for (int t = threadIdx.x; t < R; t += kThreads) {
        const int Ln = D.div_Wl.div(t);
        E[t] = D.line_off[Ln] + (t - Ln * D.Wl);
        GM_CHECK(E[t] >= 0 && E[t] <= slab_span(D));
    }
    __syncthreads();
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const bool has_abs = reach && D.absorb != nullptr;
    // the state's rows are one contiguous block: flat copies, (row, column) of the
    // lane's element advanced incrementally
    const int row0 = lane / P, col0 = lane - row0 * P, qs = 32 / P, rs = 32 - qs * P;
    const int nel = nuw * P;
    auto issue = [&](long long x, bool abs_x) {
        if (x < nx && !abs_x) {
            for (int j = lane; j < nuw; j += 32)
                cp_async8(reinterpret_cast<double*>(sorg + j), reinterpret_cast<const double*>(origins + x * nuw + j));
            const double* src = probs + x * nuw * static_cast<long long>(P);
            int row = row0, col = col0;
            for (int e = lane; e < nel; e += 32) {
                if (col < R) cp_async8(stage + row * ps + col, src + e);
                row += qs;
                col += rs;
                if (col >= P) {
                    col -= P;
                    ++row;
                }
            }
        }
        cp_async_commit();
    };
    const long long wstride = static_cast<long long>(gridDim.x) * (kThreads / 32);
    long long x = static_cast<long long>(blockIdx.x) * (kThreads / 32) + warp;
    auto absorbed_at = [&](long long xx) { return xx < nx && has_abs && D.absorb[x0 + xx] != 0; };
    bool absorbed = absorbed_at(x);
    issue(x, absorbed);
    const int j0 = lane / TPR, q = lane - j0 * TPR;
    for (; x < nx; x += wstride) {
        const bool abs_next = absorbed_at(x + wstride); // loaded early: the next issue needs it
        cp_async_wait<0>();
        __syncwarp();
        if (!absorbed) {
            for (int j = j0; j - j0 < nuw; j += RPP) { // pass 1: RPP rows at a time (warp-uniform trip count)
                const bool valid = j < nuw;
                const long long r = x * nuw + (valid ? j : 0); // local row
                double s = 0.0;
                if (valid) {
                    GM_CHECK_SLAB(D, sorg[j]);
                    const double* pr = stage + j * ps;
                    const double* vb = V + sorg[j];
                    int t = q;
                    for (; t + (U - 1) * TPR < R; t += U * TPR) {
                        double v[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) v[u] = ldg_at(vb, E[t + u * TPR]);
#pragma unroll
                        for (int u = 0; u < U; ++u) s = fma(pr[t + u * TPR], v[u], s);
                    }
                    for (; t < R; t += TPR) s = fma(pr[t], ldg_at(vb, E[t]), s);
                }
                for (int off = TPR >> 1; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (valid && q == 0) {
                    const double vr = reach ? s + t0x[r] : s;
                    vrow[j] = vr;
                    v_in[r] = vr;
                }
            }
        } else {
            for (int j = lane; j < nuw; j += 32) v_in[x * nuw + j] = 0.0;
        }
        __syncwarp();                 // row values written, the stage read
        issue(x + wstride, abs_next); // the next state's rows land during pass 2
        // pass 2 (synthesis.cpp:112-142), as k_maxmin<32>
        double best = -INFINITY;
        uint32_t bu = 0, bw = 0;
        if (!absorbed) {
            for (int iu = lane; iu < nu; iu += 32) {
                double mn = INFINITY;
                uint32_t mw = 0;
                const double* qv = vrow + iu * nw;
                for (int iw = 0; iw < nw; ++iw) {
                    const double v = qv[iw];
                    if (v < mn) {
                        mn = v;
                        mw = static_cast<uint32_t>(iw);
                    }
                }
                if (mn > best) {
                    best = mn;
                    bu = static_cast<uint32_t>(iu);
                    bw = mw;
                }
            }
        }
        for (int off = 16; off >= 1; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const uint32_t ou = __shfl_xor_sync(0xffffffffu, bu, off);
            const uint32_t ow = __shfl_xor_sync(0xffffffffu, bw, off);
            if (ob > best || (ob == best && ou < bu)) {
                best = ob;
                bu = ou;
                bw = ow;
            }
        }
        if (lane == 0) {
            const double vx = absorbed ? 0.0 : smin(1.0, smax(0.0, best));
            v_out[x] = vx;
            mirror_store(mir, x0 + x, vx);
            if (pol) pol[x] = absorbed ? 0u : bu;
            if (wst) wst[x] = absorbed ? 0u : bw;
        }
        __syncwarp(); // vrow is rewritten by the next state's pass 1
        absorbed = abs_next;
    }
    cp_async_wait<0>();
}

// min over w (strict <, ascending), then max over u (strict >, ascending):
// lowest-index ties (synthesis.cpp:112-142). L lanes per state.
template <int L>
__global__ void __launch_bounds__(kThreads) k_maxmin(GmDev D, long long x0, long long nx,
                                                    const double* __restrict__ v_in,
                                                    double* __restrict__ v_out,
                                                    uint32_t* __restrict__ pol,
                                                    uint32_t* __restrict__ wst, GmMirror mir) {
    const long long gt = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long xi = gt / L;
    const int lane = static_cast<int>(gt % L);
    const bool valid = xi < nx;
    const long long ix = x0 + xi;
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    const bool absorbed = valid && reach && D.absorb != nullptr && D.absorb[ix];
    double best = -INFINITY;
    uint32_t bu = 0, bw = 0; // policy / worst_dist are uint32 tables (synthesis.hpp:21)
    if (valid && !absorbed) {
        const double* base = v_in + xi * D.n_u * D.n_w;
        for (long long iu = lane; iu < D.n_u; iu += L) {
            double mn = INFINITY;
            uint32_t mw = 0;
            const double* q = base + iu * D.n_w;
            for (long long iw = 0; iw < D.n_w; ++iw) {
                const double v = q[iw];
                if (v < mn) {
                    mn = v;
                    mw = static_cast<uint32_t>(iw);
                }
            }
            if (mn > best) {
                best = mn;
                bu = static_cast<uint32_t>(iu);
                bw = mw;
            }
        }
    }
    if (L > 1) {
        for (int off = L >> 1; off >= 1; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const uint32_t ou = __shfl_xor_sync(0xffffffffu, bu, off);
            const uint32_t ow = __shfl_xor_sync(0xffffffffu, bw, off);
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
        mirror_store(mir, ix, 0.0);
        if (pol) pol[xi] = 0;
        if (wst) wst[xi] = 0;
        return;
    }
    v_out[xi] = smin(1.0, smax(0.0, best));
    mirror_store(mir, ix, v_out[xi]);
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
        if (zt || za) probs[(r_lo + rl) * D.pitch + (e - rl * D.R)] = 0.0;
    }
}


// ---------------------------------------------------------------------------
// Closed-loop Monte Carlo (sim.cpp:16-101). Each run draws from its own
// Philox4x32-10 stream keyed by derive_stream_seed(seed, run) (common.hpp:74-79),
// so batches are reproducible for any launch shape. The reference draws from
// libstdc++'s mt19937_64 + distributions; only the distributions agree, so
// parity is statistical (tests/test_gpu_sim.py).
// ---------------------------------------------------------------------------

struct Philox {
    uint32_t k0, k1, c0 = 0, c1 = 0;
    uint64_t buf[2];
    int left = 0;
    __device__ Philox(uint64_t key) : k0(static_cast<uint32_t>(key)), k1(static_cast<uint32_t>(key >> 32)) {}
    __device__ void refill() {
        uint32_t x0 = c0, x1 = c1, x2 = 0, x3 = 0, a = k0, b = k1;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t h0 = __umulhi(0xD2511F53u, x0), l0 = 0xD2511F53u * x0;
            const uint32_t h1 = __umulhi(0xCD9E8D57u, x2), l1 = 0xCD9E8D57u * x2;
            const uint32_t y0 = h1 ^ x1 ^ a, y1 = l1, y2 = h0 ^ x3 ^ b, y3 = l0;
            x0 = y0; x1 = y1; x2 = y2; x3 = y3;
            a += 0x9E3779B9u;
            b += 0xBB67AE85u;
        }
        buf[0] = (static_cast<uint64_t>(x0) << 32) | x1;
        buf[1] = (static_cast<uint64_t>(x2) << 32) | x3;
        left = 2;
        if (++c0 == 0) ++c1;
    }
    __device__ uint64_t next() {
        if (!left) refill();
        return buf[--left];
    }
    __device__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; } // [0, 1)
    __device__ double normal() {                                                          // Box-Muller
        const double u1 = 1.0 - uniform(), u2 = uniform();
        return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    __device__ double gamma(double a) { // Marsaglia-Tsang, shape a, scale 1
        double boost = 1.0;
        if (a < 1.0) {
            boost = pow(1.0 - uniform(), 1.0 / a);
            a += 1.0;
        }
        const double d = a - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
        for (;;) {
            const double z = normal();
            double v = 1.0 + c * z;
            if (v <= 0.0) continue;
            v = v * v * v;
            const double u = 1.0 - uniform();
            if (log(u) < 0.5 * z * z + d - d * v + d * log(v)) return d * v * boost;
        }
    }
};

__device__ __forceinline__ uint64_t derive_stream_seed(uint64_t master, uint64_t stream) {
    uint64_t z = master + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// contains(grid, x) (grid.cpp:67-75) for the model's state grid
__device__ __forceinline__ bool in_region(const GmDev& D, const double* x) {
    for (int d = 0; d < D.n; ++d) {
        const double t = (x[d] - D.xlb[d]) / D.xeta[d];
        if (t < -0.5 - kIdxTol || t > static_cast<double>(D.xcount[d] - 1) + 0.5 + kIdxTol) return false;
    }
    return true;
}

__device__ __forceinline__ bool in_spec_box(int n, const double* x, const double* lo, const double* hi) {
    for (int d = 0; d < n; ++d)
        if (!(x[d] >= lo[d] && x[d] <= hi[d])) return false;
    return true;
}

// point_to_index (grid.cpp:77-96) on a region point: nearest representative, ties to +inf
__device__ __forceinline__ long long nearest_index(int n, const double* x, const double* lb, const double* eta,
                                                   const long long* count, const long long* stride) {
    long long flat = 0;
    for (int d = 0; d < n; ++d) {
        long long j = static_cast<long long>(floor((x[d] - lb[d]) / eta[d] + 0.5));
        if (j < 0) j = 0;
        if (j >= count[d]) j = count[d] - 1;
        flat += j * stride[d];
    }
    return flat;
}

__global__ void __launch_bounds__(128) k_simulate(GmDev D, SimArgs A) {
    extern __shared__ __align__(16) unsigned char sim_sm[];
    GmIns* sprog = reinterpret_cast<GmIns*>(sim_sm);
    double* slits = reinterpret_cast<double*>(sim_sm + ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16);
    for (int i = threadIdx.x; i < D.n_ins; i += blockDim.x) sprog[i] = D.prog[i];
    for (int i = threadIdx.x; i < D.n_lits; i += blockDim.x) slits[i] = D.lits[i];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= A.runs) return;
    Philox rng(derive_stream_seed(A.seed, static_cast<uint64_t>(r)));
    const int n = D.n, m = D.m, p = D.p, T = A.T;
    double x[GMD_MAXD], u[GMD_MAXD], w[GMD_MAXD], mu[GMD_MAXD];
    for (int d = 0; d < n; ++d) x[d] = A.x0[d];
    double* st = A.states ? A.states + static_cast<long long>(r) * (T + 1) * n : nullptr;
    double* in = A.inputs ? A.inputs + static_cast<long long>(r) * T * m : nullptr;
    double* ds = A.dists ? A.dists + static_cast<long long>(r) * T * p : nullptr;
    if (st)
        for (int d = 0; d < n; ++d) st[d] = x[d];
    int state = 0; // 0 open, 1 satisfied, 2 failed
    if (A.reach) { // immediate resolution at the start state; A wins over T
        if (A.has_avoid && in_spec_box(n, x, A.alo, A.ahi)) state = 2;
        else if (in_spec_box(n, x, A.tlo, A.thi)) state = 1;
    }
    int k = 0;
    while (state == 0 && k < T) {
        // query_policy(res, x, k+1)
        const long long ix = nearest_index(n, x, A.rs_lb, A.rs_eta, A.rs_count, A.rs_stride);
        long long iu = A.policy[static_cast<long long>(k) * A.rs_n + ix];
        for (int d = 0; d < A.ru_dim; ++d) {
            const long long j = iu / A.ru_stride[d];
            iu -= j * A.ru_stride[d];
            u[d] = A.ru_lb[d] + static_cast<double>(j) * A.ru_eta[d];
        }
        long long iw = 0;
        if (D.n_w > 1) {
            if (!A.worst_case) {
                iw = static_cast<long long>(rng.uniform() * static_cast<double>(D.n_w));
                if (iw >= D.n_w) iw = D.n_w - 1;
            } else {
                const long long jx = nearest_index(n, x, D.xlb, D.xeta, D.xcount, D.xstride);
                iw = A.worst[static_cast<long long>(k) * D.n_x + jx];
            }
        }
        long long rem = iw;
        for (int d = 0; d < p; ++d) {
            const long long j = rem / D.wstride[d];
            rem -= j * D.wstride[d];
            w[d] = D.wlb[d] + static_cast<double>(j) * D.weta[d];
        }
        double xi[GMD_MAXD];
        for (int d = 0; d < n; ++d) { // sample_axis (noise.cpp:277-302)
            double v;
            switch (D.family) {
                case GM_NORMAL: v = D.s[d] * 0.70710678118654752440 * rng.normal(); break; // s = sigma*sqrt2
                case GM_UNIFORM: v = D.s[d] + (D.p2[d] - D.s[d]) * rng.uniform(); break;
                case GM_EXPONENTIAL: v = -log1p(-rng.uniform()) / D.s[d]; break;
                case GM_CUSTOM: v = 0.0; break; // joint draw below
                default: {
                    const double ga = rng.gamma(D.s[d]), gb = rng.gamma(D.p2[d]);
                    v = ga / (ga + gb);
                }
            }
            xi[d] = v;
        }
        if (D.family == GM_CUSTOM) { // rejection sampling over the support (noise.cpp:335-352)
            bool acc = false;
            for (int tries = 0; tries < 1000000 && !acc; ++tries) {
                for (int d = 0; d < n; ++d) xi[d] = D.sup_lo[d] + rng.uniform() * (D.sup_hi[d] - D.sup_lo[d]);
                double pv = 0.0;
                if (!run_expr(D, sprog, slits, n, xi, nullptr, nullptr, pv)) break;
                acc = rng.uniform() * A.custom_sup <= pv;
            }
            if (!acc) {
                atomicMin(A.err, static_cast<unsigned long long>(r));
                state = 2;
                break;
            }
        }
        for (int d = 0; d < n; ++d)
            if (D.mult) xi[d] *= x[d];
        if (!run_dynamics(D, sprog, slits, x, u, w, mu)) {
            atomicMin(A.err, static_cast<unsigned long long>(r));
            state = 2;
            break;
        }
        if (in)
            for (int d = 0; d < m; ++d) in[k * m + d] = u[d];
        if (ds)
            for (int d = 0; d < p; ++d) ds[k * p + d] = w[d];
        for (int d = 0; d < n; ++d) x[d] = mu[d] + xi[d];
        ++k;
        if (st)
            for (int d = 0; d < n; ++d) st[k * n + d] = x[d];
        if (!in_region(D, x)) {
            state = 2; // left the quantized region
        } else if (A.reach) {
            if (A.has_avoid && in_spec_box(n, x, A.alo, A.ahi)) state = 2;
            else if (in_spec_box(n, x, A.tlo, A.thi)) state = 1;
        }
    }
    if (state == 0) state = A.reach ? 2 : 1; // horizon exhausted
    A.satisfied[r] = state == 1 ? 1 : 0;
    A.steps[r] = k;
}

// ---------------------------------------------------------------------------
// Custom joint densities (NoiseSpec::custom, noise.cpp:75-85, 205-250): no
// per-axis factorisation, every cell of a slab is the nested adaptive-Simpson
// integral of the pdf over the cell's preimage in noise coordinates
// (integrate_custom / adaptive_simpson, noise.cpp:208-221, 405-425), the pdf
// being the program's expression n. Device recursion mirrors the reference's
// (tolerance 1e-10 per level, depth limit 40); one warp per row.
// ---------------------------------------------------------------------------

struct CustomCtx {
    const GmDev* D;
    const GmIns* prog;
    const double* lits;
    double lo[GMD_MAXD], hi[GMD_MAXD], point[GMD_MAXD];
    bool ok, conv;
};

__device__ double custom_integrate(CustomCtx& c, int level);

__device__ __forceinline__ double custom_f(CustomCtx& c, int level, double t) {
    c.point[level] = t;
    if (level + 1 == c.D->n) {
        double v = 0.0;
        if (!run_expr(*c.D, c.prog, c.lits, c.D->n, c.point, nullptr, nullptr, v)) c.ok = false;
        return v;
    }
    return custom_integrate(c, level + 1);
}

__device__ double simpson_rec(CustomCtx& c, int level, double a, double m, double b, double fa, double fm, double fb,
                              double whole, double tol, int depth) {
    const double lm = 0.5 * (a + m), rm = 0.5 * (m + b);
    const double flm = custom_f(c, level, lm), frm = custom_f(c, level, rm);
    const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
    const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
    if (depth > 40) {
        c.conv = false;
        return left + right;
    }
    if (fabs(left + right - whole) <= 15.0 * tol) return left + right + (left + right - whole) / 15.0;
    const double lv = simpson_rec(c, level, a, lm, m, fa, flm, fm, left, tol / 2.0, depth + 1);
    const double rv = simpson_rec(c, level, m, rm, b, fm, frm, fb, right, tol / 2.0, depth + 1);
    return lv + rv;
}

__device__ double custom_integrate(CustomCtx& c, int level) {
    const double lo = smax(c.lo[level], c.D->sup_lo[level]);
    const double hi = smin(c.hi[level], c.D->sup_hi[level]);
    if (hi <= lo) return 0.0;
    const double m = 0.5 * (lo + hi);
    const double fa = custom_f(c, level, lo), fm = custom_f(c, level, m), fb = custom_f(c, level, hi);
    const double whole = (hi - lo) / 6.0 * (fa + 4.0 * fm + fb);
    return simpson_rec(c, level, lo, m, hi, fa, fm, fb, whole, 1e-10, 0);
}

// cell_probability_impl, custom branch (noise.cpp:231-249): P(mean + s o xi in box)
__device__ double custom_cell_prob(CustomCtx& c, const double* mean, const double* blo, const double* bhi,
                                   const double* x) {
    const GmDev& D = *c.D;
    for (int d = 0; d < D.n; ++d) {
        const double s = D.mult ? x[d] : 1.0;
        if (s == 0.0) {
            c.ok = false; // "multiplicative custom density degenerates at state 0"
            return 0.0;
        }
        double a = s == 1.0 ? blo[d] - mean[d] : (blo[d] - mean[d]) / s;
        double b = s == 1.0 ? bhi[d] - mean[d] : (bhi[d] - mean[d]) / s;
        if (s < 0.0) {
            const double t = a;
            a = b;
            b = t;
        }
        c.lo[d] = a;
        c.hi[d] = b;
    }
    const double p = custom_integrate(c, 0);
    return smin(1.0, smax(0.0, p));
}

// Stage (i) for custom densities: one warp per row (lane 0 runs the row
// prologue, the lanes integrate the row's cells); probs may be null (T0x only).
__global__ void __launch_bounds__(128) k_build_custom(GmDev D, long long row0, long long nrows,
                                                     long long* __restrict__ origin_out,
                                                     double* __restrict__ t0x_out, double* __restrict__ probs,
                                                     unsigned long long* err) {
    extern __shared__ __align__(16) unsigned char cu_sm[];
    GmIns* sprog = reinterpret_cast<GmIns*>(cu_sm);
    double* slits = reinterpret_cast<double*>(cu_sm + ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16);
    for (int i = threadIdx.x; i < D.n_ins; i += blockDim.x) sprog[i] = D.prog[i];
    for (int i = threadIdx.x; i < D.n_lits; i += blockDim.x) slits[i] = D.lits[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long wpb = blockDim.x >> 5;
    const int n = D.n, R = static_cast<int>(D.R);
    const bool reach = D.spec_kind != GM_SPEC_SAFETY;
    CustomCtx c;
    c.D = &D;
    c.prog = sprog;
    c.lits = slits;
    for (long long row = blockIdx.x * wpb + (threadIdx.x >> 5); row < nrows; row += gridDim.x * wpb) {
        double x[GMD_MAXD], u[GMD_MAXD], w[GMD_MAXD], mu[GMD_MAXD];
        long long ix;
        decode_row(D, row0 + row, ix, x, u, w);
        int okd = 1;
        if (lane == 0) okd = run_dynamics(D, sprog, slits, x, u, w, mu) ? 1 : 0;
        okd = __shfl_sync(0xffffffffu, okd, 0);
        if (!okd) {
            if (lane == 0) record_error(err, row0 + row);
            continue;
        }
        long long o[GMD_MAXD];
        long long flat = 0;
        for (int d = 0; d < n; ++d) {
            mu[d] = __shfl_sync(0xffffffffu, mu[d], 0);
            o[d] = slab_origin(D, d, mu[d]);
            flat += o[d] * D.xstride[d];
        }
        if (lane == 0) {
            if (origin_out) origin_out[row] = flat;
            if (t0x_out) { // box_mass over the target (abstraction.cpp:187-191, 260-266)
                double p = 0.0;
                if (!(reach && D.absorb != nullptr && D.absorb[ix])) {
                    c.ok = c.conv = true;
                    p = custom_cell_prob(c, mu, D.tlo, D.thi, x);
                    if (!c.ok || !c.conv) record_error(err, row0 + row);
                }
                t0x_out[row] = p;
            }
        }
        if (!probs) continue;
        double* out = probs + row * D.pitch;
        for (int t = lane; t < D.pitch; t += 32) {
            double v = 0.0;
            if (t < R) { // fill_row, custom branch (abstraction.cpp:164-181): slab cell t
                double blo[GMD_MAXD], bhi[GMD_MAXD];
                int rem = t;
                for (int d = n - 1; d >= 0; --d) {
                    const int q = D.div_W[d].div(rem);
                    const int j = rem - q * D.W[d];
                    rem = q;
                    const double rep = D.xlb[d] + static_cast<double>(o[d] + j) * D.xeta[d];
                    blo[d] = rep - 0.5 * D.xeta[d];
                    bhi[d] = rep + 0.5 * D.xeta[d];
                }
                c.ok = c.conv = true;
                v = custom_cell_prob(c, mu, blo, bhi, x);
                if (!c.ok || !c.conv) record_error(err, row0 + row);
            }
            out[t] = v;
        }
    }
}
} // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

namespace {
constexpr size_t kSoftSmem = 56 * 1024;   // several CTAs per SM
constexpr size_t kMidSmem = 74 * 1024;    // three CTAs per SM
constexpr size_t kHardSmem = 200 * 1024;  // one CTA per SM, last resort
}

BatchPlan plan_batches(const GmDev& D, bool ofa) {
    BatchPlan b;
    b.tpr = ofa ? D.tpr : 32;
    b.groups = kThreads / b.tpr;
    const size_t mw = static_cast<size_t>(D.sumW + 1);
    const size_t fixed = (kThreads / 32) * sizeof(double);
    const size_t table = ofa ? static_cast<size_t>(D.n_lines) * sizeof(int) : 0;
    const size_t ptable = ofa ? static_cast<size_t>(D.P_size) * sizeof(int) : 0;
    const size_t q_row = (mw + D.P_size + D.n_lines) * sizeof(double);
    const size_t p_row = (mw + D.P_size) * sizeof(double);
    const long long want = std::max(b.groups, ofa ? 2 : 8);
    struct Opt { int tab; int lsmem; size_t budget; };
    // lsmem 2: the leading-prefix offset table (P_size ints) replaces the line table
    // when the latter does not fit (C4: 62.5 KB of lines vs 12.5 KB of prefixes).
    // GM_OFA_TABLE (tuning / tests): "global" or "prefix" forces TAB_P with that table.
    static const char* ft = std::getenv("GM_OFA_TABLE");
    const int force = !ft ? -1 : (std::string(ft) == "global" ? 0 : (std::string(ft) == "prefix" ? 2 : -1));
    // GM_OFA_SMEM_KB (tuning): the OFA plans' soft shared-memory budget per CTA (rows per batch)
    static const char* osk = std::getenv("GM_OFA_SMEM_KB");
    const size_t soft = (ofa && osk) ? static_cast<size_t>(std::atoi(osk)) * 1024 : kSoftSmem;
    const Opt opts[] = {{TAB_Q, 1, soft}, {TAB_Q, 0, soft}, {TAB_P, 1, soft},
                        {TAB_P, 2, soft}, {TAB_P, 2, kMidSmem}, {TAB_P, 0, soft}, {TAB_P, 2, kHardSmem},
                        {TAB_P, 0, kHardSmem}};
    for (const Opt& o : opts) {
        const size_t per = o.tab == TAB_Q ? q_row : p_row;
        const size_t tb = (ofa && o.lsmem) ? (o.lsmem == 2 ? ptable : table) : 0;
        if (!ofa && o.lsmem) continue;
        if (ofa && force >= 0 && (o.tab != TAB_P || o.lsmem != force)) continue;
        if (fixed + tb >= o.budget) continue;
        long long rb = static_cast<long long>((o.budget - fixed - tb) / per);
        if (rb < (o.budget == kHardSmem ? 1 : want)) continue;
        rb = std::min<long long>(rb, kThreads);
        if (rb >= b.groups) rb -= rb % b.groups;
        b.rb = static_cast<int>(rb);
        b.tab = o.tab;
        b.table_in_smem = ofa ? o.lsmem : 0;
        b.smem = fixed + per * static_cast<size_t>(b.rb) + tb;
        return b;
    }
    throw std::runtime_error("row too wide for the device batch layout (" + std::to_string(p_row) +
                             " bytes of shared memory per row)");
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

template <class K>
static void allow_smem(K kernel, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

void prologue(const GmDev& D, long long row0, long long nrows, int flags, long long* origin_out,
              double* t0x_out, uint8_t* rowflag_out, double* mass_out,
              unsigned long long* d_err_row, cudaStream_t s, const void* jit) {
    if (nrows <= 0) return;
    const size_t smem = ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16 + D.n_lits * sizeof(double);
    const void* k = jit ? jit : reinterpret_cast<const void*>(&k_prologue);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    GmDev Dv = D;
    void* args[] = {&Dv, &row0, &nrows, &flags, &origin_out, &t0x_out, &rowflag_out, &mass_out, &d_err_row};
    const cudaError_t e = cudaLaunchKernel(k, dim3(grid_for(nrows, kThreads)), dim3(kThreads), args, smem, s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("prologue: ") + cudaGetErrorString(e));
    check_launch("prologue");
}

// Resident CTAs per SM of a kernel at a dynamic shared-memory size, cached: the
// occupancy query is a driver call that costs microseconds per launch (small,
// launch-bound sweeps launch two kernels per step).
static int occupancy(const void* kernel, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, size_t>, int> cache;
    const auto key = std::make_pair(kernel, smem); // every device of the node is a B200
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = per_sm;
    return per_sm;
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

// persistent grids: resident CTAs per SM x SMs, capped by the work
template <class K>
static int resident_grid(K kernel, size_t smem, long long batches, int reserve = 0) {
    int per_sm = occupancy(reinterpret_cast<const void*>(kernel), smem);
    per_sm -= reserve; // slots left for the row prologue running concurrently on the aux stream
    if (per_sm < 1) per_sm = 1;
    long long g = static_cast<long long>(per_sm) * num_sms();
    if (g > batches) g = batches;
    return static_cast<int>(std::max<long long>(g, 1));
}

// Fused stage (i): rows per batch so that the per-row tables, prologue data and
// the dynamics program fit the soft shared-memory budget.
void build_custom(const GmDev& D, long long row0, long long nrows, long long* origin_out, double* t0x_out,
                  double* probs_out, unsigned long long* d_err, cudaStream_t s) {
    if (nrows <= 0) return;
    // nested adaptive Simpson recurses up to 42 simpson_rec frames (~0.5 KB each,
    // ptxas -v) per noise dimension: the per-thread stack must hold n of those chains
    size_t stack = 0;
    cudaDeviceGetLimit(&stack, cudaLimitStackSize);
    const size_t want = 4096 + static_cast<size_t>(D.n) * 42 * 640;
    if (stack < want && cudaDeviceSetLimit(cudaLimitStackSize, want) != cudaSuccess)
        throw std::runtime_error("build_custom: cannot reserve the quadrature stack");
    const size_t smem = ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16 + D.n_lits * sizeof(double);
    const long long blocks = std::min<long long>((nrows + 3) / 4, static_cast<long long>(num_sms()) * 16);
    k_build_custom<<<static_cast<unsigned>(std::max<long long>(blocks, 1)), 128, smem, s>>>(D, row0, nrows, origin_out,
                                                                                        t0x_out, probs_out, d_err);
    check_launch("build_custom");
}

namespace {
__global__ void k_origin_minmax(const long long* __restrict__ o, const uint8_t* __restrict__ f, long long n,
                                long long* mm) {
    long long lo = LLONG_MAX, hi = -1;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        if (f[i] == 0) {
            lo = o[i] < lo ? o[i] : lo;
            hi = o[i] > hi ? o[i] : hi;
        }
    for (int off = 16; off >= 1; off >>= 1) {
        const long long ol = __shfl_xor_sync(0xffffffffu, lo, off), oh = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = ol < lo ? ol : lo;
        hi = oh > hi ? oh : hi;
    }
    if ((threadIdx.x & 31) == 0 && hi >= 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}
} // namespace

void origin_minmax(const long long* origins, const uint8_t* rowflag, long long n, long long* mm, cudaStream_t s) {
    if (n <= 0) return;
    const long long blocks = std::min<long long>((n + kThreads - 1) / kThreads, 148 * 8);
    k_origin_minmax<<<static_cast<int>(blocks), kThreads, 0, s>>>(origins, rowflag, n, mm);
    check_launch("origin_minmax");
}

int build_ctas(const GmDev& D, bool jit) {
    static const char* bc = std::getenv("GM_BUILD_CTAS"); // tuning
    if (bc) return std::max(2, std::min(6, std::atoi(bc)));
    return jit && D.R >= 512 ? 2 : 3;
}

bool build_uses_qs(const GmDev& D) { return D.n_lines <= 512 && D.n_lines * 8 < 65536 && D.Wl * 8 < 32768; }

void build(const GmDev& D, long long row0, long long nrows, long long* origin_out, double* t0x_out,
           double* probs_out, unsigned long long* d_err, cudaStream_t s, const void* const* jit_ws) {
    if (nrows <= 0) return;
    if (D.family == GM_CUSTOM) {
        build_custom(D, row0, nrows, origin_out, t0x_out, probs_out, d_err, s);
        return;
    }
    const size_t mw = static_cast<size_t>(D.sumW + 1);
    static const char* bw = std::getenv("GM_BUILD_WS"); // 0: single-role k_build
    if (!(bw && bw[0] == '0')) {
        // three-role pipelined build: layout of k_build_ws in doubles
        // GM_BUILD_OPTS (GM_DIAG builds only): 16 = per-role cycle totals (printf),
        // 32 / 64 = constant / no stores (timing only, wrong rows).
        static const char* bo2 = std::getenv("GM_BUILD_OPTS");
        const int wopts = bo2 ? std::atoi(bo2) : 0;
#ifndef GM_DIAG
        if (wopts & 112)
            throw std::runtime_error("build: GM_BUILD_OPTS (16 / 32 / 64) are diagnostics of GM_DIAG builds only");
#endif
        const bool qs = build_uses_qs(D);
        const size_t fixed_d = D.n_ins + D.n_lits + 3 + (qs ? (D.pitch + 1) / 2 + (kThreads / 32) * (D.n_lines + 1) : 0);
        // two table buffers + two prologue buffers (pro_doubles: <= (5n + 2) rb + 2 for both)
        const size_t per_d = 2 * (mw + D.P_size) + 5 * static_cast<size_t>(D.n) + 2;
        // resident CTAs per SM (AOT kernels, interpreter: 3 beats 4 by 2-4 % on C2b, 2 is 19 % slower)
        const int ctas = build_ctas(D, jit_ws && jit_ws[qs ? 1 : 0]);
        const size_t budget_d = (216 / ctas) * 1024 / sizeof(double);
        if (fixed_d < budget_d) {
            long long rb = std::min<long long>(64, static_cast<long long>((budget_d - fixed_d) / per_d));
            // consumers: one (row, axis) item per thread; at least 2 filler warps
            const int nw = kThreads / 32;
            long long npw = (rb + 31) / 32;
            long long ncw = (rb * D.n + 31) / 32;
            while (rb > 8 && npw + ncw > nw - 2) {
                --rb;
                npw = (rb + 31) / 32;
                ncw = (rb * D.n + 31) / 32;
            }
            if (npw + ncw > nw - 2) ncw = std::max<long long>(1, nw - 2 - npw);
            if (rb >= 8 && npw + ncw <= nw - 1) {
                const size_t smem = (fixed_d + per_d * static_cast<size_t>(rb)) * sizeof(double);
                const long long batches = (nrows + rb - 1) / rb;
                const void* k = (jit_ws && jit_ws[qs ? 1 : 0]) ? jit_ws[qs ? 1 : 0]
                                       : (ctas == 4 ? (qs ? reinterpret_cast<const void*>(&k_build_ws<true, 4>)
                                                          : reinterpret_cast<const void*>(&k_build_ws<false, 4>))
                                          : ctas == 5 ? (qs ? reinterpret_cast<const void*>(&k_build_ws<true, 5>)
                                                            : reinterpret_cast<const void*>(&k_build_ws<false, 5>))
                                          : (qs ? reinterpret_cast<const void*>(&k_build_ws<true, 3>)
                                                : reinterpret_cast<const void*>(&k_build_ws<false, 3>)));
                if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                const int per_sm = occupancy(k, smem);
                const long long grid = std::min<long long>(batches, static_cast<long long>(std::max(per_sm, 1)) *
                                                                        num_sms());
                GmDev Dv = D;
                int rb_i = static_cast<int>(rb), npw_i = static_cast<int>(npw), ncw_i = static_cast<int>(ncw);
                int opts_i = wopts;
                void* args[] = {&Dv,    &row0,       &nrows,    &rb_i,      &npw_i, &ncw_i,
                                &opts_i, &origin_out, &t0x_out, &probs_out, &d_err};
                note_variant(KF_BUILD, "k_build_ws<%d,%d>%s", qs ? 1 : 0, ctas,
                             (jit_ws && jit_ws[qs ? 1 : 0]) ? "+NVRTC" : "");
                const cudaError_t e = cudaLaunchKernel(k, dim3(static_cast<unsigned>(std::max<long long>(grid, 1))),
                                                       dim3(kThreads), args, smem, s);
                if (e != cudaSuccess) throw std::runtime_error(std::string("build: ") + cudaGetErrorString(e));
                check_launch("build");
                return;
            }
        }
    }
    // single-role fallback (the pipelined layout does not fit)
    const size_t fixed = (kThreads / 32 + D.n_ins + D.n_lits + 2) * sizeof(double);
    const size_t extra_row = (2 * GMD_MAXD + 1) * sizeof(double) + GMD_MAXD * sizeof(int);
    const size_t q_row = (mw + D.P_size + D.n_lines) * sizeof(double) + extra_row;
    const size_t p_row = (mw + D.P_size) * sizeof(double) + extra_row;
    int tab = -1;
    long long rb = 0;
    for (size_t budget : {static_cast<size_t>(54 * 1024), kHardSmem}) { // 4 CTAs/SM
        for (int t : {TAB_Q, TAB_P}) {
            const size_t per = t == TAB_Q ? q_row : p_row;
            if (fixed >= budget) continue;
            const long long r = static_cast<long long>((budget - fixed) / per);
            if (r >= (budget != kHardSmem ? 8 : 1)) {
                tab = t;
                rb = std::min<long long>(r, kThreads);
                break;
            }
        }
        if (tab >= 0) break;
    }
    if (tab < 0) throw std::runtime_error("row too wide for the device build layout");
    const size_t smem = fixed + (tab == TAB_Q ? q_row : p_row) * static_cast<size_t>(rb);
    const long long batches = (nrows + rb - 1) / rb;
    const GmFastDiv drb = gm_fastdiv(static_cast<uint32_t>(rb));
    note_variant(KF_BUILD, "k_build<%s>", tab == TAB_Q ? "Q" : "P");
    if (tab == TAB_Q) {
        allow_smem(k_build<TAB_Q>, smem);
        k_build<TAB_Q><<<resident_grid(k_build<TAB_Q>, smem, batches), kThreads, smem, s>>>(
            D, row0, nrows, static_cast<int>(rb), drb, origin_out, t0x_out, probs_out, d_err);
    } else {
        allow_smem(k_build<TAB_P>, smem);
        k_build<TAB_P><<<resident_grid(k_build<TAB_P>, smem, batches), kThreads, smem, s>>>(
            D, row0, nrows, static_cast<int>(rb), drb, origin_out, t0x_out, probs_out, d_err);
    }
    check_launch("build");
}

template <int TAB, int LS>
static void launch_ofa(const GmDev& D, const BatchPlan& b, long long nrows, const double* mass,
                       const long long* origin, const double* t0x, const uint8_t* rowflag, const double* V,
                       double* v_in, cudaStream_t s) {
    const long long batches = (nrows + b.rb - 1) / b.rb;
    static const char* ou = std::getenv("GM_OFA_U"); // terms in flight per lane (tuning)
    // hoisted last-axis cell (row_dot_pk, software-pipelined, 2 CTAs/SM register
    // cap): C4 14.7 -> 12.0 s, C4' 12.0 -> 9.6 s. GM_OFA_PK=1 / 0 forces it on / off.
    static const char* opk = std::getenv("GM_OFA_PK");
    const int u = ou ? std::atoi(ou) : 6; // C5: U = 4 1.23 s, 6 1.14 s, 8 1.14 s
    auto k = u == 8 ? k_expect_ofa<TAB, LS, 8> : (u == 6 ? k_expect_ofa<TAB, LS, 6> : k_expect_ofa<TAB, LS, 4>);
    // hoisted last-axis cell: U = the smallest multiple of the cell period in [4, 8]
    const int qk = D.tpr % D.Wl;
    const int period = D.Wl / std::gcd(qk == 0 ? D.Wl : qk, D.Wl);
    int up = 0;
    for (int c = 4; c <= 8 && !up; ++c)
        if (c % period == 0) up = c;
    const int pk_mode = opk ? std::atoi(opk) : -1;
    // per-row setup (U shared loads, pipeline fill) pays off on long rows only:
    // C5 (27 terms per lane) 1.154 vs 1.137 s without it
    const long long per_lane = D.R / std::max(D.tpr, 1);
    if (up && !ou && (pk_mode == 1 || (pk_mode == -1 && per_lane >= 64))) {
        k = up == 4   ? k_expect_ofa_pk<TAB, LS, 4>
            : up == 5 ? k_expect_ofa_pk<TAB, LS, 5>
            : up == 6 ? k_expect_ofa_pk<TAB, LS, 6>
            : up == 7 ? k_expect_ofa_pk<TAB, LS, 7>
                      : k_expect_ofa_pk<TAB, LS, 8>;
    }
    const bool pk = up && !ou && (pk_mode == 1 || (pk_mode == -1 && per_lane >= 64));
    note_variant(KF_EXPECT_OFA, "%s<%s,%d,%d>", pk ? "k_expect_ofa_pk" : "k_expect_ofa", TAB == TAB_Q ? "Q" : "P", LS,
                 pk ? up : u);
    allow_smem(k, b.smem);
    // GM_OFA_CARVEOUT (tuning): shared-memory share of the unified L1/shared storage, in
    // percent; more CTAs per SM against fewer L1 hits for the V gathers
    static const char* oc = std::getenv("GM_OFA_CARVEOUT");
    if (oc) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(oc));
    k<<<resident_grid(k, b.smem, batches), kThreads, b.smem, s>>>(D, nrows, b.rb, gm_fastdiv(b.rb), mass, origin,
                                                                 t0x, rowflag, V, v_in);
}

void expect_ofa(const GmDev& D, long long nrows, const double* mass, const long long* origin,
                const double* t0x, const uint8_t* rowflag, const double* V, double* v_in,
                cudaStream_t s, const OfaJit* jit) {
    if (nrows <= 0) return;
    const BatchPlan b = plan_batches(D, true);
    // packed (Q, line offset) tables, opt-in (GM_OFA_PACK=1): measured slower (C5 1.126 vs
    // 0.938 s; the per-row staging of the 16-byte entries outweighs the one saved LDS)
    static const char* opack = std::getenv("GM_OFA_PACK");
    if (jit && jit->packed && (opack && opack[0] == '1') && b.tab == TAB_Q && !std::getenv("GM_OFA_U") &&
        !(std::getenv("GM_OFA_PK") && std::getenv("GM_OFA_PK")[0] == '1')) {
        const int groups = kThreads / D.tpr;
        const size_t per_row = (static_cast<size_t>(D.sumW + 1) + D.P_size + 2 * static_cast<size_t>(D.n_lines)) * 8;
        const size_t fixed = (1 + kThreads / 32) * 8; // alignment slot + group partials
        long long rb = static_cast<long long>((kSoftSmem - fixed) / per_row);
        rb = std::min<long long>(rb, kThreads);
        if (rb >= groups) {
            rb -= rb % groups;
            const size_t smem = fixed + per_row * static_cast<size_t>(rb);
            note_variant(KF_EXPECT_OFA, "k_expect_ofa_packed<NVRTC>");
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(jit->packed, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            const long long batches = (nrows + rb - 1) / rb;
            const int grid = resident_grid(jit->packed, smem, batches);
            GmDev Dv = D;
            long long nr = nrows;
            int rbi = static_cast<int>(rb);
            GmFastDiv dv = gm_fastdiv(static_cast<uint32_t>(rb));
            void* args[] = {&Dv, &nr, &rbi, &dv, &mass, &origin, &t0x, &rowflag, &V, &v_in};
            const cudaError_t e = cudaLaunchKernel(jit->packed, dim3(grid), dim3(kThreads), args, smem, s);
            if (e != cudaSuccess) throw std::runtime_error(std::string("expect_ofa: ") + cudaGetErrorString(e));
            check_launch("expect_ofa");
            return;
        }
    }
    // per-group rows (k_expect_ofa_group: no CTA-wide batch barriers), tpr >= 32;
    // GM_OFA_GROUP=0 keeps the batched shape kernel
    static const char* ogrp = std::getenv("GM_OFA_GROUP");
    if (jit && jit->group && !(ogrp && ogrp[0] == '0') && D.tpr >= 32 && b.tab == TAB_Q && b.table_in_smem == 1 &&
        !std::getenv("GM_OFA_U") && !(std::getenv("GM_OFA_PK") && std::getenv("GM_OFA_PK")[0] == '1')) {
        const int groups = kThreads / D.tpr;
        const size_t mw = static_cast<size_t>(D.sumW + 1);
        // Layout(D, groups, TAB_Q): masses, P, Q per slot, partials, then the line table (ints)
        const size_t offR = static_cast<size_t>(groups) * (mw + D.P_size + D.n_lines);
        const size_t smem = (2 * (offR + kThreads / 32) + static_cast<size_t>(D.n_lines)) * sizeof(int);
        note_variant(KF_EXPECT_OFA, "k_expect_ofa_group<NVRTC>");
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(jit->group, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        const long long slots = (nrows + groups - 1) / groups;
        const int grid = resident_grid(jit->group, smem, slots);
        GmDev Dv = D;
        long long nr = nrows;
        int rbi = groups;
        GmFastDiv dv = gm_fastdiv(static_cast<uint32_t>(groups));
        void* args[] = {&Dv, &nr, &rbi, &dv, &mass, &origin, &t0x, &rowflag, &V, &v_in};
        const cudaError_t e = cudaLaunchKernel(jit->group, dim3(grid), dim3(kThreads), args, smem, s);
        if (e != cudaSuccess) throw std::runtime_error(std::string("expect_ofa: ") + cudaGetErrorString(e));
        check_launch("expect_ofa");
        return;
    }
    const void* jit_shape = jit ? jit->shape : nullptr;
    // the consumer compiled for this row shape (gm_ofa.cuh k_expect_ofa_shape: same
    // terms, same order) replaces k_expect_ofa<Q,1,U> unless a tuning knob asks for
    // another kernel
    static const char* ou = std::getenv("GM_OFA_U");
    static const char* opk = std::getenv("GM_OFA_PK");
    if (jit_shape && b.tab == TAB_Q && b.table_in_smem == 1 && !ou && !(opk && opk[0] == '1')) {
        note_variant(KF_EXPECT_OFA, "k_expect_ofa_shape<NVRTC>");
        if (b.smem > 48 * 1024)
            cudaFuncSetAttribute(jit_shape, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(b.smem));
        const long long batches = (nrows + b.rb - 1) / b.rb;
        const int grid = resident_grid(jit_shape, b.smem, batches);
        GmDev Dv = D;
        long long nr = nrows;
        int rb = b.rb;
        GmFastDiv dv = gm_fastdiv(static_cast<uint32_t>(b.rb));
        void* args[] = {&Dv, &nr, &rb, &dv, &mass, &origin, &t0x, &rowflag, &V, &v_in};
        const cudaError_t e = cudaLaunchKernel(jit_shape, dim3(grid), dim3(kThreads), args, b.smem, s);
        if (e != cudaSuccess) throw std::runtime_error(std::string("expect_ofa: ") + cudaGetErrorString(e));
        check_launch("expect_ofa");
        return;
    }
    if (b.tab == TAB_Q) {
        if (b.table_in_smem) launch_ofa<TAB_Q, 1>(D, b, nrows, mass, origin, t0x, rowflag, V, v_in, s);
        else launch_ofa<TAB_Q, 0>(D, b, nrows, mass, origin, t0x, rowflag, V, v_in, s);
    } else {
        if (b.table_in_smem == 1) launch_ofa<TAB_P, 1>(D, b, nrows, mass, origin, t0x, rowflag, V, v_in, s);
        else if (b.table_in_smem == 2) launch_ofa<TAB_P, 2>(D, b, nrows, mass, origin, t0x, rowflag, V, v_in, s);
        else launch_ofa<TAB_P, 0>(D, b, nrows, mass, origin, t0x, rowflag, V, v_in, s);
    }
    check_launch("expect_ofa");
}

void expect_matrix(const GmDev& D, long long row0, long long r_lo, long long r_hi,
                   const double* probs, const long long* origins, const double* t0x,
                   const double* V, double* v_in, cudaStream_t s) {
    if (r_hi <= r_lo) return;
    const size_t table = static_cast<size_t>(D.n_lines) * sizeof(int);
    const bool in_smem = table <= 48 * 1024;
    const int groups = kThreads / D.tpr;
    const long long blocks_needed = (r_hi - r_lo + groups - 1) / groups;
    static const char* force = std::getenv("GM_MATRIX_KERNEL"); // "walk": per-term slab walk
    // default: element-offset-table kernel k_expect_matrix_et (L1 data-pipe bound).
    // Measured and removed (all slower on C2b): TMA bulk rings (CTA-synchronised 25.6 ms,
    // warp-specialised 28 ms), per-warp cp.async (32.8 ms), L2 bulk prefetch, offsets in
    // registers (21.3 ms), V staged per chunk of states in shared memory (23.2 ms);
    // contiguous rows per CTA (GM_CONTIG=1): equal.
    const size_t et_smem = (kThreads / 32) * sizeof(double) + static_cast<size_t>(D.R) * sizeof(int);
    // one-thread rows (TPR 1, R < 32): warp-staged cp.async chunks (k_expect_matrix_small;
    // C2a sweep 1.0 -> 0.9 ms). GM_MATRIX_SMALL=0 off, =1 also for TPR 2 / 4 (C3n: 0.35
    // vs 0.31 ms, slower)
    static const char* msm = std::getenv("GM_MATRIX_SMALL");
    const int small_max_tpr = msm ? (msm[0] == '0' ? 0 : 4) : 1;
    if (!(force && std::string(force) == "walk") && D.tpr <= small_max_tpr) {
        // rows per warp chunk: 32 / TPR, halved until the double buffers fit 56 KB per CTA
        int rpc = 32 / static_cast<int>(D.tpr);
        auto bytes = [&](int r) {
            return static_cast<size_t>((D.R + 1) / 2 + (kThreads / 32) * 2 * r * D.pitch) * sizeof(double);
        };
        // per-CTA budget 112 KB (whole 32-row chunks: every lane has a row) and all of a
        // lane's gathers in flight at once: C2a sweep 0.95 -> 0.87 ms on one box
        // (scripts/r02_small_u.sh; 56 KB / 8 in flight before). GM_SMALL_SMEM_KB,
        // GM_SMALL_U (8, 16, 32): tuning
        static const char* skb = std::getenv("GM_SMALL_SMEM_KB");
        const size_t budget = skb ? static_cast<size_t>(std::atoi(skb)) * 1024 : 2 * kSoftSmem;
        static const char* su = std::getenv("GM_SMALL_U");
        const int U = su ? std::atoi(su) : 32;
        while (rpc > 1 && bytes(rpc) > budget) rpc /= 2;
        const int chunk_len = static_cast<int>(rpc * D.pitch);
        const size_t smem = bytes(rpc);
        if (smem <= budget) {
            const long long chunks = (r_hi - r_lo + rpc - 1) / rpc;
            const long long ctas = (chunks + kThreads / 32 - 1) / (kThreads / 32);
            note_variant(KF_EXPECT_MATRIX, "k_expect_matrix_small<%d,%d>", D.tpr, U >= 32 ? 32 : U >= 16 ? 16 : 8);
            switch (D.tpr * 64 + (U >= 32 ? 32 : U >= 16 ? 16 : 8)) {
#define GM_MS(T, UU)                                                                                          \
    case T * 64 + UU: {                                                                                       \
        auto k = k_expect_matrix_small<T, UU>;                                                                \
        allow_smem(k, smem);                                                                                  \
        k<<<resident_grid(k, smem, ctas), kThreads, smem, s>>>(D, row0, r_lo, r_hi, rpc, chunk_len, probs, origins, \
                                                              t0x, V, v_in);                                  \
        check_launch("expect_matrix");                                                                        \
        return;                                                                                               \
    }
                GM_MS(1, 8) GM_MS(2, 8) GM_MS(4, 8) GM_MS(1, 16) GM_MS(2, 16) GM_MS(4, 16) GM_MS(1, 32)
                GM_MS(2, 32) GM_MS(4, 32)
#undef GM_MS
            default: break;
            }
        }
    }
    if (!(force && std::string(force) == "walk") && et_smem <= kHardSmem) {
        const long long nuw = D.n_u * D.n_w;
        const int div32 = (row0 + r_hi <= INT_MAX && nuw <= INT_MAX) ? 1 : 0;
        const GmFastDiv dn = gm_fastdiv(static_cast<uint32_t>(div32 ? nuw : 1));
        static const char* cg = std::getenv("GM_CONTIG");
        const int flags = div32 | ((cg && std::atoi(cg)) ? 2 : 0);
        // loads in flight per lane (U) and residency (MINB, the register cap): default
        // U = 12 at 6 CTAs/SM (C2b 16.3 ms); GM_ET_VARIANT=1 (8, 6) 17.1 ms, 2 (16, 4)
        // 17.7 ms, 3 (10, 6) 17.3 ms, 4 (14, 6) 17.3 ms; (8, 8) 21.4, (16, 3) 19.2, (12, 7) 18.2,
        // (12, 5) equal (17.4 vs 17.4 at 1.5 GHz), (20, 4) 20.4
        static const char* ev = std::getenv("GM_ET_VARIANT");
        const int var = ev ? std::atoi(ev) : 0;
#define GM_ET1(T, UU, MB)                                                                                   \
    {                                                                                                       \
        auto k = k_expect_matrix_et<T, UU, MB>;                                                             \
        note_variant(KF_EXPECT_MATRIX, "k_expect_matrix_et<%d,%d,%d>", T, UU, MB);                           \
        allow_smem(k, et_smem);                                                                             \
        k<<<resident_grid(k, et_smem, blocks_needed), kThreads, et_smem, s>>>(D, row0, r_lo, r_hi, dn, flags, \
                                                                             probs, origins, t0x, V, v_in); \
        check_launch("expect_matrix");                                                                      \
        return;                                                                                             \
    }
#define GM_ET(T)                                                                                            \
    case T:                                                                                                 \
        if (var == 1) GM_ET1(T, 8, 6)                                                                       \
        if (var == 2) GM_ET1(T, 16, 4)                                                                      \
        if (var == 3) GM_ET1(T, 10, 6)                                                                      \
        if (var == 4) GM_ET1(T, 14, 6)                                                                      \
        GM_ET1(T, 12, 6)
        // TPR = 32 (R in [512, 1024)): two rows per warp by default (C2b step 17.5 -> 16.9 ms
        // on a 1.45-1.5 GHz capped box); GM_ET_VARIANT=5 = the one-row kernel
        // (et2 at (14, 6) 17.3 ms, (12, 7) 17.2, (8, 8) 17.1 vs (12, 6) 16.8)
        if (D.tpr == 32 && var == 0) {
            auto k = k_expect_matrix_et2<12, 6>;
            note_variant(KF_EXPECT_MATRIX, "k_expect_matrix_et2<12,6>");
            allow_smem(k, et_smem);
            const long long pairs = (r_hi - r_lo + 1) / 2;
            k<<<resident_grid(k, et_smem, (pairs + kThreads / 32 - 1) / (kThreads / 32)), kThreads, et_smem, s>>>(
                D, row0, r_lo, r_hi, dn, flags, probs, origins, t0x, V, v_in);
            check_launch("expect_matrix");
            return;
        }
        switch (D.tpr) {
            GM_ET(1) GM_ET(2) GM_ET(4) GM_ET(8) GM_ET(16) GM_ET(32) GM_ET(64) GM_ET(128)
        default: break;
        }
#undef GM_ET
#undef GM_ET1
    }
    const size_t smem = (kThreads / 32) * sizeof(double) + (in_smem ? table : 0);
    note_variant(KF_EXPECT_MATRIX, "k_expect_matrix<%d>", in_smem ? 1 : 0);
    if (in_smem) {
        k_expect_matrix<true><<<resident_grid(k_expect_matrix<true>, smem, blocks_needed), kThreads, smem, s>>>(
            D, row0, r_lo, r_hi, probs, origins, t0x, V, v_in);
    } else {
        k_expect_matrix<false><<<resident_grid(k_expect_matrix<false>, smem, blocks_needed), kThreads, smem, s>>>(
            D, row0, r_lo, r_hi, probs, origins, t0x, V, v_in);
    }
    check_launch("expect_matrix");
}

namespace {
__global__ void k_count_positive(const double* __restrict__ p, long long n, unsigned long long* count) {
    unsigned long long c = 0;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        c += __ldcs(p + i) > 0.0 ? 1 : 0;
    for (int off = 16; off >= 1; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}
} // namespace

namespace {
// Store ceiling probe: varied doubles (hashed index, every mantissa bit toggles) with
// 16-byte evict-first stores, grid-stride over the buffer.
__global__ void __launch_bounds__(kThreads) k_store_probe(double2* __restrict__ p, long long n2, unsigned long long seed) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
        unsigned long long z = (static_cast<unsigned long long>(i) + seed) * 0x9E3779B97F4A7C15ULL;
        z ^= z >> 29;
        const double a = __longlong_as_double(static_cast<long long>((z >> 12) | 0x3FF0000000000000ULL));
        const double b = __longlong_as_double(static_cast<long long>((z << 20 >> 12) | 0x3FF0000000000000ULL));
        __stcs(p + i, make_double2(a, b));
    }
}
} // namespace

void store_probe(double* p, long long n, unsigned long long seed, cudaStream_t s) {
    if (n < 2) return;
    const long long n2 = n / 2;
    const int blocks = std::max(1, std::min(grid_for(n2, kThreads), num_sms() * 8));
    k_store_probe<<<blocks, kThreads, 0, s>>>(reinterpret_cast<double2*>(p), n2, seed);
    check_launch("store_probe");
}

unsigned long long count_positive(const double* p, long long n, unsigned long long* d_count, cudaStream_t s) {
    cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
    if (n > 0) {
        k_count_positive<<<std::max(1, std::min(grid_for(n, kThreads), num_sms() * 8)), kThreads, 0, s>>>(p, n,
                                                                                                       d_count);
        check_launch("count_positive");
    }
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, d_count, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return h;
}

// states per CTA of k_step_small (0: not applicable). Opt-in (GM_STEP_FUSED=1): measured
// slower than expect_matrix + maxmin on the small configurations it applies to (C2a
// sweep 1.2 vs 1.0 ms, C3n 0.4 vs 0.3 ms: the CTA-wide staging and the one-thread-per-
// state pass 2 serialise more than the second launch costs)
static long long step_small_spb(const GmDev& D) {
    static const char* on = std::getenv("GM_STEP_FUSED");
    if (!(on && on[0] == '1')) return 0;
    const long long nuw = D.n_u * D.n_w;
    if (D.tpr > 32 || nuw * D.tpr > kThreads) return 0;
    const long long per_state = nuw * (D.pitch + 1) * 8;
    const long long fixed = (D.R + 1) / 2 * 8;
    return std::max<long long>(0, std::min<long long>(kThreads / (nuw * D.tpr), (48 * 1024 - fixed) / per_state));
}

bool step_small_applies(const GmDev& D) { return step_small_spb(D) >= 1; }

bool step_small(const GmDev& D, long long x0, long long nx, const double* probs, long long r_base,
                const long long* origins, const double* t0x, const double* V, double* v_in, double* v_out,
                uint32_t* pol, uint32_t* wst, cudaStream_t s) {
    const long long spb = step_small_spb(D);
    if (spb < 1 || nx <= 0) return false;
    const long long nuw = D.n_u * D.n_w;
    const long long per_state = nuw * (D.pitch + 1) * 8;
    const long long fixed = (D.R + 1) / 2 * 8;
    const size_t smem = static_cast<size_t>(fixed + spb * per_state);
    const long long chunks = (nx + spb - 1) / spb;
    note_variant(KF_EXPECT_MATRIX, "k_step_small<%d>", D.tpr);
    switch (D.tpr) {
#define GM_SS(T)                                                                                                      \
    case T: {                                                                                                         \
        auto k = k_step_small<T>;                                                                                     \
        k<<<resident_grid(k, smem, chunks), kThreads, smem, s>>>(D, x0, nx, static_cast<int>(spb), probs, r_base,     \
                                                                 origins, t0x, V, v_in, v_out, pol, wst);             \
        break;                                                                                                        \
    }
        GM_SS(1) GM_SS(2) GM_SS(4) GM_SS(8) GM_SS(16) GM_SS(32)
#undef GM_SS
    default: return false;
    }
    check_launch("step_small");
    return true;
}

// k_step_warp geometry: the row re-pitch and the per-warp shared-memory slot in
// doubles (0: not applicable). GM_STEP_WARP=0 keeps expect_matrix + maxmin.
static void step_warp_plan(const GmDev& D, int& ps, int& wslot) {
    ps = wslot = 0;
    static const char* on = std::getenv("GM_STEP_WARP");
    if (on && on[0] == '0') return;
    const long long nuw = D.n_u * D.n_w;
    if (D.tpr > 4 || nuw > 512 || D.pitch > 64) return;
    int p = static_cast<int>(D.tpr); // a multiple of TPR with an odd quotient: conflict-free row reads
    while (p < D.R || (p / D.tpr) % 2 == 0) p += static_cast<int>(D.tpr);
    const long long slot = nuw * (p + 2); // rows, row values, origins
    if (slot * 8 > 24 * 1024) return; // at least 8 warps of slots per SM
    ps = p;
    wslot = static_cast<int>(slot + (slot & 1)); // 16-byte aligned slots
}

bool step_warp_applies(const GmDev& D) {
    int ps, ws;
    step_warp_plan(D, ps, ws);
    return ws > 0;
}

bool step_warp(const GmDev& D, long long x0, long long nx, const double* probs, const long long* origins,
               const double* t0x, const double* V, double* v_in, double* v_out, uint32_t* pol, uint32_t* wst,
               cudaStream_t s, const GmMirror* mir) {
    int ps, wslot;
    step_warp_plan(D, ps, wslot);
    if (wslot <= 0 || nx <= 0) return false;
    const size_t smem = (static_cast<size_t>((D.R + 1) / 2) + static_cast<size_t>(kThreads / 32) * wslot) * 8;
    const long long ctas = (nx + kThreads / 32 - 1) / (kThreads / 32);
    // gathers in flight per lane (tuning: GM_STEP_WARP_U = 8, 16, 32)
    static const char* su = std::getenv("GM_STEP_WARP_U");
    const int U = su ? std::atoi(su) : 16;
    const void* k = nullptr;
#define GM_SW(T, UU) if (D.tpr == T && U == UU) k = reinterpret_cast<const void*>(&k_step_warp<T, UU>);
    GM_SW(1, 8) GM_SW(1, 16) GM_SW(1, 32) GM_SW(2, 8) GM_SW(2, 16) GM_SW(2, 32) GM_SW(4, 8) GM_SW(4, 16) GM_SW(4, 32)
#undef GM_SW
    if (!k) return false;
    note_variant(KF_EXPECT_MATRIX, "k_step_warp<%d,%d>", static_cast<int>(D.tpr), U);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per_sm = 0;
    // GM_STEP_WARP_CTAS / GM_STEP_WARP_CARVEOUT (tuning): resident CTAs per SM, shared-memory carveout %
    static const char* sc = std::getenv("GM_STEP_WARP_CTAS");
    static const char* sv = std::getenv("GM_STEP_WARP_CARVEOUT");
    if (sv) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(sv));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, smem);
    if (sc) per_sm = std::min(per_sm, std::atoi(sc));
    const long long grid = std::max<long long>(1, std::min<long long>(ctas, std::max(per_sm, 1) * 1LL * num_sms()));
    GmDev Dv = D;
    GmMirror m0 = mir ? *mir : GmMirror{};
    void* args[] = {&Dv, &x0, &nx, &ps, &wslot, &probs, &origins, &t0x, &V, &v_in, &v_out, &pol, &wst, &m0};
    const cudaError_t e = cudaLaunchKernel(k, dim3(static_cast<unsigned>(grid)), dim3(kThreads), args, smem, s);
    if (e != cudaSuccess) throw std::runtime_error(std::string("step_warp: ") + cudaGetErrorString(e));
    return true;
}

void maxmin(const GmDev& D, long long x0, long long nx, const double* v_in, double* v_out,
            uint32_t* pol, uint32_t* wst, cudaStream_t s, const GmMirror* mir) {
    const GmMirror m0 = mir ? *mir : GmMirror{};
    if (nx <= 0) return;
    // L lanes per state, each scanning about three inputs (lane-strided, increasing u),
    // then a lowest-index-on-ties butterfly: C2b (n_u = 25) 8 lanes
    const long long nuw = D.n_u * D.n_w;
    int L = 1;
    while (L < 32 && 2 * L <= D.n_u / 3) L *= 2;
    if (nuw <= 8) L = 1;
    note_variant(KF_MAXMIN, "k_maxmin<%d>", L);
    switch (L) {
#define GM_MM(LL)                                                                                   \
    case LL:                                                                                        \
        k_maxmin<LL><<<grid_for(nx * LL, kThreads), kThreads, 0, s>>>(D, x0, nx, v_in, v_out, pol, wst, m0); \
        break;
        GM_MM(1) GM_MM(2) GM_MM(4) GM_MM(8) GM_MM(16) GM_MM(32)
#undef GM_MM
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

void simulate(const GmDev& D, const SimArgs& A, cudaStream_t s) {
    if (A.runs <= 0) return;
    const size_t smem = ((D.n_ins * sizeof(GmIns) + 15) / 16) * 16 + D.n_lits * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_simulate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_simulate<<<(A.runs + 127) / 128, 128, smem, s>>>(D, A);
    check_launch("simulate");
}

} // namespace gmk
