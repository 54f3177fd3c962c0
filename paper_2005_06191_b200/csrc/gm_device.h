// Plain-data device descriptor shared by the host front end (C++) and the
// sm_100a kernels (CUDA). Passed to kernels by value (kernel parameter space).
#pragma once

#ifdef __CUDACC_RTC__ // run-time compilation (gm_jit.cpp): no system headers
typedef unsigned char uint8_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned long long uintptr_t;
#else
#include <stdint.h>
#endif

#define GMD_MAXD 12     // max state / input / disturbance dimensions on device
#define GMD_MAXREGS 32  // max dynamics-interpreter registers per row

enum GmFamily { GM_NORMAL = 0, GM_UNIFORM = 1, GM_EXPONENTIAL = 2, GM_BETA = 3, GM_CUSTOM = 4 };
enum GmCut { GM_CUT_NONE = 0, GM_CUT_DEGENERATE = 1, GM_CUT_RADIUS = 2 };
enum GmSpecKind { GM_SPEC_SAFETY = 0, GM_SPEC_REACH = 1, GM_SPEC_REACH_AVOID = 2 };
enum GmModeInt { GM_MODE_MATRIX_ = 0, GM_MODE_OFA_ = 1 };

// Dynamics bytecode: register machine, lazy ite through jumps.
enum GmOpCode : uint8_t {
    GI_LIT, GI_LDX, GI_LDU, GI_LDW,
    GI_ADD, GI_SUB, GI_MUL, GI_DIV, GI_POW,
    GI_LT, GI_LE, GI_GT, GI_GE, GI_EQ, GI_NE,
    GI_NEG, GI_SIN, GI_COS, GI_TAN, GI_ASIN, GI_ACOS, GI_ATAN, GI_EXP, GI_LN, GI_SQRT, GI_ABS,
    GI_MIN, GI_MAX,
    GI_JZ,   // if reg[a] == 0.0 jump to arg
    GI_JMP   // jump to arg
};

struct GmIns {
    uint8_t op;
    uint8_t dst;
    uint8_t a;
    uint8_t b;
    int32_t arg; // literal index / variable index / jump target
};

// Bounds / layout checks of the checked build (libgridmdp_b200_checked.so, -DGM_CHECKED;
// compute-sanitizer is not available on the GPU pool): a failed check prints the
// condition and traps, which surfaces as a launch failure of the calling API.
#if defined(__CUDACC__) && defined(GM_CHECKED)
#define GM_CHECK(c)                                                                                      \
    do {                                                                                                 \
        if (!(c)) {                                                                                      \
            printf("GM_CHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__,            \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                         \
            __trap();                                                                                    \
        }                                                                                                \
    } while (0)
__device__ __forceinline__ unsigned gm_dyn_smem_bytes() {
    unsigned r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
#else
#define GM_CHECK(c) \
    do {            \
    } while (0)
#endif

// Device error codes recorded per failing row
enum GmDevErr { GE_NONE = 0, GE_EXPR = 1, GE_BETA = 2 };

// Division by a loop-invariant divisor d >= 1 for 0 <= n < 2^31:
// q = (umulhi(n, m) + n) >> s with s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1.
struct GmFastDiv {
    uint32_t d, m, s;
#ifdef __CUDACC__
    __device__ __forceinline__ int div(int n) const {
        const uint32_t t = __umulhi(static_cast<uint32_t>(n), m);
        return static_cast<int>((static_cast<uint64_t>(t) + static_cast<uint32_t>(n)) >> s);
    }
#endif
};

#ifndef __CUDACC_RTC__
static inline GmFastDiv gm_fastdiv(uint32_t d) {
    GmFastDiv f;
    f.d = d ? d : 1;
    uint32_t s = 0;
    while ((1ULL << s) < f.d) ++s;
    f.s = s;
    f.m = static_cast<uint32_t>(((1ULL << 32) * ((1ULL << s) - f.d)) / f.d + 1);
    return f;
}
#endif

struct GmDev {
    int n, m, p;             // state / input / disturbance dims
    int family, mult, cut;   // noise family, multiplicative flag, GmCut
    int spec_kind, has_avoid;
    int tpr;                 // threads per row in the expected-value kernels
    int n_ins, n_lits, nregs;
    long long n_x, n_u, n_w, rows, R;
    long long pitch;         // row stride of stored matrices in doubles (R padded to an aligned granule)

    long long xcount[GMD_MAXD], xstride[GMD_MAXD];
    long long ustride[GMD_MAXD], wstride[GMD_MAXD];
    double xlb[GMD_MAXD], xeta[GMD_MAXD];
    double ulb[GMD_MAXD], ueta[GMD_MAXD];
    double wlb[GMD_MAXD], weta[GMD_MAXD];

    double radius[GMD_MAXD];
    double s[GMD_MAXD];      // normal: sigma*sqrt(2) (noise.cpp:96); else param1
    double inv_s[GMD_MAXD];  // normal: 1 / s (the device scales erf arguments by a multiply)
    double p2[GMD_MAXD];     // uniform b / beta beta
    double tlo[GMD_MAXD], thi[GMD_MAXD], alo[GMD_MAXD], ahi[GMD_MAXD];
    double sup_lo[GMD_MAXD], sup_hi[GMD_MAXD]; // custom density support (noise coordinates)
    int W[GMD_MAXD];
    int mass_off[GMD_MAXD + 1];

    // slab layout: virtual leading axis when n == 1, so every row factors as
    // p(a, j, k) = (P[a] * mm[j]) * ml[k] with P the prefix product over the
    // leading axes (abstraction.cpp:150-159 association).
    int sumW;                // sum of W over real axes
    int s_axes;              // number of axes in the prefix table (n_eff - 2)
    int P_size;              // prod of W over the prefix axes
    int Wm, Wl;              // W of the last two (effective) axes
    int n_lines;             // R / Wl
    int mm_off, ml_off;      // offsets of the last two axes' masses (n == 1: mm_off = sumW, a 1.0 slot)
    GmFastDiv div_Wm, div_Wl, div_lines, div_P, div_mw; // n / d for n < 2^31 by multiply-shift
    GmFastDiv div_W[GMD_MAXD];
    // prefix-table index a = sum_d j_d * Ps[d] over the s_axes leading axes (last fastest)
    int Ps[GMD_MAXD];
    GmFastDiv div_Ps[GMD_MAXD];
    // row decode by multiply-shift when every row index is < 2^31 (idx32)
    int idx32;
    GmFastDiv div_nw, div_nu, div_xs[GMD_MAXD], div_us[GMD_MAXD], div_ws[GMD_MAXD];

    int entry[GMD_MAXD + 2]; // bytecode offsets of the n dynamics expressions (+ the custom pdf at n)
    const GmIns* prog;
    const double* lits;
    const int* line_off;     // n_lines relative flat offsets of slab lines
    const unsigned char* absorb; // n_x flags (reach specs), may be null
    // stage (i): optional second destinations of the origins / target-hit values of a
    // build launch (launch-relative, like its origin_out / t0x_out): pinned host memory
    // the kernel writes directly (gm_build_shard_host), or null
    long long* origin_host;
    double* t0x_host;
};
