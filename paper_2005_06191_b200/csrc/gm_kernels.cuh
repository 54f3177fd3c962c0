// Launch interface of the sm_100a kernels (gm_kernels.cu). Host C++ only sees
// plain pointers, sizes and a cudaStream_t.
#pragma once

#include "gm_device.h"

#include <cuda_runtime.h>
#include <stdint.h>

namespace gmk {

// Pass-2 epilogue stores of a step's values into other devices' value tables (the
// multi-device "store" transport, gm_multi.cpp): value of absolute state x also goes
// to dst[i][x] for lo[i] <= x < hi[i] (peer memory over NVLink / NVSwitch).
constexpr int kMaxMirrors = 8;
struct GmMirror {
    int n = 0;
    double* dst[kMaxMirrors] = {};
    long long lo[kMaxMirrors] = {}, hi[kMaxMirrors] = {};
};

// row flags written by the row prologue
enum : uint8_t { RF_ABSORBED = 1, RF_ERROR = 2 };
// prologue options
enum : int { PF_SKIP_ABSORBED = 1, PF_T0X = 2, PF_MASSES = 4 };

// kernel families (timing / launch accounting)
enum Family { KF_PROLOGUE = 0, KF_BUILD = 1, KF_MASK = 2, KF_EXPECT_MATRIX = 3, KF_EXPECT_OFA = 4,
              KF_MAXMIN = 5, KF_MISC = 6, KF_COUNT = 7 };

struct BatchPlan {
    int tpr, groups, rb;     // threads per row, row groups per CTA, rows per CTA batch
    int tab;                 // 0: line-prefix table per row, 1: leading-prefix table per row
    int table_in_smem;       // 0: global line table; 1: line table in smem; 2: prefix table in smem
    size_t smem;             // dynamic shared memory bytes
};
BatchPlan plan_batches(const GmDev& D, bool ofa);

// Name of the kernel variant the last launch of a family used (e.g.
// "k_expect_ofa_pk<P,2,5>"), "" if none: tests check which path really ran.
const char* last_variant(int family);

void absorb_flags(const GmDev& D, uint8_t* d_flags, cudaStream_t s);
// Both passes of one stored-matrix step for states [x0, x0+nx) in one kernel when a
// state's rows fit a CTA (k_step_small); probs/origins/t0x are the matrix's arrays,
// r_base the matrix row of state x0's first row. False: not applicable (the caller
// runs expect_matrix + maxmin).
// the whole step with one warp per state (k_step_warp): R < 64 (TPR <= 4), a state's
// rows within 24 KB of shared memory; probs/origins/t0x start at x0's first row
bool step_warp_applies(const GmDev& D);
bool step_warp(const GmDev& D, long long x0, long long nx, const double* probs, const long long* origins,
               const double* t0x, const double* V, double* v_in, double* v_out, uint32_t* pol, uint32_t* wst,
               cudaStream_t s, const GmMirror* mir = nullptr);
bool step_small_applies(const GmDev& D);
bool step_small(const GmDev& D, long long x0, long long nx, const double* probs, long long r_base,
                const long long* origins, const double* t0x, const double* V, double* v_in, double* v_out,
                uint32_t* pol, uint32_t* wst, cudaStream_t s);
// Writes n (even) varied doubles (a store-bandwidth probe, not a result).
void store_probe(double* p, long long n, unsigned long long seed, cudaStream_t s);
void zero_absorbing(const GmDev& D, double* d_v, cudaStream_t s);

// Row prologue (RowKernel::compute + fill_axis_masses + box_mass,
// abstraction.cpp:72-146,187-191) for rows [row0, row0+nrows): origins (flat),
// per-axis cell masses (structure of arrays, pitch nrows), target-hit masses.
// jit: run-time compiled k_prologue (gm_jit.cpp) or nullptr for the interpreter kernel.
void prologue(const GmDev& D, long long row0, long long nrows, int flags, long long* origin_out,
              double* t0x_out, uint8_t* rowflag_out, double* mass_out,
              unsigned long long* d_err_row, cudaStream_t s, const void* jit = nullptr);

// Fused stage (i) (build_matrix body, abstraction.cpp:211-223): rows
// [row0, row0+nrows) -> origins, stored rows (and target-hit masses if t0x_out).
// Stage (i) for custom joint densities (nested quadrature per cell, k_build_custom);
// probs_out may be null (origins and target-hit masses only).
void build_custom(const GmDev& D, long long row0, long long nrows, long long* origin_out, double* t0x_out,
                  double* probs_out, unsigned long long* d_err, cudaStream_t s);
// Whether build() uses the per-warp line-prefix variant k_build_ws<true>.
bool build_uses_qs(const GmDev& D);
// Resident k_build_ws CTAs per SM (its register cap): GM_BUILD_CTAS, else 2 for the
// run-time compiled kernel on rows of >= 512 entries (store-bound: C2b 19.35 ->
// 18.6 ms, C5 shard 19.1 -> 18.3 ms, no spills), else 3 (C1, R = 169: 4.06 vs 4.43 ms).
int build_ctas(const GmDev& D, bool jit);
// min / max of the flat slab origins of rows whose flag is 0 (not absorbed, no error);
// mm[0] (init LLONG_MAX) and mm[1] (init -1) accumulate across calls
void origin_minmax(const long long* origins, const uint8_t* rowflag, long long n, long long* mm, cudaStream_t s);
// jit_ws: run-time compiled k_build_ws<false>, k_build_ws<true> (gm_jit.cpp) or nullptr.
void build(const GmDev& D, long long row0, long long nrows, long long* origin_out, double* t0x_out,
           double* probs_out, unsigned long long* d_err, cudaStream_t s, const void* const* jit_ws = nullptr);

// Expected value per row, on the fly (synthesis.cpp:100-104) from prologue data.
// run-time compiled OFA consumers for the model's row shape (gm_ofa.cuh), or null
struct OfaJit {
    const void* shape = nullptr;  // k_expect_ofa_shape
    const void* packed = nullptr; // k_expect_ofa_packed
    const void* group = nullptr;  // k_expect_ofa_group
};
void expect_ofa(const GmDev& D, long long nrows, const double* mass, const long long* origin,
                const double* t0x, const uint8_t* rowflag, const double* V, double* v_in,
                cudaStream_t s, const OfaJit* jit = nullptr);

// Expected value per row from a stored matrix (synthesis.cpp:95-99); row0 is the
// absolute index of the matrix's first row, rows [row0+r_lo, row0+r_hi) are processed
// and v_in is indexed from r_lo.
void expect_matrix(const GmDev& D, long long row0, long long r_lo, long long r_hi,
                   const double* probs, const long long* origins, const double* t0x,
                   const double* V, double* v_in, cudaStream_t s);

// min over disturbances, max over inputs per state (synthesis.cpp:112-142).
void maxmin(const GmDev& D, long long x0, long long nx, const double* v_in, double* v_out,
            uint32_t* pol, uint32_t* wst, cudaStream_t s, const GmMirror* mir = nullptr);

// Number of stored probabilities > 0 in n doubles (export_prism header, io.cpp:296-298).
unsigned long long count_positive(const double* p, long long n, unsigned long long* d_count, cudaStream_t s);

// mask_absorbing (abstraction.cpp:273-344) over stored rows.
void mask(const GmDev& D, long long r_lo, long long nrows, double* probs, const long long* origins,
          const uint8_t* inT, const uint8_t* inA, const long long* axis_off, cudaStream_t s);

// Closed-loop Monte Carlo (simulate / roll_one, sim.cpp:16-101): one thread per
// run. Grids of the synthesis result (query_policy, synthesis.cpp:230-239) next to
// the model's (GmDev: dynamics, noise, disturbance grid, region check).
struct SimArgs {
    int runs, T, reach, has_avoid, worst_case;
    double custom_sup; // custom densities: rejection envelope (custom_sup_estimate, noise.cpp:307-333)
    unsigned long long seed;
    double x0[GMD_MAXD];
    double tlo[GMD_MAXD], thi[GMD_MAXD], alo[GMD_MAXD], ahi[GMD_MAXD]; // result spec boxes
    // result grids: states (point_to_index) and inputs (index_to_point)
    double rs_lb[GMD_MAXD], rs_eta[GMD_MAXD];
    long long rs_count[GMD_MAXD], rs_stride[GMD_MAXD];
    double ru_lb[GMD_MAXD], ru_eta[GMD_MAXD];
    long long ru_stride[GMD_MAXD];
    int ru_dim;
    long long rs_n; // result states (column pitch of policy / worst_dist)
    const uint32_t* policy; // [k][rs_n] (column-major n_x x T)
    const uint32_t* worst;  // [k][n_x] of the model's state grid
    // outputs (trajectories optional, [run][k][d])
    unsigned char* satisfied;
    int* steps;
    double* states;
    double* inputs;
    double* dists;
    unsigned long long* err; // lowest run hitting a dynamics domain error
};
void simulate(const GmDev& D, const SimArgs& A, cudaStream_t s);

} // namespace gmk
