/*
 * gm_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * Plain C11, compiled by oracle/Makefile into oracle/_build/libgm_oracle.so.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as the checker. The product (libgridmdp_b200.so) never calls it.
 *
 * It restates, with the reference's exact operation order (unfused mul+add,
 * glibc libm, serial slab-order dot products), the functions of
 * /root/reference/proj/src:
 *   grid.cpp:12-45           counts / strides
 *   expr.cpp:106-288,404-480 expression grammar and evaluation
 *   noise.cpp:92-180,223-258,375-403  masses, radii, box mass, inc_beta
 *   abstraction.cpp:16-48,72-191,197-344  extents, memory, RowKernel, build, T0x, mask
 *   synthesis.cpp:18-143,165-195  dot_slab, bellman_impl, run_backward
 *   spec.cpp:51-60           absorbing states
 * Pinned against the reference itself: tests/test_oracle.py compares it with
 * the golden fixtures produced by oracle/_ref (the reference compiled here).
 */
#ifndef GM_ORACLE_H
#define GM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OC_MAXD 12

typedef struct oc_desc {
    int n, m, p; /* state / input / disturbance dims (p may be 0) */
    const double *xlb, *xub, *xeta;
    const double *ulb, *uub, *ueta;
    const double *wlb, *wub, *weta;
    const char* const* dyn; /* n expression texts */
    int n_const;
    const char* const* const_names;
    const double* const_vals;
    int family; /* 0 normal, 1 uniform, 2 exponential, 3 beta */
    int mult;   /* multiplicative noise */
    double gamma;
    const double *p1, *p2; /* sigma|a|rate|alpha ; b|beta */
    int spec_kind; /* 0 safety, 1 reachability, 2 reach-avoid */
    int horizon;
    int has_target, has_avoid;
    const double *tlo, *thi, *alo, *ahi;
} oc_desc;

typedef struct oc_model oc_model;

/* return codes: 0 ok, 2 config/parse, 3 memory, 4 domain */
int oc_model_new(const oc_desc* d, oc_model** out, char* err, int errlen);
void oc_model_free(oc_model* m);
/* n_x, n_u, n_w, rows, R, then W[0..n) ; memory_estimate (0 on overflow) */
void oc_sizes(const oc_model* m, int64_t* out, uint64_t* mem_estimate);
void oc_absorbing(const oc_model* m, uint8_t* flags);
int oc_build_matrix(oc_model* m, int64_t r0, int64_t r1, int64_t* origins, double* probs, int threads,
                    char* err, int errlen);
int oc_target_hit(oc_model* m, int64_t r0, int64_t r1, double* t0x, int threads, char* err, int errlen);
void oc_mask(const oc_model* m, int64_t rows, const int64_t* origins, double* probs);
/* One backward step for states [x0,x1): probs/origins/t0x index rows from x0*n_u*n_w
 * (matrix mode) or are NULL (on the fly). v_in_out (optional) receives the per-row
 * expected values. */
int oc_bellman_step(oc_model* m, const double* probs, const int64_t* origins, const double* t0x,
                    int64_t x0, int64_t x1, const double* v_next, double* v_out, uint32_t* pol,
                    uint32_t* wst, double* v_in_out, int threads, char* err, int errlen);
/* run_backward over all states: values n_x*(T+1) column-major, pol/wst n_x*T. */
int oc_synthesize(oc_model* m, int matrix_mode, double* values, uint32_t* pol, uint32_t* wst, int threads,
                  char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
