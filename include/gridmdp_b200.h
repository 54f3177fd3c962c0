/*
 * gridmdp_b200.h — C ABI of the B200-native AMYTISS engine (libgridmdp_b200.so).
 *
 * Drop-in boundary for the reference's two data-parallel stages. Every entry
 * point below names the reference C++ interface it replaces (paths relative to
 * /root/reference/proj). Signatures use plain pointers, sizes and opaque
 * handles only; no C++ or torch types cross this boundary.
 *
 *   stage (i)  MDP construction   build_matrix / build_target_hit / mask_absorbing
 *   stage (ii) Bellman synthesis  synthesize / synthesize_with_matrix / bellman_step
 *
 * Error model: every call returns a gm_code and fills an optional gm_status.
 * Codes mirror the reference's exception taxonomy (include/gridmdp/common.hpp:16-41)
 * and the CLI exit codes it maps them to (tools/gridmdp_main.cpp:204-226):
 *   GM_ERR_CONFIG (ConfigError, ParseError)  -> exit 2
 *   GM_ERR_MEMORY (MemoryError)              -> exit 3
 *   GM_ERR_DOMAIN (DomainError)              -> exit 4
 *   GM_ERR_RANGE  (std::out_of_range)        -> exit 4
 *   GM_ERR_IO     (IoError)                  -> exit 5
 *   GM_ERR_OTHER / GM_ERR_CUDA               -> exit 1
 * Messages reproduce the reference's text (e.g. a device-side domain error is
 * re-evaluated on the host for the lowest failing row, abstraction.cpp:93-101).
 *
 * There is no CPU fallback: every compute entry point needs a CUDA device and
 * returns GM_ERR_CUDA when none is usable.
 */
#ifndef GRIDMDP_B200_H
#define GRIDMDP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GM_MAX_DIMS 12

typedef enum gm_code {
    GM_OK = 0,
    GM_ERR_OTHER = 1,
    GM_ERR_CONFIG = 2,
    GM_ERR_MEMORY = 3,
    GM_ERR_DOMAIN = 4,
    GM_ERR_IO = 5,
    GM_ERR_RANGE = 6,
    GM_ERR_CUDA = 7
} gm_code;

typedef struct gm_status {
    int32_t code;          /* gm_code */
    int32_t is_parse;      /* 1 when the ConfigError is an expression ParseError */
    int64_t first_bad_row; /* lowest failing row of a device domain error, else -1 */
    char msg[2048];
} gm_status;

typedef enum gm_mode { GM_MODE_MATRIX = 0, GM_MODE_OFA = 1 } gm_mode;          /* synthesis.hpp:12 */
typedef enum gm_spec_kind { GM_SAFETY = 0, GM_REACH = 1, GM_REACH_AVOID = 2 } gm_spec_kind; /* spec.hpp:12 */

typedef struct gm_model gm_model;   /* SystemModel + Spec + SynthesisOptions (model.hpp:15, spec.hpp:14) */
typedef struct gm_matrix gm_matrix; /* device-resident TransitionMatrix row range (abstraction.hpp:22) */
typedef struct gm_result gm_result; /* SynthesisResult (synthesis.hpp:28-40), host tables */
typedef struct gm_sim gm_sim;       /* TrajectoryBatch (sim.hpp:24-27), host copy */

/* CLI/config overrides (tools/gridmdp_main.cpp:20-41); negative / NULL = keep config value. */
typedef struct gm_overrides {
    int32_t threads;
    int32_t time_steps;
    int64_t mem_budget;
    int64_t seed;
    int32_t runs;
    const char* mode;   /* "matrix" | "ofa" */
    const char* output;
} gm_overrides;

/* Sizes of print_sizes (tools/gridmdp_main.cpp:43-54) plus device-layout facts. */
typedef struct gm_sizes {
    int32_t n_dim, m_dim, p_dim;
    int64_t n_states, n_inputs, n_disturbances, pairs, rows, row_width;
    int64_t counts[GM_MAX_DIMS];
    int64_t strides[GM_MAX_DIMS];
    int64_t extents[GM_MAX_DIMS];   /* window_extents, abstraction.cpp:16-35 */
    uint64_t memory_estimate;       /* memory_estimate, abstraction.cpp:37-48 */
    int32_t spec_kind, horizon, mode, threads;
    double gamma;
    int64_t mem_budget;
    int32_t rows_per_thread_group;  /* device reduction width (identical in matrix and OFA) */
    int32_t size_overflow;          /* rows or memory_estimate overflow 64 bits (both set to 0) */
} gm_sizes;

/* ---------------------------------------------------------------- front end */

/* load_config + build_model + build_spec + build_options (config.hpp:55-70). */
gm_code gm_model_load(const char* path, const gm_overrides* ov, gm_model** out, gm_status* st);
/* parse_config from text (config.hpp:56); `name` prefixes error messages. */
gm_code gm_model_parse(const char* text, const char* name, const gm_overrides* ov, gm_model** out,
                       gm_status* st);
void gm_model_free(gm_model* m);

/* ---- the reference's in-memory types (for adapters that already hold a
 * SystemModel / Spec / SynthesisOptions, e.g. INTEGRATION.md's drop-in of
 * synthesize(const SystemModel&, const Spec&, const SynthesisOptions&)) ---- */

/* Expr::Node (expr.hpp:36-52); op numbers follow Expr::Op (expr.hpp:38-45):
 * add sub mul div pow lt le gt ge eq ne neg sin cos tan asin acos atan exp ln
 * sqrt abs min max ite literal variable = 0..26; var_class 0 x / 1 u / 2 w. */
typedef struct gm_expr_node {
    int32_t op;
    int32_t var_class;
    int32_t var_index;
    int32_t kid[3];
    double value;
} gm_expr_node;
/* One Expr: its flat node pool (children before parents) and root (expr.hpp:48-49). */
typedef struct gm_expr_desc {
    const gm_expr_node* nodes;
    int32_t n_nodes;
    int32_t root;
} gm_expr_desc;
/* UniformGrid (grid.hpp:16-46) as made by make_grid(lb, ub, eta); dim 0 = the one-point grid. */
typedef struct gm_grid_desc {
    int32_t dim;
    const double* lb;
    const double* ub;
    const double* eta;
} gm_grid_desc;
/* NoiseFamily (noise.hpp:12). */
typedef enum gm_noise_family {
    GM_NOISE_NORMAL = 0, GM_NOISE_UNIFORM = 1, GM_NOISE_EXPONENTIAL = 2, GM_NOISE_BETA = 3, GM_NOISE_CUSTOM = 4
} gm_noise_family;
/* SystemModel (model.hpp:15-33) + Spec (spec.hpp:14-20) + SynthesisOptions (synthesis.hpp:14-18). */
typedef struct gm_model_desc {
    gm_grid_desc state, input, disturbance;
    const gm_expr_desc* dynamics;   /* one per state dimension */
    int32_t n_dynamics;
    /* NoiseSpec (noise.hpp:24-66): family, mode (0 additive, 1 multiplicative), gamma,
     * param1 (sigma / a / rate / alpha) and param2 (b / beta; NULL otherwise), noise_dim
     * entries each. Custom densities: the joint pdf as an expression over x0..x{n-1}
     * (the noise coordinates) and its support box in param1 / param2. */
    int32_t noise_family;
    int32_t noise_mode;
    double gamma;
    int32_t noise_dim;
    const double* param1;
    const double* param2;
    gm_expr_desc custom_pdf;
    /* Spec: kind (gm_spec_kind), horizon, target / avoid boxes (NULL = empty). */
    int32_t spec_kind;
    int32_t horizon;
    const double* target_lo;
    const double* target_hi;
    const double* avoid_lo;
    const double* avoid_hi;
    /* SynthesisOptions: mode (gm_mode), threads (host side only), memory budget. */
    int32_t mode;
    int32_t threads;
    uint64_t mem_budget;
} gm_model_desc;

/* make_model (model.cpp:15-29) + validate_spec from the reference's in-memory types:
 * the grids, the dynamics' node pools, the noise and the spec are copied. */
gm_code gm_model_create(const gm_model_desc* desc, gm_model** out, gm_status* st);
/* save_config (config.hpp:59-60, config.cpp:270-310) of a model made from configuration text. */
gm_code gm_model_save_config(const gm_model* m, const char* path, gm_status* st);

/* Replaces the model's Spec (make_safety/make_reachability/make_reach_avoid, spec.hpp:24-26).
 * target/avoid are n_dim-long [lo, hi] vectors, or NULL for an absent box. */
gm_code gm_model_set_spec(gm_model* m, int32_t kind, int32_t horizon, const double* target_lo,
                          const double* target_hi, const double* avoid_lo, const double* avoid_hi,
                          gm_status* st);
/* Replaces mode / memory budget (SynthesisOptions, synthesis.hpp:14-18). */
gm_code gm_model_set_options(gm_model* m, int32_t mode, int64_t mem_budget, gm_status* st);

/* window_extents + memory_estimate + n_rows (abstraction.hpp:127-131, model.hpp:27-33). */
gm_code gm_model_sizes(const gm_model* m, gm_sizes* out, gm_status* st);
/* Per-state absorbing flags (absorbing_states, spec.cpp:51-60), n_states bytes. */
gm_code gm_absorbing_states(gm_model* m, uint8_t* flags_out, gm_status* st);
/* Host evaluation of mu = f(x,u,w) for one row (dynamics_image, model.cpp:33-38). */
gm_code gm_dynamics_image(const gm_model* m, int64_t row, double* mu_out, gm_status* st);
/* exec.output of the configuration after overrides ("" when unset). */
const char* gm_model_output_path(const gm_model* m);
/* Number of dynamics bytecode instructions (for tests / reporting). */
int64_t gm_model_program_size(const gm_model* m);
/* Dynamics compilation (eval_node, expr.cpp:404-501, compiled instead of
 * interpreted): 1 if the last row-kernel launch of this model used the
 * run-time compiled kernels, 0 if it used the bytecode interpreter (reason in
 * why, e.g. NVRTC missing or GM_JIT=0). compile_s: NVRTC + load seconds. */
int32_t gm_model_jit_status(const gm_model* m, double* compile_s, char* why, int64_t why_len);
/* Compiles (does not load) one run-time kernel of this model with NVRTC: kind 0
 * k_prologue, 1 / 2 the build kernel without / with per-warp line prefixes, 3 the
 * OFA consumer specialised to the row shape (k_expect_ofa_shape).
 * Needs NVRTC but no GPU; GM_ERR_OTHER carries the compiler log on failure. */
gm_code gm_model_jit_compile(const gm_model* m, int32_t kind, double* seconds, gm_status* st);

/* --------------------------------------------------------------- devices */

/* Selects the CUDA device used by subsequent calls on this host thread. */
gm_code gm_set_device(int32_t device, gm_status* st);
/* Makes the model issue all its device work on `stream` (a cudaStream_t of the
 * current device, e.g. the caller's torch stream; NULL is the legacy default
 * stream). use_own != 0 restores the model's own stream instead. */
gm_code gm_model_set_stream(gm_model* m, void* stream, int32_t use_own, gm_status* st);
/* Number of kernel launches issued by this library since load (process-wide). */
int64_t gm_launch_count(void);
/* Device time of the last launch of each kernel family, ms (0 if none).
 * family: 0 build, 1 target-hit, 2 mask, 3 expect-matrix, 4 expect-ofa, 5 maxmin. */
double gm_last_kernel_ms(int32_t family);
/* Kernel variant the last launch of a family used, e.g. "k_expect_ofa_pk<P,2,5>" or
 * "k_build_ws<1,3>+NVRTC"; "" before the first launch. */
const char* gm_last_kernel_variant(int32_t family);
/* Enables per-launch CUDA-event timing of the kernel families above (default off). */
void gm_enable_kernel_timing(int32_t on);
/* Sum of device ms per family since the last reset, and the launch count per family. */
double gm_kernel_ms_total(int32_t family);
int64_t gm_kernel_launches(int32_t family);
void gm_reset_kernel_stats(void);

/* ------------------------------------------------------------- stage (i) */

/* build_matrix (abstraction.hpp:112, abstraction.cpp:197-225) restricted to rows
 * [row_begin, row_end) (whole matrix: 0, rows). Unmasked. Device-resident. */
gm_code gm_build_matrix(gm_model* m, int64_t row_begin, int64_t row_end, gm_matrix** out,
                        gm_status* st);
/* mask_absorbing (abstraction.hpp:121, abstraction.cpp:322-344); idempotent. */
gm_code gm_mask_absorbing(gm_model* m, gm_matrix* tm, gm_status* st);
/* build_target_hit (abstraction.hpp:117, abstraction.cpp:246-271) for rows
 * [row_begin,row_end) into host memory (row_end-row_begin doubles). */
gm_code gm_build_target_hit(gm_model* m, int64_t row_begin, int64_t row_end, double* t0x_out,
                            gm_status* st);
/* Copies rows [row_begin,row_end) (absolute row indices inside the matrix's range)
 * of origins (int64) and probabilities (row-major R doubles) to host memory. */
gm_code gm_matrix_copy_rows(const gm_matrix* tm, int64_t row_begin, int64_t row_end,
                            int64_t* origins_out, double* probs_out, gm_status* st);
/* Copies the target-hit vector a shard build fused into the matrix (rows as above);
 * GM_ERR_CONFIG when the matrix carries none. */
gm_code gm_matrix_copy_t0x(const gm_matrix* tm, int64_t row_begin, int64_t row_end, double* t0x_out,
                           gm_status* st);
/* Device pointers and row range of a matrix (for stream-level callers). Row r of
 * d_probs starts at d_probs + (r - row_begin) * gm_matrix_pitch(tm): rows are padded
 * with zeros to an aligned stride (>= row_width). */
gm_code gm_matrix_info(const gm_matrix* tm, int64_t* row_begin, int64_t* row_end,
                       int64_t* row_width, const double** d_probs, const int64_t** d_origins,
                       gm_status* st);
/* Row stride of the device payload in doubles. */
int64_t gm_matrix_pitch(const gm_matrix* tm);
/* write_matrix (io.hpp:19, io.cpp:236-256): the raw `gridmdp-matrix 1` container. */
gm_code gm_matrix_write(const gm_matrix* tm, const gm_model* m, const char* path, gm_status* st);
/* export_prism (io.hpp:21, io.cpp:289-317): PRISM explicit transitions
 * "n_states n_rows n_transitions" then "src choice dst prob" for prob > 0, streamed
 * from the device-resident matrix (the nonzero count is reduced on the device). */
gm_code gm_matrix_write_prism(const gm_matrix* tm, const gm_model* m, const char* path, gm_status* st);
void gm_matrix_free(gm_matrix* tm);
/* read_matrix (io.hpp:18, io.cpp:258-283): a `gridmdp-matrix 1` container onto the
 * current device (rows padded to the device pitch), e.g. for gm_synthesize_with_matrix.
 * The container's grid / input / disturbance counts / window are checked against the
 * model when the matrix is used with it. */
gm_code gm_matrix_read(const char* path, gm_matrix** out, gm_status* st);
/* A host TransitionMatrix (abstraction.hpp:22-65: origins int64[rows], row-major
 * probs f64[rows x R]) onto the current device for the model's rows [row_begin,
 * row_begin + rows); R must equal the model's row width. */
gm_code gm_matrix_upload(const gm_model* m, int64_t row_begin, int64_t rows, const int64_t* origins,
                         const double* probs, gm_matrix** out, gm_status* st);

/* ------------------------------------------------------------ stage (ii) */

/* bellman_step (synthesis.hpp:58, synthesis.cpp:147-161): one backward step with a
 * caller-supplied v_next (host, n_states doubles). tm NULL = on-the-fly (OFA).
 * For reach specs with a matrix, tm must be masked and t0x (host, one double per
 * row of tm) supplies the target-hit vector; NULL reuses / builds tm's own.
 * policy_out / wstar_out may be NULL. */
gm_code gm_bellman_step(gm_model* m, gm_matrix* tm, const double* t0x, const double* v_next,
                        double* v_out, uint32_t* policy_out, uint32_t* wstar_out, gm_status* st);

/* Device-level sharded step for multi-GPU drivers: states [x_begin,x_end) of the
 * backward step, reading the FULL v_next (device, n_states doubles, absorbing
 * entries already zero for reach specs) and writing v_out/policy/wstar for the
 * shard (device, x_end-x_begin entries). tm NULL = OFA; otherwise tm must cover
 * exactly the shard's rows and carry its target-hit vector (gm_build_shard).
 * `stream` is a cudaStream_t (NULL = default stream). Asynchronous. */
gm_code gm_step_device(gm_model* m, gm_matrix* tm, int64_t x_begin, int64_t x_end,
                       const double* d_v_next, double* d_v_out, uint32_t* d_policy,
                       uint32_t* d_wstar, void* stream, gm_status* st);
/* Matrix for the rows of states [x_begin,x_end), masked-equivalent and with its
 * target-hit vector fused into the same build kernel (synthesize_with_matrix prologue,
 * synthesis.cpp:199-212). When *out is not NULL the matrix is rebuilt in place,
 * reusing its device buffers. */
gm_code gm_build_shard(gm_model* m, int64_t x_begin, int64_t x_end, gm_matrix** out,
                       gm_status* st);
/* gm_build_shard that also delivers the shard's origins (and, for reach specs, the
 * target-hit vector) into host memory: the rows are built in slices and each slice's
 * metadata is copied while the next slice builds (pass pinned buffers for the copies
 * to overlap; GM_BUILD_HOST_DIRECT=1 with pinned buffers makes the build kernel write
 * them to the host itself instead). Either output may be NULL. */
gm_code gm_build_shard_host(gm_model* m, int64_t state_begin, int64_t state_end, gm_matrix** out,
                            int64_t* origins_out, double* t0x_out, gm_status* st);
/* Halo of a shard (SURVEY.md §8 e): the flat state interval [*lo, *hi) that the
 * backward step of states [x_begin, x_end) reads from v_next. Slab origins do not
 * depend on the step (abstraction.cpp:103-120), so the interval is the rows'
 * [min origin, max origin + last slab offset]; rows of absorbed states (skipped
 * by the step for reach specs, synthesis.cpp:86-89) do not count. Drives the
 * multi-GPU V exchange: ranks send each other only these ranges when they are
 * much smaller than the grid, otherwise the V shards are all-gathered. */
gm_code gm_shard_reach(gm_model* m, int64_t x_begin, int64_t x_end, int64_t* lo, int64_t* hi,
                       gm_status* st);
/* OFA steps through gm_step_device keep the row prologue results (per-axis cell
 * masses, origins, T0x, row flags: Σ W_d + 3 values per row, never the R-wide rows)
 * of the stepped rows on the device, so the following steps of a sweep only recompute
 * the rows' products and dot them with V. This releases them (call at the start of a
 * sweep of new data, or to return the memory; gm_synthesize manages its own). */
gm_code gm_model_release_ofa_cache(gm_model* m, gm_status* st);
/* Per-row expected values of the model's most recent step (the v_in workspace of
 * bellman_impl, synthesis.cpp:69-109), rows of the stepped states; n doubles. */
gm_code gm_copy_row_values(gm_model* m, double* out, int64_t n, gm_status* st);
/* Checks (after a stream sync) whether a device domain error was recorded and
 * raises it with the reference's message. */
gm_code gm_check_device_errors(gm_model* m, gm_status* st);
/* Zeroes absorbing states of a device V vector in place (reach specs only). */
gm_code gm_zero_absorbing_device(gm_model* m, double* d_v, void* stream, gm_status* st);

/* synthesize (synthesis.hpp:46, synthesis.cpp:214-228) in the model's mode. */
gm_code gm_synthesize(gm_model* m, gm_result** out, gm_status* st);
/* Device time (CUDA events on the model's stream) of the model's last gm_synthesize:
 * stage (i) (0 in OFA mode) and the T backward steps, ms. */
gm_code gm_model_last_times(const gm_model* m, double* build_ms, double* sweep_ms, gm_status* st);
/* synthesize_with_matrix (synthesis.hpp:51, synthesis.cpp:199-212); t0x may be NULL
 * (built on demand), host array of tm rows otherwise. */
gm_code gm_synthesize_with_matrix(gm_model* m, gm_matrix* tm, const double* t0x,
                                  gm_result** out, gm_status* st);

/* Result tables (SynthesisResult): values n_states x (T+1) column-major f64,
 * policy / worst_dist n_states x T column-major u32, absorbing n_states u8 (reach) */
gm_code gm_result_shape(const gm_result* r, int64_t* n_states, int32_t* horizon,
                        int32_t* has_absorbing, int32_t* mode, gm_status* st);
gm_code gm_result_copy(const gm_result* r, double* values, uint32_t* policy, uint32_t* worst,
                       uint8_t* absorbing, gm_status* st);
/* The result's own tables (same layouts as gm_result_copy), valid until
 * gm_result_free: zero-copy access for bindings (absorbing NULL if empty). */
gm_code gm_result_data(const gm_result* r, const double** values, const uint32_t** policy,
                       const uint32_t** worst, const uint8_t** absorbing, gm_status* st);
/* Builds a result from caller tables (e.g. a multi-GPU driver's gathered tables). */
gm_code gm_result_from_tables(const gm_model* m, const double* values, const uint32_t* policy,
                              const uint32_t* worst, gm_result** out, gm_status* st);
/* write_results (io.hpp:13, io.cpp:142-179): the `gridmdp-results 1` container. */
gm_code gm_result_write(const gm_result* r, const char* path, gm_status* st);
void gm_result_free(gm_result* r);

/* read_results (io.hpp:14, io.cpp:181-230): a `gridmdp-results 1` container. */
gm_code gm_result_read(const char* path, gm_result** out, gm_status* st);
/* query_policy (synthesis.hpp:66, synthesis.cpp:230-239): the input vector prescribed
 * at continuous state x (n = state dim) and step k (1 <= k <= horizon) into u_out
 * (input dim doubles); GM_ERR_RANGE outside the quantized region or the horizon. */
gm_code gm_query_policy(const gm_result* r, const double* x, int32_t n, int32_t k, double* u_out,
                        gm_status* st);
/* values(point_to_index(state_grid, x), k) (gridmdp_main.cpp:133-134 value_at_x0). */
gm_code gm_result_value_at(const gm_result* r, const double* x, int32_t n, int32_t k, double* v, gm_status* st);

/* ----------------------------------------------------------- simulation */

/* exec.runs / exec.seed of the configuration after overrides (config.hpp:40-41). */
gm_code gm_model_sim_defaults(const gm_model* m, int32_t* runs, uint64_t* seed, gm_status* st);
/* simulate (sim.hpp:42-44, sim.cpp:16-101): closed-loop Monte Carlo of `runs`
 * rollouts from x0 under the result's policy and spec, one GPU thread per run;
 * worst_case selects DisturbanceMode::worst_case. Runs use independent streams
 * split from `seed` (derive_stream_seed, common.hpp:74-79) on a Philox
 * generator, so batches are reproducible but not the reference's mt19937_64
 * draws (statistical parity). want_traj records states/inputs/disturbances. */
gm_code gm_simulate(gm_model* m, const gm_result* res, const double* x0, int32_t n_x0, int32_t runs,
                    uint64_t seed, int32_t worst_case, int32_t want_traj, gm_sim** out, gm_status* st);
/* empirical_rate (sim.cpp:103-108) with the run count and satisfied count. */
gm_code gm_sim_summary(const gm_sim* s, int32_t* runs, int64_t* satisfied, double* rate, gm_status* st);
/* Per-run flags / step counts and trajectories ([run][k][d]: T+1 state rows,
 * T input and disturbance rows per run; rows past a run's steps are unused). */
gm_code gm_sim_copy(const gm_sim* s, uint8_t* satisfied, int32_t* steps, double* states, double* inputs,
                    double* dists, gm_status* st);
/* write_trajectory_csv (sim.hpp:48-50, sim.cpp:117-154). */
gm_code gm_sim_write_csv(const gm_sim* s, const char* path, gm_status* st);
void gm_sim_free(gm_sim* s);

/* ------------------------------------------------ multi-GPU, one process */

/* The reference's execution substrate is parallel_for over contiguous row
 * ranges (include/gridmdp/parallel.hpp:23-51) under run_backward
 * (src/synthesis.cpp:165-195); the engine's multi-GPU equivalent shards the
 * states into contiguous flat-index ranges, one host thread and one stream per
 * device, and exchanges V between steps (SURVEY.md §8 e). */
typedef enum gm_exchange {
    GM_XCHG_AUTO = 0,      /* halo when it moves at most half the all-gather's states */
    GM_XCHG_HALO = 1,      /* only the cutoff-bounded halos (gm_shard_reach) */
    GM_XCHG_ALLGATHER = 2  /* every shard to every device after each step */
} gm_exchange;
typedef enum gm_transport {
    GM_XPORT_NCCL = 0,     /* ncclAllGather / ncclSend+ncclRecv (NVLink / NVSwitch); distinct devices */
    GM_XPORT_PEER = 1,     /* cudaMemcpyPeerAsync after a host barrier; any device list, repeats allowed */
    GM_XPORT_STORE = 2     /* no copy: the Bellman pass-2 epilogue stores each value straight into the
                              value tables of the devices that read it (peer memory over NVLink /
                              NVSwitch), then per-step events; <= 9 devices, peer access required,
                              repeats allowed */
} gm_transport;

typedef struct gm_multi_stats {
    double build_ms;           /* stage (i) device time, max over devices (matrix mode) */
    double sweep_ms;           /* T backward steps incl. V exchanges, device time, max over devices */
    int64_t halo_states;       /* V entries one step moves with the halo plan (all devices) */
    int64_t allgather_states;  /* V entries one step moves with the all-gather */
    int32_t exchange_used;     /* GM_XCHG_HALO or GM_XCHG_ALLGATHER (0 for one device) */
    int32_t transport_used;    /* gm_transport */
    int32_t n_devices;
} gm_multi_stats;

/* A copy of the model's host description (grids, dynamics, noise, spec, options);
 * its device state is created on the device current at its first device call. */
gm_code gm_model_clone(const gm_model* m, gm_model** out, gm_status* st);

/* synthesize (synthesis.hpp:46, synthesis.cpp:214-228) over n_dev devices of this
 * process (devices[i], NULL = 0..n_dev-1): states split into n_dev equal
 * contiguous ranges, each device builds its rows (matrix mode) and steps its
 * states; V_{k+1} is exchanged per step by `exchange` over `transport`.
 * Results are bit-identical to gm_synthesize for any n_dev. stats may be NULL. */
gm_code gm_synthesize_multi(gm_model* m, int32_t n_dev, const int32_t* devices, int32_t exchange,
                            int32_t transport, gm_result** out, gm_multi_stats* stats, gm_status* st);

/* Measurement only: writes n varied doubles (16-byte evict-first stores) to a device
 * buffer on `stream` — the store-bandwidth ceiling stage (i) is compared with. */
gm_code gm_store_probe(double* d_buf, int64_t n, uint64_t seed, void* stream, gm_status* st);

/* Large device blocks (>= 64 MB, e.g. stored matrices) are kept for reuse after
 * release; this returns them to the driver. */
void gm_release_cached_memory(void);

#ifdef __cplusplus
}
#endif

#endif /* GRIDMDP_B200_H */
