/*
 * folp_c.h -- plain C ABI over the PDLP solve path.
 *
 * The reference exposes its solve path only as C++ (`folp::solve`,
 * /root/reference/proj/include/folp/solver.hpp:226-228) plus step-level helpers
 * (solver.hpp:121-219, termination.hpp:63-68, scaling.hpp:46-70,
 * sparse_matrix.hpp:49-79).  This header is the FFI surface a non-C++ caller
 * (ctypes, cgo, JNI) binds: plain pointers and sizes, no C++ types, no
 * exceptions crossing the boundary.  Every entry returns an int status
 * (FOLP_OK or one of the FOLP_E_* codes, which name the reference exception
 * type that the C++ API would have thrown); folp_last_error() returns the
 * message of the last failure on the calling thread.
 *
 * The same declarations are implemented twice:
 *   - libfolp_b200.so : the B200 engine (CUDA kernels, prefix folp_)
 *   - oracle/_ref/libfolp_ref.so : the compiled reference, test-only
 *     (prefix folp_ref_, see oracle/ref_capi.cpp)
 */
#ifndef FOLP_C_H_
#define FOLP_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map 1:1 onto folp exception types, types.hpp:30-75) -- */
enum {
  FOLP_OK = 0,
  FOLP_E_INVALID_ARGUMENT = 1,  /* std::invalid_argument (check_params, ...) */
  FOLP_E_RUNTIME = 2,           /* any other std::exception                 */
  FOLP_E_CUDA = 3,              /* CUDA runtime / driver failure             */
  FOLP_E_NOMEM = 4,             /* device or host allocation failed          */
  FOLP_E_DIMENSION_MISMATCH = 10,
  FOLP_E_EMPTY_MATRIX = 11,
  FOLP_E_UNSUPPORTED_NORM = 12,
  FOLP_E_NONPOSITIVE_WEIGHT = 13,
  FOLP_E_NONPOSITIVE_RADIUS = 14,
  FOLP_E_STEP_UNDERFLOW = 15,
  FOLP_E_NONFINITE = 16,
  FOLP_E_INFINITE_PRODUCT = 17,
  FOLP_E_NO_DEVICE = 18,        /* no CUDA device: the engine never falls back */
  FOLP_E_IO = 19                /* IoError, MpsParseError ("line N: ...")    */
};

/* TerminationReason, solver.hpp:72-80 (same order). */
enum {
  FOLP_TERM_OPTIMAL = 0,
  FOLP_TERM_ITERATION_LIMIT = 1,
  FOLP_TERM_KKT_PASS_LIMIT = 2,
  FOLP_TERM_TIME_LIMIT = 3,
  FOLP_TERM_NUMERICAL_ERROR = 4,
  FOLP_TERM_PRIMAL_INFEASIBLE = 5,
  FOLP_TERM_DUAL_UNBOUNDED = 6
};

/* StepPolicy / RestartSchemeKind, solver.hpp:31-32 (same order). */
enum { FOLP_STEP_ADAPTIVE = 0, FOLP_STEP_CONSTANT = 1, FOLP_STEP_MALITSKY_POCK = 2 };
enum { FOLP_RESTART_PDLP = 0, FOLP_RESTART_THEORY = 1, FOLP_RESTART_NONE = 2 };

/* LinearProgram (lp_model.hpp:38-54): K given in row-compressed form with
 * columns increasing inside each row, no duplicates, no explicit zeros
 * (exactly what SparseMatrix::row_start/row_cols/row_values expose).
 * Inequality rows (G x >= h) come first. */
typedef struct folp_lp_c {
  int64_t num_rows;
  int64_t num_cols;
  int64_t num_inequality_rows;
  int64_t nnz;
  const int64_t* row_start;   /* [num_rows + 1] */
  const int64_t* row_cols;    /* [nnz]          */
  const double* row_values;   /* [nnz]          */
  const double* objective;        /* c [num_cols] */
  const double* right_hand_side;  /* q [num_rows] */
  const double* variable_lower;   /* l [num_cols], -inf allowed */
  const double* variable_upper;   /* u [num_cols], +inf allowed */
  double objective_constant;
} folp_lp_c;

/* SolverParams (solver.hpp:34-70) minus the ostream pointer. */
typedef struct folp_params_c {
  double eps_optimal;
  double beta_sufficient;
  double beta_necessary;
  double beta_artificial;
  int32_t restart_scheme;
  int32_t step_policy;
  double theta_smoothing;
  double eps_zero;
  double mp_breaking_factor;
  double mp_downscaling_factor;
  double mp_interpolation_coefficient;
  int64_t evaluation_cadence;
  double kkt_pass_limit;
  int64_t iteration_limit;
  double time_limit_seconds;
  int64_t ruiz_iterations;
  int32_t use_pock_chambolle;
  int32_t scale_invariant_initial_primal_weight;
  double pc_alpha;
  int32_t use_presolve;
  int32_t verbosity;          /* logs go to stderr when > 0 */
  int32_t record_iterate_trace;
  int32_t reserved;
} folp_params_c;

/* ConvergenceInfo, termination.hpp:28-38 (same field order). */
typedef struct folp_info_c {
  double primal_objective;
  double dual_objective;
  double gap_abs;
  double primal_residual_norm;
  double dual_residual_norm;
  double norm_q;
  double norm_c;
} folp_info_c;

/* SolveResult (solver.hpp:97-115).  Vector outputs go to caller-owned
 * buffers (any may be NULL); list outputs are truncated at the given
 * capacity while the num_* counters report the full length. */
typedef struct folp_result_c {
  /* caller-owned outputs */
  double* primal_solution;   /* [num_cols of the raw LP] */
  double* dual_solution;     /* [num_rows of the raw LP] */
  double* reduced_costs;     /* [num_cols of the raw LP] */
  int64_t restart_capacity;
  int64_t* restart_iterations;
  int64_t trace_capacity;
  int64_t* trace_iteration;
  double* trace_kkt_passes;
  folp_info_c* trace_current;
  folp_info_c* trace_average;
  int64_t iterate_capacity;  /* IterateRecord list (working space) */
  int64_t* iterate_iteration;
  double* iterate_eta;
  double* iterate_primal;    /* [iterate_capacity * iterate_n] */
  double* iterate_dual;      /* [iterate_capacity * iterate_m] */
  /* scalar outputs */
  int64_t iterate_n;         /* presolved sizes of the iterate records */
  int64_t iterate_m;
  int32_t termination_reason;
  int32_t pad0;
  folp_info_c final_info;
  int64_t iterations;
  double kkt_passes;
  double wall_seconds;
  int64_t restarts;
  int64_t step_trials;
  int64_t step_condition_violations;
  int64_t num_restart_iterations;
  int64_t num_trace;
  int64_t num_iterates;
} folp_result_c;

/* ---- B200 engine (libfolp_b200.so) ------------------------------------ */

/* Defaults identical to SolverParams{}. */
void folp_params_default(folp_params_c* params);

/* folp::solve(lp, params, z0) -- solver.hpp:226-227.  x0/y0 may be NULL
 * (the solver.hpp:228 overload, z0 = 0). */
int folp_solve(const folp_lp_c* lp, const folp_params_c* params,
               const double* x0, const double* y0, folp_result_c* out);

/* SparseMatrix::multiply / multiply_transpose (sparse_matrix.hpp:49-55). */
int folp_multiply(const folp_lp_c* lp, const double* x, double* out);
int folp_multiply_transpose(const folp_lp_c* lp, const double* y, double* out);

/* rescale_problem (scaling.hpp:62-63): writes D1 [num_rows], D2 [num_cols]
 * and the scaled CSR values [nnz], c~, q~, l~, u~ (any output may be NULL). */
int folp_rescale(const folp_lp_c* lp, int64_t ruiz_iterations,
                 int32_t apply_pock_chambolle, double alpha, double* row_scale,
                 double* col_scale, double* scaled_values,
                 double* scaled_objective, double* scaled_rhs,
                 double* scaled_lower, double* scaled_upper);

/* convergence_info (termination.hpp:63-66). */
int folp_convergence_info(const folp_lp_c* lp, const double* x,
                          const double* y, folp_info_c* info);

/* normalized_duality_gap (solver.hpp:172-174). */
int folp_normalized_duality_gap(const folp_lp_c* lp, const double* x,
                                const double* y, double radius, double omega,
                                double* gap);

/* adaptive_step (solver.hpp:145-148): next point to x_next/y_next. */
int folp_adaptive_step(const folp_lp_c* lp, const double* x, const double* y,
                       double omega, double eta_hat, int64_t k,
                       double* x_next, double* y_next, double* eta_used,
                       double* eta_hat_next, int64_t* trials,
                       double* movement_sq, double* cross_term);

/* ---- resumable solve session (B200 engine only) ----------------------
 * folp_solve split into evaluation periods: create runs validate, presolve,
 * rescaling and the start evaluation; each advance runs `evaluations`
 * periods of evaluation_cadence PDHG iterations plus the evaluation /
 * restart step.  Running it to the end gives exactly folp_solve's result.
 * The timed variant brackets the work with CUDA events on the engine
 * stream and returns the device time. */
typedef struct folp_session folp_session;
int folp_session_create(const folp_lp_c* lp, const folp_params_c* params,
                        const double* x0, const double* y0,
                        folp_session** out);
int folp_session_advance(folp_session* s, int64_t evaluations,
                         int32_t* finished, double* device_ms);
/* iterations so far; summed device time and trial slots of the fused step
 * kernels (profiling is on for sessions); kernel launches so far. */
int folp_session_stats(folp_session* s, int64_t* iterations, double* loop_ms,
                       int64_t* loop_slots, int64_t* launches);
/* The shard partition the session's device context runs (0 rows, 1 columns;
 * rows for an unsharded one), -1 before a device context exists. */
int folp_session_partition(folp_session* s, int32_t* partition);
/* The session's device context (include/folp_gpu.h), NULL before one exists
 * (diagnostics: folp_gpu_debug_warp_times). */
struct folp_gpu_ctx* folp_session_context(folp_session* s);
int folp_session_result(folp_session* s, folp_result_c* out);
void folp_session_destroy(folp_session* s);

/* ---- multi-GPU row shards (include/folp_gpu.h) ----------
 * folp_solve / folp_session_create as shard `shard->rank` of
 * `shard->world`: every shard calls with the same LP, parameters and start
 * point (one process per GPU over NCCL, or one host thread per shard of an
 * in-process loopback group) and every shard receives the same result.
 * Extension of the reference API (it has no multi-GPU solve). */
struct folp_gpu_shard;
int folp_solve_sharded(const folp_lp_c* lp, const folp_params_c* params,
                       const double* x0, const double* y0,
                       const struct folp_gpu_shard* shard, folp_result_c* out);
int folp_session_create_sharded(const folp_lp_c* lp,
                                const folp_params_c* params, const double* x0,
                                const double* y0,
                                const struct folp_gpu_shard* shard,
                                folp_session** out);

/* malitsky_pock_step (solver.hpp:160-164): next point to x_next/y_next;
 * params supplies the mp_* factors. */
int folp_malitsky_pock_step(const folp_lp_c* lp, const double* x,
                            const double* y, double omega, double eta_prev,
                            double theta_prev, const folp_params_c* params,
                            double* x_next, double* y_next, double* eta_next,
                            double* theta_next, int64_t* trials);

/* ---- MPS and result I/O ---------------------------
 * parse_mps / parse_mps_file (mps.hpp:50-51), write_mps (:55),
 * result_to_json / write_result (result_io.hpp:26-31).  A parse error
 * returns FOLP_E_IO with the reference's "line N: message"; non-finite
 * matrix values FOLP_E_INVALID_ARGUMENT (SparseMatrix::from_triplets). */
typedef struct folp_mps folp_mps;
int folp_mps_parse(const char* text, int64_t length, folp_mps** out);
int folp_mps_parse_file(const char* path, folp_mps** out);
/* Views into the parsed instance, valid until folp_mps_destroy. */
int folp_mps_view(const folp_mps* mps, folp_lp_c* lp, const char** name,
                  int32_t* was_maximization);
void folp_mps_destroy(folp_mps* mps);
/* write_mps / result_to_json into a library-owned buffer (folp_buffer_free);
 * the result's trace must be complete (trace_capacity >= num_trace). */
int folp_mps_write(const folp_lp_c* lp, const char* name, char** text,
                   int64_t* length);
int folp_result_json(const folp_result_c* result, char** text, int64_t* length);
/* write_result: summary.json and the three solution files; the vectors have
 * num_cols / num_rows / num_cols entries. */
int folp_result_write(const folp_result_c* result, int64_t num_rows,
                      int64_t num_cols, const char* output_dir);
void folp_buffer_free(char* buffer);

/* Message of the last failing call on this thread ("" if none). */
const char* folp_last_error(void);

/* Engine build/device description for logs ("sm_100a, <device name>"). */
const char* folp_engine_info(void);

#ifdef __cplusplus
}
#endif

#endif /* FOLP_C_H_ */
