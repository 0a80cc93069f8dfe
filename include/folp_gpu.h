/*
 * folp_gpu.h -- the thin C ABI between the host C++ solve driver
 * (paper_2106_04756_b200/csrc/host/solver.cpp, which keeps folp::solve's
 * C++ signature, /root/reference/proj/include/folp/solver.hpp:226-228) and
 * the sm_100a CUDA engine (paper_2106_04756_b200/csrc/engine/engine.cu).
 *
 * One folp_gpu_ctx owns one presolved LP resident in HBM (CSR + CSC with
 * int32 indices, original and scaled fp64 values), every iterate buffer of
 * the PDLP loop and its own CUDA stream, so concurrent solves on one GPU
 * are independent (the reentrancy the reference bench harness relies on,
 * proj/src/bench.cpp:46-73).  Host arrays are caller-owned and copied;
 * device buffers are context-owned.  No C++ exception crosses this ABI:
 * every call returns FOLP_OK or a FOLP_E_* code from folp_c.h and
 * folp_gpu_last_error() holds the message.
 *
 * Points live in the working (scaled) space unless stated otherwise.
 */
#ifndef FOLP_GPU_H_
#define FOLP_GPU_H_

#include <stdint.h>

#include "folp_c.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct folp_gpu_ctx folp_gpu_ctx;

/* Point slots held by a context. */
enum {
  FOLP_PT_CURRENT = 0,  /* z_k of the loop (SolveDriver::current_)        */
  FOLP_PT_AVERAGE = 1,  /* materialized running average                  */
  FOLP_PT_LAST = 2,     /* last restart point (SolveDriver::last_restart_) */
  FOLP_PT_AUX = 3       /* free slot for one-shot operations              */
};

/* Chunk exit status. */
enum {
  FOLP_CHUNK_RUNNING = 0,
  FOLP_CHUNK_DONE = 1,        /* target accepted iterations reached        */
  FOLP_CHUNK_LIMIT = 2,       /* iteration or KKT-pass limit hit mid-chunk */
  FOLP_CHUNK_NONFINITE = 3,   /* pdhg_trial produced NaN/inf (solver.cpp:91-93) */
  FOLP_CHUNK_UNDERFLOW = 4    /* adaptive eta < 1e-300 (solver.cpp:196-198) */
};

/* The presolved LP (two-block form, inequality rows first).  CSR is
 * required; CSC may be NULL (then it is built from the CSR on the host,
 * columns in increasing row order like SparseMatrix::from_triplets).
 * NULL vectors are read as zeros (matrix-only contexts). */
typedef struct folp_gpu_problem {
  int64_t num_rows;
  int64_t num_cols;
  int64_t num_inequality_rows;
  int64_t nnz;
  const int64_t* row_start;
  const int64_t* row_cols;
  const double* row_values;
  const int64_t* col_start;
  const int64_t* col_rows;
  const double* col_values;
  const double* objective;
  const double* right_hand_side;
  const double* variable_lower;
  const double* variable_upper;
  double objective_constant;
} folp_gpu_problem;

/* Loop state mirrored between host and device at chunk boundaries. */
typedef struct folp_gpu_loop {
  int32_t policy;            /* FOLP_STEP_* (adaptive, constant, Malitsky-Pock) */
  int32_t status;            /* out: FOLP_CHUNK_*                         */
  int64_t target;            /* in: accepted iterations wanted            */
  int64_t accepted;          /* out                                        */
  int64_t k_total;           /* in/out: SolveDriver::k_total_              */
  int64_t t_inner;           /* in/out: SolveDriver::t_inner_              */
  int64_t step_trials;       /* in/out                                     */
  int64_t violations;        /* in/out: step_condition_violations          */
  int64_t ledger_k;          /* in/out: KktPassLedger::k_multiplies        */
  int64_t ledger_kt;         /* in/out: KktPassLedger::kt_multiplies       */
  int64_t iteration_limit;   /* in                                         */
  double kkt_pass_limit;     /* in                                         */
  double omega;              /* in: primal weight                          */
  double eta;                /* in/out: eta_hat (adaptive), eta (constant),
                                the last accepted step (Malitsky-Pock)    */
  double theta;              /* in/out: Malitsky-Pock step ratio           */
  double mp_breaking_factor; /* in: SolverParams mp_* (solver.hpp:41-43)   */
  double mp_downscaling_factor;
  double mp_interpolation_coefficient;
  double last_eta_used;      /* out                                        */
  double avg_weight;         /* out: sum of eta over the running average   */
  double last_movement;      /* out: ||z'-z||_omega^2 of the last trial    */
  double last_cross;         /* out: (y-y')'K(x'-x) of the last trial      */
  int64_t slots;             /* out: trial slots executed                  */
  const double* reduction;   /* in: [target] 1-(k+1)^-0.3 per iteration    */
  const double* growth;      /* in: [target] 1+(k+1)^-0.6 per iteration    */
} folp_gpu_loop;

/* Convergence quantities (termination.cpp:23-73) as partial sums, so the
 * host forms ConvergenceInfo with the reference's final arithmetic. */
typedef struct folp_gpu_eval {
  double c_dot_x;            /* c'x                                       */
  double q_dot_y;            /* q'y                                       */
  double bound_terms;        /* sum l_i lambda_i^+ + u_i lambda_i^-       */
  double primal_sq;          /* ||(q-Kx) with (.)^+ on >= rows||^2        */
  double dual_sq;            /* ||c - K'y - lambda||^2                    */
  double norm_q;             /* ||q||_2                                   */
  double norm_c;             /* ||c||_2                                   */
  double dual_objective;     /* q'y + const + bound terms (lp_model.cpp:150-165) */
  int32_t nonfinite;         /* point had NaN/inf (NonFiniteIterate)      */
  int32_t infinite_product;  /* lambda outside its cone (InfiniteProduct) */
} folp_gpu_eval;

/* Context lifetime. device < 0 picks $FOLP_DEVICE (default 0). */
int folp_gpu_create(const folp_gpu_problem* problem, int device,
                    folp_gpu_ctx** out);
/* Same, with the working columns renumbered: working column j is the
 * problem's column col_order[j] (a permutation of 0..n-1).  Every n-vector
 * passed to or returned by the context is in working order (the host driver
 * maps them).  Used for degree ordering of skewed columns (tree mode). */
int folp_gpu_create_ordered(const folp_gpu_problem* problem, const int64_t* col_order, int device,
                            folp_gpu_ctx** out);
void folp_gpu_destroy(folp_gpu_ctx* ctx);

/* rescale_problem (scaling.cpp:48-96) on device: ruiz_iterations Ruiz
 * (inf-norm) steps then optionally one Pock-Chambolle step; builds
 * K~ = D1 K D2, c~, q~, l~, u~.  D1/D2 are downloaded when non-NULL. */
int folp_gpu_rescale(folp_gpu_ctx* ctx, int64_t ruiz_iterations,
                     int32_t pock_chambolle, double alpha, double* row_scale,
                     double* col_scale);

/* Working-problem statistics: max|K~| (sparse_matrix.cpp:149-154) and the
 * norms used by initialize_primal_weight (solver.cpp:421-427). */
int folp_gpu_working_stats(folp_gpu_ctx* ctx, double* max_abs_entry,
                           double* norm_c, double* norm_q);

/* Scaled values and vectors of the working problem (for parity tests). */
int folp_gpu_get_working(folp_gpu_ctx* ctx, double* csr_values,
                         double* csc_values, double* objective, double* rhs,
                         double* lower, double* upper);

/* Start point in the presolved (unscaled) space: z/D then projected
 * (solver.cpp:853-865); sets CURRENT = LAST = z and clears the average. */
int folp_gpu_set_start(folp_gpu_ctx* ctx, const double* x, const double* y);

/* Raw working-space upload/download of a point slot. */
int folp_gpu_set_point(folp_gpu_ctx* ctx, int32_t which, const double* x,
                       const double* y);
int folp_gpu_get_point(folp_gpu_ctx* ctx, int32_t which, double* x,
                       double* y);

/* reduced_point (solver.cpp:495-502): unscale and clamp into the presolved
 * bounds, downloaded to x [n], y [m]. */
int folp_gpu_get_reduced_point(folp_gpu_ctx* ctx, int32_t which, double* x,
                               double* y);

/* Flush the pending averaging weight and materialize AVERAGE
 * (materialize_average, solver.cpp:509-528).  *weight = sum of etas. */
int folp_gpu_materialize_average(folp_gpu_ctx* ctx, double* weight);

/* convergence_info of a slot after reduced_point (solver.cpp:504-507).
 * raw != 0 evaluates the slot as given (already in the presolved space,
 * no unscaling or clamping), i.e. the standalone convergence_info. */
int folp_gpu_evaluate(folp_gpu_ctx* ctx, int32_t which, int32_t raw,
                      folp_gpu_eval* out);

/* linalg::all_finite of both halves of a slot (solver.cpp:731-734). */
int folp_gpu_all_finite(folp_gpu_ctx* ctx, int32_t which, int32_t* finite);

/* SparseMatrix::axis_norms (sparse_matrix.cpp:156-186) of the original
 * (working == 0) or working values; axis 0 = rows, 1 = columns. */
int folp_gpu_axis_norms(folp_gpu_ctx* ctx, int32_t axis, double p,
                        int32_t working, double* out);

/* SparseMatrix::max_abs_entry (sparse_matrix.cpp:149-154). */
int folp_gpu_max_abs_entry(folp_gpu_ctx* ctx, int32_t working, double* out);

/* Squared distances sum (x_a-x_b)^2, sum (y_a-y_b)^2 (weighted_norm and
 * diff_norm2 inputs, lp_model.cpp:167-173, linalg.hpp:47-54). */
int folp_gpu_distance(folp_gpu_ctx* ctx, int32_t a, int32_t b, double* sx,
                      double* sy);

/* normalized_duality_gap (solver.cpp:277-370) of a slot. */
int folp_gpu_ndg(folp_gpu_ctx* ctx, int32_t which, double radius,
                 double omega, double* gap);

/* Restart bookkeeping (solver.cpp:810-815): LAST = CURRENT = slot; when
 * reset_average the running average is cleared. */
int folp_gpu_restart_to(folp_gpu_ctx* ctx, int32_t which,
                        int32_t reset_average);

/* Sets LAST = CURRENT without touching the average (kNone schedule,
 * solver.cpp:771-781). */
int folp_gpu_mark_last(folp_gpu_ctx* ctx);

/* One evaluation period of the restarted loop (solver.cpp:751-798) in a
 * single asynchronous sequence with one host synchronisation:
 * materialize_average, convergence_info of CURRENT and AVERAGE and, when
 * want_gaps, restart_candidate's distances to LAST and both normalized
 * duality gaps (solver.cpp:372-393; the radius is computed on device from
 * the distances, a zero radius gives a zero gap).  gaps_valid is 0 when a
 * point is non-finite or out of its sign cone (the caller raises then). */
typedef struct folp_gpu_period {
  folp_gpu_eval current;
  folp_gpu_eval average;
  double avg_weight;
  double dist_x[2]; /* sum (x - x_last)^2 of CURRENT, AVERAGE */
  double dist_y[2]; /* sum (y - y_last)^2 of CURRENT, AVERAGE */
  double gap[2];    /* restart-candidate duality gaps of CURRENT, AVERAGE */
  int32_t gaps_valid;
  int32_t pad;
} folp_gpu_period;
int folp_gpu_evaluation_period(folp_gpu_ctx* ctx, double omega,
                               int32_t want_gaps, folp_gpu_period* out);

/* Restart commit (solver.cpp:800-815): the new reference gap
 * normalized_duality_gap(slot, radius, omega) when radius > 0 (else 0),
 * then LAST = CURRENT = slot and the average cleared; one synchronisation. */
int folp_gpu_restart_commit(folp_gpu_ctx* ctx, int32_t which, double radius,
                            double omega, double* reference_gap);

/* Runs PDHG iterations on device until loop->target steps were accepted
 * or the loop stopped (limit, non-finite, underflow).  Trials, step-size
 * decisions, the ledger and the averaging all stay on device; the host
 * sees one synchronisation per chunk. */
int folp_gpu_run_chunk(folp_gpu_ctx* ctx, folp_gpu_loop* loop);

/* Power iteration on K~'K~ (sparse_matrix.cpp:188-220) from a host start
 * vector v0 [n] (already normalised by the caller). */
int folp_gpu_spectral_norm(folp_gpu_ctx* ctx, const double* v0,
                           double relative_tol, int64_t max_iterations,
                           double* norm, int64_t* multiplies);

/* K x / K'y on the original (unscaled) or working values of the context.
 * Host vectors in, host vectors out. */
int folp_gpu_multiply(folp_gpu_ctx* ctx, int32_t working, const double* x,
                      double* out);
int folp_gpu_multiply_transpose(folp_gpu_ctx* ctx, int32_t working,
                                const double* y, double* out);

/* Reduction order of new contexts: 0 = tree (default: fast, deterministic,
 * differs from the reference's sums in the last bits), 1 = ordered (every
 * sum folded in the reference's sequential order: results bit-identical to
 * the CPU reference; parity runs).  $FOLP_REDUCTION=ordered|tree overrides. */
/* Diagnostics / tests of the exact parallel fold (engine exactfold.cuh):
 * folds `jobs` (1..4) host arrays terms[j][0..counts[j]) sequentially in
 * index order -- s = inits[j]; s += t[i] -- bit-identically to the plain loop,
 * in one cooperative launch of `grid` CTAs (0 = all co-resident).  A job with
 * init_from[j] = k >= 0 (k < j) starts from results[k] / init_div[j] instead
 * (the movement sum of solver.cpp:81-88).  reps > 0 also times that many
 * launches (ms = mean per launch).  Not part of the solve path. */
int folp_gpu_test_exact_fold(int32_t device, int32_t jobs, const double* const* terms,
                             const int64_t* counts, const double* inits,
                             const int32_t* init_from, const double* init_div,
                             int32_t grid, int32_t reps, double* results, double* ms);

void folp_gpu_set_default_reduction(int32_t ordered);
int32_t folp_gpu_reduction_ordered(const folp_gpu_ctx* ctx);
/* The mode a context created now gets (the default, or $FOLP_REDUCTION). */
int32_t folp_gpu_default_reduction(void);

/* Kernel launches issued by this context so far (for bench accounting). */
int64_t folp_gpu_launch_count(const folp_gpu_ctx* ctx);
/* Diagnostic builds only (-DFOLP_WARP_TIMES): per-warp globaltimer stamps
 * {start, units done, exit} of the most recent kernel A (slot 0) or B
 * (slot 1) launch, `max_warps` x 3 values; FOLP_E_ARG otherwise. */
int folp_gpu_debug_warp_times(folp_gpu_ctx* ctx, int32_t slot, uint64_t* out, int32_t max_warps);

/* Device time of the fused step kernels (kernel A + kernel B of every trial
 * slot) summed over all chunks since profiling was (re)enabled, measured
 * with CUDA events on the context stream around each chunk graph. */
int folp_gpu_set_profiling(folp_gpu_ctx* ctx, int32_t enabled);
int folp_gpu_chunk_timing(folp_gpu_ctx* ctx, double* chunk_ms,
                          int64_t* slots);

/* Wall time of a stretch of stream work, measured with CUDA events on the
 * context stream (start records, stop records + synchronizes). */
int folp_gpu_timer_start(folp_gpu_ctx* ctx);
int folp_gpu_timer_stop(folp_gpu_ctx* ctx, double* ms);

const char* folp_gpu_last_error(void);

/* ------------------------------------------------------------------------
 * Row shards (BASELINE.json north_star: "K is row-partitioned
 * across the 8 GPUs of one box, with NCCL over NVLink doing an allgather of
 * x before K x and a reduce-scatter/allreduce of the partial K'y and the
 * scalar reductions").  Every shard builds the full context (same LP, same
 * rescaling, bit-identical), then attaches: the PDHG loop of run_chunk works
 * on rows [r0, r1) only -- partial K'_p y_p over the shard's CSC entries,
 * all-reduce (n), replicated primal step, K_p x' + dual step on the local
 * rows, all-reduce of the 3 trial sums, identical step decision everywhere.
 * Every other engine call first reassembles y, Kx and the averaged y
 * (broadcast of each shard's rows), then runs replicated.  Collectives are
 * NCCL (one process per GPU, libnccl.so.2 loaded at run time) or an
 * in-process loopback group (one host thread per shard on one GPU; parity
 * tests).  Tree reductions only; the Malitsky-Pock policy stays single-GPU. */
#define FOLP_SHARD_NCCL 1
#define FOLP_SHARD_LOOPBACK 2
#define FOLP_NCCL_ID_BYTES 128
/* Partition axis.  ROWS (the north_star layout): rank p owns rows of K,
 * exchanges the partial K'y (n doubles) and 3 sums per trial.  COLS: rank p
 * owns columns, exchanges the partial Kx' and 2 sums (m + 2 doubles) -- the
 * cheaper exchange when m < n (configs 2, 4, 5).  AUTO: the shorter one. */
#define FOLP_SHARD_ROWS 0
#define FOLP_SHARD_COLS 1
#define FOLP_SHARD_AUTO 2

typedef struct folp_gpu_shard {
  int32_t rank;
  int32_t world;
  int32_t backend; /* FOLP_SHARD_NCCL or FOLP_SHARD_LOOPBACK */
  int32_t partition; /* FOLP_SHARD_ROWS (0), FOLP_SHARD_COLS or FOLP_SHARD_AUTO */
  unsigned char nccl_id[FOLP_NCCL_ID_BYTES]; /* folp_gpu_nccl_unique_id on rank 0 */
  void* loopback;                            /* folp_gpu_loopback_create(world) */
} folp_gpu_shard;

/* ncclGetUniqueId, to be broadcast by the caller to every rank. */
int folp_gpu_nccl_unique_id(unsigned char* out);

/* In-process group of `world` shards (one host thread each). */
int folp_gpu_loopback_create(int32_t world, void** out);
void folp_gpu_loopback_destroy(void* group);

/* Row ranges of the shards, bounds [world+1]: contiguous, balanced on
 * nonzeros + rows.  Host only. */
int folp_gpu_shard_rows(int64_t m, const int64_t* row_start, int32_t world,
                        int64_t* bounds);

/* The CSC entries of rows [r0, r1): local column starts lptr [n+1] and
 * their positions in the full CSC (pos, up to pos_capacity; may be NULL to
 * count only).  Host only. */
int folp_gpu_shard_local_csc(int64_t n, const int64_t* col_start,
                             const int64_t* col_rows, int64_t r0, int64_t r1,
                             int64_t* lptr, int64_t* pos, int64_t pos_capacity,
                             int64_t* lnnz);

/* Column partition: the CSC entries of columns [c0, c1) in CSR order
 * (local row starts lptr [m+1], their full-CSC positions in pos).  Host
 * only.  Column ranges come from folp_gpu_shard_rows(n, col_start, ...). */
int folp_gpu_shard_local_csr(int64_t m, const int64_t* col_start,
                             const int64_t* col_rows, int64_t c0, int64_t c1,
                             int64_t* lptr, int64_t* pos, int64_t pos_capacity,
                             int64_t* lnnz);

/* Turns a context into shard spec->rank of spec->world (after create and
 * rescale; the host CSR row starts and CSC of the same matrix). */
int folp_gpu_shard_attach(folp_gpu_ctx* ctx, const folp_gpu_shard* spec,
                          const int64_t* row_start, const int64_t* col_start,
                          const int64_t* col_rows);

/* *value = max over the shards (identity on an unsharded context). */
int folp_gpu_shard_max(folp_gpu_ctx* ctx, double* value);

/* The partition the context runs (FOLP_SHARD_ROWS for an unsharded one). */
int folp_gpu_shard_partition(folp_gpu_ctx* ctx, int32_t* partition);

/* r0, r1: the shard's range on its partition axis (rows or columns). */
int folp_gpu_shard_info(folp_gpu_ctx* ctx, int32_t* rank, int32_t* world,
                        int64_t* r0, int64_t* r1, int64_t* local_nnz);

#ifdef __cplusplus
}
#endif

#endif /* FOLP_GPU_H_ */
