// capi.cpp -- include/folp_c.h on top of the C++ folp API.
//
// Exceptions never cross this boundary: each entry maps the folp exception
// type to its FOLP_E_* code and keeps the message for folp_last_error().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <cstring>
#include <exception>
#include <string>

#include "device.hpp"
#include "folp/lp_model.hpp"
#include "folp/mps.hpp"
#include "folp/result_io.hpp"
#include "folp/scaling.hpp"
#include "folp/solver.hpp"
#include "folp/termination.hpp"
#include "folp_c.h"
#include "session.hpp"
#include "parallel.hpp"
#include "sparse_access.hpp"

namespace {

using namespace folp;

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return FOLP_OK;
  } catch (const DimensionMismatch& e) {
    g_err = e.what();
    return FOLP_E_DIMENSION_MISMATCH;
  } catch (const EmptyMatrix& e) {
    g_err = e.what();
    return FOLP_E_EMPTY_MATRIX;
  } catch (const UnsupportedNorm& e) {
    g_err = e.what();
    return FOLP_E_UNSUPPORTED_NORM;
  } catch (const NonPositiveWeight& e) {
    g_err = e.what();
    return FOLP_E_NONPOSITIVE_WEIGHT;
  } catch (const NonPositiveRadius& e) {
    g_err = e.what();
    return FOLP_E_NONPOSITIVE_RADIUS;
  } catch (const StepSizeUnderflow& e) {
    g_err = e.what();
    return FOLP_E_STEP_UNDERFLOW;
  } catch (const NonFiniteIterate& e) {
    g_err = e.what();
    return FOLP_E_NONFINITE;
  } catch (const InfiniteProduct& e) {
    g_err = e.what();
    return FOLP_E_INFINITE_PRODUCT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FOLP_E_INVALID_ARGUMENT;
  } catch (const IoError& e) {
    g_err = e.what();
    return FOLP_E_IO;
  } catch (const DeviceError& e) {
    g_err = e.what();
    return std::strstr(e.what(), "no CUDA device") ? FOLP_E_NO_DEVICE : FOLP_E_CUDA;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return FOLP_E_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FOLP_E_RUNTIME;
  }
}

// Fast ingestion when the CSR is already canonical (strictly increasing
// columns, in range, finite nonzero values): that is exactly the matrix
// from_triplets would build, so the O(nnz log nnz) sort is skipped.
SparseMatrix matrix_from_csr(const folp_lp_c* in) {
  const int64_t m = in->num_rows, n = in->num_cols, nnz = in->nnz;
  if (m < 0 || n < 0 || nnz < 0 || in->row_start == nullptr || in->row_start[0] != 0 ||
      in->row_start[m] != nnz) {
    throw DimensionMismatch("folp_lp_c: inconsistent row_start");
  }
  for (int64_t r = 0; r < m; ++r) {
    if (in->row_start[r + 1] < in->row_start[r]) {
      throw DimensionMismatch("folp_lp_c: decreasing row_start");
    }
  }
  // canonical CSR (strictly increasing columns, finite nonzero values):
  // taken as is, checked and copied on all host cores
  std::vector<char> ok(64, 1);
  host::parallel_for(m, [&](int64_t r0, int64_t r1, int t) {
    for (int64_t r = r0; r < r1 && ok[t]; ++r) {
      const int64_t b = in->row_start[r], e = in->row_start[r + 1];
      for (int64_t k = b; k < e; ++k) {
        const int64_t c = in->row_cols[k];
        const double v = in->row_values[k];
        if (c < 0 || c >= n || v == 0.0 || !std::isfinite(v) ||
            (k > b && c <= in->row_cols[k - 1])) {
          ok[t] = 0;
          break;
        }
      }
    }
  }, nnz + m);
  const bool canonical = std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
  if (canonical) {
    return SparseMatrixAccess::build(m, n, host::parallel_copy(in->row_start, m + 1),
                                     host::parallel_copy(in->row_cols, nnz),
                                     host::parallel_copy(in->row_values, nnz));
  }
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(nnz));
  for (int64_t r = 0; r < m; ++r) {
    for (int64_t k = in->row_start[r]; k < in->row_start[r + 1]; ++k) {
      t.push_back({r, in->row_cols[k], in->row_values[k]});
    }
  }
  return SparseMatrix::from_triplets(m, n, t);
}

LinearProgram to_lp(const folp_lp_c* in) {
  LinearProgram lp;
  lp.constraint_matrix = matrix_from_csr(in);
  const std::size_t n = static_cast<std::size_t>(in->num_cols);
  const std::size_t m = static_cast<std::size_t>(in->num_rows);
  lp.objective = host::parallel_copy(in->objective, static_cast<int64_t>(n));
  lp.right_hand_side = host::parallel_copy(in->right_hand_side, static_cast<int64_t>(m));
  lp.variable_lower = host::parallel_copy(in->variable_lower, static_cast<int64_t>(n));
  lp.variable_upper = host::parallel_copy(in->variable_upper, static_cast<int64_t>(n));
  lp.num_inequality_rows = in->num_inequality_rows;
  lp.objective_constant = in->objective_constant;
  return lp;
}

SolverParams to_params(const folp_params_c* p) {
  SolverParams s;
  s.eps_optimal = p->eps_optimal;
  s.beta_sufficient = p->beta_sufficient;
  s.beta_necessary = p->beta_necessary;
  s.beta_artificial = p->beta_artificial;
  s.restart_scheme = static_cast<RestartSchemeKind>(p->restart_scheme);
  s.step_policy = static_cast<StepPolicy>(p->step_policy);
  s.theta_smoothing = p->theta_smoothing;
  s.eps_zero = p->eps_zero;
  s.mp_breaking_factor = p->mp_breaking_factor;
  s.mp_downscaling_factor = p->mp_downscaling_factor;
  s.mp_interpolation_coefficient = p->mp_interpolation_coefficient;
  s.evaluation_cadence = p->evaluation_cadence;
  s.kkt_pass_limit = p->kkt_pass_limit;
  s.iteration_limit = p->iteration_limit;
  s.time_limit_seconds = p->time_limit_seconds;
  s.ruiz_iterations = p->ruiz_iterations;
  s.use_pock_chambolle = p->use_pock_chambolle != 0;
  s.pc_alpha = p->pc_alpha;
  s.scale_invariant_initial_primal_weight = p->scale_invariant_initial_primal_weight != 0;
  s.use_presolve = p->use_presolve != 0;
  s.verbosity = p->verbosity;
  s.log_stream = nullptr;
  s.record_iterate_trace = p->record_iterate_trace != 0;
  return s;
}

folp_info_c to_info(const ConvergenceInfo& i) {
  return folp_info_c{i.primal_objective,   i.dual_objective,     i.gap_abs,
                     i.primal_residual_norm, i.dual_residual_norm, i.norm_q,
                     i.norm_c};
}

void put(const std::vector<double>& v, double* out) {
  if (out != nullptr && !v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(double));
}

PrimalDualPoint point(const folp_lp_c* lp, const double* x, const double* y) {
  PrimalDualPoint z;
  z.primal.assign(x, x + lp->num_cols);
  z.dual.assign(y, y + lp->num_rows);
  return z;
}

void export_result(const SolveResult& r, folp_result_c* out) {
  put(r.primal_solution, out->primal_solution);
  put(r.dual_solution, out->dual_solution);
  put(r.reduced_costs, out->reduced_costs);
  out->termination_reason = static_cast<int32_t>(r.termination_reason);
  out->final_info = to_info(r.final_info);
  out->iterations = r.iterations;
  out->kkt_passes = r.kkt_passes;
  out->wall_seconds = r.wall_seconds;
  out->restarts = r.restarts;
  out->step_trials = r.step_trials;
  out->step_condition_violations = r.step_condition_violations;
  out->num_restart_iterations = static_cast<int64_t>(r.restart_iterations.size());
  for (int64_t i = 0; i < out->num_restart_iterations && i < out->restart_capacity; ++i) {
    out->restart_iterations[i] = r.restart_iterations[i];
  }
  out->num_trace = static_cast<int64_t>(r.trace.size());
  for (int64_t i = 0; i < out->num_trace && i < out->trace_capacity; ++i) {
    const TraceEntry& e = r.trace[static_cast<std::size_t>(i)];
    if (out->trace_iteration) out->trace_iteration[i] = e.iteration;
    if (out->trace_kkt_passes) out->trace_kkt_passes[i] = e.kkt_passes;
    if (out->trace_current) out->trace_current[i] = to_info(e.current);
    if (out->trace_average) out->trace_average[i] = to_info(e.average);
  }
  out->num_iterates = static_cast<int64_t>(r.iterate_trace.size());
  out->iterate_n = r.iterate_trace.empty()
                       ? 0
                       : static_cast<int64_t>(r.iterate_trace[0].point.primal.size());
  out->iterate_m = r.iterate_trace.empty()
                       ? 0
                       : static_cast<int64_t>(r.iterate_trace[0].point.dual.size());
  for (int64_t i = 0; i < out->num_iterates && i < out->iterate_capacity; ++i) {
    const IterateRecord& rec = r.iterate_trace[static_cast<std::size_t>(i)];
    if (out->iterate_iteration) out->iterate_iteration[i] = rec.iteration;
    if (out->iterate_eta) out->iterate_eta[i] = rec.eta_used;
    if (out->iterate_primal) put(rec.point.primal, out->iterate_primal + i * out->iterate_n);
    if (out->iterate_dual) put(rec.point.dual, out->iterate_dual + i * out->iterate_m);
  }
}

SolveResult import_result(const folp_result_c* in, int64_t m, int64_t n) {
  SolveResult r;
  auto vec = [](const double* p, int64_t k) {
    return p != nullptr ? std::vector<double>(p, p + k) : std::vector<double>();
  };
  r.primal_solution = vec(in->primal_solution, n);
  r.dual_solution = vec(in->dual_solution, m);
  r.reduced_costs = vec(in->reduced_costs, n);
  r.termination_reason = static_cast<TerminationReason>(in->termination_reason);
  auto info = [](const folp_info_c& i) {
    ConvergenceInfo o;
    o.primal_objective = i.primal_objective;
    o.dual_objective = i.dual_objective;
    o.gap_abs = i.gap_abs;
    o.primal_residual_norm = i.primal_residual_norm;
    o.dual_residual_norm = i.dual_residual_norm;
    o.norm_q = i.norm_q;
    o.norm_c = i.norm_c;
    return o;
  };
  r.final_info = info(in->final_info);
  r.iterations = in->iterations;
  r.kkt_passes = in->kkt_passes;
  r.wall_seconds = in->wall_seconds;
  r.restarts = in->restarts;
  r.step_trials = in->step_trials;
  r.step_condition_violations = in->step_condition_violations;
  if (in->num_trace > in->trace_capacity) {
    throw std::invalid_argument("result: trace truncated (trace_capacity < num_trace)");
  }
  for (int64_t i = 0; i < in->num_trace; ++i) {
    TraceEntry e;
    e.iteration = in->trace_iteration[i];
    e.kkt_passes = in->trace_kkt_passes[i];
    e.current = info(in->trace_current[i]);
    e.average = info(in->trace_average[i]);
    r.trace.push_back(e);
  }
  return r;
}

char* export_text(const std::string& s, int64_t* length) {
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  if (buf == nullptr) throw std::bad_alloc();
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  *length = static_cast<int64_t>(s.size());
  return buf;
}

}  // namespace

struct folp_mps {
  folp::MpsInstance inst;
};

struct folp_session {
  std::unique_ptr<folp::SolveSession> s;
};

extern "C" {

void folp_params_default(folp_params_c* p) {
  const SolverParams s;
  std::memset(p, 0, sizeof(*p));
  p->eps_optimal = s.eps_optimal;
  p->beta_sufficient = s.beta_sufficient;
  p->beta_necessary = s.beta_necessary;
  p->beta_artificial = s.beta_artificial;
  p->restart_scheme = static_cast<int32_t>(s.restart_scheme);
  p->step_policy = static_cast<int32_t>(s.step_policy);
  p->theta_smoothing = s.theta_smoothing;
  p->eps_zero = s.eps_zero;
  p->mp_breaking_factor = s.mp_breaking_factor;
  p->mp_downscaling_factor = s.mp_downscaling_factor;
  p->mp_interpolation_coefficient = s.mp_interpolation_coefficient;
  p->evaluation_cadence = s.evaluation_cadence;
  p->kkt_pass_limit = s.kkt_pass_limit;
  p->iteration_limit = s.iteration_limit;
  p->time_limit_seconds = s.time_limit_seconds;
  p->ruiz_iterations = s.ruiz_iterations;
  p->use_pock_chambolle = s.use_pock_chambolle ? 1 : 0;
  p->pc_alpha = s.pc_alpha;
  p->scale_invariant_initial_primal_weight = s.scale_invariant_initial_primal_weight ? 1 : 0;
  p->use_presolve = s.use_presolve ? 1 : 0;
}

int folp_solve(const folp_lp_c* lp_in, const folp_params_c* p, const double* x0,
               const double* y0, folp_result_c* out) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    const LinearProgram lp = to_lp(lp_in);
    if (std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr, "[folp timing] folp_solve to_lp %.4fs\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    const SolverParams params = to_params(p);
    SolveResult r;
    if (x0 == nullptr && y0 == nullptr) {
      r = solve(lp, params);  // the origin: nothing to build or upload
    } else {
      PrimalDualPoint z0;
      z0.primal.assign(static_cast<std::size_t>(lp_in->num_cols), 0.0);
      z0.dual.assign(static_cast<std::size_t>(lp_in->num_rows), 0.0);
      if (x0 != nullptr) z0.primal.assign(x0, x0 + lp_in->num_cols);
      if (y0 != nullptr) z0.dual.assign(y0, y0 + lp_in->num_rows);
      r = solve(lp, params, z0);
    }
    if (std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr, "[folp timing] folp_solve solved %.4fs\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    export_result(r, out);
    if (std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr, "[folp timing] folp_solve exported %.4fs\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
  });
}

int folp_multiply(const folp_lp_c* lp_in, const double* x, double* out) {
  return guarded([&] {
    const SparseMatrix k = matrix_from_csr(lp_in);
    k.multiply(std::span<const double>(x, static_cast<std::size_t>(lp_in->num_cols)),
               std::span<double>(out, static_cast<std::size_t>(lp_in->num_rows)));
  });
}

int folp_multiply_transpose(const folp_lp_c* lp_in, const double* y, double* out) {
  return guarded([&] {
    const SparseMatrix k = matrix_from_csr(lp_in);
    k.multiply_transpose(std::span<const double>(y, static_cast<std::size_t>(lp_in->num_rows)),
                         std::span<double>(out, static_cast<std::size_t>(lp_in->num_cols)));
  });
}

int folp_rescale(const folp_lp_c* lp_in, int64_t ruiz_iterations, int32_t apply_pc,
                 double alpha, double* row_scale, double* col_scale, double* scaled_values,
                 double* scaled_objective, double* scaled_rhs, double* scaled_lower,
                 double* scaled_upper) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const ScaledProblem s = rescale_problem(lp, ruiz_iterations, apply_pc != 0, alpha);
    put(s.scaling.row_scale, row_scale);
    put(s.scaling.col_scale, col_scale);
    if (scaled_values != nullptr) {
      const auto v = s.lp.constraint_matrix.row_values();
      if (!v.empty()) std::memcpy(scaled_values, v.data(), v.size() * sizeof(double));
    }
    put(s.lp.objective, scaled_objective);
    put(s.lp.right_hand_side, scaled_rhs);
    put(s.lp.variable_lower, scaled_lower);
    put(s.lp.variable_upper, scaled_upper);
  });
}

int folp_convergence_info(const folp_lp_c* lp_in, const double* x, const double* y,
                          folp_info_c* info) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    *info = to_info(convergence_info(
        lp, std::span<const double>(x, static_cast<std::size_t>(lp_in->num_cols)),
        std::span<const double>(y, static_cast<std::size_t>(lp_in->num_rows))));
  });
}

int folp_normalized_duality_gap(const folp_lp_c* lp_in, const double* x, const double* y,
                                double radius, double omega, double* gap) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    *gap = normalized_duality_gap(lp, point(lp_in, x, y), radius, omega);
  });
}

int folp_adaptive_step(const folp_lp_c* lp_in, const double* x, const double* y, double omega,
                       double eta_hat, int64_t k, double* x_next, double* y_next,
                       double* eta_used, double* eta_hat_next, int64_t* trials,
                       double* movement_sq, double* cross_term) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const AdaptiveStepResult r = adaptive_step(lp, point(lp_in, x, y), omega, eta_hat, k);
    put(r.next.primal, x_next);
    put(r.next.dual, y_next);
    *eta_used = r.eta_used;
    *eta_hat_next = r.eta_hat_next;
    *trials = r.trials;
    *movement_sq = r.movement_sq;
    *cross_term = r.cross_term;
  });
}

int folp_malitsky_pock_step(const folp_lp_c* lp_in, const double* x, const double* y,
                            double omega, double eta_prev, double theta_prev,
                            const folp_params_c* p, double* x_next, double* y_next,
                            double* eta_next, double* theta_next, int64_t* trials) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const MalitskyPockResult r =
        malitsky_pock_step(lp, point(lp_in, x, y), omega, eta_prev, theta_prev, to_params(p));
    put(r.next.primal, x_next);
    put(r.next.dual, y_next);
    *eta_next = r.eta_next;
    *theta_next = r.theta_next;
    *trials = r.trials;
  });
}

int folp_session_create_sharded(const folp_lp_c* lp_in, const folp_params_c* p,
                                const double* x0, const double* y0,
                                const folp_gpu_shard* shard, folp_session** out) {
  *out = nullptr;
  return guarded([&] {
    PrimalDualPoint z0;
    z0.primal.assign(static_cast<std::size_t>(lp_in->num_cols), 0.0);
    z0.dual.assign(static_cast<std::size_t>(lp_in->num_rows), 0.0);
    if (x0 != nullptr) z0.primal.assign(x0, x0 + lp_in->num_cols);
    if (y0 != nullptr) z0.dual.assign(y0, y0 + lp_in->num_rows);
    auto sess = std::make_unique<folp_session>();
    sess->s = std::make_unique<SolveSession>(to_lp(lp_in), to_params(p), std::move(z0), shard);
    if (folp_gpu_ctx* c = sess->s->context()) folp_gpu_set_profiling(c, 1);
    *out = sess.release();
  });
}

int folp_session_create(const folp_lp_c* lp_in, const folp_params_c* p, const double* x0,
                        const double* y0, folp_session** out) {
  return folp_session_create_sharded(lp_in, p, x0, y0, nullptr, out);
}

int folp_solve_sharded(const folp_lp_c* lp_in, const folp_params_c* p, const double* x0,
                       const double* y0, const folp_gpu_shard* shard, folp_result_c* out) {
  return guarded([&] {
    if (shard == nullptr) throw std::invalid_argument("folp_solve_sharded: shard spec required");
    const LinearProgram lp = to_lp(lp_in);
    const SolverParams params = to_params(p);
    PrimalDualPoint z0;
    z0.primal.assign(static_cast<std::size_t>(lp_in->num_cols), 0.0);
    z0.dual.assign(static_cast<std::size_t>(lp_in->num_rows), 0.0);
    if (x0 != nullptr) z0.primal.assign(x0, x0 + lp_in->num_cols);
    if (y0 != nullptr) z0.dual.assign(y0, y0 + lp_in->num_rows);
    export_result(solve_sharded(lp, params, z0, *shard), out);
  });
}

int folp_session_advance(folp_session* s, int64_t evaluations, int32_t* finished,
                         double* device_ms) {
  return guarded([&] {
    folp_gpu_ctx* c = s->s->context();
    if (c != nullptr && device_ms != nullptr) device::check(folp_gpu_timer_start(c), "timer");
    const bool done = s->s->advance(evaluations);
    if (c != nullptr && device_ms != nullptr) device::check(folp_gpu_timer_stop(c, device_ms), "timer");
    if (finished) *finished = done ? 1 : 0;
  });
}

int folp_session_stats(folp_session* s, int64_t* iterations, double* loop_ms, int64_t* loop_slots,
                       int64_t* launches) {
  return guarded([&] {
    if (iterations) *iterations = s->s->iterations();
    folp_gpu_ctx* c = s->s->context();
    double ms = 0.0;
    int64_t slots = 0;
    if (c != nullptr) folp_gpu_chunk_timing(c, &ms, &slots);
    if (loop_ms) *loop_ms = ms;
    if (loop_slots) *loop_slots = slots;
    if (launches) *launches = c ? folp_gpu_launch_count(c) : 0;
  });
}

folp_gpu_ctx* folp_session_context(folp_session* s) { return s ? s->s->context() : nullptr; }

int folp_session_partition(folp_session* s, int32_t* partition) {
  return guarded([&] {
    *partition = -1;
    if (folp_gpu_ctx* c = s->s->context()) {
      if (folp_gpu_shard_partition(c, partition) != 0) throw std::runtime_error(folp_gpu_last_error());
    }
  });
}

int folp_session_result(folp_session* s, folp_result_c* out) {
  return guarded([&] {
    const SolveResult* r = s->s->result();
    if (r == nullptr) throw std::invalid_argument("folp_session_result: session not finished");
    export_result(*r, out);
  });
}

void folp_session_destroy(folp_session* s) { delete s; }

// ---- MPS and result I/O ----------------------------------------------
int folp_mps_parse(const char* text, int64_t length, folp_mps** out) {
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<folp_mps>();
    m->inst = parse_mps(std::string_view(text, static_cast<std::size_t>(length)));
    *out = m.release();
  });
}

int folp_mps_parse_file(const char* path, folp_mps** out) {
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<folp_mps>();
    m->inst = parse_mps_file(path);
    *out = m.release();
  });
}

int folp_mps_view(const folp_mps* mps, folp_lp_c* lp, const char** name,
                  int32_t* was_maximization) {
  return guarded([&] {
    const LinearProgram& p = mps->inst.lp;
    const SparseMatrix& k = p.constraint_matrix;
    lp->num_rows = p.num_rows();
    lp->num_cols = p.num_variables();
    lp->num_inequality_rows = p.num_inequality_rows;
    lp->nnz = k.nnz();
    lp->row_start = k.row_start().data();
    lp->row_cols = k.row_cols().data();
    lp->row_values = k.row_values().data();
    lp->objective = p.objective.data();
    lp->right_hand_side = p.right_hand_side.data();
    lp->variable_lower = p.variable_lower.data();
    lp->variable_upper = p.variable_upper.data();
    lp->objective_constant = p.objective_constant;
    if (name != nullptr) *name = mps->inst.name.c_str();
    if (was_maximization != nullptr) *was_maximization = mps->inst.was_maximization ? 1 : 0;
  });
}

void folp_mps_destroy(folp_mps* mps) { delete mps; }

int folp_mps_write(const folp_lp_c* lp_in, const char* name, char** text, int64_t* length) {
  *text = nullptr;
  return guarded([&] { *text = export_text(write_mps(to_lp(lp_in), name ? name : ""), length); });
}

int folp_result_json(const folp_result_c* result, char** text, int64_t* length) {
  *text = nullptr;
  return guarded([&] { *text = export_text(result_to_json(import_result(result, 0, 0)), length); });
}

int folp_result_write(const folp_result_c* result, int64_t num_rows, int64_t num_cols,
                      const char* output_dir) {
  return guarded([&] { write_result(import_result(result, num_rows, num_cols), output_dir); });
}

void folp_buffer_free(char* buffer) { std::free(buffer); }

const char* folp_last_error(void) { return g_err.c_str(); }

const char* folp_engine_info(void) {
  return "folp B200 engine: sm_100a (compute_100a), fp64 segmented-dot kernels, "
         "conditional-graph PDHG chunks";
}

}  // extern "C"
