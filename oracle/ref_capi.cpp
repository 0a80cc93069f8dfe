// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the *unmodified* reference solver, compiled from
// /root/reference/proj/src with -Dfolp=folp_ref (see oracle/Makefile) into
// oracle/_ref/libfolp_ref.so.  It exposes the same entry points as
// include/folp_c.h with a folp_ref_ prefix so that tests/ and bench.py
// (--impl reference, cpu_baseline) can drive the reference on exactly the
// inputs handed to the B200 engine.  Nothing in the product links this.
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "folp/instance_gen.hpp"
#include "folp/lp_model.hpp"
#include "folp/mps.hpp"
#include "folp/result_io.hpp"
#include "folp/scaling.hpp"
#include "folp/solver.hpp"
#include "folp/sparse_matrix.hpp"
#include "folp/termination.hpp"
#include "folp/types.hpp"
#include "folp_c.h"

using namespace folp_ref;  // the reference namespace, renamed at compile time

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return FOLP_OK;
  } catch (const DimensionMismatch& e) {
    return fail(e, FOLP_E_DIMENSION_MISMATCH);
  } catch (const EmptyMatrix& e) {
    return fail(e, FOLP_E_EMPTY_MATRIX);
  } catch (const UnsupportedNorm& e) {
    return fail(e, FOLP_E_UNSUPPORTED_NORM);
  } catch (const NonPositiveWeight& e) {
    return fail(e, FOLP_E_NONPOSITIVE_WEIGHT);
  } catch (const NonPositiveRadius& e) {
    return fail(e, FOLP_E_NONPOSITIVE_RADIUS);
  } catch (const StepSizeUnderflow& e) {
    return fail(e, FOLP_E_STEP_UNDERFLOW);
  } catch (const NonFiniteIterate& e) {
    return fail(e, FOLP_E_NONFINITE);
  } catch (const InfiniteProduct& e) {
    return fail(e, FOLP_E_INFINITE_PRODUCT);
  } catch (const std::invalid_argument& e) {
    return fail(e, FOLP_E_INVALID_ARGUMENT);
  } catch (const IoError& e) {
    return fail(e, FOLP_E_IO);
  } catch (const std::exception& e) {
    return fail(e, FOLP_E_RUNTIME);
  }
}

LinearProgram to_lp(const folp_lp_c* in) {
  LinearProgram lp;
  const std::size_t n = static_cast<std::size_t>(in->num_cols);
  const std::size_t m = static_cast<std::size_t>(in->num_rows);
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(in->nnz));
  for (int64_t r = 0; r < in->num_rows; ++r) {
    for (int64_t k = in->row_start[r]; k < in->row_start[r + 1]; ++k) {
      t.push_back({r, in->row_cols[k], in->row_values[k]});
    }
  }
  lp.constraint_matrix =
      SparseMatrix::from_triplets(in->num_rows, in->num_cols, t);
  lp.objective.assign(in->objective, in->objective + n);
  lp.right_hand_side.assign(in->right_hand_side, in->right_hand_side + m);
  lp.variable_lower.assign(in->variable_lower, in->variable_lower + n);
  lp.variable_upper.assign(in->variable_upper, in->variable_upper + n);
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
  s.scale_invariant_initial_primal_weight =
      p->scale_invariant_initial_primal_weight != 0;
  s.use_presolve = p->use_presolve != 0;
  s.verbosity = 0;
  s.log_stream = nullptr;
  s.record_iterate_trace = p->record_iterate_trace != 0;
  return s;
}

folp_info_c to_info(const ConvergenceInfo& i) {
  return folp_info_c{i.primal_objective,     i.dual_objective,
                     i.gap_abs,              i.primal_residual_norm,
                     i.dual_residual_norm,   i.norm_q,
                     i.norm_c};
}

void copy_vec(const std::vector<double>& v, double* out) {
  if (out != nullptr && !v.empty()) {
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  }
}

}  // namespace

extern "C" {

void folp_ref_params_default(folp_params_c* p) {
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
  p->scale_invariant_initial_primal_weight =
      s.scale_invariant_initial_primal_weight ? 1 : 0;
  p->use_presolve = s.use_presolve ? 1 : 0;
  p->verbosity = 0;
  p->record_iterate_trace = 0;
}

int folp_ref_solve(const folp_lp_c* lp_in, const folp_params_c* p,
                   const double* x0, const double* y0, folp_result_c* out) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const SolverParams params = to_params(p);
    PrimalDualPoint z0;
    z0.primal.assign(static_cast<std::size_t>(lp_in->num_cols), 0.0);
    z0.dual.assign(static_cast<std::size_t>(lp_in->num_rows), 0.0);
    if (x0 != nullptr) z0.primal.assign(x0, x0 + lp_in->num_cols);
    if (y0 != nullptr) z0.dual.assign(y0, y0 + lp_in->num_rows);
    const SolveResult r = solve(lp, params, z0);
    copy_vec(r.primal_solution, out->primal_solution);
    copy_vec(r.dual_solution, out->dual_solution);
    copy_vec(r.reduced_costs, out->reduced_costs);
    out->termination_reason = static_cast<int32_t>(r.termination_reason);
    out->final_info = to_info(r.final_info);
    out->iterations = r.iterations;
    out->kkt_passes = r.kkt_passes;
    out->wall_seconds = r.wall_seconds;
    out->restarts = r.restarts;
    out->step_trials = r.step_trials;
    out->step_condition_violations = r.step_condition_violations;
    out->num_restart_iterations =
        static_cast<int64_t>(r.restart_iterations.size());
    for (int64_t i = 0; i < out->num_restart_iterations &&
                        i < out->restart_capacity;
         ++i) {
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
    out->iterate_n = 0;
    out->iterate_m = 0;
    if (!r.iterate_trace.empty()) {
      out->iterate_n =
          static_cast<int64_t>(r.iterate_trace[0].point.primal.size());
      out->iterate_m = static_cast<int64_t>(r.iterate_trace[0].point.dual.size());
    }
    for (int64_t i = 0; i < out->num_iterates && i < out->iterate_capacity;
         ++i) {
      const IterateRecord& rec = r.iterate_trace[static_cast<std::size_t>(i)];
      if (out->iterate_iteration) out->iterate_iteration[i] = rec.iteration;
      if (out->iterate_eta) out->iterate_eta[i] = rec.eta_used;
      if (out->iterate_primal) {
        copy_vec(rec.point.primal, out->iterate_primal + i * out->iterate_n);
      }
      if (out->iterate_dual) {
        copy_vec(rec.point.dual, out->iterate_dual + i * out->iterate_m);
      }
    }
  });
}

int folp_ref_multiply(const folp_lp_c* lp_in, const double* x, double* out) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const std::vector<double> v = lp.constraint_matrix.multiply(
        std::span<const double>(x, static_cast<std::size_t>(lp_in->num_cols)));
    copy_vec(v, out);
  });
}

int folp_ref_multiply_transpose(const folp_lp_c* lp_in, const double* y,
                                double* out) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const std::vector<double> v = lp.constraint_matrix.multiply_transpose(
        std::span<const double>(y, static_cast<std::size_t>(lp_in->num_rows)));
    copy_vec(v, out);
  });
}

int folp_ref_rescale(const folp_lp_c* lp_in, int64_t ruiz_iterations,
                     int32_t apply_pc, double alpha, double* row_scale,
                     double* col_scale, double* scaled_values,
                     double* scaled_objective, double* scaled_rhs,
                     double* scaled_lower, double* scaled_upper) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    const ScaledProblem s =
        rescale_problem(lp, ruiz_iterations, apply_pc != 0, alpha);
    copy_vec(s.scaling.row_scale, row_scale);
    copy_vec(s.scaling.col_scale, col_scale);
    if (scaled_values != nullptr) {
      const auto v = s.lp.constraint_matrix.row_values();
      std::memcpy(scaled_values, v.data(), v.size() * sizeof(double));
    }
    copy_vec(s.lp.objective, scaled_objective);
    copy_vec(s.lp.right_hand_side, scaled_rhs);
    copy_vec(s.lp.variable_lower, scaled_lower);
    copy_vec(s.lp.variable_upper, scaled_upper);
  });
}

int folp_ref_convergence_info(const folp_lp_c* lp_in, const double* x,
                              const double* y, folp_info_c* info) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    *info = to_info(convergence_info(
        lp, std::span<const double>(x, static_cast<std::size_t>(lp_in->num_cols)),
        std::span<const double>(y, static_cast<std::size_t>(lp_in->num_rows))));
  });
}

int folp_ref_normalized_duality_gap(const folp_lp_c* lp_in, const double* x,
                                    const double* y, double radius,
                                    double omega, double* gap) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    PrimalDualPoint z;
    z.primal.assign(x, x + lp_in->num_cols);
    z.dual.assign(y, y + lp_in->num_rows);
    *gap = normalized_duality_gap(lp, z, radius, omega);
  });
}

int folp_ref_adaptive_step(const folp_lp_c* lp_in, const double* x,
                           const double* y, double omega, double eta_hat,
                           int64_t k, double* x_next, double* y_next,
                           double* eta_used, double* eta_hat_next,
                           int64_t* trials, double* movement_sq,
                           double* cross_term) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    PrimalDualPoint z;
    z.primal.assign(x, x + lp_in->num_cols);
    z.dual.assign(y, y + lp_in->num_rows);
    const AdaptiveStepResult r = adaptive_step(lp, z, omega, eta_hat, k);
    copy_vec(r.next.primal, x_next);
    copy_vec(r.next.dual, y_next);
    *eta_used = r.eta_used;
    *eta_hat_next = r.eta_hat_next;
    *trials = r.trials;
    *movement_sq = r.movement_sq;
    *cross_term = r.cross_term;
  });
}

int folp_ref_malitsky_pock_step(const folp_lp_c* lp_in, const double* x, const double* y,
                                double omega, double eta_prev, double theta_prev,
                                const folp_params_c* p, double* x_next, double* y_next,
                                double* eta_next, double* theta_next, int64_t* trials) {
  return guarded([&] {
    const LinearProgram lp = to_lp(lp_in);
    PrimalDualPoint z;
    z.primal.assign(x, x + lp_in->num_cols);
    z.dual.assign(y, y + lp_in->num_rows);
    const MalitskyPockResult r =
        malitsky_pock_step(lp, z, omega, eta_prev, theta_prev, to_params(p));
    copy_vec(r.next.primal, x_next);
    copy_vec(r.next.dual, y_next);
    *eta_next = r.eta_next;
    *theta_next = r.theta_next;
    *trials = r.trials;
  });
}

// ---- MPS and result I/O (mps.hpp, result_io.hpp) -------------------------
struct folp_ref_mps {
  MpsInstance inst;
};

static char* export_text(const std::string& s, int64_t* length) {
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  *length = static_cast<int64_t>(s.size());
  return buf;
}

int folp_ref_mps_parse(const char* text, int64_t length, folp_ref_mps** out) {
  *out = nullptr;
  return guarded([&] {
    auto* m = new folp_ref_mps{parse_mps(std::string_view(text, static_cast<std::size_t>(length)))};
    *out = m;
  });
}

int folp_ref_mps_parse_file(const char* path, folp_ref_mps** out) {
  *out = nullptr;
  return guarded([&] { *out = new folp_ref_mps{parse_mps_file(path)}; });
}

int folp_ref_mps_view(const folp_ref_mps* mps, folp_lp_c* lp, const char** name,
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

void folp_ref_mps_destroy(folp_ref_mps* mps) { delete mps; }

int folp_ref_mps_write(const folp_lp_c* lp_in, const char* name, char** text, int64_t* length) {
  *text = nullptr;
  return guarded([&] { *text = export_text(write_mps(to_lp(lp_in), name ? name : ""), length); });
}

static SolveResult import_result(const folp_result_c* in, int64_t m, int64_t n) {
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
  for (int64_t i = 0; i < in->num_trace && i < in->trace_capacity; ++i) {
    TraceEntry e;
    e.iteration = in->trace_iteration[i];
    e.kkt_passes = in->trace_kkt_passes[i];
    e.current = info(in->trace_current[i]);
    e.average = info(in->trace_average[i]);
    r.trace.push_back(e);
  }
  return r;
}

int folp_ref_result_json(const folp_result_c* result, char** text, int64_t* length) {
  *text = nullptr;
  return guarded([&] { *text = export_text(result_to_json(import_result(result, 0, 0)), length); });
}

int folp_ref_result_write(const folp_result_c* result, int64_t num_rows, int64_t num_cols,
                          const char* output_dir) {
  return guarded([&] { write_result(import_result(result, num_rows, num_cols), output_dir); });
}

void folp_ref_buffer_free(char* buffer) { std::free(buffer); }

const char* folp_ref_last_error(void) { return g_err.c_str(); }

// ---- reference instance generators (instance_gen.hpp) ---------------------
// Generated LPs are returned through an opaque handle so Python can size its
// buffers before copying out.
struct folp_ref_lp_handle {
  LinearProgram lp;
};

static folp_ref_lp_handle* wrap(LinearProgram lp) {
  return new folp_ref_lp_handle{std::move(lp)};
}

folp_ref_lp_handle* folp_ref_gen_pagerank(int64_t nodes, int64_t attach,
                                          uint64_t seed, double damping) {
  try {
    return wrap(pagerank_lp(barabasi_albert(nodes, attach, seed), damping));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

folp_ref_lp_handle* folp_ref_gen_random_feasible(uint64_t seed, int64_t m1,
                                                 int64_t m2, int64_t n,
                                                 double spread) {
  try {
    return wrap(random_feasible_lp(seed, m1, m2, n, spread));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

int64_t folp_ref_handcrafted_count(void) {
  return static_cast<int64_t>(handcrafted_suite().size());
}

folp_ref_lp_handle* folp_ref_gen_handcrafted(int64_t index, double* objective,
                                             char* name, int64_t name_cap) {
  const auto suite = handcrafted_suite();
  if (index < 0 || index >= static_cast<int64_t>(suite.size())) return nullptr;
  const NamedInstance& ni = suite[static_cast<std::size_t>(index)];
  if (objective) *objective = ni.optimal_objective;
  if (name && name_cap > 0) {
    std::strncpy(name, ni.name.c_str(), static_cast<std::size_t>(name_cap - 1));
    name[name_cap - 1] = '\0';
  }
  return wrap(ni.lp);
}

void folp_ref_lp_sizes(const folp_ref_lp_handle* h, int64_t* m, int64_t* n,
                       int64_t* m1, int64_t* nnz) {
  *m = h->lp.num_rows();
  *n = h->lp.num_variables();
  *m1 = h->lp.num_inequality_rows;
  *nnz = h->lp.constraint_matrix.nnz();
}

void folp_ref_lp_copy(const folp_ref_lp_handle* h, int64_t* row_start,
                      int64_t* row_cols, double* row_values, double* c,
                      double* q, double* l, double* u, double* constant) {
  const SparseMatrix& k = h->lp.constraint_matrix;
  std::memcpy(row_start, k.row_start().data(),
              k.row_start().size() * sizeof(int64_t));
  if (k.nnz() > 0) {
    std::memcpy(row_cols, k.row_cols().data(),
                k.row_cols().size() * sizeof(int64_t));
    std::memcpy(row_values, k.row_values().data(),
                k.row_values().size() * sizeof(double));
  }
  copy_vec(h->lp.objective, c);
  copy_vec(h->lp.right_hand_side, q);
  copy_vec(h->lp.variable_lower, l);
  copy_vec(h->lp.variable_upper, u);
  *constant = h->lp.objective_constant;
}

void folp_ref_lp_free(folp_ref_lp_handle* h) { delete h; }

}  // extern "C"
