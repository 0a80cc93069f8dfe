// solver.cpp -- folp::solve on the B200.
//
// The control flow is the reference's SolveDriver
// (/root/reference/proj/src/solver.cpp:477-946): validate and presolve on
// the host, then one device context holds the presolved LP and runs
// rescaling, the restarted PDHG loop (40-iteration chunks executed as a
// conditional CUDA graph, no host round trip per iteration), the running
// average, both convergence evaluations, the normalized duality gaps and the
// restart bookkeeping.  The host keeps only scalar decisions (termination
// test, restart rule, primal-weight update, limits) and the final postsolve.
#include "folp/solver.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <ostream>
#include <random>
#include <string>
#include <thread>

#include "device.hpp"
#include "parallel.hpp"
#include "sparse_access.hpp"
#include "session.hpp"
#include "folp/linalg.hpp"
#include "folp/presolve.hpp"
#include "folp/scaling.hpp"

namespace folp {

namespace {

constexpr double kPowerTol = 1e-4;          // solver.cpp:32
constexpr Index kPowerMaxIters = 1000;      // solver.cpp:33
constexpr std::uint64_t kPowerSeed = 1;     // solver.cpp:34
constexpr double kConstantSafety = 0.9;     // solver.cpp:35

void require_point(const LinearProgram& lp, const PrimalDualPoint& z, const char* what) {
  if (static_cast<Index>(z.primal.size()) != lp.num_variables() ||
      static_cast<Index>(z.dual.size()) != lp.num_rows()) {
    throw DimensionMismatch(std::string(what) + ": point size mismatch");
  }
}

// (1 - (k+1)^-0.3, 1 + (k+1)^-0.6) for the 1-based counter k, computed with
// the host libm exactly like adaptive_step (solver.cpp:173-175).
void step_factors(Index k, double& reduction, double& growth) {
  const double kp1 = static_cast<double>(k + 1);
  reduction = 1.0 - std::pow(kp1, -0.3);
  growth = 1.0 + std::pow(kp1, -0.6);
}

void check_params(const SolverParams& p) {  // solver.cpp:447-467
  if (!(p.eps_optimal > 0.0)) throw std::invalid_argument("solve: eps_optimal must be > 0");
  if (!(p.beta_necessary > 0.0 && p.beta_necessary < p.beta_sufficient &&
        p.beta_sufficient < 1.0)) {
    throw std::invalid_argument("solve: betas must satisfy 0 < nec < suf < 1");
  }
  if (!(p.beta_artificial > 0.0 && p.beta_artificial < 1.0)) {
    throw std::invalid_argument("solve: beta_artificial must be in (0,1)");
  }
  if (!(p.theta_smoothing >= 0.0 && p.theta_smoothing <= 1.0)) {
    throw std::invalid_argument("solve: theta must be in [0,1]");
  }
  if (p.evaluation_cadence < 1) throw std::invalid_argument("solve: evaluation cadence must be >= 1");
  if (p.ruiz_iterations < 0) throw std::invalid_argument("solve: ruiz_iterations must be >= 0");
}

double violation_score(const ConvergenceInfo& info) {  // solver.cpp:469-475
  const double gap =
      info.gap_abs / (1.0 + std::fabs(info.primal_objective) + std::fabs(info.dual_objective));
  const double primal = info.primal_residual_norm / (1.0 + info.norm_q);
  const double dual = info.dual_residual_norm / (1.0 + info.norm_c);
  return std::max(gap, std::max(primal, dual));
}

std::vector<double> start_vector(Index n) {  // sparse_matrix.cpp:195-202
  std::mt19937_64 rng(kPowerSeed);
  std::vector<double> v(static_cast<std::size_t>(n));
  for (double& e : v) e = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
  double vnorm = linalg::norm2(v);
  if (vnorm == 0.0) {
    v[0] = 1.0;
    vnorm = 1.0;
  }
  linalg::scale(v, 1.0 / vnorm);
  return v;
}

// ---------------------------------------------------------------------
class Driver {
 public:
  // zero_start: the start point is the origin (z0 is not read; the device
  // zero-fills instead of receiving two uploaded vectors of zeros)
  Driver(const LinearProgram& raw, const SolverParams& params, const PrimalDualPoint& z0,
         const folp_gpu_shard* shard = nullptr, bool zero_start = false)
      : raw_(raw), p_(params), z0_(z0), zero_start_(zero_start), start_(Clock::now()), shard_(shard) {}

  ~Driver() {
    if (std::getenv("FOLP_TIMING") == nullptr) return;
    const double t0 = elapsed();
    dev_.reset();
    std::fprintf(stderr, "[folp timing] driver teardown: entered %.4f context released %.4f\n", t0, elapsed());
  }
  SolveResult run();
  // Everything before the loop (solver.cpp:818-907); a value when the solve
  // already ended (detected, trivial, optimal start).
  std::optional<SolveResult> start();
  // Runs the loop for at most `evaluations` evaluation periods.
  std::optional<SolveResult> advance(Index evaluations);
  folp_gpu_ctx* context() const { return dev_ ? dev_->get() : nullptr; }
  Index iterations() const { return k_total_; }

 private:
  using Clock = std::chrono::steady_clock;
  double elapsed() const { return std::chrono::duration<double>(Clock::now() - start_).count(); }
  // Wall clock for the time-limit decision: the max over the shards, so
  // every shard takes the same branch.
  double decision_clock() {
    double e = elapsed();
    if (shard_ != nullptr && dev_) device::check(folp_gpu_shard_max(ctx(), &e), "shard clock");
    return e;
  }
  folp_gpu_ctx* ctx() const { return dev_->get(); }

  ConvergenceInfo evaluate(int slot) {
    ConvergenceInfo info = dev_->evaluate(slot, false, work_->objective_constant);
    ledger_.add_k();
    ledger_.add_kt();
    return info;
  }
  void materialize_average() {
    device::check(folp_gpu_materialize_average(ctx(), &avg_weight_), "materialize_average");
  }
  // (sum dx^2, sum dy^2) of slot - LAST
  void distance_to_last(int slot, double& sx, double& sy) {
    device::check(folp_gpu_distance(ctx(), slot, FOLP_PT_LAST, &sx, &sy), "distance");
  }
  double ndg(int slot, double radius, double omega) {
    double gap = 0.0;
    device::check(folp_gpu_ndg(ctx(), slot, radius, omega, &gap), "normalized_duality_gap");
    ledger_.add_kt();
    ledger_.add_k();
    return gap;
  }
  static double weighted(double sx, double sy, double omega) {  // lp_model.cpp:167-173
    return std::sqrt(omega * sx + sy / omega);
  }
  double new_primal_weight(double sx, double sy, double omega_prev) const {
    // update_primal_weight (solver.cpp:429-443) on precomputed diff norms
    if (!(omega_prev > 0.0)) throw NonPositiveWeight("update_primal_weight: omega must be > 0");
    const double theta = p_.theta_smoothing;
    if (theta == 0.0) return omega_prev;
    const double dx = std::sqrt(sx), dy = std::sqrt(sy);
    if (dx > p_.eps_zero && dy > p_.eps_zero) {
      return std::exp(theta * std::log(dy / dx) + (1.0 - theta) * std::log(omega_prev));
    }
    return omega_prev;
  }

  void log_evaluation(const ConvergenceInfo& cur, const ConvergenceInfo& avg) {
    if (p_.verbosity < 2 || p_.log_stream == nullptr) return;
    char line[256];
    std::snprintf(line, sizeof(line), "%9lld %10.1f  %+.8e %+.8e  %8.2e %8.2e %8.2e",
                  static_cast<long long>(k_total_), kkt_passes(ledger_), cur.primal_objective,
                  cur.dual_objective, cur.gap_abs, cur.primal_residual_norm,
                  cur.dual_residual_norm);
    (*p_.log_stream) << line << " | avg gap " << avg.gap_abs << "\n";
  }
  void log_summary(const SolveResult& r) {
    if (p_.verbosity < 1 || p_.log_stream == nullptr) return;
    (*p_.log_stream) << "terminated: " << to_string(r.termination_reason) << "  iterations "
                     << r.iterations << "  kkt passes " << r.kkt_passes << "  objective "
                     << r.final_info.primal_objective << "  restarts " << r.restarts << "\n";
  }

  SolveResult finish(TerminationReason reason, int slot, const ConvergenceInfo& info);
  SolveResult finish_point(TerminationReason reason, PrimalDualPoint reduced,
                           const ConvergenceInfo& info);
  SolveResult finish_detected(PresolveStatus status);
  SolveResult finish_trivial();
  SolveResult finish_limit(TerminationReason reason);
  SolveResult finish_numerical_error();
  bool evaluate_and_maybe_restart(SolveResult& out);
  void record_iterate();
  void order_columns();
  // working-space column order (col_order_[i] = presolved column of working
  // column i; empty: identity) and the maps of primal vectors across it
  void primal_to_work(std::vector<double>& v) const {
    if (col_order_.empty()) return;
    std::vector<double> w = host::uninitialized_vector<double>(static_cast<int64_t>(v.size()));
    host::parallel_for(static_cast<int64_t>(w.size()), [&](int64_t b, int64_t e, int) {
      for (int64_t i = b; i < e; ++i) w[i] = v[static_cast<std::size_t>(col_order_[i])];
    });
    v.swap(w);
  }
  void primal_from_work(std::vector<double>& v) {
    if (col_order_.empty()) return;
    std::vector<double> w = host::uninitialized_vector<double>(static_cast<int64_t>(v.size()));
    host::parallel_for(static_cast<int64_t>(w.size()), [&](int64_t b, int64_t e, int) {
      for (int64_t i = b; i < e; ++i) w[static_cast<std::size_t>(col_order_[i])] = v[i];  // a permutation: disjoint
    }, static_cast<int64_t>(w.size()) * kFreshPageWork);
    v.swap(w);
    scratch_.swap(w);  // the old buffer: its pages are mapped, reused by finish_point
  }
  // A pass whose output is freshly allocated is bound by first-touch page
  // faults (~1.7 us per 4 KB page on the B200 hosts): sized for more chunks
  // than its element count alone would get.
  static constexpr int64_t kFreshPageWork = 4;
  // project_reduced_costs (lp_model.cpp:101-119) for one entry
  static double project_reduced_cost(double lo, double hi, double v) {
    const bool lower = lo > -kInf, upper = hi < kInf;
    if (!lower && !upper) return 0.0;
    if (!lower) return std::min(v, 0.0);
    if (!upper) return std::max(v, 0.0);
    return v;
  }
  std::vector<double> scratch_;

  const LinearProgram& raw_;
  SolverParams p_;
  const PrimalDualPoint& z0_;
  bool zero_start_ = false;
  Clock::time_point start_;
  const folp_gpu_shard* shard_ = nullptr;  // row shard of a multi-GPU solve

  PresolveTransform transform_;
  LinearProgram presolved_storage_;
  std::vector<Index> col_order_;   // working column order on the device (empty: identity)
  std::vector<Index> raw_degrees_; // column degrees of raw_ (from presolve)
  bool raw_on_device_ = false;      // the device matrix is raw K (column order aside)
  const LinearProgram* work_ = nullptr;  // the presolved LP (raw_ when identity)
  std::unique_ptr<device::Context> dev_;
  KktPassLedger ledger_;

  double omega_ = 1.0;
  double eta_hat_ = 1.0;
  double eta_constant_ = 1.0;
  double mp_eta_ = 1.0;    // Malitsky-Pock accepted step (solver.cpp:595)
  double mp_theta_ = 1.0;  // Malitsky-Pock step ratio (solver.cpp:596)
  double last_eta_used_ = 0.0;
  double avg_weight_ = 0.0;
  double reference_gap_ = kInf;
  std::optional<double> last_candidate_gap_;
  Index k_total_ = 0;
  Index t_inner_ = 0;
  Index n_outer_ = 0;
  SolveResult tmpl_;
  std::vector<double> red_, grow_;
  double time_chunks_ = 0.0;  // host wall time in loop chunks / evaluations
  double time_evals_ = 0.0;   // (printed at finish when FOLP_TIMING is set)
  double time_setup_ = 0.0;
  std::string setup_marks_;   // FOLP_TIMING: elapsed time at each setup stage
  void mark(const char* stage) {
    if (std::getenv("FOLP_TIMING") == nullptr) return;
    char buf[64];
    std::snprintf(buf, sizeof(buf), " %s %.4f", stage, elapsed());
    setup_marks_ += buf;
  }
};

SolveResult Driver::finish_point(TerminationReason reason, PrimalDualPoint reduced,
                                 const ConvergenceInfo& info) {
  mark("finish:point");
  SolveResult r = tmpl_;
  r.termination_reason = reason;
  r.final_info = info;
  r.iterations = k_total_;
  r.restarts = n_outer_;
  // an identity transform postsolves to the same two vectors
  const bool same_point = transform_.is_identity() &&
                          static_cast<Index>(reduced.primal.size()) == transform_.original_cols &&
                          static_cast<Index>(reduced.dual.size()) == transform_.original_rows;
  PrimalDualPoint full = same_point ? std::move(reduced)
                                    : postsolve(transform_, reduced.primal, reduced.dual);
  mark("postsolved");
  // Reduced costs on the original problem (solver.cpp:662-670): K'y on the
  // raw K.  When presolve was the identity the device already holds raw K.
  // r.reduced_costs = project_reduced_costs(raw, c - K'y): one pass on all
  // host cores straight into the result (fresh pages are touched once, in
  // parallel); a device K'y arrives in working-column order and is mapped
  // back by the same pass.
  const Index nv = raw_.num_variables();
  std::vector<double> kty;
  bool work_order = false;
  if (nv > 0) {
    if (dev_ && transform_.is_identity() && raw_on_device_) {
      kty.swap(scratch_);  // pages already touched (the reduced point's old buffer)
      if (static_cast<Index>(kty.size()) != nv) kty = host::uninitialized_vector<double>(nv);
      device::check(folp_gpu_multiply_transpose(ctx(), 0, full.dual.data(), kty.data()),
                    "reduced costs");
      work_order = !col_order_.empty();
    } else {
      kty.assign(static_cast<std::size_t>(nv), 0.0);
      raw_.constraint_matrix.multiply_transpose(full.dual, kty);
    }
  }
  mark("kty");
  ledger_.add_kt();
  r.reduced_costs = host::uninitialized_vector<double>(nv);
  host::parallel_for(nv, [&](int64_t b, int64_t e, int) {
    for (int64_t i = b; i < e; ++i) {
      const std::size_t j = work_order ? static_cast<std::size_t>(col_order_[i]) : static_cast<std::size_t>(i);
      r.reduced_costs[j] = project_reduced_cost(raw_.variable_lower[j], raw_.variable_upper[j],
                                                raw_.objective[j] - kty[i]);
    }
  }, nv * kFreshPageWork);
  r.primal_solution = std::move(full.primal);
  r.dual_solution = std::move(full.dual);
  mark("reduced costs");
  r.kkt_passes = kkt_passes(ledger_);
  r.wall_seconds = elapsed();
  log_summary(r);
  if (std::getenv("FOLP_TIMING") != nullptr) {
    std::fprintf(stderr,
                 "[folp timing] total %.4fs  setup %.4fs  chunks %.4fs  evaluations %.4fs  "
                 "iterations %lld  setup stages:%s\n",
                 r.wall_seconds, time_setup_, time_chunks_, time_evals_,
                 static_cast<long long>(r.iterations), setup_marks_.c_str());
  }
  return r;
}

SolveResult Driver::finish(TerminationReason reason, int slot, const ConvergenceInfo& info) {
  PrimalDualPoint reduced;  // both vectors filled by the download
  reduced.primal = host::uninitialized_vector<double>(work_->num_variables());
  reduced.dual = host::uninitialized_vector<double>(work_->num_rows());
  device::check(folp_gpu_get_reduced_point(ctx(), slot, reduced.primal.data(), reduced.dual.data()),
                "reduced_point");
  mark("point downloaded");
  primal_from_work(reduced.primal);
  return finish_point(reason, std::move(reduced), info);
}

SolveResult Driver::finish_detected(PresolveStatus status) {  // solver.cpp:678-692
  SolveResult r = tmpl_;
  r.termination_reason = status == PresolveStatus::kPrimalInfeasible
                             ? TerminationReason::kPrimalInfeasibleDetected
                             : TerminationReason::kDualUnboundedDetected;
  r.primal_solution.assign(static_cast<std::size_t>(raw_.num_variables()), 0.0);
  r.dual_solution.assign(static_cast<std::size_t>(raw_.num_rows()), 0.0);
  r.reduced_costs.assign(static_cast<std::size_t>(raw_.num_variables()), 0.0);
  r.kkt_passes = kkt_passes(ledger_);
  r.wall_seconds = elapsed();
  log_summary(r);
  return r;
}

SolveResult Driver::finish_trivial() {  // solver.cpp:694-701
  const ConvergenceInfo info = convergence_info(*work_, {}, {}, &ledger_);
  tmpl_.trace.push_back(TraceEntry{0, kkt_passes(ledger_), info, info});
  return finish_point(TerminationReason::kOptimal, PrimalDualPoint{}, info);
}

SolveResult Driver::finish_limit(TerminationReason reason) {  // solver.cpp:703-726
  mark("finish:limit");
  ConvergenceInfo cur, avg;
  try {
    cur = evaluate(FOLP_PT_CURRENT);
    mark("eval current");
    materialize_average();
    avg = evaluate(FOLP_PT_AVERAGE);
    mark("eval average");
  } catch (const NonFiniteIterate&) {
    return finish_numerical_error();
  }
  tmpl_.trace.push_back(TraceEntry{k_total_, kkt_passes(ledger_), cur, avg});
  if (check_termination(cur, p_.eps_optimal)) {
    return finish(TerminationReason::kOptimal, FOLP_PT_CURRENT, cur);
  }
  if (check_termination(avg, p_.eps_optimal)) {
    return finish(TerminationReason::kOptimal, FOLP_PT_AVERAGE, avg);
  }
  if (violation_score(cur) <= violation_score(avg)) return finish(reason, FOLP_PT_CURRENT, cur);
  return finish(reason, FOLP_PT_AVERAGE, avg);
}

SolveResult Driver::finish_numerical_error() {  // solver.cpp:728-749
  materialize_average();
  int32_t finite = 0;
  device::check(folp_gpu_all_finite(ctx(), FOLP_PT_AVERAGE, &finite), "all_finite");
  int slot = finite ? FOLP_PT_AVERAGE : FOLP_PT_LAST;
  ConvergenceInfo info;
  try {
    info = evaluate(slot);
  } catch (const NonFiniteIterate&) {
    slot = FOLP_PT_LAST;
    info = evaluate(slot);
  }
  tmpl_.trace.push_back(TraceEntry{k_total_, kkt_passes(ledger_), info, info});
  const TerminationReason reason = check_termination(info, p_.eps_optimal)
                                       ? TerminationReason::kOptimal
                                       : TerminationReason::kNumericalError;
  return finish(reason, slot, info);
}

void Driver::record_iterate() {
  IterateRecord rec;
  rec.iteration = k_total_;
  rec.eta_used = last_eta_used_;
  rec.point = dev_->get_point(FOLP_PT_CURRENT);
  primal_from_work(rec.point.primal);
  tmpl_.iterate_trace.push_back(std::move(rec));
}

// solver.cpp:751-816.  Returns true when the solve terminated (out is set).
bool Driver::evaluate_and_maybe_restart(SolveResult& out) {
  const bool restarts = p_.restart_scheme != RestartSchemeKind::kNone;
  folp_gpu_period period{};
  device::check(folp_gpu_evaluation_period(ctx(), omega_, restarts ? 1 : 0, &period),
                "evaluation period");
  avg_weight_ = period.avg_weight;
  const ConvergenceInfo cur = device::to_info(period.current, work_->objective_constant);
  ledger_.add_k();
  ledger_.add_kt();
  const ConvergenceInfo avg = device::to_info(period.average, work_->objective_constant);
  ledger_.add_k();
  ledger_.add_kt();
  tmpl_.trace.push_back(TraceEntry{k_total_, kkt_passes(ledger_), cur, avg});
  log_evaluation(cur, avg);
  if (check_termination(cur, p_.eps_optimal)) {
    out = finish(TerminationReason::kOptimal, FOLP_PT_CURRENT, cur);
    return true;
  }
  if (check_termination(avg, p_.eps_optimal)) {
    out = finish(TerminationReason::kOptimal, FOLP_PT_AVERAGE, avg);
    return true;
  }

  if (!restarts) {
    if (static_cast<double>(t_inner_) >= p_.beta_artificial * static_cast<double>(k_total_)) {
      double sx = 0.0, sy = 0.0;
      distance_to_last(FOLP_PT_CURRENT, sx, sy);
      omega_ = new_primal_weight(sx, sy, omega_);
      device::check(folp_gpu_mark_last(ctx()), "mark_last");
      t_inner_ = 0;
    }
    return false;
  }
  if (!period.gaps_valid) throw DeviceError("evaluation period: duality gaps missing");

  // restart_candidate (solver.cpp:372-393); the device evaluated both gaps
  // at the radius weighted(sx, sy, omega) and skipped a zero radius
  double mu[2];
  for (int i = 0; i < 2; ++i) {
    const double radius = weighted(period.dist_x[i], period.dist_y[i], omega_);
    mu[i] = period.gap[i];
    if (radius != 0.0) {
      ledger_.add_kt();
      ledger_.add_k();
    }
  }
  const int slots[2] = {FOLP_PT_CURRENT, FOLP_PT_AVERAGE};
  const int pick = mu[0] < mu[1] ? 0 : 1;  // the average wins ties
  const double gap = mu[pick];
  const RestartDecision decision =
      should_restart(gap, reference_gap_, last_candidate_gap_, t_inner_, k_total_, p_);
  if (decision == RestartDecision::kNoRestart) {
    last_candidate_gap_ = gap;
    return false;
  }
  ++n_outer_;
  tmpl_.restart_iterations.push_back(k_total_);
  const double sx = period.dist_x[pick], sy = period.dist_y[pick];
  const double omega_new = new_primal_weight(sx, sy, omega_);
  const double radius = weighted(sx, sy, omega_new);
  if (radius > 0.0) {
    ledger_.add_kt();
    ledger_.add_k();
  }
  // Same point, weight and radius as the candidate: the gap is the same
  // deterministic evaluation, so it is not repeated on device.
  const bool same = omega_new == omega_;
  double ref = 0.0;
  device::check(folp_gpu_restart_commit(ctx(), slots[pick], same ? 0.0 : radius, omega_new, &ref),
                "restart");
  reference_gap_ = radius > 0.0 ? (same ? mu[pick] : ref) : 0.0;
  omega_ = omega_new;
  avg_weight_ = 0.0;
  last_candidate_gap_.reset();
  t_inner_ = 0;
  return false;
}

// Column renumbering (tree mode, one context, $FOLP_HOT_COLUMNS=0 turns it
// off, =1 forces it): when the column degrees are strongly skewed (config
// 2's power law: max degree >= 16x the mean), the working columns are
// ordered by descending degree, so the x gathers of K x concentrate on a
// short hot prefix of x that stays in L1 (config 2: -5.9 % device time per
// evaluation period, profiles/r1_session2_experiments.md).  Columns keep
// their entries and rows their entry order (only the column numbers change),
// so every row and column dot is the caller's.  The engine renumbers on
// the device (folp_gpu_create_ordered); the host only computes the order and
// maps primal vectors at the boundary.  Ordered mode keeps the reference's
// order throughout.
void Driver::order_columns() {
  const char* env = std::getenv("FOLP_HOT_COLUMNS");
  const int mode = env != nullptr ? std::atoi(env) : -1;
  if (mode == 0 || shard_ != nullptr || folp_gpu_default_reduction() != 0) return;
  const SparseMatrix& k = work_->constraint_matrix;
  const Index n = work_->num_variables(), nnz = k.nnz();
  if (nnz == 0 || (mode != 1 && n < (Index(1) << 16))) return;
  std::vector<Index> deg;
  if (work_ == &raw_ && static_cast<Index>(raw_degrees_.size()) == n) {
    deg.swap(raw_degrees_);  // counted by presolve already
  } else {
    const std::span<const Index> cols = k.row_cols();
    deg.assign(static_cast<std::size_t>(n), 0);
    host::parallel_histogram(cols.data(), nnz, n, deg.data());
  }
  const Index max_deg = *std::max_element(deg.begin(), deg.end());
  if (mode != 1 && static_cast<double>(max_deg) < 16.0 * static_cast<double>(nnz) / static_cast<double>(n)) {
    return;
  }
  // counting sort by descending degree, stable in the column index
  std::vector<Index> first(static_cast<std::size_t>(max_deg) + 2, 0);
  for (Index j = 0; j < n; ++j) ++first[static_cast<std::size_t>(max_deg - deg[j]) + 1];
  for (std::size_t d = 1; d < first.size(); ++d) first[d] += first[d - 1];
  col_order_.assign(static_cast<std::size_t>(n), 0);
  for (Index j = 0; j < n; ++j) {
    const Index r = first[static_cast<std::size_t>(max_deg - deg[j])]++;
    col_order_[static_cast<std::size_t>(r)] = j;
  }
}

SolveResult Driver::run() {  // solver.cpp:818-946
  if (auto done = start()) return std::move(*done);
  return std::move(*advance(std::numeric_limits<Index>::max()));
}

std::optional<SolveResult> Driver::start() {
  check_params(p_);
  if (p_.restart_scheme == RestartSchemeKind::kTheory) {
    p_.beta_sufficient = 0.37;
    p_.beta_necessary = 0.37;
  }
  if (const auto issue = validate(raw_)) {
    if (issue->kind == ValidationIssue::Kind::kBoundViolation) {
      return finish_detected(PresolveStatus::kPrimalInfeasible);
    }
    throw std::invalid_argument("solve: invalid program: " + issue->message);
  }

  mark("validated");
  if (p_.use_presolve) {
    PresolveResult pre = detail::presolve_for_solve(raw_, &raw_degrees_);
    if (pre.status != PresolveStatus::kReduced) return finish_detected(pre.status);
    transform_ = std::move(pre.transform);
    if (transform_.is_identity() && pre.reduced.objective_constant == raw_.objective_constant) {
      work_ = &raw_;  // bit-identical to the rebuilt copy; skip the copy
    } else {
      presolved_storage_ = std::move(pre.reduced);
      work_ = &presolved_storage_;
    }
  } else {
    work_ = &raw_;
    transform_.original_rows = raw_.num_rows();
    transform_.original_cols = raw_.num_variables();
  }
  mark("presolved");
  if (work_->num_variables() == 0) return finish_trivial();
  raw_on_device_ = work_ == &raw_;
  order_columns();
  mark("columns ordered");

  if (p_.use_pock_chambolle) {
    const double a = p_.pc_alpha;
    if (!(a >= 0.0 && a <= 2.0)) {
      throw std::invalid_argument("pock_chambolle_step: alpha must be in [0,2]");
    }
    for (const double pn : {2.0 - a, a}) {
      if (std::isnan(pn) || (pn < 1.0 && pn != 0.0)) {
        throw UnsupportedNorm("axis_norms: p must be 0, in [1, inf), or +inf");
      }
    }
  }

  dev_ = std::make_unique<device::Context>(*work_, col_order_.empty() ? nullptr : col_order_.data());
  mark("context");
  device::check(folp_gpu_rescale(ctx(), p_.ruiz_iterations, p_.use_pock_chambolle ? 1 : 0,
                                 p_.pc_alpha, nullptr, nullptr),
                "rescale_problem");
  mark("rescaled");
  if (shard_ != nullptr) dev_->attach_shard(work_->constraint_matrix, *shard_);

  // start point into the working space, projected (solver.cpp:853-865)
  if (zero_start_) {
    // the origin restricts and permutes to the origin
    device::check(folp_gpu_set_start(ctx(), nullptr, nullptr), "start point");
  } else {
    PrimalDualPoint z = restrict_point(transform_, z0_.primal, z0_.dual);
    primal_to_work(z.primal);
    device::check(folp_gpu_set_start(ctx(), z.primal.data(), z.dual.data()), "start point");
  }

  double max_abs = 0.0, norm_c = 0.0, norm_q = 0.0;
  device::check(folp_gpu_working_stats(ctx(), &max_abs, &norm_c, &norm_q), "working stats");
  omega_ = 1.0;
  if (p_.scale_invariant_initial_primal_weight) {
    // initialize_primal_weight (solver.cpp:421-427)
    if (norm_c > p_.eps_zero && norm_q > p_.eps_zero) omega_ = norm_c / norm_q;
  }
  const bool has_entries = work_->constraint_matrix.nnz() > 0;
  if (p_.step_policy == StepPolicy::kConstant) {
    double norm = 0.0;
    if (has_entries) {
      std::vector<double> v0 = start_vector(work_->num_variables());
      primal_to_work(v0);
      int64_t mult = 0;
      device::check(folp_gpu_spectral_norm(ctx(), v0.data(), kPowerTol, kPowerMaxIters, &norm,
                                           &mult),
                    "estimate_spectral_norm");
      ledger_.add_k(mult / 2);
      ledger_.add_kt(mult / 2);
    }
    eta_constant_ = norm > 0.0 ? kConstantSafety / norm : 1.0;
  } else {
    eta_hat_ = 1.0 / (has_entries ? max_abs : 1.0);
    mp_eta_ = eta_hat_;  // solver.cpp:879-880
    mp_theta_ = 1.0;
  }

  mark("stepsize");
  time_setup_ = elapsed();
  {
    const ConvergenceInfo info0 = evaluate(FOLP_PT_CURRENT);
    tmpl_.trace.push_back(TraceEntry{0, kkt_passes(ledger_), info0, info0});
    log_evaluation(info0, info0);
    if (check_termination(info0, p_.eps_optimal)) {
      return finish(TerminationReason::kOptimal, FOLP_PT_CURRENT, info0);
    }
  }
  return std::nullopt;
}

std::optional<SolveResult> Driver::advance(Index evaluations) {
  const Index cadence = p_.evaluation_cadence;
  for (Index evals = 0;;) {
    if (evals >= evaluations) return std::nullopt;
    if (k_total_ >= p_.iteration_limit) return finish_limit(TerminationReason::kIterationLimit);
    if (kkt_passes(ledger_) >= p_.kkt_pass_limit) {
      return finish_limit(TerminationReason::kKktPassLimit);
    }
    if (decision_clock() >= p_.time_limit_seconds) {
      return finish_limit(TerminationReason::kTimeLimit);
    }

    Index target = p_.record_iterate_trace ? 1 : cadence - (t_inner_ % cadence);
    target = std::min<Index>(target, p_.iteration_limit - k_total_);
    target = std::min<Index>(target, 4096);
    folp_gpu_loop loop{};
    loop.policy = p_.step_policy == StepPolicy::kConstant       ? FOLP_STEP_CONSTANT
                  : p_.step_policy == StepPolicy::kMalitskyPock ? FOLP_STEP_MALITSKY_POCK
                                                                : FOLP_STEP_ADAPTIVE;
    loop.target = target;
    loop.k_total = k_total_;
    loop.t_inner = t_inner_;
    loop.step_trials = tmpl_.step_trials;
    loop.violations = tmpl_.step_condition_violations;
    loop.ledger_k = ledger_.k_multiplies;
    loop.ledger_kt = ledger_.kt_multiplies;
    loop.iteration_limit = p_.iteration_limit;
    loop.kkt_pass_limit = p_.kkt_pass_limit;
    loop.omega = omega_;
    loop.eta = loop.policy == FOLP_STEP_CONSTANT        ? eta_constant_
               : loop.policy == FOLP_STEP_MALITSKY_POCK ? mp_eta_
                                                        : eta_hat_;
    loop.theta = mp_theta_;
    loop.mp_breaking_factor = p_.mp_breaking_factor;
    loop.mp_downscaling_factor = p_.mp_downscaling_factor;
    loop.mp_interpolation_coefficient = p_.mp_interpolation_coefficient;
    if (loop.policy == FOLP_STEP_ADAPTIVE) {
      red_.resize(static_cast<std::size_t>(target));
      grow_.resize(static_cast<std::size_t>(target));
      for (Index i = 0; i < target; ++i) step_factors(k_total_ + i + 1, red_[i], grow_[i]);
      loop.reduction = red_.data();
      loop.growth = grow_.data();
    }
    const auto t_chunk = Clock::now();
    device::check(folp_gpu_run_chunk(ctx(), &loop), "pdhg chunk");
    time_chunks_ += std::chrono::duration<double>(Clock::now() - t_chunk).count();
    k_total_ = loop.k_total;
    t_inner_ = loop.t_inner;
    tmpl_.step_trials = loop.step_trials;
    tmpl_.step_condition_violations = loop.violations;
    ledger_.k_multiplies = loop.ledger_k;
    ledger_.kt_multiplies = loop.ledger_kt;
    if (loop.accepted > 0) last_eta_used_ = loop.last_eta_used;
    if (loop.policy == FOLP_STEP_ADAPTIVE) eta_hat_ = loop.eta;
    if (loop.policy == FOLP_STEP_MALITSKY_POCK) {
      mp_eta_ = loop.eta;
      mp_theta_ = loop.theta;
    }
    avg_weight_ = loop.avg_weight;
    if (p_.record_iterate_trace && loop.accepted > 0) record_iterate();
    if (loop.status == FOLP_CHUNK_NONFINITE || loop.status == FOLP_CHUNK_UNDERFLOW) {
      return finish_numerical_error();
    }
    if (loop.status == FOLP_CHUNK_DONE && t_inner_ % cadence == 0) {
      SolveResult out;
      ++evals;
      try {
        const auto t_eval = Clock::now();
        const bool done = evaluate_and_maybe_restart(out);
        time_evals_ += std::chrono::duration<double>(Clock::now() - t_eval).count();
        if (done) return out;
      } catch (const NonFiniteIterate&) {
        return finish_numerical_error();
      }
    }
  }
}

}  // namespace

std::string to_string(TerminationReason reason) {
  switch (reason) {
    case TerminationReason::kOptimal: return "Optimal";
    case TerminationReason::kIterationLimit: return "IterationLimit";
    case TerminationReason::kKktPassLimit: return "KktPassLimit";
    case TerminationReason::kTimeLimit: return "TimeLimit";
    case TerminationReason::kNumericalError: return "NumericalError";
    case TerminationReason::kPrimalInfeasibleDetected: return "PrimalInfeasibleDetected";
    case TerminationReason::kDualUnboundedDetected: return "DualUnboundedDetected";
  }
  return "Unknown";
}

// ---------------------------------------------------------------------
// Step-level API: the same device kernels on a one-shot context.

namespace {

struct StepOut {
  PrimalDualPoint next;
  folp_gpu_loop loop{};
};

StepOut one_step(const LinearProgram& lp, const PrimalDualPoint& z, double omega, double eta,
                 Index k, int policy, KktPassLedger* ledger, double theta = 1.0,
                 const SolverParams* mp = nullptr) {
  device::Context ctx(lp);
  ctx.set_point(FOLP_PT_CURRENT, z.primal, z.dual);
  StepOut out;
  folp_gpu_loop& loop = out.loop;
  double red = 0.0, grow = 0.0;
  step_factors(k, red, grow);
  loop.policy = policy;
  loop.theta = theta;
  if (mp != nullptr) {
    loop.mp_breaking_factor = mp->mp_breaking_factor;
    loop.mp_downscaling_factor = mp->mp_downscaling_factor;
    loop.mp_interpolation_coefficient = mp->mp_interpolation_coefficient;
  }
  loop.target = 1;
  loop.k_total = k - 1;
  loop.iteration_limit = std::numeric_limits<Index>::max();
  loop.kkt_pass_limit = kInf;
  loop.omega = omega;
  loop.eta = eta;
  loop.reduction = &red;
  loop.growth = &grow;
  device::check(folp_gpu_run_chunk(ctx.get(), &loop), "pdhg step");
  if (ledger != nullptr) {
    ledger->add_k(loop.ledger_k);
    ledger->add_kt(loop.ledger_kt);
  }
  if (loop.status == FOLP_CHUNK_NONFINITE) {
    throw NonFiniteIterate(policy == FOLP_STEP_MALITSKY_POCK
                               ? "malitsky_pock_step: non-finite iterate"
                               : "pdhg step produced a NaN or infinite iterate");
  }
  if (loop.status == FOLP_CHUNK_UNDERFLOW) {
    throw StepSizeUnderflow(policy == FOLP_STEP_MALITSKY_POCK
                                ? "malitsky_pock_step: step size underflow"
                                : "adaptive_step: step size underflow");
  }
  out.next = ctx.get_point(FOLP_PT_CURRENT);
  return out;
}

}  // namespace

PrimalDualPoint pdhg_step(const LinearProgram& lp, const PrimalDualPoint& z, double eta,
                          double omega, KktPassLedger* ledger) {
  require_point(lp, z, "pdhg_step");
  if (!(eta > 0.0)) throw std::invalid_argument("pdhg_step: eta must be > 0");
  if (!(omega > 0.0)) throw NonPositiveWeight("pdhg_step: omega must be > 0");
  return one_step(lp, z, omega, eta, 1, FOLP_STEP_CONSTANT, ledger).next;
}

double step_size_limit(const PrimalDualPoint& dz, double cross_term, double omega) {
  if (!(omega > 0.0)) throw NonPositiveWeight("step_size_limit: omega must be > 0");
  if (!(cross_term > 0.0)) return kInf;
  const double movement_sq =
      omega * linalg::norm2_squared(dz.primal) + linalg::norm2_squared(dz.dual) / omega;
  return movement_sq / (2.0 * cross_term);
}

AdaptiveStepResult adaptive_step(const LinearProgram& lp, const PrimalDualPoint& z, double omega,
                                 double eta_hat, Index k, KktPassLedger* ledger) {
  require_point(lp, z, "adaptive_step");
  if (k < 1) throw std::invalid_argument("adaptive_step: counter k is 1-based");
  if (!(eta_hat > 0.0)) throw std::invalid_argument("adaptive_step: eta_hat must be > 0");
  StepOut s = one_step(lp, z, omega, eta_hat, k, FOLP_STEP_ADAPTIVE, ledger);
  AdaptiveStepResult r;
  r.next = std::move(s.next);
  r.eta_used = s.loop.last_eta_used;
  r.eta_hat_next = s.loop.eta;
  r.trials = s.loop.step_trials;
  r.movement_sq = s.loop.last_movement;
  r.cross_term = s.loop.last_cross;
  return r;
}

MalitskyPockResult malitsky_pock_step(const LinearProgram& lp, const PrimalDualPoint& z,
                                      double omega, double eta_prev, double theta_prev,
                                      const SolverParams& params, KktPassLedger* ledger) {
  require_point(lp, z, "malitsky_pock_step");
  if (!(eta_prev > 0.0) || !(theta_prev > 0.0)) {
    throw std::invalid_argument("malitsky_pock_step: needs positive previous step size and ratio");
  }
  StepOut s = one_step(lp, z, omega, eta_prev, 1, FOLP_STEP_MALITSKY_POCK, ledger, theta_prev,
                       &params);
  MalitskyPockResult r;
  r.next = std::move(s.next);
  r.eta_next = s.loop.eta;
  r.theta_next = s.loop.theta;
  r.trials = s.loop.step_trials;
  return r;
}

double normalized_duality_gap(const LinearProgram& lp, const PrimalDualPoint& z, double radius,
                              double omega, KktPassLedger* ledger) {
  require_point(lp, z, "normalized_duality_gap");
  if (!(radius > 0.0)) throw NonPositiveRadius("normalized_duality_gap: radius must be > 0");
  if (!(omega > 0.0)) throw NonPositiveWeight("normalized_duality_gap: omega must be > 0");
  device::Context ctx(lp);
  ctx.set_point(FOLP_PT_AUX, z.primal, z.dual);
  double gap = 0.0;
  device::check(folp_gpu_ndg(ctx.get(), FOLP_PT_AUX, radius, omega, &gap), "normalized_duality_gap");
  if (ledger != nullptr) {
    ledger->add_kt();
    ledger->add_k();
  }
  return gap;
}

RestartCandidate restart_candidate(const LinearProgram& lp, const PrimalDualPoint& current,
                                   const PrimalDualPoint& average,
                                   const PrimalDualPoint& last_restart, double omega,
                                   KktPassLedger* ledger) {
  auto gap_from = [&](const PrimalDualPoint& p) {
    PrimalDualPoint diff;
    diff.primal.resize(p.primal.size());
    diff.dual.resize(p.dual.size());
    linalg::subtract(p.primal, last_restart.primal, diff.primal);
    linalg::subtract(p.dual, last_restart.dual, diff.dual);
    const double radius = weighted_norm(diff, omega);
    if (radius == 0.0) return 0.0;
    return normalized_duality_gap(lp, p, radius, omega, ledger);
  };
  const double mu_c = gap_from(current);
  const double mu_a = gap_from(average);
  if (mu_c < mu_a) return RestartCandidate{current, mu_c, false};
  return RestartCandidate{average, mu_a, true};
}

RestartDecision should_restart(double mu_candidate, double reference_gap,
                               std::optional<double> last_candidate_gap, Index t_inner,
                               Index k_total, const SolverParams& params) {
  // solver.cpp:395-419: the stricter beta triggers alone, the looser one only
  // gates the no-progress test.
  const double strong = std::min(params.beta_necessary, params.beta_sufficient);
  const double gate = std::max(params.beta_necessary, params.beta_sufficient);
  if (mu_candidate <= strong * reference_gap) return RestartDecision::kSufficient;
  if (mu_candidate <= gate * reference_gap && last_candidate_gap.has_value() &&
      mu_candidate > *last_candidate_gap) {
    return RestartDecision::kNecessaryNoProgress;
  }
  if (static_cast<double>(t_inner) >= params.beta_artificial * static_cast<double>(k_total)) {
    return RestartDecision::kArtificial;
  }
  return RestartDecision::kNoRestart;
}

double initialize_primal_weight(std::span<const double> c, std::span<const double> q,
                                double eps_zero) {
  const double nc = linalg::norm2(c), nq = linalg::norm2(q);
  return (nc > eps_zero && nq > eps_zero) ? nc / nq : 1.0;
}

double update_primal_weight(const PrimalDualPoint& z_new, const PrimalDualPoint& z_old,
                            double omega_prev, double theta, double eps_zero) {
  if (!(omega_prev > 0.0)) throw NonPositiveWeight("update_primal_weight: omega must be > 0");
  if (theta == 0.0) return omega_prev;
  const double dx = linalg::diff_norm2(z_new.primal, z_old.primal);
  const double dy = linalg::diff_norm2(z_new.dual, z_old.dual);
  if (dx > eps_zero && dy > eps_zero) {
    return std::exp(theta * std::log(dy / dx) + (1.0 - theta) * std::log(omega_prev));
  }
  return omega_prev;
}

SolveResult solve(const LinearProgram& lp_raw, const SolverParams& params,
                  const PrimalDualPoint& z0) {
  return Driver(lp_raw, params, z0).run();
}

SolveResult solve_sharded(const LinearProgram& lp_raw, const SolverParams& params,
                          const PrimalDualPoint& z0, const folp_gpu_shard& shard) {
  if (params.step_policy == StepPolicy::kMalitskyPock) {
    throw std::invalid_argument("solve_sharded: the Malitsky-Pock policy runs on one GPU only");
  }
  return Driver(lp_raw, params, z0, &shard).run();
}

// ---- resumable session (include/folp_c.h folp_session_*) -------------
struct SolveSession::Impl {
  LinearProgram lp;
  SolverParams params;
  PrimalDualPoint z0;
  std::optional<folp_gpu_shard> shard;
  std::unique_ptr<Driver> driver;
  std::optional<SolveResult> result;
};

SolveSession::SolveSession(LinearProgram lp, const SolverParams& params, PrimalDualPoint z0,
                           const folp_gpu_shard* shard)
    : impl_(new Impl{std::move(lp), params, std::move(z0), std::nullopt, nullptr, std::nullopt}) {
  if (shard != nullptr) impl_->shard = *shard;
  impl_->driver = std::make_unique<Driver>(impl_->lp, impl_->params, impl_->z0,
                                           impl_->shard ? &*impl_->shard : nullptr);
  impl_->result = impl_->driver->start();
}

SolveSession::~SolveSession() = default;

bool SolveSession::advance(Index evaluations) {
  if (!impl_->result) impl_->result = impl_->driver->advance(evaluations);
  return impl_->result.has_value();
}

bool SolveSession::finished() const { return impl_->result.has_value(); }
Index SolveSession::iterations() const { return impl_->driver->iterations(); }
folp_gpu_ctx* SolveSession::context() const { return impl_->driver->context(); }
const SolveResult* SolveSession::result() const {
  return impl_->result ? &*impl_->result : nullptr;
}

SolveResult solve(const LinearProgram& lp_raw, const SolverParams& params) {
  const PrimalDualPoint origin;  // not read: the device zero-fills the start point
  return Driver(lp_raw, params, origin, nullptr, true).run();
}

}  // namespace folp
