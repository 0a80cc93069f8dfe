// termination.cpp -- convergence_info on the B200; the termination test and
// the SGM10 statistic are scalar host code
// (/root/reference/proj/src/termination.cpp:23-92).
#include "folp/termination.hpp"

#include <cmath>

#include "device.hpp"

namespace folp {

ConvergenceInfo convergence_info(const LinearProgram& lp, std::span<const double> x,
                                 std::span<const double> y, KktPassLedger* ledger) {
  if (static_cast<Index>(x.size()) != lp.num_variables() ||
      static_cast<Index>(y.size()) != lp.num_rows()) {
    throw DimensionMismatch("convergence_info: point size mismatch");
  }
  if (lp.num_variables() == 0 && lp.num_rows() == 0) {
    // The empty program (everything presolved away): nothing to launch.
    ConvergenceInfo info;
    info.primal_objective = lp.objective_constant;
    info.dual_objective = lp.objective_constant;
    if (ledger != nullptr) {
      ledger->add_k();
      ledger->add_kt();
    }
    return info;
  }
  device::Context ctx(lp);
  ctx.set_point(FOLP_PT_AUX, x, y);
  try {
    ConvergenceInfo info = ctx.evaluate(FOLP_PT_AUX, true, lp.objective_constant);
    if (ledger != nullptr) {
      ledger->add_k();
      ledger->add_kt();
    }
    return info;
  } catch (const InfiniteProduct&) {
    if (ledger != nullptr) {  // the reference charges before dual_objective throws
      ledger->add_k();
      ledger->add_kt();
    }
    throw;
  }
}

bool check_termination(const ConvergenceInfo& info, double eps) {
  const double obj_scale = 1.0 + std::fabs(info.dual_objective) + std::fabs(info.primal_objective);
  const bool gap_ok = info.gap_abs <= eps * obj_scale;
  const bool primal_ok = info.primal_residual_norm <= eps * (1.0 + info.norm_q);
  const bool dual_ok = info.dual_residual_norm <= eps * (1.0 + info.norm_c);
  return gap_ok && primal_ok && dual_ok;
}

double sgm10(std::span<const double> values, double shift) {
  if (values.empty()) throw std::invalid_argument("sgm10: empty input");
  double log_sum = 0.0;
  for (const double v : values) log_sum += std::log(v + shift);
  return std::exp(log_sum / static_cast<double>(values.size())) - shift;
}

}  // namespace folp
