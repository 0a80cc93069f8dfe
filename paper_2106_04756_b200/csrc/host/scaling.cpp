// scaling.cpp -- Ruiz + Pock-Chambolle preconditioning through the device
// row/column-scaling kernels (/root/reference/proj/src/scaling.cpp:32-112).
#include "folp/scaling.hpp"

#include <cmath>

#include "device.hpp"
#include "sparse_access.hpp"

namespace folp {

namespace {

std::vector<double> inverse_sqrt(std::vector<double> norms) {
  for (double& v : norms) v = v > 0.0 ? 1.0 / std::sqrt(v) : 1.0;
  return norms;
}

void check_alpha(double alpha) {
  if (!(alpha >= 0.0 && alpha <= 2.0)) {
    throw std::invalid_argument("pock_chambolle_step: alpha must be in [0,2]");
  }
  const double row_p = 2.0 - alpha;
  for (const double p : {row_p, alpha}) {
    if (std::isnan(p) || (p < 1.0 && p != 0.0)) {
      throw UnsupportedNorm("axis_norms: p must be 0, in [1, inf), or +inf");
    }
  }
}

}  // namespace

std::pair<std::vector<double>, std::vector<double>> ruiz_step(const SparseMatrix& k) {
  return {inverse_sqrt(k.axis_norms(Axis::kRows, kInf)),
          inverse_sqrt(k.axis_norms(Axis::kCols, kInf))};
}

std::pair<std::vector<double>, std::vector<double>> pock_chambolle_step(const SparseMatrix& k,
                                                                        double alpha) {
  if (!(alpha >= 0.0 && alpha <= 2.0)) {
    throw std::invalid_argument("pock_chambolle_step: alpha must be in [0,2]");
  }
  return {inverse_sqrt(k.axis_norms(Axis::kRows, 2.0 - alpha)),
          inverse_sqrt(k.axis_norms(Axis::kCols, alpha))};
}

ScaledProblem rescale_problem(const LinearProgram& lp, Index ruiz_iterations,
                              bool apply_pock_chambolle, double alpha) {
  if (apply_pock_chambolle) check_alpha(alpha);
  const Index m = lp.num_rows();
  const Index n = lp.num_variables();
  ScaledProblem out;
  out.scaling = DiagonalScaling::identity(m, n);
  LinearProgram& s = out.lp;
  s.num_inequality_rows = lp.num_inequality_rows;
  s.objective_constant = lp.objective_constant;
  s.objective.resize(static_cast<std::size_t>(n));
  s.variable_lower.resize(static_cast<std::size_t>(n));
  s.variable_upper.resize(static_cast<std::size_t>(n));
  s.right_hand_side.resize(static_cast<std::size_t>(m));
  std::vector<double> csr(static_cast<std::size_t>(lp.constraint_matrix.nnz()));
  std::vector<double> csc(csr.size());
  device::Context ctx(lp);
  device::check(folp_gpu_rescale(ctx.get(), ruiz_iterations, apply_pock_chambolle ? 1 : 0, alpha,
                                 out.scaling.row_scale.data(), out.scaling.col_scale.data()),
                "rescale_problem");
  device::check(folp_gpu_get_working(ctx.get(), csr.data(), csc.data(), s.objective.data(),
                                     s.right_hand_side.data(), s.variable_lower.data(),
                                     s.variable_upper.data()),
                "rescale_problem");
  s.constraint_matrix =
      SparseMatrixAccess::with_values(lp.constraint_matrix, std::move(csr), std::move(csc));
  return out;
}

PrimalDualPoint unscale_point(const DiagonalScaling& scaling, const PrimalDualPoint& z_scaled) {
  if (z_scaled.primal.size() != scaling.col_scale.size() ||
      z_scaled.dual.size() != scaling.row_scale.size()) {
    throw DimensionMismatch("unscale_point: size mismatch");
  }
  PrimalDualPoint z = z_scaled;
  for (std::size_t i = 0; i < z.primal.size(); ++i) z.primal[i] *= scaling.col_scale[i];
  for (std::size_t j = 0; j < z.dual.size(); ++j) z.dual[j] *= scaling.row_scale[j];
  return z;
}

}  // namespace folp
