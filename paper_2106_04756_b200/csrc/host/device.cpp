// device.cpp -- host wrappers over the engine C ABI.
#include "device.hpp"

#include <cmath>

#include "folp/sparse_matrix.hpp"

namespace folp::device {

void raise(int code, const std::string& where) {
  const std::string msg = where + ": " + folp_gpu_last_error();
  switch (code) {
    case FOLP_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case FOLP_E_EMPTY_MATRIX: throw EmptyMatrix(msg);
    case FOLP_E_UNSUPPORTED_NORM: throw UnsupportedNorm(msg);
    case FOLP_E_NONPOSITIVE_WEIGHT: throw NonPositiveWeight(msg);
    case FOLP_E_NONPOSITIVE_RADIUS: throw NonPositiveRadius(msg);
    case FOLP_E_STEP_UNDERFLOW: throw StepSizeUnderflow(msg);
    case FOLP_E_NONFINITE: throw NonFiniteIterate(msg);
    case FOLP_E_INFINITE_PRODUCT: throw InfiniteProduct(msg);
    case FOLP_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}

void Context::create(const SparseMatrix& k, const double* c, const double* q, const double* l,
                     const double* u, Index m1, double constant, const Index* col_order) {
  folp_gpu_problem p{};
  p.num_rows = k.num_rows();
  p.num_cols = k.num_cols();
  p.num_inequality_rows = m1;
  p.nnz = k.nnz();
  p.row_start = k.row_start().data();
  p.row_cols = k.row_cols().data();
  p.row_values = k.row_values().data();
  // The column mirror goes up only if the host already has it; otherwise
  // the engine transposes K on the device.
  if (k.has_column_mirror()) {
    p.col_start = k.col_start().data();
    p.col_rows = k.col_rows().data();
    p.col_values = k.col_values().data();
  }
  p.objective = c;
  p.right_hand_side = q;
  p.variable_lower = l;
  p.variable_upper = u;
  p.objective_constant = constant;
  // A default-constructed SparseMatrix has empty pointer vectors.
  std::vector<Index> zero_rows, zero_cols;
  if (k.row_start().empty()) {
    zero_rows.assign(static_cast<std::size_t>(k.num_rows()) + 1, 0);
    p.row_start = zero_rows.data();
  }
  if (p.col_start != nullptr && k.col_start().empty()) {
    zero_cols.assign(static_cast<std::size_t>(k.num_cols()) + 1, 0);
    p.col_start = zero_cols.data();
  }
  check(folp_gpu_create_ordered(&p, col_order, -1, &ctx_), "device context");
  m_ = k.num_rows();
  n_ = k.num_cols();
}

Context::Context(const LinearProgram& lp, const Index* col_order) {
  create(lp.constraint_matrix, lp.objective.data(), lp.right_hand_side.data(),
         lp.variable_lower.data(), lp.variable_upper.data(), lp.num_inequality_rows,
         lp.objective_constant, col_order);
}

Context::Context(const SparseMatrix& k) {
  create(k, nullptr, nullptr, nullptr, nullptr, 0, 0.0);
}

Context::~Context() {
  if (ctx_ != nullptr) folp_gpu_destroy(ctx_);
}

void Context::set_point(int which, std::span<const double> x, std::span<const double> y) {
  check(folp_gpu_set_point(ctx_, which, x.data(), y.data()), "set_point");
}

PrimalDualPoint Context::get_point(int which) {
  PrimalDualPoint z;
  z.primal.resize(static_cast<std::size_t>(n_));
  z.dual.resize(static_cast<std::size_t>(m_));
  check(folp_gpu_get_point(ctx_, which, z.primal.data(), z.dual.data()), "get_point");
  return z;
}

ConvergenceInfo to_info(const folp_gpu_eval& e, double objective_constant) {
  if (e.nonfinite) {
    throw NonFiniteIterate("convergence_info: point has NaN or inf entries");
  }
  if (e.infinite_product) {
    throw InfiniteProduct("dual_objective: lambda outside its sign cone");
  }
  // termination.cpp:43-71 final arithmetic
  ConvergenceInfo info;
  info.primal_objective = e.c_dot_x + objective_constant;
  info.dual_objective = e.dual_objective;
  info.gap_abs = std::fabs(info.dual_objective - info.primal_objective);
  info.primal_residual_norm = std::sqrt(e.primal_sq);
  info.dual_residual_norm = std::sqrt(e.dual_sq);
  info.norm_q = e.norm_q;
  info.norm_c = e.norm_c;
  return info;
}

void Context::attach_shard(const SparseMatrix& k, const folp_gpu_shard& spec) {
  check(folp_gpu_shard_attach(ctx_, &spec, k.row_start().data(), k.col_start().data(),
                              k.col_rows().data()),
        "shard attach");
}

ConvergenceInfo Context::evaluate(int which, bool raw, double objective_constant) {
  folp_gpu_eval e{};
  check(folp_gpu_evaluate(ctx_, which, raw ? 1 : 0, &e), "convergence_info");
  return to_info(e, objective_constant);
}

}  // namespace folp::device
