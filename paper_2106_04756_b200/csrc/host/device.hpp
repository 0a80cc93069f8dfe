// device.hpp -- host-side RAII over the engine's C ABI (include/folp_gpu.h).
//
// Maps FOLP_E_* status codes back onto the folp exception taxonomy
// (types.hpp), so the C++ driver keeps the reference's control flow
// (solver.cpp:920-942 catches NonFiniteIterate / StepSizeUnderflow).
#pragma once

#include <string>
#include <vector>

#include "folp/lp_model.hpp"
#include "folp/termination.hpp"
#include "folp/types.hpp"
#include "folp_gpu.h"

namespace folp::device {

[[noreturn]] void raise(int code, const std::string& where);

inline void check(int code, const char* where) {
  if (code != FOLP_OK) raise(code, where);
}

// convergence_info from the device reductions of a point; throws
// NonFiniteIterate / InfiniteProduct exactly where convergence_info would.
ConvergenceInfo to_info(const folp_gpu_eval& e, double objective_constant);

// One device context holding one LP.
class Context {
 public:
  Context() = default;
  // col_order: working column order (folp_gpu_create_ordered), or null
  explicit Context(const LinearProgram& lp, const Index* col_order = nullptr);
  // Matrix-only context (vectors read as zeros).
  explicit Context(const SparseMatrix& k);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  Context(Context&& o) noexcept : ctx_(o.ctx_), m_(o.m_), n_(o.n_) { o.ctx_ = nullptr; }

  folp_gpu_ctx* get() const { return ctx_; }
  Index rows() const { return m_; }
  Index cols() const { return n_; }

  void set_point(int which, std::span<const double> x, std::span<const double> y);
  PrimalDualPoint get_point(int which);
  // convergence_info quantities of a slot; throws NonFiniteIterate /
  // InfiniteProduct exactly where convergence_info would.
  ConvergenceInfo evaluate(int which, bool raw, double objective_constant);
  // Row shard of a multi-GPU solve (after rescale); k = the context's matrix.
  void attach_shard(const SparseMatrix& k, const folp_gpu_shard& spec);

 private:
  void create(const SparseMatrix& k, const double* c, const double* q, const double* l,
              const double* u, Index m1, double constant, const Index* col_order = nullptr);
  folp_gpu_ctx* ctx_ = nullptr;
  Index m_ = 0;
  Index n_ = 0;
};

}  // namespace folp::device
