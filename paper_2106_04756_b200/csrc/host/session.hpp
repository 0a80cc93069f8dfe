// session.hpp -- a folp::solve that can be advanced one evaluation period
// at a time (used by the C ABI folp_session_* and by bench.py to time the
// loop with CUDA events on the engine stream).  run-to-completion equals
// folp::solve exactly.
#pragma once

#include <memory>

#include "folp/presolve.hpp"
#include "folp/sharded.hpp"
#include "folp/solver.hpp"
#include "folp_gpu.h"

namespace folp {

class SolveSession {
 public:
  // shard != nullptr: this process/thread is one row shard of a multi-GPU
  // solve (include/folp_gpu.h folp_gpu_shard); every shard builds the same
  // session on the same LP.
  SolveSession(LinearProgram lp, const SolverParams& params, PrimalDualPoint z0,
               const folp_gpu_shard* shard = nullptr);
  ~SolveSession();
  // Advances by up to `evaluations` evaluation periods (evaluation_cadence
  // iterations + the evaluation/restart step each); true once finished.
  bool advance(Index evaluations);
  bool finished() const;
  Index iterations() const;
  folp_gpu_ctx* context() const;       // nullptr when no device loop ran
  const SolveResult* result() const;   // set once finished

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

// folp::solve_sharded: include/folp/sharded.hpp

namespace detail {
// presolve_for_solve that also returns the column degrees of `lp`
// (presolve.cpp; the driver's column ordering reuses them)
PresolveResult presolve_for_solve(const LinearProgram& lp, std::vector<Index>* degrees);
}  // namespace detail

}  // namespace folp
