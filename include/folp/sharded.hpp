// sharded.hpp -- folp::solve as one shard of a multi-GPU solve (B200 build
// extension; not in the reference's API).  Every shard -- one process or
// host thread per GPU -- calls it with the same LP, parameters and start
// point and receives the same SolveResult.  The shard spec (rank, world,
// partition, NCCL communicator or in-process loopback group) is the C
// struct of include/folp_gpu.h; DESIGN.md 7 describes the schedule.
#pragma once

#include "folp/solver.hpp"
#include "folp_gpu.h"

namespace folp {

SolveResult solve_sharded(const LinearProgram& lp, const SolverParams& params,
                          const PrimalDualPoint& z0, const folp_gpu_shard& shard);

}  // namespace folp
