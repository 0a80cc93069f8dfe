// shard_graphs.cuh -- row / column shards, the PDHG chunk graph and the evaluation graph.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

// ---------------------------------------------------------------------
// Row shards (north_star: K row-partitioned, all-reduce of the
// partial K'y and of the scalar sums).
__global__ void k_gather_values(double* out, const double* src, const int* pos, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[i] = src[pos[i]];
  }
}

// Contiguous row ranges with about equal nonzeros + rows (so empty rows
// still spread); monotone, covers [0, m).
std::vector<int64_t> shard_rows(int64_t m, const int64_t* row_start, int world) {
  std::vector<int64_t> b(static_cast<size_t>(world) + 1, 0);
  const double total = static_cast<double>(row_start[m]) + static_cast<double>(m);
  int64_t r = 0;
  for (int p = 1; p < world; ++p) {
    const double target = total * p / world;
    while (r < m && static_cast<double>(row_start[r]) + static_cast<double>(r) < target) ++r;
    b[p] = r;
  }
  b[world] = m;
  return b;
}

// The entries of rows [r0, r1) in CSC order: within every column the rows
// are increasing (sparse_matrix.cpp:82-102), so they form one sub-range.
// lptr [n+1] local column starts; pos = full-CSC positions of the entries.
void shard_local_csc(int64_t n, const int64_t* col_start, const int64_t* col_rows, int64_t r0,
                     int64_t r1, std::vector<int64_t>& lptr, std::vector<int64_t>& pos) {
  lptr.assign(static_cast<size_t>(n) + 1, 0);
  pos.clear();
  for (int64_t j = 0; j < n; ++j) {
    const int64_t* b = col_rows + col_start[j];
    const int64_t* e = col_rows + col_start[j + 1];
    const int64_t* lo = std::lower_bound(b, e, r0);
    const int64_t* hi = std::lower_bound(lo, e, r1);
    for (const int64_t* k = lo; k < hi; ++k) pos.push_back(k - col_rows);
    lptr[j + 1] = static_cast<int64_t>(pos.size());
  }
}

// Column partition: the entries of columns [c0, c1) in CSR order (a
// counting pass by row over the CSC range; columns ascend within each row
// because the range is walked column by column).  lptr [m+1] local row
// starts; pos = full-CSC positions of the entries.
void shard_local_csr(int64_t m, const int64_t* col_start, const int64_t* col_rows, int64_t c0,
                     int64_t c1, std::vector<int64_t>& lptr, std::vector<int64_t>& pos) {
  lptr.assign(static_cast<size_t>(m) + 1, 0);
  const int64_t k0 = col_start[c0], k1 = col_start[c1];
  for (int64_t k = k0; k < k1; ++k) ++lptr[static_cast<size_t>(col_rows[k]) + 1];
  for (int64_t i = 0; i < m; ++i) lptr[i + 1] += lptr[i];
  pos.assign(static_cast<size_t>(k1 - k0), 0);
  std::vector<int64_t> fill(lptr.begin(), lptr.end() - 1);
  for (int64_t k = k0; k < k1; ++k) pos[static_cast<size_t>(fill[col_rows[k]]++)] = k;
}

void ensure_gathered(folp_gpu_ctx* c) {
  if (!c->sharded() || !c->rows_dirty) return;
  const int cur = c->st_h->cur;
  if (c->col_part) {  // y, Kx and avg_y are replicated; x and avg_x are not
    c->comm->gather_rows(c->x[cur], c->shard_bounds, c->stream);
    c->comm->gather_rows(c->avg_x, c->shard_bounds, c->stream);
    if (c->pdual) {  // ... and with the partitioned dual epilogue Kx, avg_y are not
      c->comm->gather_rows(c->kx[cur], c->pd_bounds, c->stream);
      c->comm->gather_rows(c->avg_y, c->pd_bounds, c->stream);
    }
  } else {
    c->comm->gather_rows(c->y[cur], c->shard_bounds, c->stream);
    c->comm->gather_rows(c->kx[cur], c->shard_bounds, c->stream);
    c->comm->gather_rows(c->avg_y, c->shard_bounds, c->stream);
    if (c->pdual) c->comm->gather_rows(c->avg_x, c->pd_bounds, c->stream);  // own columns only
  }
  c->rows_dirty = false;
}

// Entry of every engine call that reads the iterate: a sharded context
// first reassembles the row-space vectors the loop kept local.
void prep(folp_gpu_ctx* c) {
  set_device(c);
  ensure_gathered(c);
}

// One sharded trial slot (see ops.cuh, "Row-sharded trial" and
// "Column-sharded trial").
void launch_shard_slot(folp_gpu_ctx* c, const LoopBufs& b) {
  ShardComm& comm = *c->comm;
  if (comm.peer) {  // the exchange fused into the partial product's epilogue
    const int par = c->peer_parity;
    c->peer_parity ^= 1;
    if (c->col_part) {
      EpiPrimal ep{b};
      ep.shard_out = c->kty_part + c->m;  // partial sx, bad: forwarded by the producer
      c->seg(c->lcols, c->csc_work, ep, 2);
      EpiShardPart sp{b, c->kty_part, nullptr, true};
      sp.outs = comm.peer_dst(par);
      sp.world = comm.world;
      sp.extra = c->kty_part + c->m;
      sp.extra_at = c->m;
      if (c->pdual) sp.own_chunk = c->pd_chunk;
      c->seg(c->lrows, c->lcsc_val, sp, 1);
      comm.peer_fence(c->stream);
      if (c->pdual) {  // own rows only, y' and the partial sums to every rank
        OpShardDualOwn od{EpiDual{b}, comm.peer_src(par), comm.peer_dst(par), c->pd_vdst};
        od.world = comm.world;
        od.rank = comm.rank;
        od.r0 = c->pd_bounds[comm.rank];
        od.m = c->m;
        c->ew(c->pd_bounds[comm.rank + 1] - od.r0, od, 3);
        comm.peer_fence(c->stream);
        k_shard_decide_rows<<<1, 1, 0, c->stream>>>(b, comm.peer_src(par), comm.world, c->m);
        ++c->launches;
        CK(cudaGetLastError());
        return;
      }
      OpShardDual od{EpiDual{b}, nullptr, nullptr};
      od.src = comm.peer_src(par);
      od.world = comm.world;
      od.m = c->m;
      c->ew(c->m, od, 3);
      return;
    }
    EpiShardPart sp{b, c->kty_part, nullptr, false};
    sp.outs = comm.peer_dst(par);
    sp.world = comm.world;
    if (c->pdual) sp.own_chunk = c->pd_chunk;
    c->seg(c->lcols, c->lcsc_val, sp, 1);
    comm.peer_fence(c->stream);
    if (c->pdual) {  // primal step on own columns, x' and its sums to every rank
      OpShardPrimalOwn op{EpiPrimal{b}, comm.peer_src(par), comm.peer_dst(par), c->pd_vdst};
      op.world = comm.world;
      op.rank = comm.rank;
      op.r0 = c->pd_bounds[comm.rank];
      op.n = c->n;
      c->ew(c->pd_bounds[comm.rank + 1] - op.r0, op, 2);
      comm.peer_fence(c->stream);
      EpiDual ed{b};
      ed.shard_peers = comm.peer_dst(par);  // its three sums to every rank's area
      ed.shard_world = comm.world;
      ed.shard_at = c->n + 2;
      c->seg(c->lrows, c->csr_work, ed, 3);
      comm.peer_fence(c->stream);
      k_shard_decide_rows<<<1, 1, 0, c->stream>>>(b, comm.peer_src(par), comm.world, c->n);
      ++c->launches;
      CK(cudaGetLastError());
      return;
    }
    OpShardPrimal op{EpiPrimal{b}, nullptr};
    op.src = comm.peer_src(par);
    op.world = comm.world;
    c->ew(c->n, op, 2);
    EpiDual ed{b};
    ed.shard_out = c->shard_sums;
    c->seg(c->lrows, c->csr_work, ed, 3);
    comm.allreduce_sum(c->shard_sums, 3, c->stream);
    k_shard_decide<<<1, 1, 0, c->stream>>>(b, c->shard_sums);
    ++c->launches;
    CK(cudaGetLastError());
    return;
  }
  if (c->col_part) {
    EpiPrimal ep{b};
    ep.shard_out = c->kty_part + c->m;  // partial sx, bad ride with the partial Kx'
    c->seg(c->lcols, c->csc_work, ep, 2);
    c->seg(c->lrows, c->lcsc_val, EpiShardPart{b, c->kty_part, nullptr, true}, 1);
    c->comm->allreduce_sum(c->kty_part, c->m + 2, c->stream);
    c->ew(c->m, OpShardDual{EpiDual{b}, c->kty_part, c->kty_part + c->m}, 3);
    return;
  }
  c->seg(c->lcols, c->lcsc_val, EpiShardPart{b, c->kty_part, nullptr, false}, 1);
  c->comm->allreduce_sum(c->kty_part, c->n, c->stream);
  c->ew(c->n, OpShardPrimal{EpiPrimal{b}, c->kty_part}, 2);
  EpiDual ed{b};
  ed.shard_out = c->shard_sums;
  c->seg(c->lrows, c->csr_work, ed, 3);
  c->comm->allreduce_sum(c->shard_sums, 3, c->stream);
  k_shard_decide<<<1, 1, 0, c->stream>>>(b, c->shard_sums);
  ++c->launches;
  CK(cudaGetLastError());
}

// One trial slot of a step policy: adaptive / constant = {A; B},
// Malitsky-Pock = {MP-A (first trial only); MP-E; MP-B; MP-C}.
void launch_slot(folp_gpu_ctx* c, int policy, const LoopBufs& b) {
  if (policy == FOLP_STEP_MALITSKY_POCK) {
    c->seg(c->cols, c->csc_work, EpiMpPrimal{b}, 2, 0);
    c->ew(c->n, OpMpExtrapolate{b}, 5, 1);
    c->seg(c->rows, c->csr_work, EpiMpDual{b}, 3, 1);
    c->seg(c->cols, c->csc_work, EpiMpCheck{b}, 6, 0);
  } else {
    // programmatic dependent launches: each product starts while the
    // previous one drains (FOLP_PDL=0 disables)
    const char* env = std::getenv("FOLP_PDL");
    c->pdl = env == nullptr || std::atoi(env) > 0;
    // ordered mode: the products only store their terms; one cooperative
    // k_exact_fold folds them exactly in the reference's order and decides
    const bool fold = c->ordered && c->fold_grid > 0 && !c->sharded();
    // tree mode, plain (unsharded, unwindowed) products: kernel A leaves its
    // two sums as CTA partials for kernel B's last CTA (segdot.cuh
    // DeferredSums; FOLP_DEFER_A=0 keeps kernel A's own last-CTA pass)
    const char* denv = std::getenv("FOLP_DEFER_A");
    const bool defer_a = !c->ordered && !c->sharded() && c->brows.windows == 0 &&
                         c->bcols.windows == 0 && (denv == nullptr || std::atoi(denv) > 0);
    try {
      c->defer_tail = fold;
      c->a_defer = defer_a;
      axis_product(c, false, true, EpiPrimal{b}, 2, 0);
      c->a_defer = false;
      EpiDual ed{b};
      if (defer_a) {
        ed.a_partials = c->partials_a;
        ed.a_np = c->a_np;
      }
      if (c->sell && c->sell_packed && !c->sharded() && c->brows.windows == 0) {
        c->seg(c->rows_sell, c->csr_work, ed, 3, 1);  // SELL-32 groups (sell.cuh)
      } else {
        axis_product(c, true, true, ed, 3, 1);
      }
      c->defer_tail = false;
      if (fold) c->launch_trial_fold(b);
    } catch (...) {
      c->pdl = false;
      c->defer_tail = false;
      c->a_defer = false;
      throw;
    }
    c->pdl = false;
  }
}

// Trial slots per iteration of the chunk graph's WHILE body: a slot whose
// loop already stopped is a pair of early-exit launches, and within the
// body the products chain by programmatic dependent launches
// (FOLP_BODY_SLOTS, default 2).
int body_slots() {
  const char* env = std::getenv("FOLP_BODY_SLOTS");
  return env ? std::max(1, std::atoi(env)) : 2;
}

// Builds the chunk graph of a policy: WHILE(running) { trial slot }.
void build_chunk_graph(folp_gpu_ctx* c, int policy) {
  c->graph_tried[policy] = true;
  if (std::getenv("FOLP_NO_GRAPH") != nullptr) return;
  cudaGraph_t graph = nullptr;
  if (cudaGraphCreate(&graph, 0) != cudaSuccess) return;
  cudaGraphConditionalHandle handle;
  bool ok = cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault) ==
            cudaSuccess;
  cudaGraphNodeParams cp = {};
  cudaGraphNode_t node;
  if (ok) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    ok = cudaGraphAddNode(&node, graph, nullptr, 0, &cp) == cudaSuccess;
  }
  if (ok) {
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    ok = cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeRelaxed) == cudaSuccess;
    if (ok) {
      const LoopBufs b = c->loop_bufs(handle, 1);
      const int64_t before = c->launches;
      try {
        const int reps = policy == FOLP_STEP_MALITSKY_POCK ? 1 : body_slots();
        for (int r = 0; r < reps; ++r) launch_slot(c, policy, b);
        c->body_slots[policy] = reps;
      } catch (...) {
        ok = false;
      }
      c->launches = before;
      cudaGraph_t captured = nullptr;
      ok = (cudaStreamEndCapture(c->stream, &captured) == cudaSuccess) && ok;
    }
  }
  if (ok) ok = cudaGraphInstantiate(&c->chunk_exec[policy], graph, 0) == cudaSuccess;
  cudaGetLastError();  // clear a failed optional path
  if (graph) cudaGraphDestroy(graph);
  c->graph_ok[policy] = ok;
  if (!ok && c->chunk_exec[policy]) {
    cudaGraphExecDestroy(c->chunk_exec[policy]);
    c->chunk_exec[policy] = nullptr;
  }
}

// The evaluation period's device work (average, both evaluations, both
// distances, both duality-gap setups, inits, the cooperative bisection and
// the result read-back) captured once per CURRENT parity; omega and the
// averaging weights are read on device at launch.  Replaces ~20 host-side
// launches per period.  Tree mode, gaps wanted, Kx of CURRENT cached.
void build_eval_graph(folp_gpu_ctx* c, int cur) {
  c->eval_tried[cur] = true;
  if (std::getenv("FOLP_EVAL_GRAPH") != nullptr && std::atoi(std::getenv("FOLP_EVAL_GRAPH")) == 0) {
    return;
  }
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  bool ok = true;
  const int64_t before = c->launches;
  c->capturing_eval = true;
  try {
    const int slots[2] = {FOLP_PT_CURRENT, FOLP_PT_AVERAGE};
    CK(cudaMemcpyAsync(c->eval_omega_d, c->eval_omega_h, sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    enqueue_average(c);
    for (int s = 0; s < 2; ++s) enqueue_evaluate(c, slots[s], 0, kResEval[s], c->kty_cache(s));
    for (int s = 0; s < 2; ++s) {
      enqueue_distance(c, slots[s], FOLP_PT_LAST, kResDist[s]);
      enqueue_ndg_setup(c, slots[s], s, 1.0, c->kty_cache(s));
      enqueue_ndg_init(c, s, kResDist[s], 0.0, 1.0);
    }
    enqueue_ndg_solve(c, {true, true}, {1.0, 1.0});
    CK(cudaMemcpyAsync(c->res_h, c->res, kResUsed * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
  } catch (...) {
    ok = false;
  }
  c->capturing_eval = false;
  c->launches = before;
  ok = (cudaStreamEndCapture(c->stream, &graph) == cudaSuccess) && ok;
  if (ok) ok = cudaGraphInstantiate(&c->eval_exec[cur], graph, 0) == cudaSuccess;
  cudaGetLastError();
  if (graph) cudaGraphDestroy(graph);
  if (!ok && c->eval_exec[cur]) {
    cudaGraphExecDestroy(c->eval_exec[cur]);
    c->eval_exec[cur] = nullptr;
  }
}
