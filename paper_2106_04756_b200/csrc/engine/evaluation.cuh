// evaluation.cuh -- the evaluation period: convergence info, distances, duality gaps, restarts.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

// ---------------------------------------------------------------------
// Evaluation period (solver.cpp:751-816) as one asynchronous sequence.
// Result-slot blocks of the period's reductions:
constexpr int kResEval[2] = {32, 44};  // [0] c'x [1] q'y [2] non-finite [3] primal^2
                                        // [4] dual^2 [5] bound terms [6] inf product
                                        // [10] dual objective (ordered)
constexpr int kResNorms = 56;           // ||q||^2, ||c||^2
constexpr int kResDist[2] = {60, 62};   // sum dx^2, sum dy^2 to LAST
constexpr int kResNdg[2] = {64, 74};    // duality-gap setup sums (10 each)
constexpr int kResUsed = 84;
static_assert(kResUsed <= kResSlots, "result slots");

// Bracket of one normalized_duality_gap evaluation from its setup sums
// (solver.cpp:318-355).  The radius is either given or the weighted
// distance to LAST of restart_candidate (solver.cpp:378-386; a zero radius
// gives a zero gap there without evaluating).
__global__ void k_ndg_init(NdgState* st, const double* sums, const double* dist, double radius,
                           double omega, const double* omega_dev) {
  if (omega_dev != nullptr) omega = *omega_dev;
  NdgState s{};
  s.omega = omega;
  s.winv = 1.0 / omega;
  const double r = dist != nullptr ? sqrt(omega * dist[0] + dist[1] / omega) : radius;
  s.radius = r;
  if (r == 0.0 || sums[0] + sums[5] == 0.0) {  // solver.cpp:324
    s.done = 1;
    s.result = 0.0;
    *st = s;
    return;
  }
  if (sums[2] + sums[7] == 0.0) {  // bounded corner, solver.cpp:339-341
    const double norm_sq = sums[3] + sums[8];
    if (sqrt(norm_sq) <= r * (1.0 + 1e-12)) {
      s.done = 1;
      s.result = (sums[4] + sums[9]) / r;
      *st = s;
      return;
    }
  }
  s.nu_lo = 0.0;
  s.nu_hi = sqrt(sums[1] + sums[6]) / r;
  ndg_candidates(s.nu_lo, s.nu_hi, s.nu);
  ndg_reciprocals(&s);
  *st = s;
}

// Tree-mode bisection of up to two duality gaps in ONE cooperative launch
// (solver.cpp:356-368).  Every pass evaluates the 7 midpoints of the next
// 3 levels per scratch set; the block partials are published, the grid
// synchronizes once, and every block sums the partials in the same order
// and replays the same decisions, so the bisection state never leaves
// shared memory until the end.  Replaces up to ~70 launches per period.
//
// Active sets: an element whose clamping state cannot change inside the
// current bracket [nu_lo, nu_hi] (clamped at nu_hi, hence over the whole
// bracket; or free at nu_lo, hence free over it; or g = 0) leaves the
// per-midpoint work for good -- its terms are the closed forms w*c^2, g*c
// (clamped) and g^2/(w*nu^2), g^2/(w*nu) (free), kept as three running sums
// Q, H, S per thread.  Each block compacts its own element range in place
// (index list in global memory, order preserved), so after the first pass
// only the elements with a breakpoint inside the bracket are read again;
// once no block has any left, ndg_finish_analytic ends the bisection from
// Q, H, S.
constexpr int kBisectThreads = 512;
constexpr int kBisectBatch = 4;  // tiles per super-tile in bisect_sweep
// per set: ||d||_w^2 and g'd per midpoint over the active elements, the
// number of active elements kept, and the running Q, H, S of the retired ones
constexpr int kBisectVals = 2 * kNuCands + 4;

struct BisectArgs {
  int64_t n, total;
  const double* g[2];
  const double* lo[2];
  const double* hi[2];
  NdgState* ns[2];
  int active[2];
  int* list[2];      // [total] per set: the blocks' active element lists
  double* partials;  // [2 parity][2 sets][kBisectVals][grid]
  int* compact[2];   // [kBisectSmall] per set: the last active elements, block 0's
  int small_limit;   // switch to one block at <= this many active elements (0: never)
};

// Once at most kBisectSmall elements of every running set still have a
// breakpoint inside the bracket, they are gathered into one list and block
// 0 finishes the bisection alone: a pass then costs one block's sweep over
// a few thousand L2-resident elements instead of a grid-wide sync.
constexpr int kBisectSmall = 4096;

// One pass over a set's active elements (tree mode): retire the elements
// whose clamping cannot change inside the bracket into the closed-form sums
// (fq, fh, fs), accumulate ||d||_w^2 and g'd at the candidates for the rest,
// and compact the list in place (order preserved).  Returns the kept count
// (the same in every thread of the block).
__device__ __forceinline__ int bisect_sweep(const BisectArgs& a, const NdgState& st, int s,
                                            int* list, int cnt, bool first, int64_t b0,
                                            double (&acc)[2 * kNuCands], double& fq, double& fh,
                                            double& fs, int* wcount) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int R = kBisectBatch;
  constexpr int W = kBisectThreads / 32;
  const double* g = a.g[s];
  const double* lo = a.lo[s];
  const double* hi = a.hi[s];
  const double omega = st.omega, winv = st.winv;
  int kept = 0;
  // Super-tiles of R x kBisectThreads elements: every index, then every
  // element load of the super-tile is issued before any is used (a pass over
  // a few thousand elements is a chain of dependent L2 round trips
  // otherwise), one barrier publishes the R tiles' keep counts, one more
  // closes the compaction.  Thread tid still visits k = tid, tid + T, ... in
  // order, so the sums and the kept list are those of a tile-by-tile sweep.
  for (int t0 = 0; t0 < cnt; t0 += R * kBisectThreads) {
    int iv[R];
    double gv[R], lov[R], hiv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = t0 + r * kBisectThreads + tid;
      iv[r] = k < cnt ? (first ? static_cast<int>(b0 + k) : list[k]) : -1;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = iv[r];
      gv[r] = 0.0;
      lov[r] = 0.0;
      hiv[r] = INFINITY;
      if (i >= 0) {
        gv[r] = g[i];
        lov[r] = lo[i];
        if (i < a.n) hiv[r] = hi[i];
      }
    }
    unsigned keepmask = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = iv[r];
      const double gs = gv[r];
      bool keep = false;
      if (i >= 0 && gs != 0.0) {
        const bool primal = i < a.n;
        const double w = primal ? omega : winv;
        const double los = lov[r];
        const double his = hiv[r];
        const int side = primal ? 0 : 1;
        const double ulo = gs * st.rcp_lo[side];  // |u| largest at nu_lo
        const double uhi = gs * st.rcp_hi[side];
        const bool clamped_lo = ulo < los || ulo > his;
        const bool clamped_hi = uhi < los || uhi > his;
        if (clamped_hi) {  // clamped over the whole bracket
          const double cv = uhi > his ? his : los;
          fq += w * cv * cv;
          fh += gs * cv;
        } else if (!clamped_lo) {  // free over the whole bracket
          fs += gs * gs * (primal ? winv : omega);
        } else {
          keep = true;
          const double* rcp = primal ? st.rcp_primal : st.rcp_dual;
#pragma unroll
          for (int p = 0; p < kNuCands; ++p) {
            const double d = ref_min(ref_max(gs * rcp[p], los), his);
            acc[2 * p] += w * d * d;
            acc[2 * p + 1] += gs * d;
          }
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) wcount[r * W + warp] = __popc(bal);
      if (keep) keepmask |= 1u << r;
    }
    // in-place, order-preserving compaction: every read of this super-tile
    // precedes the barrier, every write lands below t0 + R * kBisectThreads
    __syncthreads();
    int off = kept;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const unsigned bal = __ballot_sync(0xffffffffu, (keepmask >> r) & 1u);
      int before = 0, tile = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const int c = wcount[r * W + w];
        if (w < warp) before += c;
        tile += c;
      }
      if ((keepmask >> r) & 1u) list[off + before + __popc(bal & ((1u << lane) - 1u))] = iv[r];
      off += tile;
    }
    kept = off;
    __syncthreads();
  }
  return kept;
}

__global__ void __launch_bounds__(kBisectThreads) k_ndg_bisect(BisectArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ NdgState st[2];
  __shared__ double wsum[kBisectThreads / 32][2][kBisectVals];
  __shared__ double tot[2][kBisectVals];
  __shared__ int wcount[kBisectBatch * kBisectThreads / 32];
  __shared__ int kept_count[2];
  __shared__ int s_off[2];
  __shared__ double base[2][3];  // block 0 alone: the grid's Q, H, S at the switch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x;
  const int64_t chunk = (a.total + nb - 1) / nb;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t own = b0 < a.total ? (a.total - b0 < chunk ? a.total - b0 : chunk) : 0;
  if (tid < 2) {
    st[tid] = *a.ns[tid];
    if (!a.active[tid]) st[tid].done = 1;
    kept_count[tid] = static_cast<int>(own);
  }
  double fq[2] = {0.0, 0.0}, fh[2] = {0.0, 0.0}, fs[2] = {0.0, 0.0};
  __syncthreads();
  bool first = true, alone = false;
#ifdef FOLP_BISECT_TIMES
  unsigned long long t_prev = global_ns();
  int pass_no = 0;
#endif
  for (int parity = 0;; parity ^= 1) {
    const bool run[2] = {st[0].done == 0, st[1].done == 0};
    if (!run[0] && !run[1]) break;  // same state in every block
    double acc[2][2 * kNuCands];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int k = 0; k < 2 * kNuCands; ++k) acc[s][k] = 0.0;
    int kept_s[2] = {0, 0};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (!run[s]) continue;
      int* list = alone ? a.compact[s] : a.list[s] + b0;
      kept_s[s] = bisect_sweep(a, st[s], s, list, kept_count[s], first, b0, acc[s], fq[s], fh[s],
                               fs[s], wcount);
    }
    __syncthreads();
    if (tid < 2 && run[tid]) kept_count[tid] = kept_s[tid];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
#pragma unroll
      for (int k = 0; k < kBisectVals; ++k) {
        double v = k < 2 * kNuCands ? acc[s][k]
                 : k == 2 * kNuCands ? 0.0
                 : k == 2 * kNuCands + 1 ? fq[s]
                 : k == 2 * kNuCands + 2 ? fh[s]
                                         : fs[s];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) wsum[warp][s][k] = v;
      }
    }
    __syncthreads();
    double* part = a.partials + static_cast<size_t>(parity) * 2 * kBisectVals * nb;
    if (alone) {
      // block 0 alone: block totals are the totals (plus the grid's
      // retired sums at the switch)
      if (tid < 2 * kBisectVals) {
        const int s = tid / kBisectVals, k = tid % kBisectVals;
        double v = 0.0;
        if (k == 2 * kNuCands) {
          v = static_cast<double>(kept_s[s]);
        } else {
          for (int w = 0; w < kBisectThreads / 32; ++w) v += wsum[w][s][k];
          if (k > 2 * kNuCands) v += base[s][k - 2 * kNuCands - 1];
        }
        tot[s][k] = v;
      }
    } else {
      if (tid < 2 * kBisectVals) {
        const int s = tid / kBisectVals, k = tid % kBisectVals;
        double v = 0.0;
        if (k == 2 * kNuCands) {
          v = static_cast<double>(kept_s[s]);
        } else {
          for (int w = 0; w < kBisectThreads / 32; ++w) v += wsum[w][s][k];
        }
        part[static_cast<size_t>(tid) * nb + blockIdx.x] = v;
      }
      grid.sync();
      // every block: totals in block order, one warp per (set, value) pair
      for (int pair = warp; pair < 2 * kBisectVals; pair += kBisectThreads / 32) {
        const double* src = part + static_cast<size_t>(pair) * nb;
        double v = 0.0;
        for (int b = lane; b < nb; b += 32) v += src[b];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) tot[pair / kBisectVals][pair % kBisectVals] = v;
      }
    }
    __syncthreads();
    if (tid < 2 && run[tid]) {
      const double q = tot[tid][2 * kNuCands + 1], h = tot[tid][2 * kNuCands + 2];
      const double sf = tot[tid][2 * kNuCands + 3];
      double nsq[kNuCands], gd[kNuCands];
      for (int p = 0; p < kNuCands; ++p) {
        const double nu = st[tid].nu[p];
        nsq[p] = tot[tid][2 * p] + (q + sf / (nu * nu));
        gd[p] = tot[tid][2 * p + 1] + (h + sf / nu);
      }
      if (!alone) st[tid].grid_passes += 1;
      ndg_replay(&st[tid], nsq, gd, kNuLevels, false);
      // no breakpoint inside this pass's bracket: none inside the narrower one
      if (!st[tid].done && tot[tid][2 * kNuCands] == 0.0) ndg_finish_analytic(&st[tid], q, h, sf);
    }
    first = false;
    __syncthreads();
    // the next candidates' reciprocals, one division per thread
    if (tid < 2 * kNdgRcp && run[tid / kNdgRcp] && !st[tid / kNdgRcp].done) {
      ndg_reciprocal(&st[tid / kNdgRcp], tid % kNdgRcp);
    }
    __syncthreads();
#ifdef FOLP_BISECT_TIMES
    if (blockIdx.x == 0 && tid == 0 && pass_no < kBisectTimeSlots) {
      const unsigned long long t = global_ns();
      g_bisect_times[pass_no][0] += t - t_prev;
      g_bisect_times[pass_no][1] += 1;
      g_bisect_times[pass_no][2] += alone ? 1 : 0;
      t_prev = t;
    }
    ++pass_no;
#endif
    if (!alone && a.small_limit > 0) {
      // every block sees the same totals, so all take the same branch
      bool go = st[0].done == 0 || st[1].done == 0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (st[s].done == 0 && tot[s][2 * kNuCands] > static_cast<double>(a.small_limit)) go = false;
      }
      if (go) {
        if (tid < 2) {  // this block's offset in the gathered list
          int off = 0;
          for (int b = 0; b < static_cast<int>(blockIdx.x); ++b) {
            off += static_cast<int>(part[static_cast<size_t>(tid * kBisectVals + 2 * kNuCands) * nb + b]);
          }
          s_off[tid] = off;
          base[tid][0] = tot[tid][2 * kNuCands + 1];
          base[tid][1] = tot[tid][2 * kNuCands + 2];
          base[tid][2] = tot[tid][2 * kNuCands + 3];
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (st[s].done) continue;
          const int* own_list = a.list[s] + b0;
          for (int k = tid; k < kept_count[s]; k += kBisectThreads) {
            a.compact[s][s_off[s] + k] = own_list[k];
          }
        }
        grid.sync();
        if (blockIdx.x != 0) return;
        if (tid < 2) kept_count[tid] = static_cast<int>(tot[tid][2 * kNuCands]);
#pragma unroll
        for (int s = 0; s < 2; ++s) fq[s] = fh[s] = fs[s] = 0.0;  // now in base[]
        alone = true;
        __syncthreads();
      }
    }
  }
  if (blockIdx.x == 0 && tid < 2 && a.active[tid]) *a.ns[tid] = st[tid];
}

__global__ void k_clear_pending(DevState* st) { st->pending = 0.0; }

void enqueue_average(folp_gpu_ctx* c) {
  DevState* st = c->st_h;
  OpAverage op{};
  op.n = c->n;
  op.m1 = c->m1;
  op.x = c->cur_x();
  op.y = c->cur_y();
  op.ax = c->avg_x;
  op.ay = c->avg_y;
  op.l = c->lw;
  op.u = c->uw;
  op.pending = st->pending;
  op.copy_current = st->avg_weight <= 0.0 ? 1 : 0;
  op.inv = st->avg_weight > 0.0 ? 1.0 / st->avg_weight : 0.0;
  op.out_x = c->avgp_x;
  op.out_y = c->avgp_y;
  if (c->capturing_eval) {
    // graph: the weights are read on device at run time, then pending is
    // cleared there (the host mirror is cleared before the launch)
    op.st = c->st_d;
    c->ew(c->n + c->m, op, 6);
    k_clear_pending<<<1, 1, 0, c->stream>>>(c->st_d);
    ++c->launches;
    CK(cudaGetLastError());
    return;
  }
  c->ew(c->n + c->m, op, 6);
  st->pending = 0.0;
  c->push_state();
}

// convergence_info reductions of a slot into the block at res[base].
// kty_out (tree mode): keep K'y of the presolved point for enqueue_ndg_setup.
void enqueue_evaluate(folp_gpu_ctx* c, int which, int raw, int base, double* kty_out = nullptr) {
  OpEvalPoint op{};
  op.raw = raw != 0 ? 1 : 0;
  op.n = c->n;
  op.m = c->m;
  op.xs = c->slot_x(which);
  op.ys = c->slot_y(which);
  op.d1 = c->d1;
  op.d2 = c->d2;
  op.l = c->l0;
  op.u = c->u0;
  op.c = c->c0;
  op.q = c->q0;
  op.xr = c->xr;
  op.yr = c->yr;
  op.result = c->res + base;
  c->ew(c->n + c->m, op, 7);
  axis_product(c, true, false, EpiPrimalResidual{c->xr, c->q0, c->m1, c->res + base + 3}, 8);
  EpiDualResidual dres{c->yr, c->c0, c->l0, c->u0, c->res + base + 4};
  dres.q_dot_y = c->res + base + 1;
  dres.constant = c->objective_constant;
  dres.dual_objective = c->res + base + 10;
  dres.kty_out = raw == 0 ? kty_out : nullptr;
  axis_product(c, false, false, dres, 9);
  if (!c->norms_ready) {
    c->ew(c->m, OpNormSq{c->q0, c->res + kResNorms}, 10);
    c->ew(c->n, OpNormSq{c->c0, c->res + kResNorms + 1}, 11);
  }
}

// Reads a block written by enqueue_evaluate (after the sync).
void read_evaluate(folp_gpu_ctx* c, int base, folp_gpu_eval* out) {
  if (!c->norms_ready) {
    c->norm_q_sq = c->res_h[kResNorms];
    c->norm_c_sq = c->res_h[kResNorms + 1];
    c->norms_ready = true;
  }
  const double* r = c->res_h + base;
  out->c_dot_x = r[0];
  out->q_dot_y = r[1];
  out->nonfinite = r[2] != 0.0 ? 1 : 0;
  out->primal_sq = r[3];
  out->dual_sq = r[4];
  out->bound_terms = r[5];
  out->infinite_product = r[6] != 0.0 ? 1 : 0;
  out->norm_q = std::sqrt(c->norm_q_sq);
  out->norm_c = std::sqrt(c->norm_c_sq);
  // lp_model.cpp:154-163; ordered mode folded it term by term on device
  out->dual_objective =
      c->ordered ? r[10] : (out->q_dot_y + c->objective_constant) + out->bound_terms;
}

void enqueue_distance(folp_gpu_ctx* c, int a, int b, int base) {
  OpDistance op{c->n, c->slot_x(a), c->slot_x(b), c->slot_y(a), c->slot_y(b), c->res + base};
  c->ew(c->n + c->m, op, 12);
}

// g, lo, hi of a slot into scratch set s with the setup sums
// (solver.cpp:300-342); Kx of the point is cached for CURRENT and kept for
// AVERAGE (a restart to it reuses it).
// kty_raw: K'y of the same point from enqueue_evaluate (tree mode), so the
// working-space K~'y~ is D2 (K'y) elementwise instead of a column product.
void enqueue_ndg_setup(folp_gpu_ctx* c, int which, int s, double omega,
                       const double* kty_raw = nullptr) {
  const int64_t n = c->n, m = c->m;
  double* px = c->slot_x(which);
  double* py = c->slot_y(which);
  double* sums = c->res + kResNdg[s];
  EpiNdgPrimal ep{py, px, c->cw, c->lw, c->uw, omega, c->g[s], c->lo[s], c->hi[s], sums};
  if (c->capturing_eval) ep.omega_dev = c->eval_omega_d;
  if (kty_raw != nullptr) {
    c->ew(n, OpNdgPrimalRaw{kty_raw, c->d2, ep}, 13, 0);
  } else {
    axis_product(c, false, true, ep, 13, 0);
  }
  EpiNdgDual ed{};
  ed.x = px;
  ed.y = py;
  ed.q = c->qw;
  ed.m1 = c->m1;
  ed.winv = 1.0 / omega;
  ed.g = c->g[s] + n;
  ed.lo = c->lo[s] + n;
  ed.result = sums;
  ed.primal_terms = c->terms[0];
  ed.n = n;
  if (c->capturing_eval) ed.omega_dev = c->eval_omega_d;
  if (which == FOLP_PT_CURRENT && c->kx_valid) {
    ed.kx_out = nullptr;
    c->ew(m, OpNdgDualCached{c->kx[c->st_h->cur], ed}, 14, 1);
  } else {
    ed.kx_out = which == FOLP_PT_AVERAGE ? c->kx_avg : c->kx_aux;
    axis_product(c, true, true, ed, 14, 1);
  }
}

void enqueue_ndg_init(folp_gpu_ctx* c, int s, int dist_base, double radius, double omega) {
  const double* dist = dist_base >= 0 ? c->res + dist_base : nullptr;
  k_ndg_init<<<1, 1, 0, c->stream>>>(c->ndg_d + s, c->res + kResNdg[s], dist, radius, omega,
                                     c->capturing_eval ? c->eval_omega_d : nullptr);
  ++c->launches;
  CK(cudaGetLastError());
}

// One bisection pass (3 levels in tree mode, 1 in ordered mode); a no-op
// once the bisection of that scratch set is done.
void enqueue_ndg_pass(folp_gpu_ctx* c, int s, double omega) {
  OpNdgPass pass{};
  pass.n = c->n;
  pass.total = c->n + c->m;
  pass.g = c->g[s];
  pass.lo = c->lo[s];
  pass.hi = c->hi[s];
  pass.omega = omega;
  pass.winv = 1.0 / omega;
  pass.ns = c->ndg_d + s;
  c->ew(c->n + c->m, pass, 15);
}

// Passes before the first look: 42 tree levels / 48 ordered levels cover
// a typical evaluation (the bracket starts at ||g|| / r, the stop is 1e-10 r).
int ndg_first_batch(const folp_gpu_ctx* c) { return c->ordered ? 48 : 14; }
int ndg_next_batch(const folp_gpu_ctx* c) { return c->ordered ? 16 : 5; }

// Starts the bisections of the wanted scratch sets and queues the readback
// of their states: tree mode runs them to the end in one cooperative
// launch, ordered mode (one reference level per pass) queues a first batch.
void enqueue_ndg_solve(folp_gpu_ctx* c, const bool (&want)[2], const double (&omega)[2]);

void fetch_ndg(folp_gpu_ctx* c) {
  CK(cudaMemcpyAsync(c->ndg_h, c->ndg_d, 2 * sizeof(NdgState), cudaMemcpyDeviceToHost, c->stream));
}

// After a synchronized fetch: runs more passes on the scratch sets still
// bisecting until all wanted ones are done.
void finish_ndg(folp_gpu_ctx* c, const bool (&want)[2], const double (&omega)[2]) {
  for (int round = 0; round < 256; ++round) {
    bool pending = false;
    for (int s = 0; s < 2; ++s) pending = pending || (want[s] && !c->ndg_h[s].done);
    if (!pending) return;
    const int batch = ndg_next_batch(c);
    for (int i = 0; i < batch; ++i) {
      for (int s = 0; s < 2; ++s) {
        if (want[s] && !c->ndg_h[s].done) enqueue_ndg_pass(c, s, omega[s]);
      }
    }
    fetch_ndg(c);
    CK(cudaStreamSynchronize(c->stream));
  }
  throw EngineError(FOLP_E_RUNTIME, "normalized_duality_gap: bisection stalled");
}

void check_ndg_args(double radius, double omega) {
  if (!(radius > 0.0)) {
    throw EngineError(FOLP_E_NONPOSITIVE_RADIUS, "normalized_duality_gap: radius must be > 0");
  }
  if (!(omega > 0.0)) {
    throw EngineError(FOLP_E_NONPOSITIVE_WEIGHT, "normalized_duality_gap: omega must be > 0");
  }
}

void enqueue_ndg_solve(folp_gpu_ctx* c, const bool (&want)[2], const double (&omega)[2]) {
  if (c->ordered || !c->coop_ok) {
    // ordered mode, or no cooperative launch on this device/context: passes
    // of OpNdgPass (finish_ndg continues them after the read-back)
    for (int i = 0, e = ndg_first_batch(c); i < e; ++i) {
      for (int s = 0; s < 2; ++s) {
        if (want[s]) enqueue_ndg_pass(c, s, omega[s]);
      }
    }
  } else {
    BisectArgs a{};
    a.n = c->n;
    a.total = c->n + c->m;
    for (int s = 0; s < 2; ++s) {
      a.g[s] = c->g[s];
      a.lo[s] = c->lo[s];
      a.hi[s] = c->hi[s];
      a.ns[s] = c->ndg_d + s;
      a.active[s] = want[s] ? 1 : 0;
    }
    a.partials = c->partials;
    a.list[0] = c->ndg_list;
    a.list[1] = c->ndg_list + a.total;
    a.compact[0] = c->ndg_compact;
    a.compact[1] = c->ndg_compact + kBisectSmall;
    {
      const char* env = std::getenv("FOLP_BISECT_SMALL");  // 0: grid-wide to the end
      a.small_limit = env ? std::min(std::max(0, std::atoi(env)), kBisectSmall) : kBisectSmall;
    }
    int& grid = c->bisect_grid;
    if (grid == 0) {  // co-resident by construction (cooperative launch)
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ndg_bisect, kBisectThreads, 0));
      grid = std::max(1, std::min(c->sms * std::max(occ, 1), std::min(c->sms * 2, kMaxGrid / 2)));
      // small problems: no more CTAs than 4 elements per thread -- a
      // cooperative launch holds every CTA it spans, so concurrent solves of
      // small programs would otherwise serialize on the whole GPU
      const int64_t want = (c->n + c->m + int64_t(kBisectThreads) * 4 - 1) / (int64_t(kBisectThreads) * 4);
      grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, want)));
      if (const char* env = std::getenv("FOLP_BISECT_GRID")) {  // experiments
        grid = std::max(1, std::min(grid, std::atoi(env)));
      }
    }
    void* args[] = {&a};
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_ndg_bisect),
                                                      dim3(grid), dim3(kBisectThreads), args, 0,
                                                      c->stream);
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported ||
        e == cudaErrorNotPermitted) {
      cudaGetLastError();
      c->coop_ok = false;  // e.g. under MPS: fall back to pass kernels from now on
      enqueue_ndg_solve(c, want, omega);
      return;
    }
    CK(e);
    ++c->launches;
  }
  fetch_ndg(c);
}

// restart_to without the sync: copies of the restart point (solver.cpp:805-813).
void enqueue_restart(folp_gpu_ctx* c, int which, int reset_average) {
  DevState* st = c->st_h;
  if (which != FOLP_PT_CURRENT) {
    copy_d2d(c, c->cur_x(), c->slot_x(which), c->n);
    copy_d2d(c, c->cur_y(), c->slot_y(which), c->m);
    if (which == FOLP_PT_AVERAGE) {
      copy_d2d(c, c->kx[st->cur], c->kx_avg, c->m);
      c->kx_valid = true;
    } else {
      refresh_kx(c);
    }
  }
  copy_d2d(c, c->last_x, c->cur_x(), c->n);
  copy_d2d(c, c->last_y, c->cur_y(), c->m);
  if (reset_average) zero_average(c);
  c->push_state();
}
