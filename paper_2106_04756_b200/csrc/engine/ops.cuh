// ops.cuh -- epilogues and elementwise operators of the PDLP loop.
//
// Each struct is a value type passed by value as a kernel parameter; its
// prepare() runs once per CTA and caches the loop scalars from the device
// state.  Arithmetic follows the reference expression by expression (the
// file is compiled with -fmad=false, so a*b+c is two roundings exactly like
// the reference's x86-64 -O2 build, which emits no FMA).
//
// Reductions go through a sink `acc.add(k, index, term)`: tree mode sums in
// registers (then per-CTA partials, see segdot.cuh); ordered mode stores the
// term per index and finalize_ordered() folds the terms with one thread in
// exactly the reference's sequential order, including the orders that span
// two kernels (movement = sum dy^2 / omega + sum omega dx^2, solver.cpp:76-88;
// dual objective = q'y + const + sum bound*lambda, lp_model.cpp:154-163;
// the duality-gap sums over (x; y), solver.cpp:318-369).
#pragma once

#include <cuda_runtime.h>

#include "segdot.cuh"

#include <cooperative_groups.h>

namespace folpgpu {

// Chunk status values (mirror folp_gpu.h).
constexpr int kRunning = 0;
constexpr int kDone = 1;
constexpr int kLimit = 2;
constexpr int kNonFinite = 3;
constexpr int kUnderflow = 4;

constexpr double kStepSizeFloor = 1e-300;  // solver.cpp:31

// Device-resident loop state.  Host mirrors it at chunk boundaries.
struct alignas(8) DevState {
  int32_t running;   // slot kernels work only while 1
  int32_t status;
  int32_t cur;       // parity of the CURRENT buffers
  int32_t policy;    // 0 adaptive, 1 constant
  int64_t target;
  int64_t accepted;
  int64_t k_total;
  int64_t k_chunk0;  // k_total at chunk start (factor-table origin)
  int64_t t_inner;
  int64_t trials_iter;
  int64_t step_trials;
  int64_t violations;
  int64_t ledger_k;
  int64_t ledger_kt;
  int64_t iteration_limit;
  int64_t slots;     // trial slots executed (diagnostics)
  double kkt_pass_limit;
  double omega;
  double eta;        // step of the next trial
  double eta_hat;
  double last_eta_used;
  double avg_weight;
  double pending;    // eta of the accepted iterate not yet folded into avg
  double sx;         // sum omega*dx*dx of the current trial (kernel A)
  double bad_a;      // non-finite x' entries of the current trial
  double cross;      // last trial diagnostics
  double movement;
  // Malitsky-Pock policy (solver.cpp:202-275)
  double mp_theta;   // theta of the last accepted step
  double mp_eta_hat; // candidate step of the current trial
  double mp_dy_sq;   // ||dy||^2 of the current trial
  double mp_break, mp_down, mp_interp;
};

static_assert(sizeof(DevState) % 8 == 0, "DevState is copied as 8-byte words");

// a[i] for i in {0, 1} without dynamic indexing (which would force the
// parameter struct into local memory).
template <class T>
__device__ __forceinline__ T pick(const T (&a)[2], int i) {
  return i ? a[1] : a[0];
}

// Buffers of the loop, fixed for the context lifetime.
struct LoopBufs {
  double* x[2];
  double* y[2];
  double* kx[2];
  double* avg_x;
  double* avg_y;
  const double* c;   // working (scaled) problem
  const double* l;
  const double* u;
  const double* q;
  int64_t m1;
  int64_t n;
  DevState* st;
  const double* red;   // per-iteration factor tables of the chunk
  const double* grow;
  const double* a_terms;  // ordered mode: kernel A's omega*dx*dx terms
  double* mp_ext;         // Malitsky-Pock: extrapolated primal [n]
  double* mp_dy;          // Malitsky-Pock: dual difference [m]
  cudaGraphConditionalHandle cond;
  int use_cond;
  // uniform working bounds (every l_j, or every u_j, the same value -- x >= 0
  // with no upper bound in configs 3 and 5): the primal steps take the
  // constant instead of streaming the array (16 B per column less)
  double l_const, u_const;
  int l_uni, u_uni;
};

// ---------------------------------------------------------------------
// Kernel A: K'y of the current dual, fused primal projected step
// (pdhg_trial, solver.cpp:58-63) + lazy averaging of the previous accepted
// primal (accumulate_average, solver.cpp:530-538) + omega*dx*dx
// (solver.cpp:84-88) and the finiteness flag (solver.cpp:91-93).
struct EpiPrimal {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  static constexpr int kTrace = 0;  // FOLP_WARP_TIMES slot
  LoopBufs b;
  const double* xc;
  double* xn;
  double* avg;
  const double* yv;
  double tau, omega, pend;

  __device__ bool prepare() {
    const DevState* st = b.st;
    if (!st->running) return false;
    const int cur = st->cur;
    xc = pick(b.x, cur);
    xn = pick(b.x, cur ^ 1);
    yv = pick(b.y, cur);
    avg = b.avg_x;
    omega = st->omega;
    tau = st->eta / omega;  // solver.cpp:53
    pend = st->pending;
    return true;
  }
  __device__ const double* vec() const { return yv; }
  struct Pre {
    double x, c, l, u, a;
  };
  __device__ Pre load(int j) const {
    return Pre{xc[j], b.c[j], b.l_uni ? b.l_const : b.l[j], b.u_uni ? b.u_const : b.u[j],
               pend != 0.0 ? avg[j] : 0.0};
  }
  template <class Acc>
  __device__ void apply(int j, double kty, const Pre& o, Acc& acc) const {
    const double xj = o.x;
    if (pend != 0.0) avg[j] = o.a + pend * xj;
    const double v = xj - tau * (o.c - kty);
    const double xv = ref_min(ref_max(v, o.l), o.u);
    xn[j] = xv;
    const double dx = xv - xj;
    acc.add(0, j, omega * dx * dx);
    acc.add(1, j, isfinite(xv) ? 0.0 : 1.0);
  }
  double* shard_out = nullptr;  // column shard: local sums for the all-reduce
  __device__ void finalize(const double (&tot)[K]) const {
    if (shard_out != nullptr) {
      shard_out[0] = tot[0];
      shard_out[1] = tot[1];
      return;
    }
    b.st->sx = tot[0];
    b.st->bad_a = tot[1];
  }
  // kernel B folds the omega*dx*dx terms after its own (solver.cpp:83-88)
  __device__ void finalize_ordered(const double* t, int64_t n) const {
    b.st->bad_a = any_nonzero(t + n, n) ? 1.0 : 0.0;
  }
};

// The adaptive step-size rule (adaptive_step, solver.cpp:173-199) and the
// loop bookkeeping, run by one thread once a trial's sums are known.
// `st` is the device state or the last CTA's shared copy of it; `rg`, when
// given, holds this trial's red / grow factors (loaded in parallel).
__device__ __forceinline__ void decide_trial_on(const LoopBufs& b, DevState* st, double cross,
                                                double movement, bool bad, const double* rg) {
  st->slots += 1;
  st->pending = 0.0;  // consumed by kernels A and B of this slot
  const double eta = st->eta;
  st->cross = cross;
  st->movement = movement;
  st->trials_iter += 1;
  if (bad) {
    st->status = kNonFinite;
    st->running = 0;
  } else {
    bool accept = true;
    double eta_next = eta;
    if (st->policy == 0) {
      const int64_t ki = st->k_total - st->k_chunk0;
      const double eta_bar = cross > 0.0 ? movement / (2.0 * cross) : INFINITY;
      const double a = (rg ? rg[0] : b.red[ki]) * eta_bar;
      const double g = (rg ? rg[1] : b.grow[ki]) * eta;
      eta_next = (g < a) ? g : a;  // std::min(a, g)
      accept = eta <= eta_bar;
    }
    if (accept) {
      st->k_total += 1;
      st->t_inner += 1;
      st->accepted += 1;
      st->step_trials += st->trials_iter;
      st->ledger_kt += 1;                   // K'y of the current point
      st->ledger_k += 1 + st->trials_iter;  // Kx + one Kx' per trial
      if (st->policy == 0 && cross > 0.0 && 2.0 * eta * cross > movement * (1.0 + 1e-9)) {
        st->violations += 1;  // solver.cpp:618-621
      }
      st->trials_iter = 0;
      st->last_eta_used = eta;
      st->avg_weight += eta;
      st->pending = eta;
      if (st->policy == 0) {
        st->eta_hat = eta_next;
        st->eta = eta_next;
      }
      st->cur ^= 1;
      if (st->accepted >= st->target) {
        st->status = kDone;
        st->running = 0;
      } else if (st->k_total >= st->iteration_limit ||
                 0.5 * static_cast<double>(st->ledger_k + st->ledger_kt) >= st->kkt_pass_limit) {
        st->status = kLimit;
        st->running = 0;
      }
    } else {
      st->eta = eta_next;
      if (eta_next < kStepSizeFloor) {
        st->status = kUnderflow;
        st->running = 0;
      }
    }
  }
  if (b.use_cond) cudaGraphSetConditional(b.cond, st->running ? 1u : 0u);
}
__device__ __forceinline__ void decide_trial(const LoopBufs& b, double cross, double movement,
                                             bool bad) {
  decide_trial_on(b, b.st, cross, movement, bad, nullptr);
}

// Kernel B: K x' of the trial primal, fused dual projected step with the
// extrapolation 2Kx'-Kx (solver.cpp:70-75), cross term and movement
// (solver.cpp:76-83), lazy averaging of the previous accepted dual, and the
// step-size decision in the last CTA.  Kx' is kept as the next Kx
// (bit-identical to recomputing it: the product is deterministic).
struct EpiDual {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
  static constexpr int kTrace = 1;  // FOLP_WARP_TIMES slot
  LoopBufs b;
  const double* yc;
  double* yn;
  const double* kxc;
  double* kxn;
  const double* xv;
  double sigma, pend;

  __device__ bool prepare() {
    const DevState* st = b.st;
    if (!st->running) return false;
    const int cur = st->cur;
    yc = pick(b.y, cur);
    yn = pick(b.y, cur ^ 1);
    kxc = pick(b.kx, cur);
    kxn = pick(b.kx, cur ^ 1);
    xv = pick(b.x, cur ^ 1);
    sigma = st->eta * st->omega;  // solver.cpp:54
    pend = st->pending;
    return true;
  }
  __device__ const double* vec() const { return xv; }
  struct Pre {
    double y, kx, q, a;
  };
  __device__ Pre load(int i) const {
    return Pre{yc[i], kxc[i], b.q[i], pend != 0.0 ? b.avg_y[i] : 0.0};
  }
  template <class Acc>
  __device__ void apply(int i, double kx_next, const Pre& o, Acc& acc) const {
    const double yi = o.y;
    if (pend != 0.0) b.avg_y[i] = o.a + pend * yi;
    const double kxi = o.kx;
    const double extrapolated = 2.0 * kx_next - kxi;
    double v = yi + sigma * (o.q - extrapolated);
    if (i < b.m1) v = ref_max(v, 0.0);
    yn[i] = v;
    kxn[i] = kx_next;
    const double dy = v - yi;
    acc.add(0, i, dy * (kxi - kx_next));
    acc.add(1, i, dy * dy);
    acc.add(2, i, isfinite(v) ? 0.0 : 1.0);
  }
  double* shard_out = nullptr;  // row shard: local sums for the all-reduce
  // row shard, partitioned primal epilogue: the sums go to slot `rank` of
  // every rank's area at [shard_at, shard_at + 3)
  double* const* shard_peers = nullptr;
  int shard_world = 0;
  int64_t shard_at = 0;
  __device__ bool shard_sums(const double (&tot)[K]) const {
    if (shard_peers != nullptr) {
      for (int r = 0; r < shard_world; ++r)
        for (int k = 0; k < K; ++k) shard_peers[r][shard_at + k] = tot[k];
      return true;
    }
    if (shard_out != nullptr) {
      for (int k = 0; k < K; ++k) shard_out[k] = tot[k];
      return true;
    }
    return false;
  }
  __device__ void finalize(const double (&tot)[K]) const {
    if (shard_sums(tot)) return;
    const DevState* st = b.st;
    double movement = tot[1] / st->omega;  // solver.cpp:83
    movement = movement + st->sx;
    decide_trial(b, tot[0], movement, st->bad_a != 0.0 || tot[2] != 0.0);
  }
  // kernel A's deferred sums (segdot.cuh DeferredSums): its CTA partials,
  // summed by this kernel's highest-numbered CTA at its start into the state
  static constexpr int kDeferredK = 2;  // EpiPrimal::K
  const double* a_partials = nullptr;
  int a_np = 0;
  __device__ const double* deferred_partials() const { return a_partials; }
  __device__ int deferred_np() const { return a_np; }
  __device__ void store_deferred(const double (&tot)[kDeferredK]) const {
    b.st->sx = tot[0];     // EpiPrimal::finalize
    b.st->bad_a = tot[1];
  }
  // the decision on the last CTA's shared copy of the state (segdot.cuh StateTail)
  static constexpr int kStateWords = sizeof(DevState) / 8;
  __device__ unsigned long long* state_words() const {
    return reinterpret_cast<unsigned long long*>(b.st);
  }
  __device__ void tail_aux(double* rg) const {  // this trial's step factors
    const DevState* st = b.st;
    if (__ldcg(&st->policy) == 0) {
      const int64_t ki = __ldcg(&st->k_total) - __ldcg(&st->k_chunk0);
      rg[0] = b.red[ki];
      rg[1] = b.grow[ki];
    }
  }
  __device__ void finalize_state(const double (&tot)[K], unsigned long long* words,
                                 const double* rg) const {
    if (shard_sums(tot)) return;
    DevState* st = reinterpret_cast<DevState*>(words);
    double movement = tot[1] / st->omega;  // solver.cpp:83
    movement = movement + st->sx;
    decide_trial_on(b, st, tot[0], movement, st->bad_a != 0.0 || tot[2] != 0.0, rg);
  }
  __device__ void finalize_ordered(const double* t, int64_t m) const {
    const DevState* st = b.st;
    const double cross = fold(0.0, t, m);       // solver.cpp:80
    double movement = fold(0.0, t + m, m);      // solver.cpp:81
    movement /= st->omega;                      // solver.cpp:83
    movement = fold(movement, b.a_terms, b.n);  // solver.cpp:84-88
    const bool bad = st->bad_a != 0.0 || any_nonzero(t + 2 * m, m);
    decide_trial(b, cross, movement, bad);
  }
};

// Ordered mode's trial decision after the exact parallel folds
// (exactfold.cuh k_exact_fold): jobs {cross = sum dy*(Kx-Kx') over m,
// sum dy^2 over m, movement = (sum dy^2)/omega + sum omega*dx^2 over n},
// each the reference's sequential fold bit for bit (solver.cpp:76-88);
// flag arrays = kernel A's and kernel B's non-finite markers (:91-93).
struct FinTrial {
  LoopBufs b;
  __device__ bool prepare() const { return __ldcg(&b.st->running) != 0; }
  __device__ void finalize(const double* r, int, unsigned flags) const {
    decide_trial(b, r[0], r[2], flags != 0u);
  }
};

// ---------------------------------------------------------------------
// Row-sharded trial (north_star: K row-partitioned across the
// GPUs, all-reduce of the partial K'y and of the scalar reductions).  Rank p
// owns rows [r0, r1): y, Kx and the averaged y of those rows; x, c, l, u and
// the primal step are replicated.  One trial =
//   EpiShardPart (partial K'_p y_p over the local CSC) -> all-reduce (n)
//   OpShardPrimal (kernel A's epilogue on the summed K'y, replicated)
//   EpiDual over the local rows with shard_out        -> all-reduce (3)
//   k_shard_decide (kernel B's finalize on the global sums)
// Every rank holds bit-identical replicated data and sums, so every rank
// takes the same decisions.
// Partial product of the own block, stored (no reduction): K'_p y_p over
// the local CSC (row partition), or K_p x'_p over the local CSR of the own
// columns (column partition, of the TRIAL primal).
struct EpiShardPart {
  static constexpr int K = 1;
  static constexpr bool kReduce = false;
  LoopBufs b;
  double* out;
  const double* v;
  bool trial_x;
  // peer exchange (ShardComm::peer): the partial goes straight to slot
  // `rank` of all `world` receive areas; segment 0's unit also forwards the
  // two primal sums kernel A left at extra[0..1] (column partition)
  double* const* outs = nullptr;
  int world = 0;
  const double* extra = nullptr;
  int64_t extra_at = 0;
  // partitioned dual epilogue (column partition): row j's partial goes to
  // its owner's area only, owner = j / own_chunk (0: every rank's)
  int64_t own_chunk = 0;
  __device__ bool prepare() {
    if (!b.st->running) return false;
    v = trial_x ? pick(b.x, b.st->cur ^ 1) : pick(b.y, b.st->cur);
    return true;
  }
  __device__ const double* vec() const { return v; }
  struct Pre {};
  __device__ Pre load(int) const { return Pre{}; }
  template <class Acc>
  __device__ void apply(int j, double dot, const Pre&, Acc&) const {
    if (outs == nullptr) {
      out[j] = dot;
      return;
    }
    if (own_chunk > 0) {
      const int64_t o = j / own_chunk;
      outs[o < world ? o : world - 1][j] = dot;
    } else {
      for (int r = 0; r < world; ++r) outs[r][j] = dot;
    }
    if (j == 0 && extra != nullptr) {
      const double e0 = extra[0], e1 = extra[1];
      for (int r = 0; r < world; ++r) {
        outs[r][extra_at] = e0;
        outs[r][extra_at + 1] = e1;
      }
    }
  }
  __device__ void finalize(const double (&)[K]) const {}
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// Sum of the `world` peer slots at i, in rank order (every rank the same).
__device__ __forceinline__ double sum_slots(const double* const* src, int world, int64_t i) {
  double v = src[0][i];
  for (int r = 1; r < world; ++r) v += src[r][i];
  return v;
}

struct OpShardPrimal {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  EpiPrimal e;
  const double* kty;
  const double* const* src = nullptr;  // peer exchange: the partials' slots
  int world = 0;
  __device__ bool prepare() { return e.prepare(); }
  template <class Acc>
  __device__ void apply(int64_t j, Acc& acc) const {
    const int jj = static_cast<int>(j);
    e.apply(jj, src != nullptr ? sum_slots(src, world, j) : kty[jj], e.load(jj), acc);
  }
  __device__ void finalize(const double (&tot)[K]) const { e.finalize(tot); }
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

__global__ void k_shard_decide(LoopBufs b, const double* sums) {
  const DevState* st = b.st;
  if (!st->running) return;
  double movement = sums[1] / st->omega;  // solver.cpp:83, on the global sums
  movement = movement + st->sx;
  decide_trial(b, sums[0], movement, st->bad_a != 0.0 || sums[2] != 0.0);
}

// Column-sharded trial (the partition on the shorter axis
// when m < n: the exchange is then m + 2 doubles instead of n).  Rank p owns
// columns [c0, c1): x, the averaged x and c, l, u of those columns; y, Kx and
// the dual step are replicated.  One trial =
//   EpiPrimal over the own CSC columns, sums to shard_out (partial sx, bad)
//   EpiShardPart: partial K_p x'_p over the own block in CSR order
//   all-reduce (m + 2: the partial Kx' and the two primal sums)
//   OpShardDual: kernel B's epilogue on the summed Kx' over all rows
//     (replicated), whose finalize takes the step decision.
struct OpShardDual {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
  EpiDual e;
  const double* kx;
  const double* a_sums;  // global sx, bad of kernel A
  const double* const* src = nullptr;  // peer exchange: slots [0, m) Kx', [m, m+2) sx, bad
  int world = 0;
  int64_t m = 0;
  __device__ bool prepare() { return e.prepare(); }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    const int ii = static_cast<int>(i);
    e.apply(ii, src != nullptr ? sum_slots(src, world, i) : kx[ii], e.load(ii), acc);
  }
  __device__ void finalize(const double (&tot)[K]) const {
    const DevState* st = e.b.st;
    const double sx = src != nullptr ? sum_slots(src, world, m) : a_sums[0];
    const double bad = src != nullptr ? sum_slots(src, world, m + 1) : a_sums[1];
    double movement = tot[1] / st->omega;  // solver.cpp:83, on the global sums
    movement = movement + sx;
    decide_trial(e.b, tot[0], movement, bad != 0.0 || tot[2] != 0.0);
  }
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// Partitioned dual epilogue of the column partition (peer exchange; DESIGN
// 7): rank p owns rows [r0, r1) = [p c, (p+1) c).  The partial products
// reached their owner only (EpiShardPart own_chunk), so the owner sums the
// W slots of its rows in rank order, runs kernel B's epilogue on them --
// y', Kx', the lazy average, the trial sums over its rows -- and stores y'
// straight into every rank's y' vector and its three partial sums into
// slot p of every rank's area at [m + 2, m + 5).  After the second fence
// k_shard_decide_rows folds the W partial sums in rank order (identical on
// every rank) and decides.  The replicated epilogue ran all m rows on every
// rank; this one runs m / W (config 4 at W = 8: 1.2 GB -> 150 MB per rank
// and trial).
struct OpShardDualOwn {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
  EpiDual e;
  const double* const* src;   // this rank's W slots (current parity)
  double* const* sdst;        // slot `rank` of every rank's area (current parity)
  double* const* ydst2;       // [2][W] every rank's y[0], y[1]
  double* const* ydst = nullptr;
  int world = 0, rank = 0;
  int64_t r0 = 0, m = 0;
  __device__ bool prepare() {
    if (!e.prepare()) return false;
    ydst = ydst2 + (e.b.st->cur ^ 1) * world;
    return true;
  }
  template <class Acc>
  __device__ void apply(int64_t k, Acc& acc) const {
    const int i = static_cast<int>(r0 + k);
    e.apply(i, sum_slots(src, world, i), e.load(i), acc);
    const double v = e.yn[i];
    for (int r = 0; r < world; ++r) {
      if (r != rank) ydst[r][i] = v;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    for (int r = 0; r < world; ++r) {
      for (int k = 0; k < K; ++k) sdst[r][m + 2 + k] = tot[k];
    }
  }
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// The row partition's counterpart (DESIGN 7): rank p owns columns [r0, r1)
// (equal chunks); the partial K'y of every column reached its owner only,
// the owner sums the W slots in rank order, runs kernel A's epilogue on its
// columns, stores x' into every rank's x' vector and its two sums (sx, bad)
// into slot p of every rank's area at [n, n + 2).  EpiDual over the own
// rows then adds its three sums at [n + 2, n + 5) (shard_peers) and
// k_shard_decide_rows(..., n) folds all five in rank order.
struct OpShardPrimalOwn {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  EpiPrimal e;
  const double* const* src;   // this rank's W slots (current parity)
  double* const* sdst;        // slot `rank` of every rank's area (current parity)
  double* const* xdst2;       // [2][W] every rank's x[0], x[1]
  double* const* xdst = nullptr;
  int world = 0, rank = 0;
  int64_t r0 = 0, n = 0;
  __device__ bool prepare() {
    if (!e.prepare()) return false;
    xdst = xdst2 + (e.b.st->cur ^ 1) * world;
    return true;
  }
  template <class Acc>
  __device__ void apply(int64_t k, Acc& acc) const {
    const int j = static_cast<int>(r0 + k);
    e.apply(j, sum_slots(src, world, j), e.load(j), acc);
    const double v = e.xn[j];
    for (int r = 0; r < world; ++r) {
      if (r != rank) xdst[r][j] = v;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    for (int r = 0; r < world; ++r) {
      for (int k = 0; k < K; ++k) sdst[r][n + k] = tot[k];
    }
  }
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

__global__ void k_shard_decide_rows(LoopBufs b, const double* const* src, int world, int64_t m) {
  const DevState* st = b.st;
  if (!st->running) return;
  const double sx = sum_slots(src, world, m), bad = sum_slots(src, world, m + 1);
  const double cross = sum_slots(src, world, m + 2), dy2 = sum_slots(src, world, m + 3);
  const double flag = sum_slots(src, world, m + 4);
  double movement = dy2 / st->omega;  // solver.cpp:83, on the global sums
  movement = movement + sx;
  decide_trial(b, cross, movement, bad != 0.0 || flag != 0.0);
}

// ---------------------------------------------------------------------
// Small problems (config 1: 10^4 nonzeros): a whole chunk of trials in ONE
// launch of one thread-block cluster; kernel A and kernel B become
// cluster-wide phases: every CTA reduces its units, CTA 0 folds the CTAs'
// partials (distributed shared memory, rank order) and the multi-part slots
// and runs the epilogue's finalize (kernel B: the step decision), cluster
// barriers order the phases.  No kernel boundary or graph node per trial --
// at this size the two-kernel trial is launch / tail bound.
template <int NT>
__global__ void __launch_bounds__(NT) k_chunk_cluster(LoopBufs b, SegPlan rows, SegPlan cols,
                                                      const double* csr_val, const double* csc_val,
                                                      double* multi_scratch) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int ncta = static_cast<int>(cl.num_blocks());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double wbuf[NT / 32][kWarpTile];
  __shared__ double scratch[NT / 32][kMaxAcc];
  __shared__ double parts[16 * kMaxAcc];  // CTA 0: partials of every CTA
  __shared__ int running;
  double* parts0 = cl.map_shared_rank(parts, 0);
  const int u = rank * (NT / 32) + warp;  // this warp's unit in each plan
  ResidentUnit ua, ub;
  load_resident(cols, csc_val, u, lane, ua);
  load_resident(rows, csr_val, u, lane, ub);
  auto fold = [&](double* tot, int K, const SegPlan& p) {
    for (int k = 0; k < K; ++k) {
      double v = 0.0;
      for (int r = 0; r < ncta; ++r) v += parts[r * kMaxAcc + k];
      for (int q = 0; q < p.n_multi; ++q) v += multi_scratch[q * K + k];
      tot[k] = v;
    }
  };
  for (;;) {
    if (threadIdx.x == 0) running = b.st->running;
    __syncthreads();
    if (!running) break;
    EpiPrimal ea{b};
    ea.prepare();
    cluster_product<NT>(cols, ua, u, ea, rank, wbuf[warp], scratch, multi_scratch, parts0);
    cl.sync();
    if (rank == 0 && threadIdx.x == 0) {
      double t[EpiPrimal::K];
      fold(t, EpiPrimal::K, cols);
      ea.finalize(t);
    }
    cl.sync();
    EpiDual eb{b};
    eb.prepare();
    cluster_product<NT>(rows, ub, u, eb, rank, wbuf[warp], scratch, multi_scratch, parts0);
    cl.sync();
    if (rank == 0 && threadIdx.x == 0) {
      double t[EpiDual::K];
      fold(t, EpiDual::K, rows);
      eb.finalize(t);  // decide_trial: accept / shrink / stop
    }
    cl.sync();
  }
}

// ---------------------------------------------------------------------
// Malitsky-Pock step (malitsky_pock_step// ---------------------------------------------------------------------
// Malitsky-Pock step (malitsky_pock_step, solver.cpp:202-275) as four
// kernels per trial: MP-A once per iteration (K'y, x' = clamp(x - tau(c -
// K'y)), the first step-size candidate), MP-E (extrapolation), MP-B (K w,
// dual step, dy), MP-C (K'dy and the breaking test).
struct EpiMpPrimal {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  LoopBufs b;
  const double* xc;
  double* xn;
  const double* yv;
  double tau, pend;
  __device__ bool prepare() {
    const DevState* st = b.st;
    if (!st->running || st->trials_iter != 0) return false;  // once per iteration
    const int cur = st->cur;
    xc = pick(b.x, cur);
    xn = pick(b.x, cur ^ 1);
    yv = pick(b.y, cur);
    tau = st->eta / st->omega;  // solver.cpp:219: eta_prev / omega
    pend = st->pending;
    return true;
  }
  __device__ const double* vec() const { return yv; }
  struct Pre {
    double x, c, l, u, a;
  };
  __device__ Pre load(int j) const {
    return Pre{xc[j], b.c[j], b.l_uni ? b.l_const : b.l[j], b.u_uni ? b.u_const : b.u[j],
               pend != 0.0 ? b.avg_x[j] : 0.0};
  }
  template <class Acc>
  __device__ void apply(int j, double kty, const Pre& o, Acc& acc) const {
    if (pend != 0.0) b.avg_x[j] = o.a + pend * o.x;
    const double v = o.x - tau * (o.c - kty);
    const double xv = ref_min(ref_max(v, o.l), o.u);
    xn[j] = xv;
    acc.add(0, j, isfinite(xv) ? 0.0 : 1.0);
  }
  __device__ void start(bool bad) const {
    DevState* st = b.st;
    if (bad) {  // solver.cpp:226-228
      st->status = kNonFinite;
      st->running = 0;
      if (b.use_cond) cudaGraphSetConditional(b.cond, 0u);
      return;
    }
    const double eta_prev = st->eta;  // solver.cpp:230-233
    st->mp_eta_hat =
        eta_prev + st->mp_interp * (sqrt(1.0 + st->mp_theta) - 1.0) * eta_prev;
  }
  __device__ void finalize(const double (&tot)[K]) const { start(tot[0] != 0.0); }
  __device__ void finalize_ordered(const double* t, int64_t n) const {
    start(any_nonzero(t, n));
  }
};

struct OpMpExtrapolate {
  static constexpr int K = 1;
  static constexpr bool kReduce = false;
  LoopBufs b;
  const double* xc;
  const double* xn;
  double theta_hat;
  __device__ bool prepare() {
    const DevState* st = b.st;
    if (!st->running) return false;
    xc = pick(b.x, st->cur);
    xn = pick(b.x, st->cur ^ 1);
    theta_hat = st->eta / st->mp_eta_hat;  // solver.cpp:241
    return true;
  }
  template <class Acc>
  __device__ void apply(int64_t i, Acc&) const {
    b.mp_ext[i] = xn[i] + theta_hat * (xn[i] - xc[i]);  // solver.cpp:244
  }
  __device__ void finalize(const double (&)[K]) const {}
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

struct EpiMpDual {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  LoopBufs b;
  const double* yc;
  double* yn;
  double sigma, pend;
  __device__ bool prepare() {
    const DevState* st = b.st;
    if (!st->running) return false;
    yc = pick(b.y, st->cur);
    yn = pick(b.y, st->cur ^ 1);
    sigma = st->omega * st->mp_eta_hat;  // solver.cpp:249
    pend = st->trials_iter == 0 ? st->pending : 0.0;
    return true;
  }
  __device__ const double* vec() const { return b.mp_ext; }
  struct Pre {
    double y, q, a;
  };
  __device__ Pre load(int i) const {
    return Pre{yc[i], b.q[i], pend != 0.0 ? b.avg_y[i] : 0.0};
  }
  template <class Acc>
  __device__ void apply(int i, double kw, const Pre& o, Acc& acc) const {
    if (pend != 0.0) b.avg_y[i] = o.a + pend * o.y;
    double v = o.y + sigma * (o.q - kw);  // solver.cpp:252-255
    if (i < b.m1) v = ref_max(v, 0.0);
    yn[i] = v;
    const double dy = v - o.y;
    b.mp_dy[i] = dy;
    acc.add(0, i, dy * dy);
    acc.add(1, i, isfinite(v) ? 0.0 : 1.0);
  }
  __device__ void store(double dy_sq, bool bad) const {
    DevState* st = b.st;
    st->mp_dy_sq = dy_sq;
    if (bad) {  // solver.cpp:257-259
      st->status = kNonFinite;
      st->running = 0;
      if (b.use_cond) cudaGraphSetConditional(b.cond, 0u);
    }
  }
  __device__ void finalize(const double (&tot)[K]) const { store(tot[0], tot[1] != 0.0); }
  __device__ void finalize_ordered(const double* t, int64_t m) const {
    store(fold(0.0, t, m), any_nonzero(t + m, m));
  }
};

struct EpiMpCheck {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  LoopBufs b;
  __device__ bool prepare() { return b.st->running != 0; }
  __device__ const double* vec() const { return b.mp_dy; }
  struct Pre {};
  __device__ Pre load(int) const { return Pre{}; }
  template <class Acc>
  __device__ void apply(int j, double ktdy, const Pre&, Acc& acc) const {
    acc.add(0, j, ktdy * ktdy);
  }
  __device__ void decide(double ktdy_sq) const {
    DevState* st = b.st;
    st->slots += 1;
    st->trials_iter += 1;
    st->pending = 0.0;
    const double eta_hat = st->mp_eta_hat;
    // solver.cpp:263-269: eta_hat ||K'dy|| <= breaking ||dy||
    if (eta_hat * sqrt(ktdy_sq) <= st->mp_break * sqrt(st->mp_dy_sq)) {
      const double theta_hat = st->eta / eta_hat;
      st->k_total += 1;
      st->t_inner += 1;
      st->accepted += 1;
      st->step_trials += st->trials_iter;
      st->ledger_kt += 1 + st->trials_iter;  // K'y, then K'dy per trial
      st->ledger_k += st->trials_iter;       // K w per trial
      st->trials_iter = 0;
      st->eta = eta_hat;
      st->mp_theta = theta_hat;
      st->last_eta_used = eta_hat;
      st->avg_weight += eta_hat;
      st->pending = eta_hat;
      st->cur ^= 1;
      if (st->accepted >= st->target) {
        st->status = kDone;
        st->running = 0;
      } else if (st->k_total >= st->iteration_limit ||
                 0.5 * static_cast<double>(st->ledger_k + st->ledger_kt) >= st->kkt_pass_limit) {
        st->status = kLimit;
        st->running = 0;
      }
    } else {
      st->mp_eta_hat = eta_hat * st->mp_down;  // solver.cpp:270-273
      if (st->mp_eta_hat < kStepSizeFloor) {
        st->status = kUnderflow;
        st->running = 0;
      }
    }
    if (b.use_cond) cudaGraphSetConditional(b.cond, st->running ? 1u : 0u);
  }
  __device__ void finalize(const double (&tot)[K]) const { decide(tot[0]); }
  __device__ void finalize_ordered(const double* t, int64_t n) const { decide(fold(0.0, t, n)); }
};

// ---------------------------------------------------------------------
// Plain products (no reduction): out = K v.
struct EpiStore {
  static constexpr int K = 1;
  static constexpr bool kReduce = false;
  const double* v;
  double* out;
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return v; }
  struct Pre {};
  __device__ Pre load(int) const { return Pre{}; }
  template <class Acc>
  __device__ void apply(int s, double dot, const Pre&, Acc&) const {
    out[s] = dot;
  }
  __device__ void finalize(const double (&)[K]) const {}
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// ---------------------------------------------------------------------
// Window-blocked products (tree mode, gathered vector larger than L2): the
// entries of every segment are split by gather index into windows that fit
// in L2 and the product runs one phase per window (config 4's
// 320 MB x makes every random gather an HBM sector read).  Phases before the
// last accumulate each segment's dot in `carry`; the last one runs the real
// epilogue on carry + its own window's dot.  Sums stay deterministic (window
// dots in window order), not sequential.
template <class Epi>
struct EpiCarry {
  static constexpr int K = 1;
  static constexpr bool kReduce = false;
  Epi inner;            // gathered vector and running flag only
  const double* carry;  // nullptr in the first phase
  double* out;
  __device__ bool prepare() { return inner.prepare(); }
  __device__ const double* vec() const { return inner.vec(); }
  struct Pre {
    double c;
  };
  __device__ Pre load(int s) const { return Pre{carry != nullptr ? carry[s] : 0.0}; }
  template <class Acc>
  __device__ void apply(int s, double dot, const Pre& p, Acc&) const {
    out[s] = p.c + dot;
  }
  __device__ void finalize(const double (&)[K]) const {}
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

template <class Epi>
struct EpiCarryIn {
  static constexpr int K = Epi::K;
  static constexpr bool kReduce = Epi::kReduce;
  Epi inner;
  const double* carry;
  __device__ bool prepare() { return inner.prepare(); }
  __device__ const double* vec() const { return inner.vec(); }
  struct Pre {
    typename Epi::Pre p;
    double c;
  };
  __device__ Pre load(int s) const { return Pre{inner.load(s), carry[s]}; }
  template <class Acc>
  __device__ void apply(int s, double dot, const Pre& p, Acc& acc) const {
    inner.apply(s, p.c + dot, p.p, acc);
  }
  __device__ void finalize(const double (&t)[K]) const { inner.finalize(t); }
  __device__ void finalize_ordered(const double* t, int64_t n) const { inner.finalize_ordered(t, n); }
};

// out = K v plus the power-iteration reductions v'out and ||out||^2
// (estimate_spectral_norm, sparse_matrix.cpp:206-211).
struct EpiStoreDotNorm {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  const double* v;      // gathered vector
  const double* w;      // vector dotted with the product
  double* out;
  double* result;       // [2]
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return v; }
  struct Pre {
    double w;
  };
  __device__ Pre load(int s) const { return Pre{w[s]}; }
  template <class Acc>
  __device__ void apply(int s, double dot, const Pre& o, Acc& acc) const {
    out[s] = dot;
    acc.add(0, s, o.w * dot);
    acc.add(1, s, dot * dot);
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
  }
  __device__ void finalize_ordered(const double* t, int64_t n) const {
    result[0] = fold(0.0, t, n);
    result[1] = fold(0.0, t + n, n);
  }
  // ordered mode through the exact parallel fold (exactfold.cuh)
  __host__ void fold_plan(const double* t, int64_t n, FoldJobs& f) const {
    f.count = 2;
    f.job[0] = FoldJob{t, n, 0.0, -1, 1.0, nullptr, nullptr};
    f.job[1] = FoldJob{t + n, n, 0.0, -1, 1.0, nullptr, nullptr};
  }
  __device__ void finalize_exact(const double* r, unsigned) const {
    result[0] = r[0];
    result[1] = r[1];
  }
};

// ---------------------------------------------------------------------
// convergence_info (termination.cpp:23-73) on the presolved, unscaled
// problem.  Step 1 (elementwise over n+m): reduced_point (solver.cpp:495-502)
// x = clamp(D2 x~, l, u), y = D1 y~; c'x, q'y; finiteness.
struct OpEvalPoint {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
  int64_t n, m;
  int raw;           // 1: point already in the presolved space
  const double* xs;  // working-space point
  const double* ys;
  const double* d1;
  const double* d2;
  const double* l;   // presolved bounds / data
  const double* u;
  const double* c;
  const double* q;
  double* xr;        // out: reduced point
  double* yr;
  double* result;    // [3] c'x, q'y, nonfinite count
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    if (i < n) {
      const double v = raw ? xs[i] : ref_min(ref_max(xs[i] * d2[i], l[i]), u[i]);
      xr[i] = v;
      acc.add(0, i, c[i] * v);
      acc.add(1, i, 0.0);
      acc.add(2, i, isfinite(v) ? 0.0 : 1.0);
    } else {
      const int64_t j = i - n;
      const double v = raw ? ys[j] : ys[j] * d1[j];
      yr[j] = v;
      acc.add(0, i, 0.0);
      acc.add(1, i, q[j] * v);
      acc.add(2, i, isfinite(v) ? 0.0 : 1.0);
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
    result[2] = tot[2];
  }
  __device__ void finalize_ordered(const double* t, int64_t tot) const {
    result[0] = fold(0.0, t, n);            // linalg::dot(c, x)
    result[1] = fold(0.0, t + tot + n, m);  // linalg::dot(q, y)
    result[2] = any_nonzero(t + 2 * tot, tot) ? 1.0 : 0.0;
  }
  __host__ void fold_plan(const double* t, int64_t tot, FoldJobs& f) const {
    f.count = 2;
    f.job[0] = FoldJob{t, n, 0.0, -1, 1.0, nullptr, nullptr};
    f.job[1] = FoldJob{t + tot + n, m, 0.0, -1, 1.0, nullptr, nullptr};
    f.nflags = 1;
    f.flag[0] = t + 2 * tot;
    f.flag_n[0] = tot;
    f.flag_group[0] = 0;
  }
  __device__ void finalize_exact(const double* r, unsigned flags) const {
    result[0] = r[0];
    result[1] = r[1];
    result[2] = (flags & 1u) ? 1.0 : 0.0;
  }
};

// Step 2 (rows, original values): primal residual (termination.cpp:54-61).
struct EpiPrimalResidual {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  const double* xr;
  const double* q;
  int64_t m1;
  double* result;  // [1]
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return xr; }
  struct Pre {
    double q;
  };
  __device__ Pre load(int i) const { return Pre{q[i]}; }
  template <class Acc>
  __device__ void apply(int i, double kx, const Pre& o, Acc& acc) const {
    double v = o.q - kx;
    if (i < m1) v = ref_max(v, 0.0);
    acc.add(0, i, v * v);
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
  __device__ void finalize_ordered(const double* t, int64_t m) const {
    result[0] = fold(0.0, t, m);
  }
  __host__ void fold_plan(const double* t, int64_t m, FoldJobs& f) const {
    f.count = 1;
    f.job[0] = FoldJob{t, m, 0.0, -1, 1.0, nullptr, nullptr};
  }
  __device__ void finalize_exact(const double* r, unsigned) const { result[0] = r[0]; }
};

// Step 3 (columns, original values): reduced costs, dual residual and the
// bound terms of the dual objective (termination.cpp:46-68,
// lp_model.cpp:129-165).
struct EpiDualResidual {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
  const double* yr;
  const double* c;
  const double* l;
  const double* u;
  double* result;          // [3] dual_sq, bound terms, infinite-product count
  const double* q_dot_y;   // ordered mode: q'y from step 1
  double constant;         // ordered mode: objective constant
  double* dual_objective;  // ordered mode: q'y + const + sum bound*lambda
  double* kty_out = nullptr;  // tree mode: K'y of the presolved point, kept for the gap setup
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return yr; }
  struct Pre {
    double c, l, u;
  };
  __device__ Pre load(int j) const { return Pre{c[j], l[j], u[j]}; }
  template <class Acc>
  __device__ void apply(int j, double kty, const Pre& o, Acc& acc) const {
    if (kty_out != nullptr) kty_out[j] = kty;
    const double r = o.c - kty;
    const double lj = o.l, uj = o.u;
    const bool has_lower = lj > -INFINITY;
    const bool has_upper = uj < INFINITY;
    double lambda;
    if (!has_lower && !has_upper) {
      lambda = 0.0;
    } else if (!has_lower) {
      lambda = ref_min(r, 0.0);
    } else if (!has_upper) {
      lambda = ref_max(r, 0.0);
    } else {
      lambda = r;
    }
    const double d = r - lambda;
    acc.add(0, j, d * d);
    double bt = 0.0, inf = 0.0;
    if (lambda != 0.0) {
      const double bound = lambda > 0.0 ? lj : uj;
      if (!isfinite(bound)) {
        inf = 1.0;
      } else {
        bt = bound * lambda;
      }
    }
    acc.add(1, j, bt);
    acc.add(2, j, inf);
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
    result[2] = tot[2];
  }
  __device__ void finalize_ordered(const double* t, int64_t n) const {
    result[0] = fold(0.0, t, n);
    result[1] = 0.0;
    result[2] = any_nonzero(t + 2 * n, n) ? 1.0 : 0.0;
    // lp_model.cpp:154-163: value = q'y + const, then += bound*lambda in order
    double v = *q_dot_y + constant;
    for (int64_t j = 0; j < n; ++j) {
      const double bt = ld_cg(&t[n + j]);
      if (bt != 0.0) v += bt;
    }
    *dual_objective = v;
  }
  // The bound terms are folded including the zero ones (the reference skips
  // lambda == 0): adding +0.0 changes a partial sum only when it is -0.0, so
  // the two agree except possibly in the sign of an exactly-zero objective.
  __host__ void fold_plan(const double* t, int64_t nn, FoldJobs& f) const {
    f.count = 2;
    f.job[0] = FoldJob{t, nn, 0.0, -1, 1.0, nullptr, nullptr};
    f.job[1] = FoldJob{t + nn, nn, constant, -1, 1.0, nullptr, q_dot_y};
    f.nflags = 1;
    f.flag[0] = t + 2 * nn;
    f.flag_n[0] = nn;
    f.flag_group[0] = 0;
  }
  __device__ void finalize_exact(const double* r, unsigned flags) const {
    result[0] = r[0];
    result[1] = 0.0;
    result[2] = (flags & 1u) ? 1.0 : 0.0;
    *dual_objective = r[1];
  }
};

// ---------------------------------------------------------------------
// normalized_duality_gap (solver.cpp:277-370), setup of g, lo, hi over the
// n primal coordinates (columns: K'y) and the m dual ones (rows: Kx), with
// the reductions of the any-gradient test, sum g^2/w and the nu -> 0
// "bounded" corner (solver.cpp:318-342).
// terms: [0] g!=0, [1] g*g/w, [2] non-finite corner, [3] w*d*d, [4] g*d
__device__ __forceinline__ void ndg_terms(double gj, double w, double d, double (&t)[5]) {
  t[0] = gj != 0.0 ? 1.0 : 0.0;
  t[1] = gj * gj / w;
  if (!isfinite(d)) {
    t[2] = 1.0;
    t[3] = 0.0;
    t[4] = 0.0;
  } else {
    t[2] = 0.0;
    t[3] = w * d * d;
    t[4] = gj * d;
  }
}

struct EpiNdgPrimal {
  static constexpr int K = 5;
  static constexpr bool kReduce = true;
  const double* y;   // gathered
  const double* x;
  const double* c;
  const double* l;
  const double* u;
  double omega;
  double* g;
  double* lo;
  double* hi;
  double* result;
  const double* omega_dev = nullptr;  // graph-captured evaluation: omega read on device
  __device__ bool prepare() {
    if (omega_dev != nullptr) omega = *omega_dev;
    return true;
  }
  __device__ const double* vec() const { return y; }
  struct Pre {
    double x, c, l, u;
  };
  __device__ Pre load(int j) const { return Pre{x[j], c[j], l[j], u[j]}; }
  template <class Acc>
  __device__ void apply(int j, double kty, const Pre& o, Acc& acc) const {
    const double gj = kty - o.c;
    const double loj = ref_min(0.0, o.l - o.x);
    const double hij = ref_max(0.0, o.u - o.x);
    g[j] = gj;
    lo[j] = loj;
    hi[j] = hij;
    const double d = gj > 0.0 ? hij : (gj < 0.0 ? loj : 0.0);
    double t[5];
    ndg_terms(gj, omega, d, t);
#pragma unroll
    for (int k = 0; k < 5; ++k) acc.add(k, j, t[k]);
  }
  __device__ void finalize(const double (&tot)[K]) const {
#pragma unroll
    for (int k = 0; k < K; ++k) result[k] = tot[k];
  }
  // the dual half folds both halves in (x; y) order
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

struct EpiNdgDual {
  static constexpr int K = 5;
  static constexpr bool kReduce = true;
  const double* x;   // gathered
  const double* y;
  const double* q;
  int64_t m1;
  double winv;       // 1/omega, computed once like solver.cpp:313
  double* g;         // dual part (already offset by n)
  double* lo;
  double* kx_out;    // Kx of the point (kept for a restart to it)
  double* result;    // [10]: primal half [0..5), dual half [5..10)
  const double* primal_terms;  // ordered mode: EpiNdgPrimal's terms [5 n]
  int64_t n;
  const double* omega_dev = nullptr;  // graph-captured evaluation: 1/omega on device
  __device__ bool prepare() {
    if (omega_dev != nullptr) winv = 1.0 / *omega_dev;
    return true;
  }
  __device__ const double* vec() const { return x; }
  struct Pre {
    double y, q;
  };
  __device__ Pre load(int i) const { return Pre{y[i], q[i]}; }
  template <class Acc>
  __device__ void apply(int i, double kx, const Pre& o, Acc& acc) const {
    if (kx_out != nullptr) kx_out[i] = kx;
    const double gi = o.q - kx;
    const double loi = i < m1 ? ref_min(0.0, -o.y) : -INFINITY;
    g[i] = gi;
    lo[i] = loi;
    const double d = gi > 0.0 ? INFINITY : (gi < 0.0 ? loi : 0.0);
    double t[5];
    ndg_terms(gi, winv, d, t);
#pragma unroll
    for (int k = 0; k < 5; ++k) acc.add(k, i, t[k]);
  }
  __device__ void finalize(const double (&tot)[K]) const {
#pragma unroll
    for (int k = 0; k < K; ++k) result[k + 5] = tot[k];
  }
  // both halves, (x; y) order; the primal slots [0..5) carry the totals
  __device__ void finalize_ordered(const double* t, int64_t m) const {
    const double* p = primal_terms;
    result[0] = (any_nonzero(p, n) || any_nonzero(t, m)) ? 1.0 : 0.0;
    result[1] = fold(fold(0.0, p + n, n), t + m, m);          // solver.cpp:322
    result[2] = (any_nonzero(p + 2 * n, n) || any_nonzero(t + 2 * m, m)) ? 1.0 : 0.0;
    result[3] = fold(fold(0.0, p + 3 * n, n), t + 3 * m, m);  // solver.cpp:338
    result[4] = fold(fold(0.0, p + 4 * n, n), t + 4 * m, m);  // linalg::dot(g, d)
    for (int k = 5; k < 10; ++k) result[k] = 0.0;
  }
  __host__ void fold_plan(const double* t, int64_t m, FoldJobs& f) const {
    const double* p = primal_terms;
    f.count = 6;
    for (int h = 0; h < 3; ++h) {  // (x; y) folds of terms 1, 3, 4
      const int k = h == 0 ? 1 : h + 2;
      f.job[2 * h] = FoldJob{p + k * n, n, 0.0, -1, 1.0, nullptr, nullptr};
      f.job[2 * h + 1] = FoldJob{t + k * m, m, 0.0, 2 * h, 1.0, nullptr, nullptr};
    }
    f.nflags = 4;
    f.flag[0] = p;          f.flag_n[0] = n; f.flag_group[0] = 0;  // g != 0
    f.flag[1] = t;          f.flag_n[1] = m; f.flag_group[1] = 0;
    f.flag[2] = p + 2 * n;  f.flag_n[2] = n; f.flag_group[2] = 1;  // non-finite corner
    f.flag[3] = t + 2 * m;  f.flag_n[3] = m; f.flag_group[3] = 1;
  }
  __device__ void finalize_exact(const double* r, unsigned flags) const {
    result[0] = (flags & 1u) ? 1.0 : 0.0;
    result[1] = r[1];
    result[2] = (flags & 2u) ? 1.0 : 0.0;
    result[3] = r[3];
    result[4] = r[5];
    for (int k = 5; k < 10; ++k) result[k] = 0.0;
  }
};

// Same as EpiNdgDual but with Kx already cached (the loop keeps Kx of the
// current point), so it runs elementwise without touching K.
struct OpNdgDualCached {
  static constexpr int K = 5;
  static constexpr bool kReduce = true;
  const double* kx;
  EpiNdgDual e;
  __device__ bool prepare() { return e.prepare(); }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    e.apply(static_cast<int>(i), kx[i], e.load(static_cast<int>(i)), acc);
  }
  __device__ void finalize(const double (&tot)[K]) const { e.finalize(tot); }
  __device__ void finalize_ordered(const double* t, int64_t m) const {
    e.finalize_ordered(t, m);
  }
  __host__ void fold_plan(const double* t, int64_t m, FoldJobs& f) const { e.fold_plan(t, m, f); }
  __device__ void finalize_exact(const double* r, unsigned flags) const { e.finalize_exact(r, flags); }
};

// EpiNdgPrimal without touching K (tree mode): the working-space K~'y~ of
// the point is D2 (K' y) with y = D1 y~ the presolved dual that
// convergence_info has just multiplied (EpiDualResidual::kty_out) -- the
// same product up to rounding, one elementwise pass instead of a column
// product.
struct OpNdgPrimalRaw {
  static constexpr int K = 5;
  static constexpr bool kReduce = true;
  const double* kty_raw;
  const double* d2;
  EpiNdgPrimal e;
  __device__ bool prepare() { return e.prepare(); }
  template <class Acc>
  __device__ void apply(int64_t j, Acc& acc) const {
    const int jj = static_cast<int>(j);
    e.apply(jj, d2[j] * kty_raw[j], e.load(jj), acc);
  }
  __device__ void finalize(const double (&tot)[K]) const { e.finalize(tot); }
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// Bisection state of one normalized_duality_gap evaluation.
constexpr int kNuLevels = 3;                     // bisection levels per pass
constexpr int kNuCands = (1 << kNuLevels) - 1;   // 7 candidate multipliers
struct NdgState {
  double nu_lo;
  double nu_hi;
  double radius;
  double result;   // g'd / r once done
  double nu[kNuCands];  // candidates of the next pass (heap order)
  double rcp_primal[kNuCands];  // tree mode: RN(1 / (nu * omega))
  double rcp_dual[kNuCands];    // tree mode: RN(1 / (nu * (1/omega)))
  double omega, winv;
  double rcp_lo[2], rcp_hi[2];  // tree mode: RN(1 / (nu_lo|hi * w)), primal / dual
  int32_t it;      // bisection iterations consumed (<= 200)
  int32_t done;
  int32_t passes;
  int32_t grid_passes;  // tree-mode cooperative passes that synchronized the grid
};

#ifdef FOLP_BISECT_TIMES
// Diagnostic build: block 0's %globaltimer at the start and after each pass,
// summed per pass index over launches ([k][0] ns, [k][1] launches, [k][2]
// launches in which block 0 ran pass k alone); read by the context's timing print.
constexpr int kBisectTimeSlots = 32;
__device__ unsigned long long g_bisect_times[kBisectTimeSlots][3];
#endif

// Heap-ordered tree of the next kNuLevels bisection midpoints below
// [lo, hi]: node i covers [a_i, b_i] with nu_i = 0.5 * (a_i + b_i)
// (solver.cpp:360); children 2i+1 = [a_i, nu_i], 2i+2 = [nu_i, b_i].
// Same IEEE operations on host and device.
__host__ __device__ inline void ndg_candidates(double lo, double hi, double* nu) {
  double a[kNuCands], b[kNuCands];
  a[0] = lo;
  b[0] = hi;
  for (int i = 0; i < kNuCands; ++i) {
    nu[i] = 0.5 * (a[i] + b[i]);
    if (2 * i + 2 < kNuCands) {
      a[2 * i + 1] = a[i];
      b[2 * i + 1] = nu[i];
      a[2 * i + 2] = nu[i];
      b[2 * i + 2] = b[i];
    }
  }
}

__host__ __device__ inline void ndg_reciprocals(NdgState* st) {
  for (int i = 0; i < kNuCands; ++i) {
    st->rcp_primal[i] = 1.0 / (st->nu[i] * st->omega);
    st->rcp_dual[i] = 1.0 / (st->nu[i] * st->winv);
  }
  st->rcp_lo[0] = 1.0 / (st->nu_lo * st->omega);
  st->rcp_lo[1] = 1.0 / (st->nu_lo * st->winv);
  st->rcp_hi[0] = 1.0 / (st->nu_hi * st->omega);
  st->rcp_hi[1] = 1.0 / (st->nu_hi * st->winv);
}

// Tree mode: once no element changes its clamping state inside the bracket
// [nu_lo, nu_hi], ||d(nu)||_w^2 = Q + S / nu^2 and g'd(nu) = H + S / nu
// exactly there (Q, H: the clamped elements' w c^2 and g c; S: the free
// elements' g^2 / w), so the remaining levels of the reference bisection
// (solver.cpp:356-368) are replayed from these three sums without another
// pass over the data.
__device__ inline void ndg_finish_analytic(NdgState* st, double q, double h, double sfree) {
  const double r = st->radius;
  const double r2 = r * r;
  double lo_ = st->nu_lo, hi_ = st->nu_hi;
  while (!st->done) {
    const double nu = 0.5 * (lo_ + hi_);
    const double nsq = q + sfree / (nu * nu);
    const double gd = h + sfree / nu;
    st->it += 1;
    if (fabs(sqrt(nsq) - r) <= 1e-10 * r || st->it >= 200) {
      st->result = gd / r;
      st->done = 1;
    } else if (nsq > r2) {
      lo_ = nu;
    } else {
      hi_ = nu;
    }
  }
  st->nu_lo = lo_;
  st->nu_hi = hi_;
}

// Replays `levels` levels of the reference bisection (solver.cpp:356-368)
// from per-node sums (heap order) and leaves the next bracket.
__device__ inline void ndg_replay(NdgState* st, const double* norm_sq, const double* gd,
                                  int levels, bool reciprocals = true) {
  const double r = st->radius;
  const double r2 = r * r;
  double lo_ = st->nu_lo, hi_ = st->nu_hi;
  int node = 0;
  st->passes += 1;
  for (int level = 0; level < levels; ++level) {
    const int evaluated = node;
    st->it += 1;
    if (fabs(sqrt(norm_sq[evaluated]) - r) <= 1e-10 * r) {
      st->result = gd[evaluated] / r;
      st->done = 1;
      return;
    }
    if (norm_sq[evaluated] > r2) {
      lo_ = st->nu[evaluated];
      node = 2 * node + 2;
    } else {
      hi_ = st->nu[evaluated];
      node = 2 * node + 1;
    }
    if (st->it >= 200) {  // loop exhausted: d holds the last evaluation
      st->result = gd[evaluated] / r;
      st->done = 1;
      return;
    }
  }
  st->nu_lo = lo_;
  st->nu_hi = hi_;
  ndg_candidates(lo_, hi_, st->nu);
  if (reciprocals) ndg_reciprocals(st);
}

// ndg_reciprocals' value j (0..kNdgRcp-1) alone -- the same IEEE operations,
// so threads can share the work.
constexpr int kNdgRcp = 2 * kNuCands + 4;
__device__ inline void ndg_reciprocal(NdgState* st, int j) {
  if (j < kNuCands) {
    st->rcp_primal[j] = 1.0 / (st->nu[j] * st->omega);
  } else if (j < 2 * kNuCands) {
    st->rcp_dual[j - kNuCands] = 1.0 / (st->nu[j - kNuCands] * st->winv);
  } else if (j < 2 * kNuCands + 2) {
    st->rcp_lo[j - 2 * kNuCands] = 1.0 / (st->nu_lo * (j == 2 * kNuCands ? st->omega : st->winv));
  } else {
    st->rcp_hi[j - 2 * kNuCands - 2] = 1.0 / (st->nu_hi * (j == 2 * kNuCands + 2 ? st->omega : st->winv));
  }
}

// One bisection pass.  Tree mode: ||d(nu)||_w^2 and g'd(nu) for the 7 nodes
// of the next 3 levels (one read of g, lo, hi).  Ordered mode: the first
// node only, folded in (x; y) order -- one reference iteration per pass.
struct OpNdgPass {
  static constexpr int K = 2 * kNuCands;
  static constexpr bool kReduce = true;
  int64_t n, total;
  const double* g;
  const double* lo;
  const double* hi;  // primal part only; dual hi = +inf
  double omega, winv;
  NdgState* ns;

  // the weights come from the bisection state (set by k_ndg_init), so a
  // captured evaluation graph never bakes a stale omega into the pass
  __device__ bool prepare() {
    if (ns->done != 0) return false;
    omega = ns->omega;
    winv = ns->winv;
    return true;
  }
  template <class Acc>
  __device__ void apply(int64_t s, Acc& acc) const {
    const double gs = g[s];
    const bool primal = s < n;
    const double w = primal ? omega : winv;
    const double los = lo[s];
    const double his = primal ? hi[s] : INFINITY;
    const double* nu = ns->nu;
    if constexpr (Acc::kOrdered) {
      // exactly the reference's quotient g / (nu * w) (solver.cpp:349)
      const double unclamped = gs / (__ldg(&nu[0]) * w);
      const double d = ref_min(ref_max(unclamped, los), his);
      acc.add(0, s, w * d * d);
      acc.add(1, s, gs * d);
    } else {
      // tree mode: g * RN(1 / (nu * w)) -- within 1.5 ulp of the quotient,
      // far below the tree-order noise; no per-element division
      const double* rcp = primal ? ns->rcp_primal : ns->rcp_dual;
#pragma unroll
      for (int p = 0; p < kNuCands; ++p) {
        const double unclamped = gs * __ldg(&rcp[p]);
        const double d = ref_min(ref_max(unclamped, los), his);
        acc.add(2 * p, s, w * d * d);
        acc.add(2 * p + 1, s, gs * d);
      }
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    double nsq[kNuCands], gd[kNuCands];
    for (int p = 0; p < kNuCands; ++p) {
      nsq[p] = tot[2 * p];
      gd[p] = tot[2 * p + 1];
    }
    ndg_replay(ns, nsq, gd, kNuLevels);
  }
  __device__ void finalize_ordered(const double* t, int64_t tot_n) const {
    const double norm_sq = fold(0.0, t, tot_n);
    const double gd = fold(0.0, t + tot_n, tot_n);
    ndg_replay(ns, &norm_sq, &gd, 1);
  }
  __host__ void fold_plan(const double* t, int64_t tot_n, FoldJobs& f) const {
    f.count = 2;
    f.job[0] = FoldJob{t, tot_n, 0.0, -1, 1.0, nullptr, nullptr};
    f.job[1] = FoldJob{t + tot_n, tot_n, 0.0, -1, 1.0, nullptr, nullptr};
  }
  __device__ void finalize_exact(const double* r, unsigned) const { ndg_replay(ns, &r[0], &r[1], 1); }
};

// ---------------------------------------------------------------------
// Squared distances of two points: [0] sum (xa-xb)^2, [1] sum (ya-yb)^2.
struct OpDistance {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
  int64_t n;
  const double* xa;
  const double* xb;
  const double* ya;
  const double* yb;
  double* result;
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    if (i < n) {
      const double d = xa[i] - xb[i];
      acc.add(0, i, d * d);
      acc.add(1, i, 0.0);
    } else {
      const double d = ya[i - n] - yb[i - n];
      acc.add(0, i, 0.0);
      acc.add(1, i, d * d);
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
  }
  __device__ void finalize_ordered(const double* t, int64_t tot) const {
    result[0] = fold(0.0, t, n);
    result[1] = fold(0.0, t + tot + n, tot - n);
  }
  __host__ void fold_plan(const double* t, int64_t tot, FoldJobs& f) const {
    f.count = 2;
    f.job[0] = FoldJob{t, n, 0.0, -1, 1.0, nullptr, nullptr};
    f.job[1] = FoldJob{t + tot + n, tot - n, 0.0, -1, 1.0, nullptr, nullptr};
  }
  __device__ void finalize_exact(const double* r, unsigned) const {
    result[0] = r[0];
    result[1] = r[1];
  }
};

// Fold the pending eta*z into the running sums and materialize the
// average (solver.cpp:509-538).
struct OpAverage {
  static constexpr int K = 1;
  static constexpr bool kReduce = false;
  int64_t n, m1;
  const double* x;
  const double* y;
  double* ax;
  double* ay;
  const double* l;
  const double* u;
  double pending;
  double inv;      // 1 / avg_weight
  int copy_current;  // avg_weight <= 0: the average is the current point
  double* out_x;
  double* out_y;
  const DevState* st = nullptr;  // graph-captured evaluation: weights read on device
  __device__ bool prepare() {
    if (st != nullptr) {
      pending = st->pending;
      copy_current = st->avg_weight <= 0.0 ? 1 : 0;
      inv = st->avg_weight > 0.0 ? 1.0 / st->avg_weight : 0.0;
    }
    return true;
  }
  template <class Acc>
  __device__ void apply(int64_t i, Acc&) const {
    if (i < n) {
      double s = ax[i];
      if (pending != 0.0) {
        s += pending * x[i];
        ax[i] = s;
      }
      out_x[i] = copy_current ? x[i] : ref_min(ref_max(s * inv, l[i]), u[i]);
    } else {
      const int64_t j = i - n;
      double s = ay[j];
      if (pending != 0.0) {
        s += pending * y[j];
        ay[j] = s;
      }
      double v = s * inv;
      if (j < m1) v = ref_max(v, 0.0);
      out_y[j] = copy_current ? y[j] : v;
    }
  }
  __device__ void finalize(const double (&)[K]) const {}
  __device__ void finalize_ordered(const double*, int64_t) const {}
};

// Ordered mode through the exact parallel fold: an epilogue / operator with
// fold_plan (host: the folds of its stored terms) and finalize_exact
// (device: the same results as finalize_ordered) is finalized by a
// k_exact_fold<FinExact<E>> launch instead of one thread's sequential folds.
template <class E>
struct FinExact {
  E e;
  __device__ bool prepare() { return e.prepare(); }
  __device__ void finalize(const double* r, int, unsigned flags) const { e.finalize_exact(r, flags); }
};
template <class E, class = void>
struct HasFoldPlan : std::false_type {};
template <class E>
struct HasFoldPlan<E, std::void_t<decltype(&E::fold_plan)>> : std::true_type {};

}  // namespace folpgpu
