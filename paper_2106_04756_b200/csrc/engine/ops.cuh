// ops.cuh -- epilogues and elementwise operators of the PDLP loop.
//
// Each struct is a value type passed by value as a kernel parameter; its
// prepare() runs once per CTA and caches the loop scalars from the device
// state.  Arithmetic follows the reference expression by expression (the
// file is compiled with -fmad=false, so a*b+c is two roundings exactly like
// the reference's x86-64 -O2 build, which emits no FMA).
#pragma once

#include <cuda_runtime.h>

#include "segdot.cuh"

namespace folpgpu {

// Chunk status values (mirror folp_gpu.h).
constexpr int kRunning = 0;
constexpr int kDone = 1;
constexpr int kLimit = 2;
constexpr int kNonFinite = 3;
constexpr int kUnderflow = 4;

constexpr double kStepSizeFloor = 1e-300;  // solver.cpp:31

// Device-resident loop state.  Host mirrors it at chunk boundaries.
struct DevState {
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
};

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
  DevState* st;
  const double* red;   // per-iteration factor tables of the chunk
  const double* grow;
  cudaGraphConditionalHandle cond;
  int use_cond;
};

// ---------------------------------------------------------------------
// Kernel A: K'y of the current dual, fused primal projected step
// (pdhg_trial, solver.cpp:58-63) + lazy averaging of the previous accepted
// primal (accumulate_average, solver.cpp:530-538) + sum omega*dx*dx
// (solver.cpp:84-88) and the finiteness flag (solver.cpp:91-93).
struct EpiPrimal {
  static constexpr int K = 2;
  static constexpr bool kReduce = true;
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
    return Pre{xc[j], b.c[j], b.l[j], b.u[j], pend != 0.0 ? avg[j] : 0.0};
  }
  __device__ void apply(int j, double kty, const Pre& o, double (&acc)[K]) const {
    const double xj = o.x;
    if (pend != 0.0) avg[j] = o.a + pend * xj;
    const double v = xj - tau * (o.c - kty);
    const double xv = ref_min(ref_max(v, o.l), o.u);
    xn[j] = xv;
    const double dx = xv - xj;
    acc[0] += omega * dx * dx;
    if (!isfinite(xv)) acc[1] += 1.0;
  }
  __device__ void finalize(const double (&tot)[K]) const {
    b.st->sx = tot[0];
    b.st->bad_a = tot[1];
  }
};

// Kernel B: K x' of the trial primal, fused dual projected step with the
// extrapolation 2Kx'-Kx (solver.cpp:70-75), cross term and movement
// (solver.cpp:76-83), lazy averaging of the previous accepted dual, and the
// adaptive step-size decision (adaptive_step, solver.cpp:173-199) in the
// last CTA.  Kx' is kept as the next Kx (bit-identical to recomputing it,
// because the product is deterministic).
struct EpiDual {
  static constexpr int K = 3;
  static constexpr bool kReduce = true;
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
  __device__ void apply(int i, double kx_next, const Pre& o, double (&acc)[K]) const {
    const double yi = o.y;
    if (pend != 0.0) b.avg_y[i] = o.a + pend * yi;
    const double kxi = o.kx;
    const double extrapolated = 2.0 * kx_next - kxi;
    double v = yi + sigma * (o.q - extrapolated);
    if (i < b.m1) v = ref_max(v, 0.0);
    yn[i] = v;
    kxn[i] = kx_next;
    const double dy = v - yi;
    acc[0] += dy * (kxi - kx_next);
    acc[1] += dy * dy;
    if (!isfinite(v)) acc[2] += 1.0;
  }
  __device__ void finalize(const double (&tot)[K]) const {
    DevState* st = b.st;
    st->slots += 1;
    st->pending = 0.0;  // consumed by kernels A and B of this slot
    const double cross = tot[0];
    const double omega = st->omega;
    const double eta = st->eta;
    double movement = tot[1];
    movement = movement / omega;  // solver.cpp:83
    movement = movement + st->sx;
    st->cross = cross;
    st->movement = movement;
    st->trials_iter += 1;
    if (st->bad_a != 0.0 || tot[2] != 0.0) {
      st->status = kNonFinite;
      st->running = 0;
    } else {
      bool accept = true;
      double eta_next = eta;
      if (st->policy == 0) {
        const int64_t ki = st->k_total - st->k_chunk0;
        const double eta_bar =
            cross > 0.0 ? movement / (2.0 * cross) : __longlong_as_double(0x7ff0000000000000LL);
        const double a = b.red[ki] * eta_bar;
        const double g = b.grow[ki] * eta;
        eta_next = (g < a) ? g : a;  // std::min(a, g)
        accept = eta <= eta_bar;
      }
      if (accept) {
        st->k_total += 1;
        st->t_inner += 1;
        st->accepted += 1;
        st->step_trials += st->trials_iter;
        st->ledger_kt += 1;                    // K'y of the current point
        st->ledger_k += 1 + st->trials_iter;   // Kx + one Kx' per trial
        if (st->policy == 0 && cross > 0.0 &&
            2.0 * eta * cross > movement * (1.0 + 1e-9)) {
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
                   0.5 * static_cast<double>(st->ledger_k + st->ledger_kt) >=
                       st->kkt_pass_limit) {
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
  __device__ void apply(int s, double dot, const Pre&, double (&)[K]) const { out[s] = dot; }
  __device__ void finalize(const double (&)[K]) const {}
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
  __device__ void apply(int s, double dot, const Pre& o, double (&acc)[K]) const {
    out[s] = dot;
    acc[0] += o.w * dot;
    acc[1] += dot * dot;
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
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
  __device__ void apply(int64_t i, double (&acc)[K]) const {
    if (i < n) {
      const double v = raw ? xs[i] : ref_min(ref_max(xs[i] * d2[i], l[i]), u[i]);
      xr[i] = v;
      acc[0] += c[i] * v;
      if (!isfinite(v)) acc[2] += 1.0;
    } else {
      const int64_t j = i - n;
      const double v = raw ? ys[j] : ys[j] * d1[j];
      yr[j] = v;
      acc[1] += q[j] * v;
      if (!isfinite(v)) acc[2] += 1.0;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
    result[2] = tot[2];
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
  __device__ void apply(int i, double kx, const Pre& o, double (&acc)[K]) const {
    double v = o.q - kx;
    if (i < m1) v = ref_max(v, 0.0);
    acc[0] += v * v;
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
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
  double* result;  // [3] dual_sq, bound terms, infinite-product count
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return yr; }
  struct Pre {
    double c, l, u;
  };
  __device__ Pre load(int j) const { return Pre{c[j], l[j], u[j]}; }
  __device__ void apply(int j, double kty, const Pre& o, double (&acc)[K]) const {
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
    acc[0] += d * d;
    if (lambda != 0.0) {
      const double bound = lambda > 0.0 ? lj : uj;
      if (!isfinite(bound)) {
        acc[2] += 1.0;
      } else {
        acc[1] += bound * lambda;
      }
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
    result[2] = tot[2];
  }
};

// ---------------------------------------------------------------------
// normalized_duality_gap (solver.cpp:277-370), setup of g, lo, hi over the
// n primal coordinates (columns: K'y) and the m dual ones (rows: Kx), with
// the reductions of the any-gradient test, sum g^2/w and the nu -> 0
// "bounded" corner (solver.cpp:318-342).
// acc: [0] #g!=0, [1] sum g*g/w, [2] #non-finite corner, [3] sum w*d*d,
//      [4] sum g*d
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
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return y; }
  struct Pre {
    double x, c, l, u;
  };
  __device__ Pre load(int j) const { return Pre{x[j], c[j], l[j], u[j]}; }
  __device__ void apply(int j, double kty, const Pre& o, double (&acc)[K]) const {
    const double gj = kty - o.c;
    const double loj = ref_min(0.0, o.l - o.x);
    const double hij = ref_max(0.0, o.u - o.x);
    g[j] = gj;
    lo[j] = loj;
    hi[j] = hij;
    const double w = omega;
    if (gj != 0.0) acc[0] += 1.0;
    acc[1] += gj * gj / w;
    const double d = gj > 0.0 ? hij : (gj < 0.0 ? loj : 0.0);
    if (!isfinite(d)) {
      acc[2] += 1.0;
    } else {
      acc[3] += w * d * d;
      acc[4] += gj * d;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    for (int k = 0; k < K; ++k) result[k] = tot[k];
  }
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
  double* result;
  __device__ bool prepare() { return true; }
  __device__ const double* vec() const { return x; }
  struct Pre {
    double y, q;
  };
  __device__ Pre load(int i) const { return Pre{y[i], q[i]}; }
  __device__ void apply(int i, double kx, const Pre& o, double (&acc)[K]) const {
    if (kx_out != nullptr) kx_out[i] = kx;
    const double gi = o.q - kx;
    const double loi = i < m1 ? ref_min(0.0, -o.y) : -INFINITY;
    g[i] = gi;
    lo[i] = loi;
    const double w = winv;
    if (gi != 0.0) acc[0] += 1.0;
    acc[1] += gi * gi / w;
    const double d = gi > 0.0 ? INFINITY : (gi < 0.0 ? loi : 0.0);
    if (!isfinite(d)) {
      acc[2] += 1.0;
    } else {
      acc[3] += w * d * d;
      acc[4] += gi * d;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    for (int k = 0; k < K; ++k) result[k] = tot[k];
  }
};

// Same as EpiNdgDual but with Kx already cached (the loop keeps Kx of the
// current point), so it runs elementwise without touching K.
struct OpNdgDualCached {
  static constexpr int K = 5;
  static constexpr bool kReduce = true;
  const double* kx;
  EpiNdgDual e;
  __device__ bool prepare() { return true; }
  __device__ void apply(int64_t i, double (&acc)[K]) const {
    e.apply(static_cast<int>(i), kx[i], e.load(static_cast<int>(i)), acc);
  }
  __device__ void finalize(const double (&tot)[K]) const { e.finalize(tot); }
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
  int32_t it;      // bisection iterations consumed (<= 200)
  int32_t done;
  int32_t passes;
  int32_t pad;
};

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

// One bisection pass: evaluates ||d(nu)||_w^2 and g'd(nu) for the 7 nodes of
// the next 3 bisection levels (one read of g, lo, hi), then the last CTA
// replays the reference's sequential bisection (solver.cpp:356-368) on them
// and leaves the next candidates in the state.
struct OpNdgPass {
  static constexpr int K = 2 * kNuCands;
  static constexpr bool kReduce = true;
  int64_t n, total;
  const double* g;
  const double* lo;
  const double* hi;  // primal part only; dual hi = +inf
  double omega, winv;
  NdgState* ns;

  __device__ bool prepare() { return ns->done == 0; }
  __device__ void apply(int64_t s, double (&acc)[K]) const {
    const double gs = g[s];
    const bool primal = s < n;
    const double w = primal ? omega : winv;
    const double los = lo[s];
    const double his = primal ? hi[s] : INFINITY;
    const double* nu = ns->nu;
#pragma unroll
    for (int p = 0; p < kNuCands; ++p) {
      const double unclamped = gs / (__ldg(&nu[p]) * w);  // solver.cpp:349
      const double d = ref_min(ref_max(unclamped, los), his);
      acc[2 * p] += w * d * d;
      acc[2 * p + 1] += gs * d;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    NdgState* st = ns;
    const double r = st->radius;
    const double r2 = r * r;
    double lo_ = st->nu_lo, hi_ = st->nu_hi;
    int node = 0;
    st->passes += 1;
    for (int level = 0; level < kNuLevels; ++level) {
      const double norm_sq = tot[2 * node];
      const int evaluated = node;
      st->it += 1;
      if (fabs(sqrt(norm_sq) - r) <= 1e-10 * r) {
        st->result = tot[2 * evaluated + 1] / r;
        st->done = 1;
        return;
      }
      if (norm_sq > r2) {
        lo_ = st->nu[node];
        node = 2 * node + 2;
      } else {
        hi_ = st->nu[node];
        node = 2 * node + 1;
      }
      if (st->it >= 200) {  // loop exhausted: d holds the last evaluation
        st->result = tot[2 * evaluated + 1] / r;
        st->done = 1;
        return;
      }
    }
    st->nu_lo = lo_;
    st->nu_hi = hi_;
    ndg_candidates(lo_, hi_, st->nu);
  }
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
  __device__ void apply(int64_t i, double (&acc)[K]) const {
    if (i < n) {
      const double d = xa[i] - xb[i];
      acc[0] += d * d;
    } else {
      const double d = ya[i - n] - yb[i - n];
      acc[1] += d * d;
    }
  }
  __device__ void finalize(const double (&tot)[K]) const {
    result[0] = tot[0];
    result[1] = tot[1];
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
  __device__ bool prepare() { return true; }
  __device__ void apply(int64_t i, double (&)[K]) const {
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
};

}  // namespace folpgpu
