// exactfold.cuh -- the reference's sequential fold, bit for bit, in parallel.
//
// The reference folds every reduction left to right with one IEEE rounding
// per addition (linalg.hpp:25-61; the cross term and movement of
// solver.cpp:76-88; norms, objectives and the duality-gap sums):
//     s = init;  for i in [0, n):  s = fl(s + t[i])
// Any parallel summation re-associates that and changes the last bits, and
// PDHG's adaptive step rule amplifies them (tools/noise_floor.py: 3e-5 by
// iteration 100 on config 2).  This kernel reproduces the sequential result
// EXACTLY while doing almost all the work in parallel.
//
// Why it works.  Let S_i be the sequential partial sum before step i and u
// the spacing of doubles in S_i's binade [2^E, 2^(E+1)).  If S_i and the
// exact S_i + t[i] lie in the same binade (same sign), rounding happens on
// the grid of multiples of u, S_i is on that grid, so
//     fl(S_i + t[i]) = S_i + u * N_i,   N_i = nearest integer to t[i]/u,
// and N_i does not depend on S_i (unless t[i]/u is exactly half an integer:
// a tie, whose round-to-even depends on S_i's last bit).  A run of such
// "regular" steps on one grid is therefore an exact integer sum of the N_i,
// which can be computed in any order.  Whether a step is regular only needs
// the binade of S_i, which an approximate prefix P_i decides whenever P_i is
// farther than a rigorous error bound D from every binade boundary (and from
// zero).  Every other step is a "breakpoint": an *event* (irregular step or
// tie: performed as the real floating-point addition) or a *flush* (the grid
// changes between two regular steps).
//
// Three phases, one cooperative launch:
//   1. every CTA sums its contiguous range of each job approximately (and
//      the absolute values, for D); grid-wide sync;
//   2. every thread walks its contiguous sub-range with the approximate
//      prefix P: classifies each step, accumulates the N_i of regular steps
//      (wrapping 64-bit integers -- only differences inside one segment are
//      ever used, and those are < 2^54), records breakpoints in its CTA's
//      list (sorted by index);
//   3. the last CTA to finish replays only the breakpoints, in order, with
//      the exact running sum:  S += u(S) * (C_bp - C_prev) (exact: the
//      result is the representable S_bp), then S = fl(S + t) for events.
//      A CTA whose breakpoints overflow the list is folded step by step.
// Error bound (global step i, Higham's recursive-summation bound, with a
// factor 2 of slack): |S_i - P_i| <= (i + depth) * 2^-51 * (|init| +
// sum_{k<=i} |t_k|), depth covering the scan tree.  Non-finite terms or sums
// near the overflow threshold fall back to the plain sequential fold.
//
// Used by the ordered (bit-exact) reduction mode of the PDHG loop
// (ops.cuh EpiDual::finalize_ordered) and tested in tests/test_gpu_exact_fold.py
// against a sequential fold on adversarial inputs.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace folpgpu {

constexpr int kFoldBlock = 256;
constexpr int kFoldWarps = kFoldBlock / 32;
constexpr int kFoldMaxJobs = 4;
constexpr int kFoldBpCap = 128;  // breakpoints per CTA range and job
constexpr int kFoldIrregular = -100000;
constexpr int kFoldAfterEvent = -100001;

struct FoldBp {
  int64_t i;               // global step index
  unsigned long long c;    // N-prefix of the CTA's regular steps before step i (wrapping)
  double t;                // the term (events)
  int event;               // 1 real addition, 0 grid flush
  int thread;              // owner thread (phase 2 fix-up), then unused
};

struct FoldJob {
  const double* t;
  int64_t n;
  double init;
  int init_from;     // -1, or an earlier job whose result / divisor is this job's init
  double init_div;
  const double* init_div_dev;  // non-null: the divisor is read here (device state)
};

struct FoldJobs {
  FoldJob job[kFoldMaxJobs];
  int count;
  const double* flag[2];  // 0/1 arrays OR-ed into finalize's `flagged` (non-finite iterates)
  int64_t flag_n[2];
};

__device__ __forceinline__ double fold_divisor(const FoldJob& jb) {
  return jb.init_div_dev != nullptr ? __ldcg(jb.init_div_dev) : jb.init_div;
}

struct FoldScratch {
  double* cta_sum;                // [kFoldMaxJobs][cap]
  double* cta_abs;                // [kFoldMaxJobs][cap]
  unsigned long long* cta_ntot;   // [kFoldMaxJobs][cap]
  int* cta_nbp;                   // [kFoldMaxJobs][cap]  (-1 dense)
  int* cta_bad;                   // [kFoldMaxJobs][cap]
  int* cta_flag;                  // [cap] flag arrays non-zero in the CTA's range
  FoldBp* bps;                    // [kFoldMaxJobs][cap][kFoldBpCap]
  double* results;                // [kFoldMaxJobs]
  unsigned* counter;              // last-CTA ticket, zero between launches
  int cap;                        // CTAs the scratch is sized for
};

__device__ __forceinline__ int fold_binade(double a) {  // a > 0, finite
  return static_cast<int>((__double_as_longlong(a) >> 52) & 0x7ff) - 1023;
}
__device__ __forceinline__ double fold_pow2(int e) {  // 2^e, -1022 <= e <= 1023
  return __longlong_as_double(static_cast<long long>(e + 1023) << 52);
}

// Regular-step test of step i with approximate prefix P (|P - S_i| <= D):
// returns the grid exponent E and sets N, or kFoldIrregular.
__device__ __forceinline__ int fold_classify(double P, double t, double D, long long& N) {
  const double Q = P + t;
  const double aP = fabs(P), aQ = fabs(Q);
  if (!(aP > 0.0) || !(aQ > 0.0) || !isfinite(Q) || !isfinite(D)) return kFoldIrregular;
  if ((P > 0.0) != (Q > 0.0)) return kFoldIrregular;
  const int E = fold_binade(aP);
  if (E < -960 || E > 1000) return kFoldIrregular;
  const double lo = fold_pow2(E), hi = fold_pow2(E + 1), u = fold_pow2(E - 52);
  const double d = D + 4.0 * u;  // slack for the roundings of the tests themselves
  if (aP - d < lo || aP + d >= hi) return kFoldIrregular;
  if (aQ - d < lo || aQ + d >= hi) return kFoldIrregular;
  const double r = t * fold_pow2(52 - E);  // t / u, exact (power-of-two scaling)
  if (r - floor(r) == 0.5) return kFoldIrregular;  // tie: rounding depends on S_i
  N = __double2ll_rn(r);
  return E;
}

// S + u(S) * d, exact when the true result is the representable next
// partial sum (regular steps on S's grid).
__device__ __forceinline__ double fold_jump(double S, unsigned long long d) {
  if (d == 0ull) return S;
  const int E = fold_binade(fabs(S));
  return S + fold_pow2(E - 52) * static_cast<double>(static_cast<long long>(d));
}

// block-wide sum (all threads get it); scratch >= kFoldWarps doubles
__device__ __forceinline__ double fold_block_sum(double v, double* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kFoldWarps; ++w) s += scratch[w];
  return s;
}

// exclusive block scan of a double (approximate) and a wrapping u64
__device__ __forceinline__ double fold_block_exscan(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  double base = 0.0;
  for (int w = 0; w < warp; ++w) base += scratch[w];
  return base + inc - v;
}
__device__ __forceinline__ unsigned long long fold_block_exscan_u64(unsigned long long v,
                                                                    unsigned long long* scratch,
                                                                    unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  unsigned long long base = 0, all = 0;
  for (int w = 0; w < kFoldWarps; ++w) {
    if (w < warp) base += scratch[w];
    all += scratch[w];
  }
  *total = all;
  return base + inc - v;
}

__device__ __forceinline__ void fold_range(int64_t n, int G, int b, int64_t& lo, int64_t& hi) {
  const int64_t R = (n + G - 1) / G;
  lo = R * b < n ? R * b : n;
  hi = lo + R < n ? lo + R : n;
}

// Replays one job's breakpoints (one warp; lane 0 holds the result).
__device__ double fold_chain(const FoldJob& jb, int j, double S, const FoldScratch& sc, int G) {
  const int lane = threadIdx.x & 31;
  const int64_t n = jb.n;
  // non-finite terms or an overflow-scale sum: the plain sequential fold
  bool slow = false;
  double abs_all = fabs(S);
  for (int b0 = 0; b0 < G; b0 += 32) {
    const int b = b0 + lane;
    const bool bad = b < G && __ldcg(&sc.cta_bad[j * sc.cap + b]) != 0;
    double a = b < G ? __ldcg(&sc.cta_abs[j * sc.cap + b]) : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    abs_all += a;
    if (__any_sync(0xffffffffu, bad)) slow = true;
  }
  if (slow || !(abs_all < 1e300)) {
    if (lane == 0) {
      for (int64_t i = 0; i < n; ++i) S += __ldcg(&jb.t[i]);
    }
    return __shfl_sync(0xffffffffu, S, 0);
  }
  unsigned long long Cc = 0, Cbase = 0;
  for (int b0 = 0; b0 < G; b0 += 32) {
    const int b = b0 + lane;
    const int nb = b < G ? __ldcg(&sc.cta_nbp[j * sc.cap + b]) : 0;
    const unsigned long long tot = b < G ? __ldcg(&sc.cta_ntot[j * sc.cap + b]) : 0ull;
    unsigned long long inc = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += o;
    }
    const unsigned long long base_l = Cbase + inc - tot;
    unsigned mask = __ballot_sync(0xffffffffu, nb != 0);
    while (mask) {
      const int L = __ffs(mask) - 1;
      mask &= mask - 1;
      const int bb = b0 + L;
      const unsigned long long base = __shfl_sync(0xffffffffu, base_l, L);
      const int cnt = __shfl_sync(0xffffffffu, nb, L);
      const unsigned long long tb = __shfl_sync(0xffffffffu, tot, L);
      if (cnt < 0) {  // dense CTA range: fold it step by step from the exact sum
        int64_t lo, hi;
        fold_range(n, G, bb, lo, hi);
        if (lane == 0) {
          S = fold_jump(S, base - Cc);
          for (int64_t i = lo; i < hi; ++i) S += __ldcg(&jb.t[i]);
        }
        S = __shfl_sync(0xffffffffu, S, 0);
        Cc = base + tb;
        continue;
      }
      const FoldBp* list = sc.bps + (static_cast<int64_t>(j) * sc.cap + bb) * kFoldBpCap;
      for (int k0 = 0; k0 < cnt; k0 += 32) {
        unsigned long long mc = 0;
        double mt = 0.0;
        int mev = 0;
        if (k0 + lane < cnt) {
          mc = __ldcg(&list[k0 + lane].c);
          mt = __ldcg(&list[k0 + lane].t);
          mev = __ldcg(&list[k0 + lane].event);
        }
        const int kn = cnt - k0 < 32 ? cnt - k0 : 32;
        for (int k = 0; k < kn; ++k) {
          const unsigned long long c = base + __shfl_sync(0xffffffffu, mc, k);
          const double t = __shfl_sync(0xffffffffu, mt, k);
          const int ev = __shfl_sync(0xffffffffu, mev, k);
          S = fold_jump(S, c - Cc);
          if (ev) S = S + t;
          Cc = c;
        }
      }
    }
    Cbase += __shfl_sync(0xffffffffu, inc, 31);
  }
  return fold_jump(S, Cbase - Cc);
}

// Fin::prepare() (every CTA; false = skip the launch) and
// Fin::finalize(const double* results, int count, bool flagged) on thread 0
// of the last CTA after every job is folded (`flagged`: a flag array held a
// non-zero entry).
template <class Fin>
__global__ void __launch_bounds__(kFoldBlock) k_exact_fold(FoldJobs jobs, FoldScratch sc, Fin fin) {
  namespace cg = cooperative_groups;
  if (!fin.prepare()) return;  // every CTA agrees (loop slot disabled)
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  __shared__ double s_red[kFoldWarps];
  __shared__ unsigned long long s_u64[kFoldWarps];
  __shared__ FoldBp s_bp[kFoldBpCap];
  __shared__ int s_nbp;
  __shared__ int s_last;
  __shared__ double s_init[kFoldMaxJobs];
  __shared__ double s_einit[kFoldMaxJobs];

  // ---- phase 1: approximate sums of each CTA range ----------------------
  double tsum[kFoldMaxJobs], tabs[kFoldMaxJobs];
#pragma unroll
  for (int j = 0; j < kFoldMaxJobs; ++j) {
    tsum[j] = 0.0;
    tabs[j] = 0.0;
    if (j >= jobs.count) continue;
    const FoldJob& jb = jobs.job[j];
    int64_t lo, hi;
    fold_range(jb.n, G, b, lo, hi);
    const int64_t r = (hi - lo + kFoldBlock - 1) / kFoldBlock;
    const int64_t a = lo + r * tid < hi ? lo + r * tid : hi;
    const int64_t e = a + r < hi ? a + r : hi;
    bool bad = false;
    for (int64_t i = a; i < e; ++i) {
      const double t = __ldcg(&jb.t[i]);
      tsum[j] += t;
      tabs[j] += fabs(t);
      bad |= !isfinite(t);
    }
    const double cs = fold_block_sum(tsum[j], s_red);
    const double ca = fold_block_sum(tabs[j], s_red);
    const int nbad = __syncthreads_or(bad);
    if (tid == 0) {
      sc.cta_sum[j * sc.cap + b] = cs;
      sc.cta_abs[j * sc.cap + b] = ca;
      sc.cta_bad[j * sc.cap + b] = nbad;
    }
  }
  {
    bool fl = false;
    for (int f = 0; f < 2; ++f) {
      if (jobs.flag[f] == nullptr) continue;
      int64_t lo, hi;
      fold_range(jobs.flag_n[f], G, b, lo, hi);
      for (int64_t i = lo + tid; i < hi; i += kFoldBlock) fl |= __ldcg(&jobs.flag[f][i]) != 0.0;
    }
    const int any = __syncthreads_or(fl);
    if (tid == 0) sc.cta_flag[b] = any;
  }
  cg::this_grid().sync();

  // ---- phase 2: classify, integer sums, breakpoints ----------------------
  // approximate inits (dependent jobs: source total / divisor) and their error
  if (tid < 32) {
    for (int j = 0; j < jobs.count; ++j) {
      const FoldJob& jb = jobs.job[j];
      double init = jb.init, einit = 0.0;
      if (jb.init_from >= 0) {
        const int s = jb.init_from;
        double tot = 0.0, ab = 0.0;
        for (int c = tid; c < G; c += 32) {
          tot += __ldcg(&sc.cta_sum[s * sc.cap + c]);
          ab += __ldcg(&sc.cta_abs[s * sc.cap + c]);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          tot += __shfl_xor_sync(0xffffffffu, tot, off);
          ab += __shfl_xor_sync(0xffffffffu, ab, off);
        }
        const double src_init = s_init[s];
        const double Dsrc = (static_cast<double>(jobs.job[s].n) + G + 2048.0) * 0x1p-51 *
                                (fabs(src_init) + ab) * 1.01 + s_einit[s];
        const double dv = fold_divisor(jb);
        init = (src_init + tot) / dv;
        einit = (Dsrc / fabs(dv)) * 1.01 + fabs(init) * 0x1p-50;
      }
      if (tid == 0) {
        s_init[j] = init;
        s_einit[j] = einit;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int j = 0; j < jobs.count; ++j) {
    const FoldJob& jb = jobs.job[j];
    int64_t lo, hi;
    fold_range(jb.n, G, b, lo, hi);
    // prefix of the preceding CTA ranges (and of their absolute values)
    double pre = 0.0, pab = 0.0;
    for (int c = tid; c < b; c += kFoldBlock) {
      pre += __ldcg(&sc.cta_sum[j * sc.cap + c]);
      pab += __ldcg(&sc.cta_abs[j * sc.cap + c]);
    }
    pre = fold_block_sum(pre, s_red);
    pab = fold_block_sum(pab, s_red);
    const double tpre = fold_block_exscan(tsum[j], s_red);
    const double tpab = fold_block_exscan(tabs[j], s_red);
    if (tid == 0) s_nbp = 0;
    __syncthreads();
    const int64_t r = (hi - lo + kFoldBlock - 1) / kFoldBlock;
    const int64_t a = lo + r * tid < hi ? lo + r * tid : hi;
    const int64_t e = a + r < hi ? a + r : hi;
    const double init = s_init[j];
    double P = init + pre + tpre;
    const double absend = fabs(init) + pab + tpab + tabs[j];
    const double D = (static_cast<double>(e) + G + 2048.0) * 0x1p-51 * absend * 1.01 + s_einit[j];
    unsigned long long c = 0;
    long long N = 0;
    int Eprev = kFoldAfterEvent;  // global step 0 follows the (exact) init
    if (a > 0 && a < e) {
      const double tp = __ldcg(&jb.t[a - 1]);
      Eprev = fold_classify(P - tp, tp, D, N);
    }
    for (int64_t i = a; i < e; ++i) {
      const double t = __ldcg(&jb.t[i]);
      const int E = fold_classify(P, t, D, N);
      int bp = -1;  // -1 none, 1 event, 0 flush
      if (E == kFoldIrregular) {
        bp = 1;
      } else if (Eprev != kFoldAfterEvent && Eprev != E) {
        bp = 0;
      }
      if (bp >= 0) {
        const int k = atomicAdd(&s_nbp, 1);
        if (k < kFoldBpCap) s_bp[k] = FoldBp{i, c, t, bp, tid};
      }
      if (E != kFoldIrregular) c += static_cast<unsigned long long>(N);
      Eprev = E == kFoldIrregular ? kFoldAfterEvent : E;
      P += t;
    }
    unsigned long long ctot;
    const unsigned long long coff = fold_block_exscan_u64(c, s_u64, &ctot);
    // thread offsets for the fix-up: reuse the exclusive offsets via shared memory
    __shared__ unsigned long long s_off[kFoldBlock];
    s_off[tid] = coff;
    __syncthreads();
    const int nbp = s_nbp;
    FoldBp* out = sc.bps + (static_cast<int64_t>(j) * sc.cap + b) * kFoldBpCap;
    if (nbp <= kFoldBpCap) {
      for (int k = tid; k < nbp; k += kFoldBlock) {  // rank sort by step index
        FoldBp v = s_bp[k];
        int rank = 0;
        for (int q = 0; q < nbp; ++q) rank += s_bp[q].i < v.i ? 1 : 0;
        v.c += s_off[v.thread];
        out[rank] = v;
      }
    }
    if (tid == 0) {
      sc.cta_ntot[j * sc.cap + b] = ctot;
      sc.cta_nbp[j * sc.cap + b] = nbp <= kFoldBpCap ? nbp : -1;
    }
    __syncthreads();
  }

  // ---- phase 3: the last CTA replays the breakpoints ---------------------
  __threadfence();  // every thread's breakpoint stores, before the ticket
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd(sc.counter, 1u);
    s_last = ticket == static_cast<unsigned>(G - 1) ? 1 : 0;
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (!s_last) return;
  __shared__ double s_res[kFoldMaxJobs];
  // one warp per independent job; a dependent job follows its source in the
  // source's warp (jobs are listed after their sources)
  const int warp = tid >> 5;
  for (int j = 0; j < jobs.count; ++j) {
    int root = j;
    while (jobs.job[root].init_from >= 0) root = jobs.job[root].init_from;
    if (root % kFoldWarps != warp) continue;
    const FoldJob& jb = jobs.job[j];
    double S = jb.init;
    if (jb.init_from >= 0) S = s_res[jb.init_from] / fold_divisor(jb);
    S = fold_chain(jb, j, S, sc, G);
    if ((tid & 31) == 0) {
      s_res[j] = S;
      sc.results[j] = S;
    }
    __syncwarp();
  }
  int fl = 0;
  for (int c = tid; c < G; c += kFoldBlock) fl |= __ldcg(&sc.cta_flag[c]);
  fl = __syncthreads_or(fl);
  if (tid == 0) {
    fin.finalize(s_res, jobs.count, fl != 0);
    *sc.counter = 0u;
  }
}

// ---------------------------------------------------------------------
// The same fold by ONE warp over t[0..n) (a long segment's products, in
// global memory the warp just wrote): lane l walks the contiguous block
// [l*r, (l+1)*r); approximate prefixes from a warp scan; breakpoints into
// the warp's shared buffer (unsorted, then rank-sorted); lane 0 replays.
// Returns the sequential result in every lane.  Falls back to lane 0's plain
// fold on non-finite terms, overflow-scale sums or too many breakpoints.
constexpr int kWarpBpCap = 40;  // 2 x 40 x 24 B fits the warp's 2 KB product buffer
struct WarpBp {
  int i;                   // (step index << 1) | event
  int lane;                // owner lane (its N-prefix offset is added in the replay)
  unsigned long long c;    // N-prefix within the owner lane before the step
  double t;                // the term
};
__device__ __forceinline__ double warp_exact_fold(const double* t, int n, double init,
                                                  void* smem /* >= 2*kWarpBpCap*sizeof(WarpBp)+8 */) {
  const int lane = threadIdx.x & 31;
  WarpBp* raw = reinterpret_cast<WarpBp*>(smem);
  WarpBp* sorted = raw + kWarpBpCap;
  int* counter = reinterpret_cast<int*>(sorted + kWarpBpCap);
  const int r = (n + 31) / 32;
  const int a = min(lane * r, n), e = min(a + r, n);
  double s = 0.0, ab = 0.0;
  bool bad = false;
  for (int i = a; i < e; ++i) {
    const double v = __ldcg(&t[i]);
    s += v;
    ab += fabs(v);
    bad |= !isfinite(v);
  }
  double tot_ab = ab;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tot_ab += __shfl_xor_sync(0xffffffffu, tot_ab, off);
  if (__any_sync(0xffffffffu, bad) || !(tot_ab + fabs(init) < 1e300)) {
    double S = init;
    if (lane == 0)
      for (int i = 0; i < n; ++i) S += __ldcg(&t[i]);
    return __shfl_sync(0xffffffffu, S, 0);
  }
  double is = s, ia = ab;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double os = __shfl_up_sync(0xffffffffu, is, off);
    const double oa = __shfl_up_sync(0xffffffffu, ia, off);
    if (lane >= off) {
      is += os;
      ia += oa;
    }
  }
  if (lane == 0) *counter = 0;
  __syncwarp();
  double P = init + (is - s);
  const double D = (static_cast<double>(e) + 128.0) * 0x1p-51 * (fabs(init) + ia) * 1.01;
  unsigned long long c = 0;
  long long N = 0;
  int Eprev = kFoldAfterEvent;
  if (a > 0 && a < e) {
    const double tp = __ldcg(&t[a - 1]);
    Eprev = fold_classify(P - tp, tp, D, N);
  }
  bool over = false;
  for (int i = a; i < e; ++i) {
    const double v = __ldcg(&t[i]);
    const int E = fold_classify(P, v, D, N);
    int bp = -1;
    if (E == kFoldIrregular) bp = 1;
    else if (Eprev != kFoldAfterEvent && Eprev != E) bp = 0;
    if (bp >= 0) {
      const int k = atomicAdd(counter, 1);
      if (k < kWarpBpCap) raw[k] = WarpBp{(i << 1) | bp, lane, c, v};
      else over = true;
    }
    if (E != kFoldIrregular) c += static_cast<unsigned long long>(N);
    Eprev = E == kFoldIrregular ? kFoldAfterEvent : E;
    P += v;
  }
  // lane offsets of the N-prefix
  unsigned long long ic = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, ic, off);
    if (lane >= off) ic += o;
  }
  const unsigned long long ctot = __shfl_sync(0xffffffffu, ic, 31);
  const unsigned long long coff = ic - c;
  __syncwarp();
  const int nbp = *counter;
  if (__any_sync(0xffffffffu, over) || nbp > kWarpBpCap) {
    double S = init;
    if (lane == 0)
      for (int i = 0; i < n; ++i) S += __ldcg(&t[i]);
    return __shfl_sync(0xffffffffu, S, 0);
  }
  for (int k = lane; k < nbp; k += 32) {  // rank sort; the owner's offset added by shuffle below
    const WarpBp v = raw[k];
    int rank = 0;
    for (int q = 0; q < nbp; ++q) rank += raw[q].i < v.i ? 1 : 0;
    sorted[rank] = v;
  }
  __syncwarp();
  double S = init;
  unsigned long long Cc = 0;
  for (int k0 = 0; k0 < nbp; k0 += 32) {
    WarpBp mine{};
    if (k0 + lane < nbp) mine = sorted[k0 + lane];
    // global prefix = owner lane's offset + within-lane prefix
    const unsigned long long off_owner = __shfl_sync(0xffffffffu, coff, mine.lane);
    const unsigned long long cg_ = mine.c + off_owner;
    const int kn = min(32, nbp - k0);
    for (int k = 0; k < kn; ++k) {
      const unsigned long long cc = __shfl_sync(0xffffffffu, cg_, k);
      const double tv = __shfl_sync(0xffffffffu, mine.t, k);
      const int ev = __shfl_sync(0xffffffffu, mine.i, k) & 1;
      S = fold_jump(S, cc - Cc);
      if (ev) S = S + tv;
      Cc = cc;
    }
  }
  S = fold_jump(S, ctot - Cc);
  __syncwarp();
  return S;
}

// Plain result sink (tests, one-off folds).
struct FoldToMemory {
  __device__ bool prepare() const { return true; }
  __device__ void finalize(const double*, int, bool) const {}
};

}  // namespace folpgpu
