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
constexpr int kFoldMaxJobs = 8;
constexpr int kFoldMaxFlags = 4;
constexpr int kFoldBpCap = 512;  // breakpoints per CTA range and job (beyond: folded step by step)
constexpr int kFoldIrregular = -100000;
constexpr int kFoldAfterEvent = -100001;

struct FoldBp {
  int64_t i;               // global step index
  unsigned long long c;    // N-prefix of the CTA's regular steps before step i (wrapping)
  double t;                // the term (events)
  int type;                // 1 event (real addition), 0 grid flush
  int ebefore;             // grid exponent of the regular step i-1, kFoldAfterEvent
                           // (step i-1 was a breakpoint), or kFoldFromPrev (unresolved)
  int thread;              // owner thread (phase-2 fix-up)
  int pad;
};

// One entry of a job's replay list (phase 3): S += jv (the jump over the
// regular steps since the previous entry; NaN: jv unknown, jump by `delta`
// units of S's own grid), then the entry's own operation.
struct FoldEntry {
  double jv;
  double t;
  unsigned long long delta;
  int type;                // 0 flush, 1 event, 2 dense CTA range (fold it step by step)
  int cta;                 // type 2: the CTA whose range is folded
};

// Phase timestamps of the most recent launch (globaltimer ns; diagnostics,
// folp_gpu_test_exact_fold): start, phase 1 done, grid sync done, phase 2
// done (CTA 0); ticket, lists built, replay done (last CTA).
__device__ unsigned long long g_fold_times[8];
// zero terms at undecidable sums skipped as transparent steps (1, default)
// or folded as events (0, FOLP_FOLD_SKIP_ZEROS=0: diagnostics)
__device__ int g_fold_skip_zeros = 1;
__device__ __forceinline__ unsigned long long fold_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct FoldJob {
  const double* t;
  int64_t n;
  double init;                 // the initial value (plus *init_dev when given)
  int init_from;               // -1, or an earlier job whose result / divisor is this job's init
  double init_div;
  const double* init_div_dev;  // non-null: the divisor is read here (device state)
  const double* init_dev;      // non-null (init_from < 0): init = fl(*init_dev + init)
};

// Jobs and 0/1 flag arrays of one launch; flag array f ORs into bit
// flag_group[f] of finalize's `flags`.
struct FoldJobs {
  FoldJob job[kFoldMaxJobs];
  int count;
  const double* flag[kFoldMaxFlags];
  int64_t flag_n[kFoldMaxFlags];
  int flag_group[kFoldMaxFlags];
  int nflags;
};

__device__ __forceinline__ double fold_divisor(const FoldJob& jb) {
  return jb.init_div_dev != nullptr ? __ldcg(jb.init_div_dev) : jb.init_div;
}
__device__ __forceinline__ double fold_plain_init(const FoldJob& jb) {
  return jb.init_dev != nullptr ? __ldcg(jb.init_dev) + jb.init : jb.init;
}

struct FoldScratch {
  double* cta_sum;                // [kFoldMaxJobs][cap]
  double* cta_abs;                // [kFoldMaxJobs][cap]
  unsigned long long* cta_ntot;   // [kFoldMaxJobs][cap]
  int* cta_nbp;                   // [kFoldMaxJobs][cap]  (-1 dense)
  int* cta_bad;                   // [kFoldMaxJobs][cap]
  int* cta_laste;                 // [kFoldMaxJobs][cap]  grid of the range's last step (kFoldEmpty)
  unsigned long long* cta_lastc;  // [kFoldMaxJobs][cap]  CTA-level N-prefix of its last breakpoint
  int* cta_flag;                  // [cap] flag groups non-zero in the CTA's range (bits)
  FoldBp* bps;                    // [kFoldMaxJobs][cap][kFoldBpCap]
  FoldEntry* chain;               // [kFoldMaxJobs][cap * kFoldBpCap + 1]
  double* results;                // [kFoldMaxJobs]
  unsigned* counter;              // last-CTA ticket, zero between launches
  int cap;                        // CTAs the scratch is sized for (<= kFoldMaxCtas)
};

constexpr int kFoldFromPrev = -100002;
constexpr int kFoldEmpty = -100003;
constexpr int kFoldMaxCtas = 768;  // grid cap (the last CTA's shared-memory tables)

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
// the same jump with the grid known: u(E) * d (0 when d == 0; NaN when E unknown)
__device__ __forceinline__ double fold_jv(int E, unsigned long long d) {
  if (d == 0ull) return 0.0;
  if (E < -960 || E > 1000) return __longlong_as_double(0x7ff8000000000000ll);
  return fold_pow2(E - 52) * static_cast<double>(static_cast<long long>(d));
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

// exclusive block scan of a double (approximate)
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
// exclusive block scan (wrapping u64 sum), with the total
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
// exclusive block scan of max (int), identity `none`
__device__ __forceinline__ int fold_block_exmax(int v, int none, int* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc = max(inc, o);
  }
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  int base = none;
  for (int w = 0; w < warp; ++w) base = max(base, scratch[w]);
  const int ex = __shfl_up_sync(0xffffffffu, inc, 1);
  return max(base, lane > 0 ? ex : none);
}

__device__ __forceinline__ void fold_range(int64_t n, int G, int b, int64_t& lo, int64_t& hi) {
  const int64_t R = (n + G - 1) / G;
  lo = R * b < n ? R * b : n;
  hi = lo + R < n ? lo + R : n;
}

// Phase 3 part 1 (the whole last CTA): job j's replay list from the CTAs'
// breakpoint lists -- global N-prefixes, jump values, entry order -- into
// shared memory (ejv / et / etype, `ecap` entries) or, when longer, into
// sc.chain.  Returns the entry count (every thread); *final_jv /
// *final_delta: the jump from the last entry to the end of the array.
// Few dependent global round trips: one batch of per-CTA loads, scans in
// shared memory, then one batch of breakpoint loads spread over all threads.
constexpr int kFoldPer = kFoldMaxCtas / kFoldBlock;  // CTAs per thread
constexpr int kFoldSmemPool = 2048;                  // replay entries in shared memory, all jobs
constexpr size_t kFoldDynSmem = static_cast<size_t>(kFoldSmemPool) * 17;
__device__ int fold_build_chain(int j, const FoldScratch& sc, int G, double* final_jv,
                                unsigned long long* final_delta, double* ejv, double* et,
                                unsigned char* etype, int ecap, bool* in_smem) {
  __shared__ int s_i[kFoldWarps];
  __shared__ unsigned long long s_u[kFoldWarps];
  __shared__ unsigned long long s_base[kFoldMaxCtas];
  __shared__ unsigned long long s_prevc[kFoldMaxCtas];  // C after the previous entry-holding CTA
  __shared__ unsigned long long s_lastc[kFoldMaxCtas];  // C after this CTA's last entry
  __shared__ int s_preve[kFoldMaxCtas];                 // grid before the CTA's first step
  __shared__ int s_off[kFoldMaxCtas + 1];
  __shared__ int s_nbp[kFoldMaxCtas];
  __shared__ int s_laste[kFoldMaxCtas];
  const int tid = threadIdx.x;
  const int b0 = tid * kFoldPer;
  int nb[kFoldPer], le[kFoldPer];
  unsigned long long nt[kFoldPer], lc[kFoldPer];
#pragma unroll
  for (int q = 0; q < kFoldPer; ++q) {  // one batch of loads
    const int b = b0 + q;
    const bool in = b < G;
    nb[q] = in ? __ldcg(&sc.cta_nbp[j * sc.cap + b]) : 0;
    nt[q] = in ? __ldcg(&sc.cta_ntot[j * sc.cap + b]) : 0ull;
    le[q] = in ? __ldcg(&sc.cta_laste[j * sc.cap + b]) : kFoldEmpty;
    lc[q] = in ? __ldcg(&sc.cta_lastc[j * sc.cap + b]) : 0ull;
  }
  int cnt_local = 0, def_local = -1, defe_local = -1;
  unsigned long long ntot_local = 0;
#pragma unroll
  for (int q = 0; q < kFoldPer; ++q) {
    cnt_local += nb[q] < 0 ? 1 : nb[q];
    ntot_local += nt[q];
    if (nb[q] != 0) def_local = b0 + q;
    if (le[q] != kFoldEmpty) defe_local = b0 + q;
  }
  unsigned long long tot_all, ctot;
  const unsigned long long cbase = fold_block_exscan_u64(ntot_local, s_u, &tot_all);
  const unsigned long long obase =
      fold_block_exscan_u64(static_cast<unsigned long long>(cnt_local), s_u, &ctot);
  const int prevdef = fold_block_exmax(def_local, -1, s_i);
  const int preve = fold_block_exmax(defe_local, -1, s_i);
  {
    unsigned long long cb = cbase;
    int ob = static_cast<int>(obase);
#pragma unroll
    for (int q = 0; q < kFoldPer; ++q) {
      const int b = b0 + q;
      s_base[b] = cb;
      s_off[b] = ob;
      s_nbp[b] = nb[q];
      s_laste[b] = le[q];
      s_lastc[b] = nb[q] < 0 ? cb + nt[q] : cb + lc[q];
      cb += nt[q];
      ob += nb[q] < 0 ? 1 : nb[q];
    }
    if (tid == kFoldBlock - 1) s_off[kFoldMaxCtas] = ob;
  }
  __syncthreads();
  {
    int pd = prevdef, pe = preve;
#pragma unroll
    for (int q = 0; q < kFoldPer; ++q) {
      const int b = b0 + q;
      s_prevc[b] = pd >= 0 ? s_lastc[pd] : 0ull;
      s_preve[b] = pe >= 0 ? s_laste[pe] : kFoldAfterEvent;
      if (nb[q] != 0) pd = b;
      if (le[q] != kFoldEmpty) pe = b;
    }
    if (tid == kFoldBlock - 1) {  // the jump from the last entry to the end of the array
      const unsigned long long cend = pd >= 0 ? s_lastc[pd] : 0ull;
      const int e_end = pe >= 0 ? s_laste[pe] : kFoldAfterEvent;
      const unsigned long long d = tot_all - cend;
      *final_delta = d;
      *final_jv = fold_jv(e_end, d);
    }
  }
  __syncthreads();
  const int cnt_total = static_cast<int>(ctot);
  const bool smem = cnt_total <= ecap;
  FoldEntry* out = sc.chain + static_cast<int64_t>(j) * (static_cast<int64_t>(sc.cap) * kFoldBpCap + 1);
  for (int k = tid; k < cnt_total; k += kFoldBlock) {
    // the entry's CTA: last b with s_off[b] <= k (binary search)
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= k) lo = mid; else hi = mid - 1;
    }
    const int b = lo, q = k - s_off[b];
    double jv, t = 0.0;
    unsigned long long d;
    int type;
    if (s_nbp[b] < 0) {  // dense range: jump to its start, then fold it step by step
      d = s_base[b] - s_prevc[b];
      jv = fold_jv(s_preve[b], d);
      type = 2;
    } else {
      const FoldBp* list = sc.bps + (static_cast<int64_t>(j) * sc.cap + b) * kFoldBpCap;
      const unsigned long long c = s_base[b] + __ldcg(&list[q].c);
      const unsigned long long cprev = q == 0 ? s_prevc[b] : s_base[b] + __ldcg(&list[q - 1].c);
      int e = __ldcg(&list[q].ebefore);
      if (e == kFoldFromPrev) e = s_preve[b];
      t = __ldcg(&list[q].t);
      type = __ldcg(&list[q].type);
      d = c - cprev;
      jv = fold_jv(e, d);
    }
    if (smem) {
      ejv[k] = jv;
      et[k] = t;
      etype[k] = static_cast<unsigned char>(type);
    }
    // the global entry: the whole list when it does not fit shared memory,
    // else only what the rare paths read (NaN jumps: delta; dense: cta)
    if (!smem || isnan(jv) || type == 2) out[k] = FoldEntry{jv, t, d, type, b};
  }
  *in_smem = smem;
  __syncthreads();
  return cnt_total;
}

// Phase 3 part 2 (one thread): replays job j's entry list from the exact init.
__device__ double fold_replay(const FoldJob& jb, int j, double S, const FoldScratch& sc, int G,
                              int count, double final_jv, unsigned long long final_delta,
                              const double* ejv, const double* et, const unsigned char* etype,
                              bool smem) {
  const FoldEntry* e = sc.chain + static_cast<int64_t>(j) * (static_cast<int64_t>(sc.cap) * kFoldBpCap + 1);
  if (smem) {
#pragma unroll 4
    for (int k = 0; k < count; ++k) {
      const double jv = ejv[k];
      const int type = etype[k];
      if (isnan(jv)) {
        S = fold_jump(S, __ldcg(&e[k].delta));
      } else if (jv != 0.0) {
        S = S + jv;
      }
      if (type == 1) {
        S = S + et[k];
      } else if (type == 2) {
        int64_t lo, hi;
        fold_range(jb.n, G, __ldcg(&e[k].cta), lo, hi);
        for (int64_t i = lo; i < hi; ++i) S = S + __ldcg(&jb.t[i]);
      }
    }
  } else {
    constexpr int B = 8;
    for (int k0 = 0; k0 < count; k0 += B) {
      double vj[B], vt[B];
      int vy[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        if (k0 + q < count) {
          vj[q] = __ldcg(&e[k0 + q].jv);
          vt[q] = __ldcg(&e[k0 + q].t);
          vy[q] = __ldcg(&e[k0 + q].type);
        }
      }
#pragma unroll
      for (int q = 0; q < B; ++q) {
        if (k0 + q >= count) break;
        if (isnan(vj[q])) {
          S = fold_jump(S, __ldcg(&e[k0 + q].delta));
        } else if (vj[q] != 0.0) {
          S = S + vj[q];
        }
        if (vy[q] == 1) {
          S = S + vt[q];
        } else if (vy[q] == 2) {
          int64_t lo, hi;
          fold_range(jb.n, G, __ldcg(&e[k0 + q].cta), lo, hi);
          for (int64_t i = lo; i < hi; ++i) S = S + __ldcg(&jb.t[i]);
        }
      }
    }
  }
  if (isnan(final_jv)) return fold_jump(S, final_delta);
  return final_jv != 0.0 ? S + final_jv : S;
}

// Fin::prepare() (every CTA; false = skip the launch) and
// Fin::finalize(const double* results, int count, unsigned flags) on thread
// 0 of the last CTA after every job is folded (`flags`: bit g set when a
// flag array of group g held a non-zero entry).
template <class Fin>
__global__ void __launch_bounds__(kFoldBlock) k_exact_fold(FoldJobs jobs, FoldScratch sc, Fin fin) {
  namespace cg = cooperative_groups;
  if (!fin.prepare()) return;  // every CTA agrees (loop slot disabled)
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  if (b == 0 && tid == 0) g_fold_times[0] = fold_ns();
  __shared__ double s_red[kFoldWarps];
  __shared__ unsigned long long s_u64[kFoldWarps];
  __shared__ int s_laste_t[kFoldBlock];
  __shared__ int s_nbp;
  __shared__ int s_last;
  __shared__ double s_init[kFoldMaxJobs];
  __shared__ double s_einit[kFoldMaxJobs];

  // this thread's contiguous sub-range of job j's CTA range
  auto sub = [&](int j, int64_t& a, int64_t& e) {
    int64_t lo, hi;
    fold_range(jobs.job[j].n, G, b, lo, hi);
    const int64_t r = (hi - lo + kFoldBlock - 1) / kFoldBlock;
    a = lo + r * tid < hi ? lo + r * tid : hi;
    e = a + r < hi ? a + r : hi;
  };

  // ---- phase 1: approximate sums of each CTA range ----------------------
  for (int j = 0; j < jobs.count; ++j) {
    const double* T = jobs.job[j].t;
    int64_t a, e;
    sub(j, a, e);
    double ts = 0.0, ta = 0.0;
    bool bad = false;
    for (int64_t i = a; i < e; ++i) {
      const double t = __ldcg(&T[i]);
      ts += t;
      ta += fabs(t);
      bad |= !isfinite(t);
    }
    const double cs = fold_block_sum(ts, s_red);
    const double ca = fold_block_sum(ta, s_red);
    const int nbad = __syncthreads_or(bad);
    if (tid == 0) {
      sc.cta_sum[j * sc.cap + b] = cs;
      sc.cta_abs[j * sc.cap + b] = ca;
      sc.cta_bad[j * sc.cap + b] = nbad;
    }
  }
  {
    unsigned fl = 0;
    for (int f = 0; f < jobs.nflags; ++f) {
      int64_t lo, hi;
      fold_range(jobs.flag_n[f], G, b, lo, hi);
      bool any = false;
      for (int64_t i = lo + tid; i < hi; i += kFoldBlock) any |= __ldcg(&jobs.flag[f][i]) != 0.0;
      if (any) fl |= 1u << jobs.flag_group[f];
    }
    // OR over the CTA: bits by __syncthreads_or per group (two groups at most in use)
    unsigned all = 0;
    for (int g = 0; g < 2; ++g) all |= __syncthreads_or((fl >> g) & 1u) ? (1u << g) : 0u;
    if (tid == 0) sc.cta_flag[b] = static_cast<int>(all);
  }
  if (b == 0 && tid == 0) g_fold_times[1] = fold_ns();
  cg::this_grid().sync();
  if (b == 0 && tid == 0) g_fold_times[2] = fold_ns();

  // ---- phase 2: classify, integer sums, breakpoints ----------------------
  // approximate inits (dependent jobs: source total / divisor) and their error
  if (tid < 32) {
    for (int j = 0; j < jobs.count; ++j) {
      const FoldJob& jb = jobs.job[j];
      double init = fold_plain_init(jb), einit = 0.0;
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
    int64_t a, e;
    sub(j, a, e);
    double ts = 0.0, ta = 0.0;  // this thread's sums again (cheaper than holding them)
    for (int64_t i = a; i < e; ++i) {
      const double t = __ldcg(&jb.t[i]);
      ts += t;
      ta += fabs(t);
    }
    // prefix of the preceding CTA ranges (and of their absolute values)
    double pre = 0.0, pab = 0.0;
    for (int c = tid; c < b; c += kFoldBlock) {
      pre += __ldcg(&sc.cta_sum[j * sc.cap + c]);
      pab += __ldcg(&sc.cta_abs[j * sc.cap + c]);
    }
    pre = fold_block_sum(pre, s_red);
    pab = fold_block_sum(pab, s_red);
    const double tpre = fold_block_exscan(ts, s_red);
    const double tpab = fold_block_exscan(ta, s_red);
    if (tid == 0) s_nbp = 0;
    __syncthreads();
    const double init = s_init[j];
    double P = init + pre + tpre;
    const double absend = fabs(init) + pab + tpab + ta;
    const double D = (static_cast<double>(e) + G + 2048.0) * 0x1p-51 * absend * 1.01 + s_einit[j];
    unsigned long long c = 0;
    long long N = 0;
    int Eprev = kFoldAfterEvent;  // global step 0 follows the (exact) init
    if (a > 0 && a < e) {
      const double tp = __ldcg(&jb.t[a - 1]);
      Eprev = fold_classify(P - tp, tp, D, N);
      if (Eprev == kFoldIrregular) Eprev = kFoldFromPrev;  // unknown: the owner decides
    }
    // Zero terms are transparent (fl(S + 0) == S), so an undecidable zero step
    // -- the running sum itself at or near zero, e.g. an all-zero residual or
    // the leading zeros of a cross term -- is skipped instead of recorded as
    // an event; a CTA of such steps would otherwise overflow its breakpoint
    // list and be folded step by step.  The one exception is S == -0.0 and
    // t == +0.0 (the sum becomes +0.0), possible only while every step so
    // far added -0.0 to a -0.0 init.
    const bool zpos = jb.init_from < 0 ? !(init == 0.0 && signbit(init))
                                       : fabs(init) > s_einit[j];
    // Pass 1 classifies the thread's steps: breakpoint count, N-prefix, last
    // grid; pass 2 (after the block scans) walks them again and writes the
    // breakpoints straight to their sorted place -- sub-ranges ascend with
    // the thread index, so a thread's offset is the scan of the counts (no
    // shared list, atomics or rank sort).
    const int Einit = Eprev;
    const double Pinit = P;
    bool any = false;
    int nb = 0;
    unsigned long long lastc_local = 0;
    for (int64_t i = a; i < e; ++i) {
      const double t = __ldcg(&jb.t[i]);
      const int E = fold_classify(P, t, D, N);
      if (E == kFoldIrregular && t == 0.0 && (zpos || signbit(t)) && g_fold_skip_zeros) continue;
      any = true;
      if (E == kFoldIrregular || (Eprev != kFoldAfterEvent && Eprev != E)) {
        ++nb;
        lastc_local = c;
      }
      if (E != kFoldIrregular) c += static_cast<unsigned long long>(N);
      Eprev = E == kFoldIrregular ? kFoldAfterEvent : E;
      P += t;
    }
    s_laste_t[tid] = any ? Eprev : kFoldEmpty;
    unsigned long long ctot, btot;
    const unsigned long long coff = fold_block_exscan_u64(c, s_u64, &ctot);
    const unsigned long long boff =
        fold_block_exscan_u64(static_cast<unsigned long long>(nb), s_u64, &btot);
    if (tid == 0) {
      s_nbp = -1;
      s_last = -1;
    }
    __syncthreads();
    if (any) atomicMax(&s_nbp, tid);          // the last thread with a step
    if (nb > 0) atomicMax(&s_last, tid);      // the last thread with a breakpoint
    const bool fits = btot <= static_cast<unsigned long long>(kFoldBpCap);
    FoldBp* out = sc.bps + (static_cast<int64_t>(j) * sc.cap + b) * kFoldBpCap;
    if (fits && nb > 0) {
      // the grid before the thread's first step when it was undecidable
      int eprev_thread = kFoldAfterEvent;
      if (Einit == kFoldFromPrev) {
        eprev_thread = kFoldFromPrev;
        for (int q = tid - 1; q >= 0; --q) {
          if (s_laste_t[q] != kFoldEmpty) {
            eprev_thread = s_laste_t[q];
            break;
          }
        }
      }
      P = Pinit;
      Eprev = Einit;
      unsigned long long cc = 0;
      int k = static_cast<int>(boff);
      for (int64_t i = a; i < e; ++i) {
        const double t = __ldcg(&jb.t[i]);
        const int E = fold_classify(P, t, D, N);
        if (E == kFoldIrregular && t == 0.0 && (zpos || signbit(t)) && g_fold_skip_zeros) continue;
        int bp = -1;  // -1 none, 1 event, 0 flush
        if (E == kFoldIrregular) {
          bp = 1;
        } else if (Eprev != kFoldAfterEvent && Eprev != E) {
          bp = 0;
        }
        if (bp >= 0) {
          const int eb = Eprev == kFoldFromPrev ? eprev_thread : Eprev;
          out[k++] = FoldBp{i, cc + coff, t, bp, eb, tid, 0};
        }
        if (E != kFoldIrregular) cc += static_cast<unsigned long long>(N);
        Eprev = E == kFoldIrregular ? kFoldAfterEvent : E;
        P += t;
      }
    }
    __syncthreads();
    if (tid == 0) {
      sc.cta_ntot[j * sc.cap + b] = ctot;
      sc.cta_nbp[j * sc.cap + b] = fits ? static_cast<int>(btot) : -1;
      if (s_nbp < 0) sc.cta_laste[j * sc.cap + b] = kFoldEmpty;
      if (s_last < 0 || !fits) sc.cta_lastc[j * sc.cap + b] = 0ull;
    }
    if (tid == s_nbp) sc.cta_laste[j * sc.cap + b] = s_laste_t[tid];
    if (fits && tid == s_last) sc.cta_lastc[j * sc.cap + b] = lastc_local + coff;
    __syncthreads();
  }

  // ---- phase 3: the last CTA builds the replay lists and replays them ----
  if (b == 0 && tid == 0) g_fold_times[3] = fold_ns();
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
  if (tid == 0) g_fold_times[4] = fold_ns();
  __shared__ double s_res[kFoldMaxJobs];
  __shared__ int s_count[kFoldMaxJobs];
  __shared__ int s_slow[kFoldMaxJobs];
  __shared__ double s_fjv[kFoldMaxJobs];
  __shared__ unsigned long long s_fd[kFoldMaxJobs];
  __shared__ int s_insmem[kFoldMaxJobs];
  extern __shared__ double fold_dyn[];  // kFoldDynSmem bytes: the replay lists
  const int ecap = kFoldSmemPool / jobs.count;
  double* ejv = fold_dyn;
  double* et = fold_dyn + kFoldSmemPool;
  unsigned char* ety = reinterpret_cast<unsigned char*>(fold_dyn + 2 * kFoldSmemPool);
  for (int j = 0; j < jobs.count; ++j) {
    // non-finite terms or an overflow-scale sum: the plain sequential fold
    double ab = 0.0;
    int bad = 0;
    for (int c = tid; c < G; c += kFoldBlock) {
      ab += __ldcg(&sc.cta_abs[j * sc.cap + c]);
      bad |= __ldcg(&sc.cta_bad[j * sc.cap + c]);
    }
    ab = fold_block_sum(ab, s_red);
    bad = __syncthreads_or(bad);
    const int slow = bad || !(ab + fabs(s_init[j]) < 1e300);
    int cnt = 0;
    bool in_smem = false;
    if (!slow) {
      cnt = fold_build_chain(j, sc, G, &s_fjv[j], &s_fd[j], ejv + j * ecap, et + j * ecap,
                             ety + j * ecap, ecap, &in_smem);
    }
    if (tid == 0) {
      s_count[j] = cnt;
      s_slow[j] = slow;
      s_insmem[j] = in_smem;
    }
  }
  __syncthreads();
  if (tid == 0) g_fold_times[5] = fold_ns();
  // one thread per independent job; a dependent job follows its source
  // (jobs are listed after their sources)
  const int warp = tid >> 5;
  if ((tid & 31) == 0) {
    for (int j = 0; j < jobs.count; ++j) {
      int root = j;
      while (jobs.job[root].init_from >= 0) root = jobs.job[root].init_from;
      if (root % kFoldWarps != warp) continue;
      const FoldJob& jb = jobs.job[j];
      double S = fold_plain_init(jb);
      if (jb.init_from >= 0) S = s_res[jb.init_from] / fold_divisor(jb);
      if (s_slow[j]) {
        for (int64_t i = 0; i < jb.n; ++i) S = S + __ldcg(&jb.t[i]);
      } else {
        S = fold_replay(jb, j, S, sc, G, s_count[j], s_fjv[j], s_fd[j], ejv + j * ecap,
                        et + j * ecap, ety + j * ecap, s_insmem[j] != 0);
      }
      s_res[j] = S;
      sc.results[j] = S;
    }
  }
  __syncthreads();
  if (tid == 0) g_fold_times[6] = fold_ns();
  int fl = 0;
  for (int c = tid; c < G; c += kFoldBlock) fl |= __ldcg(&sc.cta_flag[c]);
  unsigned flags = 0;
  for (int g = 0; g < 2; ++g) flags |= __syncthreads_or((fl >> g) & 1) ? (1u << g) : 0u;
  if (tid == 0) {
    fin.finalize(s_res, jobs.count, flags);
    *sc.counter = 0u;
  }
}

// ---------------------------------------------------------------------
// The same fold by ONE warp, streaming: the dot of a long segment,
//     s = 0;  for k in [k0, k1):  s = fl(s + fl(val[k] * vec[idx[k]]))
// (sparse_matrix.cpp:112-118), in chunks of 256 products staged in the
// warp's shared buffer.  The running sum S is exact at every chunk start, so
// a chunk only needs its own approximate prefixes: lane l takes products
// [8l, 8l+8), a warp scan gives its prefix, the lane classifies its steps,
// and the breakpoints (at most 2 per lane, else the chunk is folded by lane
// 0) are replayed in order by shuffles.  Returns the sequential result in
// every lane.
template <bool PROD>
__device__ __forceinline__ double warp_exact_dot(const double* __restrict__ val,
                                                 const int* __restrict__ idx,
                                                 const double* __restrict__ vec, int k0, int k1,
                                                 double* wbuf /* 256 doubles */) {
  const int lane = threadIdx.x & 31;
  double S = 0.0;
  int Elast = kFoldAfterEvent;  // grid of the previous step (exact bookkeeping)
  for (int c0 = k0; c0 < k1; c0 += 256) {
    const int len = min(256, k1 - c0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = c0 + lane + 32 * j;
      if (k < c0 + len) wbuf[k - c0] = PROD ? val[k] : val[k] * __ldg(&vec[idx[k]]);
    }
    __syncwarp();
    const int a = min(8 * lane, len), e = min(a + 8, len);
    double sl = 0.0, al = 0.0;
    bool bad = false;
    for (int i = a; i < e; ++i) {
      const double v = wbuf[i];
      sl += v;
      al += fabs(v);
      bad |= !isfinite(v);
    }
    double is = sl, ia = al;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double os = __shfl_up_sync(0xffffffffu, is, off);
      const double oa = __shfl_up_sync(0xffffffffu, ia, off);
      if (lane >= off) {
        is += os;
        ia += oa;
      }
    }
    const bool slow_chunk = __any_sync(0xffffffffu, bad) || !(fabs(S) + __shfl_sync(0xffffffffu, ia, 31) < 1e300);
    // classify this lane's steps
    double P = S + (is - sl);
    const double D = 384.0 * 0x1p-51 * (fabs(S) + ia) * 1.01;
    long long cl = 0;             // N-prefix within the lane
    int nb = 0;                   // breakpoints of this lane (<= 2 kept)
    int bpos[2] = {0, 0}, bev[2] = {0, 0}, beb[2] = {0, 0};
    long long bc[2] = {0, 0};
    int Efirst = kFoldEmpty, Eprev = kFoldEmpty;  // kFoldEmpty: before the lane's first step
    bool first_flush_pending = false;
    int first = -1;  // the lane's first non-transparent step
    if (!slow_chunk) {
      for (int i = a; i < e; ++i) {
        const double v = wbuf[i];
        long long N = 0;
        const int E = fold_classify(P, v, D, N);
        // a zero product at an undecidable sum is transparent (S starts at
        // +0.0, so S + 0 == S always holds here)
        if (E == kFoldIrregular && v == 0.0 && g_fold_skip_zeros) continue;
        if (first < 0) first = i;
        int bp = -1;
        if (E == kFoldIrregular) {
          bp = 1;
        } else if (Eprev == kFoldEmpty) {
          first_flush_pending = true;  // decided after the shuffle of the previous lane's last grid
        } else if (Eprev != kFoldAfterEvent && Eprev != E) {
          bp = 0;
        }
        if (i == first) Efirst = E == kFoldIrregular ? kFoldAfterEvent : E;
        if (bp >= 0) {
          if (nb < 2) {
            bpos[nb] = i;
            bev[nb] = bp;
            beb[nb] = Eprev;  // kFoldEmpty: the previous lane's last grid, resolved below
            bc[nb] = cl;
          }
          ++nb;
        }
        if (E != kFoldIrregular) cl += N;
        Eprev = E == kFoldIrregular ? kFoldAfterEvent : E;
        P += v;
      }
    }
    // the previous non-empty lane's last grid (or the previous chunk's)
    int Ein = Eprev;  // this lane's last grid, kFoldEmpty if no steps
    int prevE = Elast;
    {
      // exclusive "last non-empty" scan of the lanes' last grids
      int carry = Ein;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, carry, off);
        if (lane >= off && carry == kFoldEmpty) carry = o;
      }
      const int ex = __shfl_up_sync(0xffffffffu, carry, 1);
      if (lane > 0 && ex != kFoldEmpty) prevE = ex;
      const int lastlane = __shfl_sync(0xffffffffu, carry, 31);
      if (lastlane != kFoldEmpty) Elast = lastlane;  // for the next chunk
    }
    if (!slow_chunk && first_flush_pending && first >= 0) {
      // the lane's first step is regular: a flush unless the grid continues
      // (or the previous step was a breakpoint)
      if (prevE != kFoldAfterEvent && prevE != Efirst) {
        // insert at the front
        if (nb < 2) {
          bpos[1] = bpos[0]; bev[1] = bev[0]; beb[1] = beb[0]; bc[1] = bc[0];
        }
        bpos[0] = first; bev[0] = 0; beb[0] = prevE; bc[0] = 0;
        ++nb;
      }
    }
    for (int q = 0; q < 2; ++q)
      if (beb[q] == kFoldEmpty) beb[q] = prevE;
    // lane offsets of the N-prefix
    long long ic = cl;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, ic, off);
      if (lane >= off) ic += o;
    }
    const long long coff = ic - cl, ctot = __shfl_sync(0xffffffffu, ic, 31);
    if (slow_chunk || __any_sync(0xffffffffu, nb > 2)) {
      double T = S;
      if (lane == 0)
        for (int i = 0; i < len; ++i) T = T + wbuf[i];
      S = __shfl_sync(0xffffffffu, T, 0);
      if (slow_chunk) Elast = kFoldIrregular;  // unknown: the next chunk flushes, jumps by S's grid
      __syncwarp();
      continue;
    }
    // replay: lanes in order, each lane's (<= 2) breakpoints in order
    long long Cc = 0;
    unsigned mask = __ballot_sync(0xffffffffu, nb > 0);
    while (mask) {
      const int L = __ffs(mask) - 1;
      mask &= mask - 1;
      const int cnt = __shfl_sync(0xffffffffu, nb, L);
      const long long off_l = __shfl_sync(0xffffffffu, coff, L);
      for (int q = 0; q < cnt; ++q) {
        const int pos = __shfl_sync(0xffffffffu, q ? bpos[1] : bpos[0], L);
        const int ev = __shfl_sync(0xffffffffu, q ? bev[1] : bev[0], L);
        const int eb = __shfl_sync(0xffffffffu, q ? beb[1] : beb[0], L);
        const long long c = off_l + __shfl_sync(0xffffffffu, q ? bc[1] : bc[0], L);
        const unsigned long long d = static_cast<unsigned long long>(c - Cc);
        const double jv = fold_jv(eb, d);
        S = isnan(jv) ? fold_jump(S, d) : (jv != 0.0 ? S + jv : S);
        if (ev) S = S + wbuf[pos];
        Cc = c;
      }
    }
    {
      const unsigned long long d = static_cast<unsigned long long>(ctot - Cc);
      const double jv = fold_jv(Elast, d);
      S = isnan(jv) ? fold_jump(S, d) : (jv != 0.0 ? S + jv : S);
    }
    __syncwarp();
  }
  return S;
}

// Plain result sink (tests, one-off folds).
struct FoldToMemory {
  __device__ bool prepare() const { return true; }
  __device__ void finalize(const double*, int, unsigned) const {}
};

}  // namespace folpgpu
