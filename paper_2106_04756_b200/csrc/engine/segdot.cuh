// segdot.cuh -- the one sparse-product kernel family of the engine.
//
// Every K-application of the PDLP loop is a "segmented dot": for each
// segment s (a CSR row for K x, a CSC column = row of K' for K'y),
//     dot_s = sum_{k in seg s} val[k] * vec[idx[k]]
// followed by a per-segment *epilogue* that consumes dot_s in registers
// (the fused primal / dual projected step, a residual, ...) and feeds
// per-thread reduction accumulators.  Reductions are deterministic: a fixed
// block->work mapping, fixed shuffle trees, per-block partials and a
// last-block-done final pass in index order -- no floating-point atomics, so
// a rerun is bit-identical (the reference pins that in
// proj/tests/acceptance_main.cpp:653-682).
//
// Work units (built once on the host, SegPlan) -- all warp-sized, one
// stream distributed round-robin over the warps of a persistent grid of a
// few CTAs per SM (unit u runs on warp u mod warps; plans.cuh orders the
// units so every warp gets the same work):
//   tile : consecutive segments with len <= kWarpTile packed into <=
//          kWarpTile nonzeros (CSR-stream per warp).  Lane l loads entries
//          l, l+32, ... of the tile's contiguous value/index range
//          (coalesced), issues its 8 gathers back to back and parks the
//          products in a per-warp shared-memory buffer; one lane per segment
//          then sums its products sequentially in index order -- the
//          reference's own order (sparse_matrix.cpp:112-118), so these dots
//          are bit-identical -- and runs the epilogue with operands it loaded
//          before the gathers.
//   single part {-1, -(seg+2), k0, k1}: tree mode, a segment longer than
//          the serial cap (plans.cuh), reduced by the warp; its epilogue
//          feeds the warp's own accumulators (no slot, no arrival).
//   part {-(multi+1), slot, k0, k1}: a fixed chunk (kWarpTile entries;
//          kGiantPart for giant segments)
//          of a longer segment, reduced by the warp.  The last part of a
//          segment to arrive sums the part sums in part order and runs the
//          epilogue; its reduction contribution goes to a per-segment slot so
//          the final order never depends on arrival order.
// No CTA barrier outside the reduction tail: warps overlap gathering and
// reducing, which keeps the L1 gather pipe busy (random 8-byte gathers
// saturate at ~240 G/s on B200, one L1tex wavefront per lane --
// tools/microbench/spmv_ceiling.cu -- which bounds a random-pattern SpMV
// before HBM does).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "exactfold.cuh"

namespace folpgpu {

// Checked build (lib/libfolp_b200_checked.so, -DFOLP_CHECKED): device-side
// bounds and invariant checks on the products' index arithmetic -- gather
// indices inside the gathered vector, tile / part / group ranges inside
// their buffers, reduction slots inside the partials -- trapping with the
// failing line.  compute-sanitizer is closed on this GPU pool; the checked
// library runs the GPU parity cases instead (tests/test_gpu_checked.py).
#ifdef FOLP_CHECKED
#define FOLP_DCHECK(cond)                                                            \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("folp device check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define FOLP_DCHECK(cond) ((void)0)
#endif

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
#ifdef FOLP_TILE128  // A/B builds (make variant): smaller tiles, fewer registers
constexpr int kWarpTile = 128;
#else
constexpr int kWarpTile = 256;        // nonzeros per tile / part (8 per lane)
#endif
constexpr int kGiantMin = 65536;      // segments above this use kGiantPart parts
constexpr int kGiantPart = 2048;      // nnz per part of a giant segment
constexpr int kMaxAcc = 30;           // widest reduction (bisection pass)
constexpr int kSerialCap = 128;       // tree mode, large axes: longest segment one lane sums
                                      // (with degree-ordered columns: config 2 -1.6 %, config 3 -1.4 % per trial)
constexpr int kSingleMax = 1024;      // tree mode, large axes: longest one-warp segment
#ifdef FOLP_MINB
constexpr int kPlanCtasPerSm = FOLP_MINB;
#else
constexpr int kPlanCtasPerSm = 4;     // the loop products' residency (64 registers)
#endif
constexpr double kBalanceMin = 1.04;  // round-robin CTA load imbalance worth reordering
constexpr int kSegdotCarveout = 36;   // % of the unified L1 as shared memory (engine.cu)

// std::max / std::min semantics (NaN in `a` propagates), which the
// reference's projections rely on for its NonFiniteIterate detection.
__device__ __forceinline__ double ref_max(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double ref_min(double a, double b) { return (b < a) ? b : a; }

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// Release / acquire fence at GPU scope for the last-arrival patterns (store;
// fence; atomic ticket -- ticket; fence; loads).  __threadfence() is
// fence.sc.gpu, a sequentially consistent fence the patterns do not need.
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Lane-per-segment groups (SELL-32; tree mode, the loop's row products):
// 32 consecutive segments of equal length L stored interleaved -- entry j of
// the group's segment `lane` at base + 32 j + lane -- so lane l sums its
// segment in entry order while the warp's loads of one j are consecutive.
// Chosen per group when the interleaved gathers touch far fewer sectors than
// the per-segment ones (config 5's demand rows: entry j of demand row d is
// column j*D + d, so 32 neighbouring rows gather 32 consecutive x values,
// while one row alone strides by D).  A unit {-(kSellTag + g), part, j0, j1}
// covers entries [j0, j1) of all 32 segments; the last part to arrive sums
// each lane's part sums in part order and runs the epilogue, its reduction
// terms going to slot n_multi + g (deterministic, like multi-part segments).
constexpr int kSellTag = 1 << 29;
constexpr int kSellPart = 128;     // entries per lane per unit (4096 nonzeros)
constexpr int kSellGiantMin = 4096;  // CSR rows of a SELL plan above this: 2048-entry parts
struct SellPlan {
  const int* idx = nullptr;      // [32 * sum L] interleaved gather indices
  const double* val = nullptr;   // interleaved working values
  const int* base = nullptr;     // [n_groups] first interleaved entry
  const int* row0 = nullptr;     // [n_groups] first segment
  const int* nparts = nullptr;   // [n_groups]
  const int* slot0 = nullptr;    // [n_groups] first part slot (slots hold 32 sums)
  double* part_sums = nullptr;   // [total parts * 32]
  unsigned* arrivals = nullptr;  // [n_groups], zero between launches
  int n_groups = 0;
};

// One warp unit: a tile {seg0, seg1, k0, k1} (seg0 >= 0) or a part
// {-(multi+1), first_unit_of_segment, k0, k1} of multi-part segment `multi`.
struct SegPlan {
  const int* ptr;         // [S+1]
  const int* idx;         // [nnz] gather index of each entry
  int S;
  const int4* units;      // [n_units]
  int n_units;
  const int* multi_seg;   // [n_multi] segment id of each multi-part segment
  const int* multi_parts; // [n_multi] number of parts
  const int* multi_first; // [n_multi] slot of the first part (parts' slots are consecutive)
  int n_multi;
  double* part_sums;      // [n_units] (only part slots used)
  unsigned* arrivals;     // [n_multi], zero between launches
  int vec_len = 0;        // length of the gathered vector (0: unknown; staging off)
  SellPlan sell{};        // lane-per-segment groups (n_groups = 0: none)
};

// Staged gathers: when the vector an axis gathers from fits in shared memory
// (config 5's K'y gathers y: 10,000 doubles, 80 KB), each CTA copies it once
// after griddep_wait and every gather reads shared memory -- random 8-byte
// shared loads run ~2.4x the L1tex gather rate (587 vs ~240 G/s,
// profiles/r1_ceiling_cfg4.txt) and leave the L1tex pipe to the streams.
// (Staging only the hot prefix of a degree-ordered x -- config 2's 2,048
// hottest columns take 26 % of K x's gathers -- measured 56.3 -> 75.7 us per
// trial: the shared carveout it needs takes the L1 that already held that
// prefix.)
constexpr int kStageMaxBytes = 96 * 1024;
template <int STAGE>
__device__ __forceinline__ double gather(const double* __restrict__ v, const double* sv, int i) {
  if constexpr (STAGE == 1) {
    return sv[i];
  } else {
    return __ldg(&v[i]);
  }
}

struct RedBuf {
  double* partials;   // [(gridDim.x + n_multi) * K]  (capacity `cap` slots of kMaxAcc)
  unsigned* counter;  // zero between launches (reset by the last block)
  double* terms;      // ordered mode: [K * nterm] per-segment terms
  int64_t nterm;      // ordered mode: segment (element) count
  int defer = 0;      // ordered mode: only store the terms; a k_exact_fold launch
                      // folds them and runs the finalize (exactfold.cuh)
  double* scratch = nullptr;  // ordered mode: [nnz] products of long segments
                              // (warp_exact_fold); null = one lane folds them
  int cap = 0;                // partial slots allocated (checked build; 0 = unknown)
  int tree_defer = 0;         // tree mode: store the CTA partials only; the successor
                              // kernel's last CTA sums them (DeferredSums below)
};

// Reduction sinks.  Tree mode accumulates in registers (fast, deterministic
// but not the reference's summation order); ordered mode stores each
// segment's term so one thread can fold them in the reference's sequential
// order afterwards (bit-identical to the reference, used for parity runs).
template <int K>
struct TreeAcc {
  static constexpr bool kOrdered = false;
  double v[K];
  __device__ void zero() {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = 0.0;
  }
  __device__ __forceinline__ void add(int k, int64_t, double x) { v[k] += x; }
};

template <int K>
struct OrderedAcc {
  static constexpr bool kOrdered = true;
  double* terms;
  int64_t nterm;
  __device__ void zero() {}
  __device__ __forceinline__ void add(int k, int64_t seg, double x) {
    terms[k * nterm + seg] = x;
  }
};

// fold(init, t[0..n)) in index order, one thread
__device__ __forceinline__ double fold(double init, const double* t, int64_t n) {
  double s = init;
  for (int64_t i = 0; i < n; ++i) s += ld_cg(&t[i]);
  return s;
}
__device__ __forceinline__ bool any_nonzero(const double* t, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (ld_cg(&t[i]) != 0.0) return true;
  return false;
}

// Sum over the CTA; result valid in thread 0.  Ends with a barrier so the
// scratch can be reused immediately.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += scratch[w];
  }
  __syncthreads();
  return s;
}

template <int K>
__device__ __forceinline__ void block_sum_vec(double (&acc)[K], double (*scratch)[K],
                                              double (&out)[K]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) scratch[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += scratch[w][k];
      out[k] = s;
    }
  }
  __syncthreads();
}

// Ordered mode: after every CTA stored its terms, the last CTA's thread 0
// folds them (epi.finalize_ordered).
template <class Epi>
__device__ __forceinline__ void ordered_tail(const Epi& epi, RedBuf rb) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned ticket = atomicAdd(rb.counter, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    epi.finalize_ordered(rb.terms, rb.nterm);
    *rb.counter = 0u;
  }
}

// Per-warp timeline of the loop products (diagnostic build, -DFOLP_WARP_TIMES):
// globaltimer at warp start, after its last unit, and at kernel exit, for
// the most recent launch of each traced epilogue (Epi::kTrace = 0 / 1).
constexpr int kTraceWarps = 16384;
#ifdef FOLP_WARP_TIMES
__device__ unsigned long long g_warp_times[2][kTraceWarps][4];  // + work word
__device__ unsigned long long g_tail_times[2][4];  // last CTA: ticket, sums, finalize, end
#endif
template <class E, class = void>
struct TraceSlot { static constexpr int v = -1; };
template <class E>
struct TraceSlot<E, std::void_t<decltype(E::kTrace)>> { static constexpr int v = E::kTrace; };
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
template <class Epi>
__device__ __forceinline__ void trace_tail(int which) {
#ifdef FOLP_WARP_TIMES
  constexpr int slot = TraceSlot<Epi>::v;
  if constexpr (slot >= 0) {
    if (threadIdx.x == 0) g_tail_times[slot][which] = global_ns();
  }
#else
  (void)which;
#endif
}
template <class Epi>
__device__ __forceinline__ void trace_warp(int which, unsigned long long t) {
#ifdef FOLP_WARP_TIMES
  constexpr int slot = TraceSlot<Epi>::v;
  if constexpr (slot >= 0) {
    const int w = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0 && w < kTraceWarps) g_warp_times[slot][w][which] = t;
  }
#else
  (void)which;
  (void)t;
#endif
}

// Epilogues whose finalize runs the loop's step decision on the device
// state (EpiDual) expose it as kStateWords 8-byte words: the last CTA loads
// them into shared memory with all its threads while it sums the partials,
// decides on the shared copy and writes it back -- a dozen dependent global
// round trips of one thread cost ~2.4 us per trial (tools/warp_timeline.py).
template <class E, class = void>
struct StateTail { static constexpr int words = 0; };
template <class E>
struct StateTail<E, std::void_t<decltype(E::kStateWords)>> {
  static constexpr int words = E::kStateWords;
};

// The final pass over the per-CTA partials (np slots of K values): a fixed
// thread -> slot mapping and tree, so the totals depend on the partials and
// np alone.  Result valid in thread 0.
template <int K>
__device__ __forceinline__ void sum_partials(const double* partials, int np, double (*s_vec)[K],
                                             double (&tot)[K]) {
  double part[K];
#pragma unroll
  for (int k = 0; k < K; ++k) part[k] = 0.0;
  // all of a thread's loads in flight at once (same per-thread order)
  constexpr int R = K <= 3 ? 4 : 2;
  for (int base = threadIdx.x; base < np; base += kBlock * R) {
    double v[R][K];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = base + r * kBlock;
#pragma unroll
      for (int k = 0; k < K; ++k) v[r][k] = i < np ? ld_cg(&partials[i * K + k]) : 0.0;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (base + r * kBlock < np) {
#pragma unroll
        for (int k = 0; k < K; ++k) part[k] += v[r][k];
      }
    }
  }
  block_sum_vec<K>(part, s_vec, tot);
}

// Deferred sums: a kernel whose totals only its successor's decision needs
// (kernel A's sum omega dx^2 and non-finite flag, consumed by kernel B's
// step rule) stores its CTA partials and exits -- no ticket, no last-CTA
// pass, so its successor's griddepcontrol.wait releases that much earlier.
// The successor's highest-numbered CTA sums them at its START with the same
// sum_partials (same bits) and stores the totals where the decision reads
// them -- under the product, not in its serial tail; the store precedes that
// CTA's own arrival ticket, so the last CTA's acquire covers it.  An
// epilogue that consumes such sums provides
//   static constexpr int kDeferredK;  const double* deferred_partials() const;
//   int deferred_np() const;  void store_deferred(const double (&)[kDeferredK]) const;
template <class E, class = void>
struct DeferredSums { static constexpr int k = 0; };
template <class E>
struct DeferredSums<E, std::void_t<decltype(E::kDeferredK)>> { static constexpr int k = E::kDeferredK; };
template <class Epi>
__device__ __forceinline__ void absorb_deferred_sums(const Epi& epi) {
  constexpr int DK = DeferredSums<Epi>::k;
  if constexpr (DK > 0) {
    if (blockIdx.x == gridDim.x - 1 && epi.deferred_partials() != nullptr) {  // CTA-uniform
      __shared__ double s_dvec[kWarps][DK];
      double dtot[DK];
      sum_partials<DK>(epi.deferred_partials(), epi.deferred_np(), s_dvec, dtot);
      if (threadIdx.x == 0) epi.store_deferred(dtot);
    }
  }
}

// Per-block partial + last-block-done final reduction, then epi.finalize().
template <class Epi>
__device__ __forceinline__ void reduce_tail(const Epi& epi, double (&acc)[Epi::K], RedBuf rb,
                                            int n_extra) {
  constexpr int K = Epi::K;
  __shared__ double s_vec[kWarps][K];
  __shared__ int s_last;
  double tot[K];
  block_sum_vec<K>(acc, s_vec, tot);
  FOLP_DCHECK(rb.cap == 0 || static_cast<int>(gridDim.x) + n_extra <= rb.cap);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) rb.partials[blockIdx.x * K + k] = tot[k];
    if (rb.tree_defer) {
      s_last = 0;  // the successor kernel sums the partials
    } else {
      fence_acq_rel();
      const unsigned ticket = atomicAdd(rb.counter, 1u);
      s_last = (ticket == gridDim.x - 1) ? 1 : 0;
      if (s_last) fence_acq_rel();  // acquire; the barrier below extends it to the CTA
    }
  }
  __syncthreads();
  if (!s_last) return;
  trace_tail<Epi>(0);
  constexpr int SW = StateTail<Epi>::words;
  __shared__ unsigned long long s_state[SW > 0 ? SW : 1];
  __shared__ double s_rg[2];
  if constexpr (SW > 0) {
    if (threadIdx.x < SW) s_state[threadIdx.x] = __ldcg(epi.state_words() + threadIdx.x);
    if (threadIdx.x == kBlock - 1) epi.tail_aux(s_rg);
  }
  const int np = static_cast<int>(gridDim.x) + n_extra;
  sum_partials<K>(rb.partials, np, s_vec, tot);
  trace_tail<Epi>(1);
  if (threadIdx.x == 0) {
    if constexpr (SW > 0) {
      epi.finalize_state(tot, s_state, s_rg);
    } else {
      epi.finalize(tot);
    }
    trace_tail<Epi>(2);
    *rb.counter = 0u;
  }
  if constexpr (SW > 0) {
    __syncthreads();
    if (threadIdx.x < SW) epi.state_words()[threadIdx.x] = s_state[threadIdx.x];
  }
}

// Two-phase products (gathered vector and products L2-resident): phase 1
// streams the whole axis once, prod[k] = val[k] * vec[idx[k]], with nothing
// but independent gathers in flight (4 per thread per step, 16-byte stream
// loads); phase 2 is segdot_kernel<..., PROD=true>, which reads prod[k] as a
// coalesced stream instead of gathering.  In the single-pass kernel every
// dependent load of a warp unit (indices -> gathers -> epilogue) waits
// behind the SM's whole L1tex gather queue; split, the gathers run at the
// queue's rate and phase 2's loads see a short queue.  Same products, same
// summation order: bit-identical to the single-pass kernel.
template <class Epi>
__global__ void __launch_bounds__(kBlock)
gather_products_kernel(const int* __restrict__ idx, const double* __restrict__ val,
                       int64_t nnz, double* __restrict__ out, Epi epi) {
  if (!epi.prepare()) return;
  const double* __restrict__ vec = epi.vec();
  const int64_t nq = nnz >> 2;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kBlock;
  const int4* __restrict__ idx4 = reinterpret_cast<const int4*>(idx);
  const double2* __restrict__ val2 = reinterpret_cast<const double2*>(val);
  double2* __restrict__ out2 = reinterpret_cast<double2*>(out);
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; q < nq; q += stride) {
    const int4 i = __ldcs(&idx4[q]);
    const double2 a = __ldcs(&val2[2 * q]);
    const double2 b = __ldcs(&val2[2 * q + 1]);
    const double g0 = __ldg(&vec[i.x]), g1 = __ldg(&vec[i.y]);
    const double g2 = __ldg(&vec[i.z]), g3 = __ldg(&vec[i.w]);
    out2[2 * q] = make_double2(a.x * g0, a.y * g1);
    out2[2 * q + 1] = make_double2(b.x * g2, b.y * g3);
  }
  if (blockIdx.x == 0 && threadIdx.x < (nnz & 3)) {
    const int64_t k = (nq << 2) + threadIdx.x;
    out[k] = val[k] * __ldg(&vec[idx[k]]);
  }
}

// The segmented-dot kernel.
// PROD: `val` holds the products val[k] * vec[idx[k]] (phase 2 above).
// Epi must provide:  static constexpr int K (>= 1); static constexpr bool
//   kReduce (run the reduction tail); __device__ bool prepare();
//   __device__ const double* vec() const;
//   struct Pre (epilogue operands of one segment, independent of the dot);
//   __device__ Pre load(int seg) const;
//   __device__ void apply(int seg, double dot, const Pre&, double (&acc)[K]) const;
//   __device__ void finalize(const double (&tot)[K]) const;
// Programmatic dependent launch (the PDHG loop's kernels, FOLP_PDL): a
// kernel launched with programmatic stream serialization starts while its
// predecessor drains; griddepcontrol.wait blocks until the predecessor grid
// has completed and its memory is visible (a no-op without the attribute).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// L2 prefetch of a warp unit's static streams (values, indices, segment
// bounds): issued before griddep_wait, so the first unit's stream loads
// overlap the predecessor's tail.
__device__ __forceinline__ void prefetch_unit(const SegPlan& p, const double* val, int4 d, int lane) {
  const int k0 = d.z, k1 = d.w;
  if (k1 <= k0) return;
  const char* vb = reinterpret_cast<const char*>(val + k0);
  const char* ib = reinterpret_cast<const char*>(p.idx + k0);
  const int vlines = ((k1 - k0) * 8 + 127) / 128 + 1;
  const int ilines = ((k1 - k0) * 4 + 127) / 128 + 1;
  if (lane < vlines && lane < 20) asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + 128 * lane));
  if (lane >= 20 && lane - 20 < ilines && lane < 30) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ib + 128 * (lane - 20)));
  }
  if (lane == 31 && d.x >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.ptr + d.x));
}

template <class Epi, bool ORDERED, bool PROD = false, int STAGE = 0, bool SELLU = false>
#ifdef FOLP_WARP_TIMES
#define FOLP_SEGDOT_BOUNDS __launch_bounds__(kBlock, kPlanCtasPerSm)  // same residency as the product build
#else
#ifdef FOLP_MINB  // A/B builds: CTAs per SM the compiler must fit
#define FOLP_SEGDOT_BOUNDS __launch_bounds__(kBlock, FOLP_MINB)
#else
#define FOLP_SEGDOT_BOUNDS __launch_bounds__(kBlock)
#endif
#endif
__global__ void FOLP_SEGDOT_BOUNDS
segdot_kernel(SegPlan p, const double* __restrict__ val, Epi epi, RedBuf rb) {
  constexpr int K = Epi::K;
  {
    const int u0 = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (u0 < p.n_units) prefetch_unit(p, val, p.units[u0], threadIdx.x & 31);
  }
  griddep_wait();
  griddep_launch();            // the successor may start filling freed SMs
  if (!epi.prepare()) return;  // loop slot disabled: every CTA agrees
  if constexpr (!ORDERED) absorb_deferred_sums(epi);
#ifdef FOLP_WARP_TIMES
  trace_warp<Epi>(0, global_ns());
#endif
  const double* __restrict__ vec = epi.vec();
  extern __shared__ double s_stage[];
  if constexpr (STAGE != 0) {
    const int X = p.vec_len;
    if ((reinterpret_cast<uintptr_t>(vec) & 15) == 0) {
      const double2* v2 = reinterpret_cast<const double2*>(vec);
      double2* s2 = reinterpret_cast<double2*>(s_stage);
      for (int i = threadIdx.x; i < (X >> 1); i += kBlock) s2[i] = __ldcg(&v2[i]);
      if (threadIdx.x == 0 && (X & 1)) s_stage[X - 1] = __ldcg(&vec[X - 1]);
    } else {
      for (int i = threadIdx.x; i < X; i += kBlock) s_stage[i] = __ldcg(&vec[i]);
    }
    __syncthreads();
  }
  const int* __restrict__ idx = p.idx;
  const int* __restrict__ ptr = p.ptr;
  __shared__ double s_prod[kWarps][kWarpTile];

  using Acc = std::conditional_t<ORDERED, OrderedAcc<K>, TreeAcc<K>>;
  Acc acc;
  if constexpr (ORDERED) {
    acc.terms = rb.terms;
    acc.nterm = rb.nterm;
  }
  acc.zero();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* wbuf = s_prod[warp];
  const int nw = static_cast<int>(gridDim.x) * kWarps;

  // The next unit's descriptor is loaded one unit ahead: every dependent
  // load waits behind the SM's whole gather queue, so the descriptor ->
  // indices -> gathers chain is cut to indices -> gathers.  (Prefetching the
  // index stream too -- in registers or by cp.async -- costs occupancy or
  // data-pipe wavefronts and measured slower: profiles/r1_segpipe_experiments.md.)
  int u = blockIdx.x * kWarps + warp;
  int4 d_next = u < p.n_units ? p.units[u] : make_int4(0, 0, 0, 0);
#ifdef FOLP_WARP_TIMES
  unsigned long long work = 0;  // nnz | parts << 24 | tile segments << 36 | smid << 52
#endif
  for (; u < p.n_units; u += nw) {
    const int4 d = d_next;
    if (u + nw < p.n_units) d_next = p.units[u + nw];
    const int k0 = d.z, k1 = d.w;
#ifdef FOLP_WARP_TIMES
    work += static_cast<unsigned long long>(k1 - k0) +
            (d.x < 0 ? (1ull << 24) : (static_cast<unsigned long long>(d.y - d.x) << 36));
#endif
    if constexpr (ORDERED) {  // (tree plans split long segments into parts)
      if (d.x >= 0 && k1 - k0 > kWarpTile) {
        // ordered plan: one long segment, its dot the reference's sequential
        // sum in index order -- by the whole warp through the exact fold
        // (products staged in rb.scratch), or by one lane
        if (rb.scratch != nullptr) {
          const double sum = warp_exact_dot<PROD>(val, idx, vec, k0, k1, wbuf);
          if (lane == 0) epi.apply(d.x, sum, epi.load(d.x), acc);
          __syncwarp();
        } else if (lane == 0) {
          double sum = 0.0;
          for (int k = k0; k < k1; ++k) sum += PROD ? val[k] : val[k] * vec[idx[k]];
          epi.apply(d.x, sum, epi.load(d.x), acc);
        }
        continue;
      }
    }
    if (d.x >= 0) {
      // ---------------- tile of short segments ----------------
      const int seg0 = d.x, seg1 = d.y;
      FOLP_DCHECK(seg0 <= seg1 && seg1 <= p.S && k1 - k0 <= kWarpTile && k0 <= k1);
      const int s_first = seg0 + lane;
      int b_first = 0, e_first = 0;
      typename Epi::Pre pre_first{};
      if (s_first < seg1) {
        b_first = ptr[s_first];
        e_first = ptr[s_first + 1];
        pre_first = epi.load(s_first);  // in flight with the tile's loads
      }
      double prod[kWarpTile / 32];
#pragma unroll
      for (int j = 0; j < kWarpTile / 32; ++j) {
        const int k = k0 + lane + 32 * j;
        FOLP_DCHECK(k >= k1 || p.vec_len == 0 || (idx[k] >= 0 && idx[k] < p.vec_len));
        if constexpr (PROD) {
          prod[j] = k < k1 ? val[k] : 0.0;
        } else {
          prod[j] = k < k1 ? val[k] * gather<STAGE>(vec, s_stage, idx[k]) : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < kWarpTile / 32; ++j) {
        const int k = k0 + lane + 32 * j;
        if (k < k1) wbuf[k - k0] = prod[j];
      }
      __syncwarp();
      for (int s = s_first; s < seg1; s += 32) {
        int b = b_first, e = e_first;
        typename Epi::Pre pre = pre_first;
        if (s != s_first) {
          b = ptr[s];
          e = ptr[s + 1];
          pre = epi.load(s);
        }
        double sum = 0.0;
        FOLP_DCHECK(b >= k0 && e <= k1 && b <= e);
        for (int k = b; k < e; ++k) sum += wbuf[k - k0];
        epi.apply(s, sum, pre, acc);
      }
      __syncwarp();
    } else if (SELLU && d.x <= -kSellTag) {
      // ---------------- lane-per-segment group part (SELL-32) ----------------
      const SellPlan& q = p.sell;
      const int g = -d.x - kSellTag;
      FOLP_DCHECK(g >= 0 && g < q.n_groups && d.z <= d.w);
      FOLP_DCHECK(rb.cap == 0 || static_cast<int>(gridDim.x) + p.n_multi + g < rb.cap);
      const int np = q.nparts[g];
      FOLP_DCHECK(d.y >= 0 && d.y < np);
      const int row = q.row0[g] + lane;
      const int base = q.base[g];
      typename Epi::Pre pre_one{};
      if (np == 1) pre_one = epi.load(row);  // in flight with the gathers
      // the group's reduction terms always go to its slot (a single-part
      // group too: the tail sums every group slot)
      auto finish = [&](double total, const typename Epi::Pre& pre) {
        TreeAcc<K> macc;
        macc.zero();
        epi.apply(row, total, pre, macc);
        if constexpr (Epi::kReduce) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            double v = macc.v[k];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) rb.partials[(gridDim.x + p.n_multi + g) * K + k] = v;
          }
        }
      };
      double sum = 0.0;
      {
        const int* __restrict__ qi = q.idx + base + lane;
        const double* __restrict__ qv = q.val + base + lane;
        int j = d.z;
        for (; j + 8 <= d.w; j += 8) {  // 8 independent loads per lane in flight
          int ix[8];
          double v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            ix[t] = qi[32 * (j + t)];
            v[t] = qv[32 * (j + t)];
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) sum += v[t] * gather<STAGE>(vec, s_stage, ix[t]);
        }
        for (; j < d.w; ++j) sum += qv[32 * j] * gather<STAGE>(vec, s_stage, qi[32 * j]);
      }
      if (np == 1) {
        finish(sum, pre_one);
      } else {
        const int slot = q.slot0[g] + d.y;
        q.part_sums[slot * 32 + lane] = sum;
        fence_acq_rel();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(&q.arrivals[g], 1u) == static_cast<unsigned>(np - 1) ? 1u : 0u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          fence_acq_rel();
          double total = 0.0;
          for (int pp = 0; pp < np; ++pp) total += ld_cg(&q.part_sums[(q.slot0[g] + pp) * 32 + lane]);
          finish(total, epi.load(row));
          if (lane == 0) q.arrivals[g] = 0u;
        }
      }
    } else if constexpr (!ORDERED) {
      // ---------------- part of a long segment ----------------
      const int multi = -d.x - 1;
      const bool single = d.y < 0;
      FOLP_DCHECK(single ? (-d.y - 2 < p.S) : (multi < p.n_multi && d.y < p.n_units));
      FOLP_DCHECK(single || rb.cap == 0 || static_cast<int>(gridDim.x) + multi < rb.cap);
      typename Epi::Pre pre_single{};
      if (single && lane == 0) pre_single = epi.load(-d.y - 2);  // in flight with the gathers
      double sum = 0.0;
#pragma unroll 8
      for (int k = k0 + lane; k < k1; k += 32) {
        FOLP_DCHECK(PROD || p.vec_len == 0 || (idx[k] >= 0 && idx[k] < p.vec_len));
        if constexpr (PROD) {
          sum += val[k];
        } else {
          sum += val[k] * gather<STAGE>(vec, s_stage, idx[k]);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off);
      if (single) {
        if (lane == 0) epi.apply(-d.y - 2, sum, pre_single, acc);
      } else {
        int np = 0;
        unsigned last = 0;
        if (lane == 0) {
          p.part_sums[d.y] = sum;
          fence_acq_rel();
          np = p.multi_parts[multi];
          last = atomicAdd(&p.arrivals[multi], 1u) == static_cast<unsigned>(np - 1) ? 1u : 0u;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          // The last part to arrive sums the segment's part sums with the
          // whole warp: lane l takes parts l, l + 32, ... in order, then a
          // fixed shuffle tree (deterministic, arrival order never matters).
          // One lane walking config 3's 977-part row alone was the kernel's
          // last straggler: units done p99 113 us, p100 148 us.
          np = __shfl_sync(0xffffffffu, np, 0);
          fence_acq_rel();
          const int first = p.multi_first[multi];
          double total = 0.0;
          for (int q = lane; q < np; q += 32) total += ld_cg(&p.part_sums[first + q]);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) total += __shfl_down_sync(0xffffffffu, total, off);
          if (lane == 0) {
            const int seg = p.multi_seg[multi];
            TreeAcc<K> macc;
            macc.zero();
            epi.apply(seg, total, epi.load(seg), macc);
            if constexpr (Epi::kReduce) {
#pragma unroll
              for (int k = 0; k < K; ++k) rb.partials[(gridDim.x + multi) * K + k] = macc.v[k];
            }
            p.arrivals[multi] = 0u;
          }
        }
      }
    }
  }
#ifdef FOLP_WARP_TIMES
  trace_warp<Epi>(1, global_ns());
  {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    trace_warp<Epi>(3, work | (static_cast<unsigned long long>(smid) << 52));
  }
#endif
  if constexpr (Epi::kReduce) {
    if constexpr (ORDERED) {
      if (!rb.defer) ordered_tail(epi, rb);
    } else {
      reduce_tail(epi, acc.v, rb, p.n_multi + p.sell.n_groups);
    }
  }
#ifdef FOLP_WARP_TIMES
  trace_warp<Epi>(2, global_ns());
#endif
}

// Two-entry segments, one thread per segment (tree mode, the loop's
// products).  An axis whose every segment holds exactly two entries -- the
// columns of a node-arc incidence matrix: transportation, assignment and
// network-flow LPs; config 5 has 16M of them -- needs no unit plan, segment
// bounds or shared memory: segment s owns entries 2s and 2s+1, so a thread
// reads its indices as one int2 and its values as one double2 (consecutive
// threads, consecutive 8 / 16 bytes), and the kernel is a stream of
// independent loads, two segments per thread in flight.  Through the warp
// tiles the same axis ran at 57 % of the HBM peak: a lane owned four
// segments of a 128-segment tile one after the other, each with its own
// dependent operand loads behind the tile's shared-memory round trip.
// The dot is 0 + p0 + p1 in entry order, as in the tiles (bit-identical).
// The first round's entries are static data and are loaded BEFORE
// griddepcontrol.wait, under the predecessor's tail.  Plain read-only loads:
// evict-first (ld.global.cs) streams measured 466 vs 424 us per config-5
// trial, a 256-byte L2 prefetch hint, 4 or 8 CTAs per SM and a 2.7x larger
// grid no change (profiles/r2_experiments_s4.md).
template <class Epi>
__global__ void __launch_bounds__(kBlock)
pair_kernel(int S, const int* __restrict__ idx, const double* __restrict__ val, int vec_len, Epi epi,
            RedBuf rb) {
  constexpr int K = Epi::K;
  const int2* __restrict__ idx2 = reinterpret_cast<const int2*>(idx);
  const double2* __restrict__ val2 = reinterpret_cast<const double2*>(val);
  const int stride = static_cast<int>(gridDim.x) * kBlock;
  int s = static_cast<int>(blockIdx.x) * kBlock + threadIdx.x;
  int2 ia = make_int2(0, 0), ib = make_int2(0, 0);
  double2 va = make_double2(0.0, 0.0), vb = make_double2(0.0, 0.0);
  if (s < S) {
    ia = __ldg(&idx2[s]);
    va = __ldg(&val2[s]);
  }
  if (s < S - stride) {
    ib = __ldg(&idx2[s + stride]);
    vb = __ldg(&val2[s + stride]);
  }
  griddep_wait();
  griddep_launch();
  if (!epi.prepare()) return;
  absorb_deferred_sums(epi);
  const double* __restrict__ vec = epi.vec();
  TreeAcc<K> acc;
  acc.zero();
  (void)vec_len;
  for (; s < S; s += 2 * stride) {
    const bool two = s < S - stride;
    const typename Epi::Pre pa = epi.load(s);
    typename Epi::Pre pb{};
    if (two) pb = epi.load(s + stride);
    FOLP_DCHECK(vec_len == 0 || (ia.x >= 0 && ia.x < vec_len && ia.y >= 0 && ia.y < vec_len));
    FOLP_DCHECK(!two || vec_len == 0 || (ib.x >= 0 && ib.x < vec_len && ib.y >= 0 && ib.y < vec_len));
    const double ga0 = __ldg(&vec[ia.x]), ga1 = __ldg(&vec[ia.y]);
    double gb0 = 0.0, gb1 = 0.0;
    if (two) {
      gb0 = __ldg(&vec[ib.x]);
      gb1 = __ldg(&vec[ib.y]);
    }
    // the next round's entries, in flight across this round's epilogues
    const int sn = s + 2 * stride;
    int2 na = make_int2(0, 0), nb = make_int2(0, 0);
    double2 wa = make_double2(0.0, 0.0), wb = make_double2(0.0, 0.0);
    if (sn < S) {
      na = __ldg(&idx2[sn]);
      wa = __ldg(&val2[sn]);
    }
    if (sn < S - stride) {
      nb = __ldg(&idx2[sn + stride]);
      wb = __ldg(&val2[sn + stride]);
    }
    double dot = 0.0;
    dot += va.x * ga0;
    dot += va.y * ga1;
    epi.apply(s, dot, pa, acc);
    if (two) {
      dot = 0.0;
      dot += vb.x * gb0;
      dot += vb.y * gb1;
      epi.apply(s + stride, dot, pb, acc);
    }
    ia = na;
    ib = nb;
    va = wa;
    vb = wb;
  }
  if constexpr (Epi::kReduce) reduce_tail(epi, acc.v, rb, 0);
}

// A warp's unit of one plan held in registers for a whole chunk (small
// problems: every warp of the cluster owns at most one unit per product, so
// its descriptor, index stream, values and segment bounds never change
// between trials and only the gathers and epilogue operands are loaded).
struct ResidentUnit {
  int4 d;
  int b, e;  // this lane's segment bounds (tiles)
  int ix[kWarpTile / 32];
  double v[kWarpTile / 32];
};

__device__ __forceinline__ void load_resident(const SegPlan& p, const double* __restrict__ val,
                                              int u, int lane, ResidentUnit& r) {
  r.d = u < p.n_units ? p.units[u] : make_int4(0, 0, 0, 0);
  r.b = r.e = 0;
#pragma unroll
  for (int j = 0; j < kWarpTile / 32; ++j) {
    const int k = r.d.z + lane + 32 * j;
    r.ix[j] = k < r.d.w ? p.idx[k] : 0;
    r.v[j] = k < r.d.w ? val[k] : 0.0;
  }
  if (r.d.x >= 0 && r.d.x + lane < r.d.y) {
    r.b = p.ptr[r.d.x + lane];
    r.e = p.ptr[r.d.x + lane + 1];
  }
}

// One product by a thread-block cluster from resident units (at most one per
// warp); the CTA's partial sums go to CTA 0's `parts[rank]` (distributed
// shared memory), folded there in rank order.
template <int NT, class Epi>
__device__ void cluster_product(const SegPlan& p, const ResidentUnit& r, int u, const Epi& epi,
                                int rank, double* wbuf, double (*scratch)[kMaxAcc],
                                double* multi_out, double* parts0) {
  constexpr int K = Epi::K;
  constexpr int NW = NT / 32;
  constexpr int J = kWarpTile / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* __restrict__ vec = epi.vec();
  TreeAcc<K> acc;
  acc.zero();
  const int4 d = r.d;
  if (u < p.n_units && d.x >= 0) {
    // tile: gathers and this lane's operands in one round
    const int s_first = d.x + lane;
    typename Epi::Pre pre_first{};
    if (s_first < d.y) pre_first = epi.load(s_first);
    double prod[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = d.z + lane + 32 * j;
      prod[j] = k < d.w ? r.v[j] * __ldg(&vec[r.ix[j]]) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = d.z + lane + 32 * j;
      if (k < d.w) wbuf[k - d.z] = prod[j];
    }
    __syncwarp();
    for (int s = s_first; s < d.y; s += 32) {
      int b = r.b, e = r.e;
      typename Epi::Pre pre = pre_first;
      if (s != s_first) {
        b = p.ptr[s];
        e = p.ptr[s + 1];
        pre = epi.load(s);
      }
      double sum = 0.0;
      for (int k = b; k < e; ++k) sum += wbuf[k - d.z];
      epi.apply(s, sum, pre, acc);
    }
    __syncwarp();
  } else if (u < p.n_units) {
    // part of a long segment (<= kWarpTile entries at this size)
    const int multi = -d.x - 1;
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int k = d.z + lane + 32 * j;
      if (k < d.w) sum += r.v[j] * __ldg(&vec[r.ix[j]]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off);
    const int np = p.multi_parts[multi];
    unsigned last = 0;
    if (lane == 0) {
      p.part_sums[d.y] = sum;
      __threadfence();
      last = atomicAdd(&p.arrivals[multi], 1u) == static_cast<unsigned>(np - 1) ? 1u : 0u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence();
      double total = 0.0;
      const int first = p.multi_first[multi];
      for (int q = lane; q < np; q += 32) total += ld_cg(&p.part_sums[first + q]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) total += __shfl_down_sync(0xffffffffu, total, off);
      if (lane == 0) {
        const int seg = p.multi_seg[multi];
        TreeAcc<K> macc;
        macc.zero();
        epi.apply(seg, total, epi.load(seg), macc);
#pragma unroll
        for (int k = 0; k < K; ++k) multi_out[multi * K + k] = macc.v[k];
        p.arrivals[multi] = 0u;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc.v[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) scratch[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += scratch[w][threadIdx.x];
    parts0[rank * kMaxAcc + threadIdx.x] = v;  // remote store into CTA 0
  }
}

// Elementwise kernel with the same deterministic reduction tail.
// Op must provide K (>= 1), kReduce, prepare(), apply(i, acc), finalize(tot),
// finalize_ordered(terms, n).
template <class Op, bool ORDERED>
__global__ void __launch_bounds__(kBlock) elementwise_kernel(int64_t n, Op op, RedBuf rb) {
  constexpr int K = Op::K;
  if (!op.prepare()) return;
  using Acc = std::conditional_t<ORDERED, OrderedAcc<K>, TreeAcc<K>>;
  Acc acc;
  if constexpr (ORDERED) {
    acc.terms = rb.terms;
    acc.nterm = rb.nterm;
  }
  acc.zero();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kBlock;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; i < n; i += stride) {
    op.apply(i, acc);
  }
  if constexpr (Op::kReduce) {
    if constexpr (ORDERED) {
      if (!rb.defer) ordered_tail(op, rb);
    } else {
      reduce_tail(op, acc.v, rb, 0);
    }
  }
}

}  // namespace folpgpu
