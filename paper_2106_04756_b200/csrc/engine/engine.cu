// engine.cu -- the sm_100a PDLP engine behind include/folp_gpu.h.
//
// Data layout in HBM (one context = one presolved LP):
//   CSR  : int32 row_ptr[m+1], int32 col[nnz], fp64 val_orig[nnz], val_work[nnz]
//   CSC  : int32 col_ptr[n+1], int32 row[nnz], fp64 val_orig[nnz], val_work[nnz]
//          (CSC = CSR of K', columns in increasing row order, so K'y is the
//           same row-dot kernel as Kx; indices shared by both value sets)
//   vectors: presolved c,q,l,u and scaled c~,q~,l~,u~, D1, D2; iterate
//          double buffers x[2], y[2], Kx[2]; average sums; AVERAGE, LAST,
//          AUX points; evaluation / duality-gap scratch.
// All fp64, structure-of-arrays, 256-byte aligned by cudaMalloc.
//
// Compiled with -fmad=false (see Makefile): every a*b+c is two IEEE
// roundings like the reference's x86-64 build.
//
// One translation unit; the engine's parts are fragments included below in
// dependency order:
//   segdot.cuh         the segmented-dot kernel family (warp units, tails)
//   ops.cuh            PDLP epilogues / elementwise ops, the cluster loop
//   comm.cuh           NCCL and loopback collectives of the row shards
//   memory.cuh         device / pinned block cache
//   setup_kernels.cuh  scaling, start / reduced point, small utilities
//   (here)             folp_gpu_ctx: the context and its launchers
//   plans.cuh          unit plans, uploads, device CSR->CSC transpose
//   blocked.cuh        window-blocked products, per-axis scaling primitives
//   evaluation.cuh     evaluation period, duality gaps, restarts
//   shard_graphs.cuh   row-shard slot, chunk graph, evaluation graph
//   (here)             the extern "C" API of include/folp_gpu.h
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <map>
#include <functional>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "folp_gpu.h"
#include "../host/parallel.hpp"
#include "ops.cuh"
#include "exactfold.cuh"

#include <cooperative_groups.h>
#include <cub/cub.cuh>

using namespace folpgpu;

namespace {

thread_local std::string g_err;

struct EngineError : std::runtime_error {
  int code;
  EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      throw EngineError(e_ == cudaErrorMemoryAllocation ? FOLP_E_NOMEM        \
                                                        : FOLP_E_CUDA,        \
                        std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                         \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return FOLP_OK;
  } catch (const EngineError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return FOLP_E_NOMEM;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FOLP_E_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FOLP_E_RUNTIME;
  }
}

#include "comm.cuh"
#include "memory.cuh"
#include "setup_kernels.cuh"

// ---------------------------------------------------------------------
struct PlanDev {
  SegPlan sp{};
  int pair_len = 0;  // 2: every segment holds exactly two entries (pair_kernel)
  std::vector<void*> owned;
  const int* long_segs = nullptr;  // segments above kLongSeq entries (sequential norms)
  int n_long = 0;
};

// Window-blocked copy of one axis for the PDHG loop (EpiCarry / EpiCarryIn).
struct BlockedAxis {
  int windows = 0;                 // 0: the axis is not blocked
  int64_t window = 0;              // gather indices per window
  std::vector<PlanDev> plans;      // one unit plan per window
  int* idx = nullptr;              // index stream, window-major
  double* val = nullptr;           // working values, window-major
  double* val_orig = nullptr;      // original values, window-major (evaluations)
  double* carry = nullptr;         // per-segment partial dots
  std::vector<void*> owned;
};

bool g_default_ordered = false;
std::mutex g_occ_mu;
std::map<std::pair<const void*, int>, int> g_occ;  // (kernel, dynamic smem) -> CTAs per SM

int occupancy(const void* fn, int smem = 0) {
  std::lock_guard<std::mutex> lk(g_occ_mu);
  const auto key = std::make_pair(fn, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  if (smem > 0) {  // opt in once for the largest staging any context may use (static + dynamic > 48 KB)
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            std::max(smem, kStageMaxBytes)));
  }
  int b = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kBlock, smem));
  if (b < 1) b = 1;
  g_occ[key] = b;
  return b;
}

constexpr double kL2PersistFill = 1.0;  // share of the persisting carve-out the loop's streams may pin
constexpr int kResSlots = 96;
constexpr int kCounters = 16;
constexpr int kMaxGrid = 148 * 8;
constexpr int kSmallThreads = 256;   // k_chunk_cluster CTA
constexpr int kSmallCluster = 8;     // CTAs in its cluster (portable size)

}  // namespace

struct folp_gpu_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  int64_t m = 0, n = 0, m1 = 0, nnz = 0;
  double objective_constant = 0.0;

  int *csr_ptr = nullptr, *csr_col = nullptr, *csc_ptr = nullptr, *csc_row = nullptr;
  bool l2_window = false;  // the loop's streams hold an L2 persisting window
  struct Staged { void* pinned; double* host_dst; size_t bytes; };
  std::vector<Staged> staged;  // staged vector copies in flight (plans.cuh upload / download)
  double *csr_orig = nullptr, *csc_orig = nullptr, *csr_work = nullptr, *csc_work = nullptr;
  PlanDev rows, cols;

  double *c0, *q0, *l0, *u0;
  double *cw, *qw, *lw, *uw, *d1, *d2;
  double *x[2], *y[2], *kx[2];
  double *avg_x, *avg_y;
  double *avgp_x, *avgp_y, *last_x, *last_y, *aux_x, *aux_y;
  double *mp_ext, *mp_dy;  // Malitsky-Pock scratch
  double *kx_avg;   // K~ x of AVERAGE (filled by the duality gap)
  double *kx_aux;
  double* kty_raw[2] = {nullptr, nullptr};  // tree mode: K'y of CURRENT / AVERAGE in a period
  // the evaluation period's K'y cache for set s (tree mode, unsharded; else null)
  double* kty_cache(int s) const {
    return (!ordered && !sharded() && std::getenv("FOLP_NDG_RAW") == nullptr) ? kty_raw[s] : nullptr;
  }
  double *xr, *yr;  // reduced point scratch
  double *g[2], *lo[2], *hi[2];  // duality-gap scratch per candidate (CURRENT, AVERAGE)
  double *partials;
  unsigned* counters;
  double* res;      // small result slots
  double* res_h;    // pinned mirror
  DevState* st_d;
  DevState* st_h;   // pinned
  NdgState* ndg_d;  // [2]
  NdgState* ndg_h;  // [2], pinned
  double *red_d, *grow_d;
  double *red_h, *grow_h;  // pinned
  int64_t table_cap = 0;
  bool kx_valid = false;
  bool ordered = false;     // bit-exact reference summation order (parity runs)
  double* terms[2] = {nullptr, nullptr};  // ordered mode term regions
  bool norms_ready = false;
  double norm_q_sq = 0.0, norm_c_sq = 0.0;
  int max_giant = 0;
  int bisect_grid = 0;
  int* ndg_list = nullptr;        // k_ndg_bisect active lists [2][n + m]
  int* ndg_compact = nullptr;     // k_ndg_bisect block 0's gathered lists [2][kBisectSmall]
  bool coop_ok = true;            // cooperative launches available (else OpNdgPass passes)
  // evaluation period as a CUDA graph, one per CURRENT buffer parity
  cudaGraphExec_t eval_exec[2] = {nullptr, nullptr};
  bool eval_tried[2] = {false, false};
  bool capturing_eval = false;    // enqueue_*: read omega / weights on device
  double* eval_omega_h = nullptr;  // pinned: omega of the next graph launch
  double* eval_omega_d = nullptr;
  bool small_loop = false;        // k_chunk_cluster (tree mode, <= one unit per warp)
  double* small_multi = nullptr;  // its multi-part epilogue slots
  int64_t ndg_count = 0, ndg_passes = 0, ndg_levels = 0, ndg_grid_passes = 0;  // FOLP_TIMING statistics
  void* loop_block = nullptr;  // K~ values + indices of CSR and CSC (one block)
  size_t loop_block_bytes = 0;
  double* prod = nullptr;      // two-phase products (gather_products_kernel), nnz + 8

  // shard: rows [r0, r1) of K~ are this shard's, or columns
  // [r0, r1) under the column partition
  std::unique_ptr<ShardComm> comm;
  bool col_part = false;
  std::vector<int64_t> shard_bounds;  // [world + 1]
  int64_t r0 = 0, r1 = 0, lnnz = 0;
  PlanDev lrows, lcols;               // rows: own CSR rows, local CSC; cols: local CSR, own CSC columns
  BlockedAxis brows, bcols;           // window-blocked loop copies (large vectors)
  bool blocked_checked = false;
  PlanDev rows_sell;                  // the loop's K x' with SELL-32 groups (sell.cuh)
  bool sell = false, sell_packed = false, sell_coalesced = false;
  int* lcsc_ptr = nullptr;
  int* lcsc_row = nullptr;
  int* lcsc_pos = nullptr;            // local CSC entry -> full CSC position
  double* lcsc_val = nullptr;
  double* kty_part = nullptr;
  int peer_parity = 0;  // receive-area parity of the next peer exchange
  // partitioned epilogue over the peer exchange (DESIGN 7): the column
  // partition's dual step on own rows, the row partition's primal step on
  // own columns -- [pd_bounds[rank], pd_bounds[rank+1]) of equal chunks
  bool pdual = false;
  int64_t pd_chunk = 0;
  std::vector<int64_t> pd_bounds;
  double** pd_vdst = nullptr;  // device [2][W]: every rank's y[0], y[1] (cols) / x[0], x[1] (rows)
  bool hot_columns = false;  // created with a degree order (folp_gpu_create_ordered)
  double* shard_sums = nullptr;
  bool shard_values_ready = false;
  bool rows_dirty = false;            // partitioned vectors outside [r0, r1) stale
  bool sharded() const { return comm != nullptr; }

  cudaGraphExec_t chunk_exec[3] = {nullptr, nullptr, nullptr};  // per step policy
  bool graph_tried[3] = {false, false, false};
  bool graph_ok[3] = {false, false, false};
  int body_slots[3] = {1, 1, 1};  // trial slots per WHILE-body iteration
  int64_t launches = 0;
  bool profiling = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, tev0 = nullptr, tev1 = nullptr;
  double chunk_ms_total = 0.0;
  int64_t chunk_slots_total = 0;

  std::vector<void*> owned;

  template <class T>
  T* alloc(size_t count) {
    T* p = dalloc<T>(count);
    owned.push_back(p);
    return p;
  }

  double* cur_x() { return x[st_h->cur]; }
  double* cur_y() { return y[st_h->cur]; }
  double* slot_x(int which) {
    switch (which) {
      case FOLP_PT_CURRENT: return cur_x();
      case FOLP_PT_AVERAGE: return avgp_x;
      case FOLP_PT_LAST: return last_x;
      case FOLP_PT_AUX: return aux_x;
    }
    throw std::invalid_argument("unknown point slot");
  }
  double* slot_y(int which) {
    switch (which) {
      case FOLP_PT_CURRENT: return cur_y();
      case FOLP_PT_AVERAGE: return avgp_y;
      case FOLP_PT_LAST: return last_y;
      case FOLP_PT_AUX: return aux_y;
    }
    throw std::invalid_argument("unknown point slot");
  }

  int ew_grid(int64_t count, const void* fn) {
    const int64_t need = (count + kBlock - 1) / kBlock;
    const int64_t cap = static_cast<int64_t>(sms) * occupancy(fn);
    return static_cast<int>(std::max<int64_t>(1, std::min(need, std::min<int64_t>(cap, kMaxGrid))));
  }
  int simple_grid(int64_t count) {
    const int64_t need = (count + kBlock - 1) / kBlock;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, sms * 8)));
  }
  RedBuf red(int counter) {
    RedBuf rb{partials, counters + counter, nullptr, 0};
    rb.cap = partial_cap;
    return rb;
  }
  int partial_cap = 0;  // slots (of kMaxAcc doubles) in `partials`
  // kernel A's deferred sums (segdot.cuh DeferredSums): its own partial
  // slots, the slot count of its last launch, and the switch launch_slot sets
  double* partials_a = nullptr;
  int a_np = 0;
  bool a_defer = false;

  // exact parallel fold (exactfold.cuh) of ordered mode's trial sums
  FoldScratch fold{};
  int fold_grid = 0;         // co-resident CTAs of k_exact_fold (0: not available)
  bool defer_tail = false;   // ordered products store terms only (the fold finalizes)
  double* oprod = nullptr;   // ordered mode: long-segment products (warp_exact_fold)
  void alloc_fold() {
    int per_sm = 0;
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_exact_fold<FinTrial>),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFoldDynSmem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_exact_fold<FinTrial>, kFoldBlock, kFoldDynSmem) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      return;
    }
    if (const char* env = std::getenv("FOLP_FOLD_SKIP_ZEROS")) {
      const int v = std::atoi(env) != 0 ? 1 : 0;
      CK(cudaMemcpyToSymbol(g_fold_skip_zeros, &v, sizeof v));
    }
    int G = std::min(sms * per_sm, kFoldMaxCtas);
    if (const char* env = std::getenv("FOLP_FOLD_GRID")) G = std::max(1, std::min(G, std::atoi(env)));
    fold.cap = G;
    fold.cta_sum = alloc<double>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_abs = alloc<double>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_ntot = alloc<unsigned long long>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_nbp = alloc<int>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_bad = alloc<int>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_flag = alloc<int>(G);
    fold.cta_laste = alloc<int>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.cta_lastc = alloc<unsigned long long>(static_cast<size_t>(kFoldMaxJobs) * G);
    fold.bps = alloc<FoldBp>(static_cast<size_t>(kFoldMaxJobs) * G * kFoldBpCap);
    fold.chain = alloc<FoldEntry>(static_cast<size_t>(kFoldMaxJobs) * (static_cast<size_t>(G) * kFoldBpCap + 1));
    fold.results = alloc<double>(kFoldMaxJobs);
    fold.counter = alloc<unsigned>(1);
    CK(cudaMemsetAsync(fold.counter, 0, sizeof(unsigned), stream));
    fold_grid = G;
  }
  // Ordered finalize of E through the exact parallel fold: e's stored terms
  // (t, nterm as finalize_ordered sees them) folded by k_exact_fold<FinExact<E>>.
  template <class E>
  void launch_exact(const E& e, const double* t, int64_t nterm) {
    using Fin = FinExact<E>;
    const void* fn = reinterpret_cast<const void*>(k_exact_fold<Fin>);
    static std::mutex mu;
    static std::unordered_map<int, int> grid_of;  // device -> co-resident CTAs
    int G = 0;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = grid_of.find(device);
      if (it == grid_of.end()) {
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kFoldDynSmem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFoldBlock, kFoldDynSmem));
        it = grid_of.emplace(device, std::max(1, per_sm) * sms).first;
      }
      G = std::min(it->second, fold.cap);
    }
    FoldJobs fj{};
    e.fold_plan(t, nterm, fj);
    Fin fin{e};
    void* args[] = {&fj, &fold, &fin};
    CK(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kFoldBlock), args, kFoldDynSmem, stream));
    ++launches;
  }

  // the trial's three folds + decision (replaces EpiDual::finalize_ordered)
  void launch_trial_fold(const LoopBufs& b) {
    FoldJobs fj{};
    fj.count = 3;
    fj.job[0] = FoldJob{terms[1], m, 0.0, -1, 1.0, nullptr, nullptr};      // cross (solver.cpp:80)
    fj.job[1] = FoldJob{terms[1] + m, m, 0.0, -1, 1.0, nullptr, nullptr};  // sum dy^2 (:81)
    fj.job[2] = FoldJob{terms[0], n, 0.0, 1, 1.0, &st_d->omega, nullptr};  // /omega + sum omega dx^2 (:83-88)
    fj.nflags = 2;
    fj.flag[0] = terms[0] + n;
    fj.flag_n[0] = n;
    fj.flag[1] = terms[1] + 2 * m;
    fj.flag_n[1] = m;
    FinTrial fin{b};
    void* args[] = {&fj, &fold, &fin};
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_exact_fold<FinTrial>),
                                   dim3(fold_grid), dim3(kFoldBlock), args, kFoldDynSmem, stream));
    ++launches;
  }

  // Launch of a segdot kernel; with `pdl` (the PDHG loop's products, see
  // segdot.cuh griddep_wait) as a programmatic dependent launch.
  bool pdl = false;
  // Staged gathers (segdot.cuh) for the loop's own axis plans when the
  // gathered vector fits kStageMaxBytes; FOLP_STAGE=1 enables.  Off by
  // default: on config 5 (y = 80 KB) two CTAs per SM fit next to the copy,
  // and the halved occupancy costs the streams more than the shared-memory
  // gathers save (K'y + primal step 530 -> 608 us per trial).
  int stage_env = -1;
  bool stage_ok(const PlanDev& p) {
    if (stage_env < 0) {
      const char* env = std::getenv("FOLP_STAGE");
      stage_env = env != nullptr ? std::atoi(env) : 0;
    }
    return stage_env != 0 && (&p == &rows || &p == &cols) && p.sp.vec_len > 0 &&
           p.sp.vec_len * static_cast<int64_t>(sizeof(double)) <= kStageMaxBytes;
  }
  // Axes of two-entry segments (segdot.cuh pair_kernel): the loop's own
  // products in tree mode; FOLP_PAIRS=0 keeps the warp tiles.
  int pairs_env = -1;
  template <class Epi>
  bool pairs_ok(const PlanDev& p) {
    if (pairs_env < 0) {
      const char* env = std::getenv("FOLP_PAIRS");
      pairs_env = env != nullptr ? std::atoi(env) : 1;
    }
    const bool ok = pairs_env != 0 && TraceSlot<Epi>::v >= 0 && p.pair_len == 2 && (&p == &rows || &p == &cols);
    if (ok && !pairs_said && std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr, "[folp timing] pair kernel on the axis of %d two-entry segments\n", p.sp.S);
      pairs_said = true;
    }
    return ok;
  }
  bool pairs_said = false;
  template <class Epi>
  void launch_pairs(const PlanDev& p, const double* val, const Epi& epi, RedBuf rb) {
    auto fn = pair_kernel<Epi>;
    const int64_t need = (static_cast<int64_t>(p.sp.S) + 2 * kBlock - 1) / (2 * kBlock);
    const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, fn, p.sp.S, p.sp.idx, val, p.sp.vec_len, epi, rb));
    last_np = grid;
  }
  template <class Epi, bool ORD, bool PR, int ST = 0, bool SE = false>
  void launch_segdot(int grid, const SegPlan& sp, const double* val, const Epi& epi, RedBuf rb,
                     int smem = 0) {
    auto fn = segdot_kernel<Epi, ORD, PR, ST, SE>;
    // L1 / shared split: the smallest shared carveout that still holds
    // kPlanCtasPerSm CTAs leaves the most L1 to the gathers (config 2's
    // degree-ordered hot prefix: 59.7 -> 57.6 us per trial; config 3 250.2
    // -> 243.2 us; config 5 unchanged); window-blocked contexts keep the
    // driver's choice (config 4 loses 25 % with the small carveout).
    // FOLP_CARVEOUT=% forces one split everywhere, -1 = driver default.
    // Set per launch (a launch attribute, captured into graph nodes too), so
    // concurrent contexts of both kinds never share mutable state.
    const char* env = std::getenv("FOLP_CARVEOUT");
    const bool windowed = brows.windows > 0 || bcols.windows > 0;
    const int want = ST != 0 ? 100 : env != nullptr ? std::atoi(env) : (!windowed ? kSegdotCarveout : -1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (want >= 0) {
      attr[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
      attr[na].val.sharedMemCarveout = static_cast<unsigned>(want);
      ++na;
    }
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, fn, sp, val, epi, rb));
  }

  template <class Epi>
  void seg(const PlanDev& p, const double* val, const Epi& epi, int counter, int region = 1) {
    RedBuf rb = red(counter);
    const int64_t need = (static_cast<int64_t>(p.sp.n_units) + kWarps - 1) / kWarps;
    if constexpr (std::is_same_v<Epi, EpiPrimal>) {
      if (a_defer && !ordered) {
        rb.partials = partials_a;
        rb.tree_defer = 1;
      }
    }
    if (ordered) {
      rb.terms = terms[region];
      rb.nterm = p.sp.S;
      rb.defer = defer_tail ? 1 : 0;
      rb.scratch = oprod;
      bool exact = false;
      if constexpr (HasFoldPlan<Epi>::value) exact = fold_grid > 0 && !defer_tail;
      if (exact) rb.defer = 1;
      auto fn = segdot_kernel<Epi, true>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      launch_segdot<Epi, true, false>(grid, p.sp, val, epi, rb);
      if constexpr (HasFoldPlan<Epi>::value) {
        if (exact) launch_exact(epi, terms[region], p.sp.S);
      }
    } else if (prod != nullptr && (&p == &rows || &p == &cols)) {
      // two phases (segdot.cuh): gathers over the whole axis, then the
      // segmented sums and the epilogue over the product stream
      auto gn = gather_products_kernel<Epi>;
      const int64_t quads = (nnz >> 2) + 1;
      const int ggrid = ew_grid(quads, reinterpret_cast<const void*>(gn));
      gn<<<ggrid, kBlock, 0, stream>>>(p.sp.idx, val, nnz, prod, epi);
      auto fn = segdot_kernel<Epi, false, true>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      launch_segdot<Epi, false, true>(grid, p.sp, prod, epi, rb);
      last_np = grid + p.sp.n_multi + p.sp.sell.n_groups;
      ++launches;
    } else if (pairs_ok<Epi>(p)) {
      if constexpr (TraceSlot<Epi>::v >= 0) launch_pairs(p, val, epi, rb);
    } else if (p.sp.sell.n_groups > 0) {
      // a plan with SELL-32 groups (sell.cuh)
      auto fn = segdot_kernel<Epi, false, false, 0, true>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      launch_segdot<Epi, false, false, 0, true>(grid, p.sp, val, epi, rb);
      last_np = grid + p.sp.n_multi + p.sp.sell.n_groups;
    } else if (stage_ok(p)) {
      // the gathered vector in shared memory (segdot.cuh, staged gathers)
      auto fn = segdot_kernel<Epi, false, false, 1>;
      const int smem = p.sp.vec_len * static_cast<int>(sizeof(double));
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn), smem);
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      launch_segdot<Epi, false, false, 1>(grid, p.sp, val, epi, rb, smem);
      last_np = grid + p.sp.n_multi + p.sp.sell.n_groups;
    } else {
      auto fn = segdot_kernel<Epi, false>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      launch_segdot<Epi, false, false>(grid, p.sp, val, epi, rb);
      last_np = grid + p.sp.n_multi + p.sp.sell.n_groups;
    }
    ++launches;
    CK(cudaGetLastError());
    if constexpr (std::is_same_v<Epi, EpiPrimal>) {
      if (rb.tree_defer) a_np = last_np;
    }
  }
  int last_np = 0;  // partial slots of the last tree-mode product launch

  template <class Op>
  void ew(int64_t count, const Op& op, int counter, int region = 1) {
    RedBuf rb = red(counter);
    if (ordered) {
      rb.terms = terms[region];
      rb.nterm = count;
      bool exact = false;
      if constexpr (HasFoldPlan<Op>::value) exact = fold_grid > 0;
      if (exact) rb.defer = 1;
      auto fn = elementwise_kernel<Op, true>;
      const int grid = ew_grid(count, reinterpret_cast<const void*>(fn));
      fn<<<grid, kBlock, 0, stream>>>(count, op, rb);
      if constexpr (HasFoldPlan<Op>::value) {
        if (exact) launch_exact(op, terms[region], count);
      }
    } else {
      auto fn = elementwise_kernel<Op, false>;
      const int grid = ew_grid(count, reinterpret_cast<const void*>(fn));
      fn<<<grid, kBlock, 0, stream>>>(count, op, rb);
    }
    ++launches;
    CK(cudaGetLastError());
  }

  void fetch_res(int count) {
    CK(cudaMemcpyAsync(res_h, res, count * sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
  void push_state() {
    CK(cudaMemcpyAsync(st_d, st_h, sizeof(DevState), cudaMemcpyHostToDevice, stream));
  }
  void pull_state() {
    CK(cudaMemcpyAsync(st_h, st_d, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }
  LoopBufs loop_bufs(cudaGraphConditionalHandle h, int use_cond) {
    LoopBufs b{};
    b.x[0] = x[0];
    b.x[1] = x[1];
    b.y[0] = y[0];
    b.y[1] = y[1];
    b.kx[0] = kx[0];
    b.kx[1] = kx[1];
    b.avg_x = avg_x;
    b.avg_y = avg_y;
    b.c = cw;
    b.l = lw;
    b.u = uw;
    b.q = qw;
    b.m1 = m1;
    b.n = n;
    b.a_terms = terms[0];
    b.mp_ext = mp_ext;
    b.mp_dy = mp_dy;
    b.st = st_d;
    b.red = red_d;
    b.grow = grow_d;
    b.cond = h;
    b.use_cond = use_cond;
    b.l_const = l_const;
    b.u_const = u_const;
    b.l_uni = l_uni;
    b.u_uni = u_uni;
    return b;
  }
  // uniform working bounds (LoopBufs l_uni / u_uni), checked once after rescaling
  bool bounds_checked = false;
  double l_const = 0.0, u_const = 0.0;
  int l_uni = 0, u_uni = 0;

  ~folp_gpu_ctx() {
    if (ndg_count > 0 && std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr,
                   "[folp timing] duality gaps %lld: %.1f passes (%.1f grid-wide), %.1f bisection levels each\n",
                   static_cast<long long>(ndg_count), static_cast<double>(ndg_passes) / ndg_count,
                   static_cast<double>(ndg_grid_passes) / ndg_count,
                   static_cast<double>(ndg_levels) / ndg_count);
#ifdef FOLP_BISECT_TIMES
      unsigned long long bt[kBisectTimeSlots][3];
      if (cudaMemcpyFromSymbol(bt, g_bisect_times, sizeof bt) == cudaSuccess) {
        for (int k = 0; k < kBisectTimeSlots && bt[k][1] > 0; ++k) {
          std::fprintf(stderr, "[folp timing] bisection pass %d: %.2f us avg over %llu launches (%llu alone)\n", k,
                       1e-3 * static_cast<double>(bt[k][0]) / static_cast<double>(bt[k][1]), bt[k][1], bt[k][2]);
        }
      }
#endif
    }
    if (fold_grid > 0 && std::getenv("FOLP_FOLD_TIMES") != nullptr) {
      unsigned long long tt[8];
      if (cudaMemcpyFromSymbol(tt, g_fold_times, sizeof tt) == cudaSuccess) {
        std::fprintf(stderr, "[fold times us, last trial] phase1 %.2f sync %.2f phase2 %.2f ticket %.2f lists %.2f replay %.2f\n",
                     1e-3 * (tt[1] - tt[0]), 1e-3 * (tt[2] - tt[1]), 1e-3 * (tt[3] - tt[2]),
                     1e-3 * (double)(long long)(tt[4] - tt[3]), 1e-3 * (tt[5] - tt[4]), 1e-3 * (tt[6] - tt[5]));
      }
    }
    const bool timing = std::getenv("FOLP_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    if (device >= 0) cudaSetDevice(device);
    for (auto& e : chunk_exec)
      if (e) cudaGraphExecDestroy(e);
    for (auto& e : eval_exec)
      if (e) cudaGraphExecDestroy(e);
    const double t_graphs = since();
    block_free(eval_omega_h);
    if (stream) cudaStreamSynchronize(stream);  // cached blocks must be idle
    for (const Staged& sg : staged) block_free(sg.pinned);
    const double t_sync = since();
    for (void* p : owned) block_free(p);
    for (void* p : rows.owned) block_free(p);
    for (void* p : cols.owned) block_free(p);
    for (void* p : lrows.owned) block_free(p);
    for (void* p : lcols.owned) block_free(p);
    for (BlockedAxis* ax : {&brows, &bcols}) {
      for (PlanDev& pl : ax->plans)
        for (void* p : pl.owned) block_free(p);
      for (void* p : ax->owned) block_free(p);
    }
    comm.reset();
    block_free(res_h);
    block_free(st_h);
    block_free(ndg_h);
    block_free(red_h);
    block_free(grow_h);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (tev0) cudaEventDestroy(tev0);
    if (tev1) cudaEventDestroy(tev1);
    const double t_free = since();
    if (stream) cudaStreamDestroy(stream);
    // lines this context pinned go back to normal (a later, larger context
    // would otherwise stream past a carve-out full of dead lines)
    if (l2_window) cudaCtxResetPersistingL2Cache();
    if (timing) {
      std::fprintf(stderr, "[folp timing] engine destroy: graphs %.4f sync %.4f blocks %.4f stream %.4f\n",
                   t_graphs, t_sync, t_free, since());
    }
  }
};

namespace {

#include "plans.cuh"
#include "sell.cuh"
#include "blocked.cuh"
#include "evaluation.cuh"
#include "shard_graphs.cuh"

}  // namespace

// =====================================================================
extern "C" {

const char* folp_gpu_last_error(void) { return g_err.c_str(); }

int folp_gpu_create(const folp_gpu_problem* p, int device, folp_gpu_ctx** out) {
  return folp_gpu_create_ordered(p, nullptr, device, out);
}

int folp_gpu_create_ordered(const folp_gpu_problem* p, const int64_t* col_order, int device,
                            folp_gpu_ctx** out) {
  *out = nullptr;
  return guarded([&] {
    if (p->num_rows < 0 || p->num_cols < 0 || p->nnz < 0 ||
        p->num_inequality_rows < 0 || p->num_inequality_rows > p->num_rows) {
      throw EngineError(FOLP_E_DIMENSION_MISMATCH, "folp_gpu_create: bad dimensions");
    }
    if (p->nnz >= (int64_t(1) << 31) || p->num_rows >= (int64_t(1) << 31) ||
        p->num_cols >= (int64_t(1) << 31)) {
      throw EngineError(FOLP_E_INVALID_ARGUMENT, "folp_gpu_create: sizes exceed int32 indexing");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw EngineError(FOLP_E_NO_DEVICE, "folp_gpu_create: no CUDA device visible");
    }
    const bool timing = std::getenv("FOLP_TIMING") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::string marks;
    auto mark = [&](const char* stage) {
      if (!timing) return;
      char buf[64];
      std::snprintf(buf, sizeof(buf), " %s %.4f", stage,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      marks += buf;
    };
    std::unique_ptr<folp_gpu_ctx> c(new folp_gpu_ctx());
    c->device = pick_device(device);
    c->ordered = folp_gpu_default_reduction() != 0;
    if (const char* env = std::getenv("FOLP_NO_COOP")) c->coop_ok = std::atoi(env) == 0;
    set_device(c.get());
    CK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreate(&c->tev0));
    CK(cudaEventCreate(&c->tev1));
    mark("stream");
    const int64_t m = p->num_rows, n = p->num_cols, nnz = p->nnz;
    c->m = m;
    c->n = n;
    c->m1 = p->num_inequality_rows;
    c->nnz = nnz;
    c->objective_constant = p->objective_constant;

    std::vector<int64_t> cs;
    const int64_t *col_start = p->col_start, *col_rows = p->col_rows;
    const double* col_values = p->col_values;
    // No column mirror from the host: transpose on the device (below).
    const bool device_csc =
        col_order != nullptr || col_start == nullptr || col_rows == nullptr || col_values == nullptr;
    // working column j = caller's column col_order[j]: indices renumbered
    // on device right after their upload, the CSC built from the
    // renumbered CSR, c / l / u gathered (host vectors map at the boundary)
    int* order_d = nullptr;
    int* rank_d = nullptr;
    if (col_order != nullptr && n > 0) {
      std::vector<int> ord(static_cast<size_t>(n)), rnk(static_cast<size_t>(n), -1);
      for (int64_t j = 0; j < n; ++j) {
        const int64_t o = col_order[j];
        if (o < 0 || o >= n || rnk[static_cast<size_t>(o)] >= 0) {
          throw EngineError(FOLP_E_INVALID_ARGUMENT, "folp_gpu_create_ordered: not a permutation");
        }
        ord[static_cast<size_t>(j)] = static_cast<int>(o);
        rnk[static_cast<size_t>(o)] = static_cast<int>(j);
      }
      order_d = c->alloc<int>(n);
      rank_d = c->alloc<int>(n);
      c->hot_columns = true;
      CK(cudaMemcpy(order_d, ord.data(), n * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(rank_d, rnk.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    }

    // value / index streams padded by 8 entries: bulk tiles are staged in
    // 16-byte-aligned windows that may run up to 3 entries past the end
    c->csr_ptr = c->alloc<int>(m + 1);
    c->csc_ptr = c->alloc<int>(n + 1);
    c->csr_orig = c->alloc<double>(nnz + 8);
    c->csc_orig = c->alloc<double>(nnz + 8);
    {
      // The loop's streams -- working values and indices of both layouts --
      // in ONE block, so a single L2 access-policy window can cover them.
      const size_t vb = (static_cast<size_t>(nnz + 8) * sizeof(double) + 255) / 256 * 256;
      const size_t ib = (static_cast<size_t>(nnz + 8) * sizeof(int) + 255) / 256 * 256;
      char* blk = c->alloc<char>(2 * vb + 2 * ib);
      c->csr_work = reinterpret_cast<double*>(blk);
      c->csc_work = reinterpret_cast<double*>(blk + vb);
      c->csr_col = reinterpret_cast<int*>(blk + 2 * vb);
      c->csc_row = reinterpret_cast<int*>(blk + 2 * vb + ib);
      c->loop_block = blk;
      c->loop_block_bytes = 2 * vb + 2 * ib;
    }
    // the CSR streams: narrowed / copied into pinned blocks by all host
    // threads, then one DMA each (pageable copies ran at ~8 GB/s: 7 ms of
    // config 2's end-to-end solve)
    std::vector<void*> pinned;
    auto stage_in = [&](void* dst, const void* src, int64_t count, bool narrow) {
      if (count <= 0) return;
      const size_t bytes = static_cast<size_t>(count) * (narrow ? sizeof(int) : sizeof(double));
      void* h = block_alloc(bytes, true);
      pinned.push_back(h);
      folp::host::parallel_for(count, [&](int64_t b, int64_t e, int) {
        if (narrow) {
          const int64_t* s64 = static_cast<const int64_t*>(src);
          int* d32 = static_cast<int*>(h);
          for (int64_t i = b; i < e; ++i) d32[i] = static_cast<int>(s64[i]);
        } else {
          std::memcpy(static_cast<double*>(h) + b, static_cast<const double*>(src) + b,
                      static_cast<size_t>(e - b) * sizeof(double));
        }
      });
      CK(cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, c->stream));
    };
    auto release_pinned = [&] {
      cudaStreamSynchronize(c->stream);
      for (void* h : pinned) block_free(h);
      pinned.clear();
    };
    {
      const int64_t cap = std::min<int64_t>(std::max<int64_t>({m + 1, n + 1, nnz}), int64_t(1) << 26);
      int64_t* stage = dalloc<int64_t>(cap);
      try {
        upload_index(c.get(), p->row_start, c->csr_ptr, m + 1, stage, cap);
        if (nnz < (int64_t(1) << 20)) {
          upload_index(c.get(), p->row_cols, c->csr_col, nnz, stage, cap);
        } else {
          stage_in(c->csr_col, p->row_cols, nnz, true);
        }
        if (rank_d != nullptr && nnz > 0) {
          k_renumber<<<c->simple_grid(nnz), kBlock, 0, c->stream>>>(c->csr_col, rank_d, nnz);
          ++c->launches;
          CK(cudaGetLastError());
        }
        if (!device_csc) {
          upload_index(c.get(), col_start, c->csc_ptr, n + 1, stage, cap);
          upload_index(c.get(), col_rows, c->csc_row, nnz, stage, cap);
        }
        CK(cudaStreamSynchronize(c->stream));
      } catch (...) {
        block_free(stage);
        release_pinned();
        throw;
      }
      block_free(stage);
    }
    mark("indices");
    // the rows plan (and the SELL groups) on a second host thread while this
    // one uploads the values, transposes on the device and plans the columns
    std::exception_ptr rows_err;
    SellHost sh;
    std::thread rows_worker([&] {
      try {
        CK(cudaSetDevice(c->device));
        build_plan(c.get(), p->row_start, m, nnz, c->csr_ptr, c->csr_col, c->rows);
        if (!c->ordered && col_order == nullptr && nnz > 0 && p->row_cols != nullptr) {
          sh = detect_sell(p->row_start, p->row_cols, m, nnz);
          if (!sh.row0.empty()) build_sell_plan(c.get(), p->row_start, m, nnz, sh, c->rows_sell);
        }
      } catch (...) {
        rows_err = std::current_exception();
      }
    });
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{rows_worker};
    try {
      if (nnz < (int64_t(1) << 20) || p->row_values == nullptr) {
        upload(c.get(), c->csr_orig, p->row_values, nnz);
      } else {
        stage_in(c->csr_orig, p->row_values, nnz, false);
      }
    } catch (...) {
      release_pinned();
      throw;
    }
    if (device_csc) {
      device_transpose(c.get(), cs);
      col_start = cs.data();
    } else {
      upload(c.get(), c->csc_orig, col_values, nnz);
    }
    copy_d2d(c.get(), c->csr_work, c->csr_orig, nnz);
    copy_d2d(c.get(), c->csc_work, c->csc_orig, nnz);
    release_pinned();

    mark("values");
    build_plan(c.get(), col_start, n, nnz, c->csc_ptr, c->csc_row, c->cols);
    rows_worker.join();
    if (rows_err) std::rethrow_exception(rows_err);
    c->rows.sp.vec_len = static_cast<int>(std::min<int64_t>(n, INT32_MAX));
    c->cols.sp.vec_len = static_cast<int>(std::min<int64_t>(m, INT32_MAX));
    if (!sh.row0.empty()) {
      c->sell = true;
      c->sell_coalesced = sh.gathers_coalesced;
      if (timing) {
        std::fprintf(stderr, "[folp timing] SELL-32: %zu row groups, %lld entries, coalesced %d\n",
                     sh.row0.size(), static_cast<long long>(sh.nnz), sh.gathers_coalesced ? 1 : 0);
      }
    }

    mark("plans");
    auto vn = [&] { return c->alloc<double>(n); };
    auto vm = [&] { return c->alloc<double>(m); };
    c->c0 = vn(); c->l0 = vn(); c->u0 = vn(); c->q0 = vm();
    c->cw = vn(); c->lw = vn(); c->uw = vn(); c->qw = vm();
    c->d1 = vm(); c->d2 = vn();
    c->x[0] = vn(); c->x[1] = vn();
    c->y[0] = vm(); c->y[1] = vm();
    c->kx[0] = vm(); c->kx[1] = vm();
    c->avg_x = vn(); c->avg_y = vm();
    c->avgp_x = vn(); c->avgp_y = vm();
    c->last_x = vn(); c->last_y = vm();
    c->aux_x = vn(); c->aux_y = vm();
    c->kx_avg = vm(); c->kx_aux = vm();
    c->mp_ext = vn(); c->mp_dy = vm();
    c->xr = vn(); c->yr = vm();
    for (int s = 0; s < 2; ++s) {
      c->g[s] = c->alloc<double>(n + m);
      c->lo[s] = c->alloc<double>(n + m);
      c->hi[s] = vn();
    }
    if (!c->ordered) {
      c->kty_raw[0] = vn();
      c->kty_raw[1] = vn();
      c->ndg_list = c->alloc<int>(2 * static_cast<size_t>(n + m) + 2);
      c->ndg_compact = c->alloc<int>(2 * static_cast<size_t>(kBisectSmall));
    }
    c->partials = c->alloc<double>(static_cast<size_t>(kMaxGrid + c->max_giant + 8) * kMaxAcc);
    c->partial_cap = kMaxGrid + c->max_giant + 8;
    c->partials_a = c->alloc<double>(static_cast<size_t>(c->partial_cap) * EpiPrimal::K);
    if (c->ordered) {
      c->terms[0] = c->alloc<double>(5 * std::max(n, m) + 8);
      c->terms[1] = c->alloc<double>(5 * (n + m) + 8);
      // exact parallel folds of the trial sums (exactfold.cuh); FOLP_EXACT_FOLD=0
      // keeps the one-thread sequential folds
      const char* env = std::getenv("FOLP_EXACT_FOLD");
      if (env == nullptr || std::atoi(env) != 0) {
        c->alloc_fold();
        c->oprod = c->alloc<double>(static_cast<size_t>(nnz) + 8);
      }
    }
    {
      const char* env = std::getenv("FOLP_SMALL_LOOP");
      // every warp of the cluster owns at most one unit of each product
      const int warps = kSmallCluster * (kSmallThreads / 32);
      c->small_loop = !c->ordered && nnz > 0 && c->rows.sp.n_units <= warps &&
                      c->cols.sp.n_units <= warps && (env == nullptr || std::atoi(env) > 0);
      c->small_multi = c->alloc<double>(
          static_cast<size_t>(std::max(c->rows.sp.n_multi, c->cols.sp.n_multi) + 1) * kMaxAcc);
    }
    {
      // Two-phase products (FOLP_TWO_PHASE=1 always, =2 when the product
      // stream fits L2 next to the gathered vector; default off: measured
      // 1.6x slower on config 2 -- profiles/r1_two_phase.md; tree mode only).
      const char* env = std::getenv("FOLP_TWO_PHASE");
      const int mode = env ? std::atoi(env) : 0;
      const bool fits = static_cast<double>(nnz) * 8.0 <= 48.0 * (1 << 20);
      if (!c->ordered && !c->small_loop && nnz > 0 && (mode == 1 || (mode == 2 && fits))) {
        c->prod = c->alloc<double>(nnz + 8);
      }
    }
    c->counters = c->alloc<unsigned>(kCounters);
    CK(cudaMemsetAsync(c->counters, 0, kCounters * sizeof(unsigned), c->stream));
    c->res = c->alloc<double>(kResSlots);
    halloc(&c->res_h, kResSlots);
    halloc(&c->eval_omega_h, 1);
    c->eval_omega_d = c->alloc<double>(1);
    c->st_d = c->alloc<DevState>(1);
    halloc(&c->st_h, 1);
    std::memset(c->st_h, 0, sizeof(DevState));
    c->ndg_d = c->alloc<NdgState>(2);
    halloc(&c->ndg_h, 2);
    c->table_cap = 4096;
    c->red_d = c->alloc<double>(c->table_cap);
    c->grow_d = c->alloc<double>(c->table_cap);
    halloc(&c->red_h, c->table_cap);
    halloc(&c->grow_h, c->table_cap);

    mark("buffers");
    upload(c.get(), c->c0, p->objective, n);
    upload(c.get(), c->l0, p->variable_lower, n);
    upload(c.get(), c->u0, p->variable_upper, n);
    if (order_d != nullptr) {
      for (double* v : {c->c0, c->l0, c->u0}) {
        copy_d2d(c.get(), c->xr, v, n);  // xr: scratch until the first evaluation
        k_gather_order<<<c->simple_grid(n), kBlock, 0, c->stream>>>(c->xr, order_d, v, n);
        ++c->launches;
        CK(cudaGetLastError());
      }
    }
    upload(c.get(), c->q0, p->right_hand_side, m);
    // Identity scaling until folp_gpu_rescale: working problem = presolved.
    copy_d2d(c.get(), c->cw, c->c0, n);
    copy_d2d(c.get(), c->lw, c->l0, n);
    copy_d2d(c.get(), c->uw, c->u0, n);
    copy_d2d(c.get(), c->qw, c->q0, m);
    k_fill<<<c->simple_grid(m), kBlock, 0, c->stream>>>(c->d1, m, 1.0);
    k_fill<<<c->simple_grid(n), kBlock, 0, c->stream>>>(c->d2, n, 1.0);
    c->launches += 2;
    for (int i = 0; i < 2; ++i) {
      if (n) CK(cudaMemsetAsync(c->x[i], 0, n * sizeof(double), c->stream));
      if (m) CK(cudaMemsetAsync(c->y[i], 0, m * sizeof(double), c->stream));
      if (m) CK(cudaMemsetAsync(c->kx[i], 0, m * sizeof(double), c->stream));
    }
    zero_average(c.get());
    sync_transfers(c.get());
    const char* l2env = std::getenv("FOLP_L2_PERSIST");
    if (l2env == nullptr || std::atoi(l2env) > 0) {
      // keep the loop's streams in L2 (persisting lines) across trials
      int max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
      // Only when the block (nearly) fits the persisting carve-out.  A larger
      // block keeps a random ~max_persist of its lines pinned and leaves the
      // rest of the L2 to every other stream: measured per trial, config 5
      // (768 MB block) 426.7 us with the window vs 284.6 us without, config
      // 3 (480 MB) 306.8 vs 249.7 us; config 2 (84 MB, fits) 56.0 vs 58.0 us.
      // FOLP_L2_PERSIST=2 forces the window.
      const bool fits = c->loop_block_bytes <= static_cast<size_t>(max_persist) + (static_cast<size_t>(max_persist) >> 2);
      if (max_persist > 0 && max_window > 0 && (fits || (l2env != nullptr && std::atoi(l2env) > 1))) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(max_persist));
        cudaStreamAttrValue attr{};
        const size_t bytes = std::min(c->loop_block_bytes, static_cast<size_t>(max_window));
        attr.accessPolicyWindow.base_ptr = c->loop_block;
        attr.accessPolicyWindow.num_bytes = bytes;
        // the fraction of the window's lines that persist (the rest stream);
        // FOLP_L2_HIT_RATIO overrides
        double ratio = std::min(1.0, kL2PersistFill * static_cast<double>(max_persist) / bytes);
        if (const char* renv = std::getenv("FOLP_L2_HIT_RATIO")) ratio = std::min(1.0, std::max(0.0, std::atof(renv)));
        attr.accessPolicyWindow.hitRatio = static_cast<float>(ratio);
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
        c->l2_window = true;
        cudaGetLastError();
        if (timing) {
          std::fprintf(stderr, "[folp timing] L2 persist: max %d B, window max %d B, block %zu B\n",
                       max_persist, max_window, c->loop_block_bytes);
        }
      }
    }
    mark("vectors");
    if (timing) std::fprintf(stderr, "[folp timing] engine create:%s\n", marks.c_str());
    *out = c.release();
  });
}

void folp_gpu_destroy(folp_gpu_ctx* ctx) { delete ctx; }

int folp_gpu_rescale(folp_gpu_ctx* c, int64_t ruiz_iterations, int32_t pock_chambolle,
                     double alpha, double* row_scale, double* col_scale) {
  return guarded([&] {
    prep(c);
    c->shard_values_ready = false;
    if (c->blocked_checked && (c->brows.windows > 0 || c->bcols.windows > 0)) {
      throw std::invalid_argument("rescale: the loop's blocked copies are already built");
    }
    const int64_t m = c->m, n = c->n, nnz = c->nnz;
    double* cum1 = c->d1;
    double* cum2 = c->d2;
    k_fill<<<c->simple_grid(m), kBlock, 0, c->stream>>>(cum1, m, 1.0);
    k_fill<<<c->simple_grid(n), kBlock, 0, c->stream>>>(cum2, n, 1.0);
    c->launches += 2;
    copy_d2d(c, c->csr_work, c->csr_orig, nnz);
    copy_d2d(c, c->csc_work, c->csc_orig, nnz);
    double* step1 = c->yr;  // scratch m
    double* step2 = c->xr;  // scratch n
    auto apply_step = [&] {
      k_recip_sqrt_cum<<<c->simple_grid(m), kBlock, 0, c->stream>>>(step1, cum1, (int)m);
      k_recip_sqrt_cum<<<c->simple_grid(n), kBlock, 0, c->stream>>>(step2, cum2, (int)n);
      // working = working.scaled(step1, step2)   (scaling.cpp:57)
      axis_scale(c, true, c->csr_work, c->csr_work, step1, step2);
      axis_scale(c, false, c->csc_work, c->csc_work, step2, step1);
      c->launches += 2;
      CK(cudaGetLastError());
    };
    for (int64_t it = 0; it < ruiz_iterations; ++it) {
      // ruiz_step (scaling.cpp:32-36): inf-norms of the running matrix.
      axis_absmax(c, true, c->csr_work, step1);
      axis_absmax(c, false, c->csc_work, step2);
      apply_step();
    }
    if (pock_chambolle) {
      // pock_chambolle_step (scaling.cpp:38-46)
      const double row_p = 2.0 - alpha;
      axis_pnorm(c, true, c->csr_work, row_p, step1);
      axis_pnorm(c, false, c->csc_work, alpha, step2);
      apply_step();
    }
    // K~ = K .scaled(D1, D2) from the original values in one shot (scaling.cpp:75-76)
    axis_scale(c, true, c->csr_orig, c->csr_work, cum1, cum2);
    axis_scale(c, false, c->csc_orig, c->csc_work, cum2, cum1);
    k_scale_vectors<<<c->simple_grid(n + m), kBlock, 0, c->stream>>>(
        n, m, c->c0, c->l0, c->u0, c->q0, cum1, cum2, c->cw, c->lw, c->uw, c->qw);
    c->launches += 1;
    CK(cudaGetLastError());
    download(c, row_scale, cum1, m);
    download(c, col_scale, cum2, n);
    sync_transfers(c);
    c->kx_valid = false;
  });
}

int folp_gpu_working_stats(folp_gpu_ctx* c, double* max_abs_entry, double* norm_c,
                           double* norm_q) {
  return guarded([&] {
    prep(c);
    const int nb = std::min<int64_t>(c->sms * 4, std::max<int64_t>(1, (c->nnz + kBlock - 1) / kBlock));
    k_absmax_blocks<<<nb, kBlock, 0, c->stream>>>(c->csr_work, c->nnz, c->partials);
    k_absmax_all<<<1, kBlock, 0, c->stream>>>(c->partials, nb, c->res + 0);
    c->launches += 2;
    c->ew(c->n, OpNormSq{c->cw, c->res + 1}, 4);
    c->ew(c->m, OpNormSq{c->qw, c->res + 2}, 5);
    c->fetch_res(3);
    if (max_abs_entry) *max_abs_entry = c->res_h[0];
    if (norm_c) *norm_c = std::sqrt(c->res_h[1]);
    if (norm_q) *norm_q = std::sqrt(c->res_h[2]);
  });
}

int folp_gpu_get_working(folp_gpu_ctx* c, double* csr_values, double* csc_values,
                         double* objective, double* rhs, double* lower, double* upper) {
  return guarded([&] {
    prep(c);
    download(c, csr_values, c->csr_work, c->nnz);
    download(c, csc_values, c->csc_work, c->nnz);
    download(c, objective, c->cw, c->n);
    download(c, rhs, c->qw, c->m);
    download(c, lower, c->lw, c->n);
    download(c, upper, c->uw, c->n);
    sync_transfers(c);
  });
}

int folp_gpu_set_start(folp_gpu_ctx* c, const double* x0, const double* y0) {
  return guarded([&] {
    prep(c);
    upload(c, c->aux_x, x0, c->n);
    upload(c, c->aux_y, y0, c->m);
    k_start_point<<<c->simple_grid(c->n + c->m), kBlock, 0, c->stream>>>(
        c->n, c->m, c->m1, c->aux_x, c->aux_y, c->d1, c->d2, c->lw, c->uw, c->cur_x(),
        c->cur_y(), c->last_x, c->last_y);
    ++c->launches;
    CK(cudaGetLastError());
    zero_average(c);
    refresh_kx(c);
    sync_transfers(c);
  });
}

int folp_gpu_set_point(folp_gpu_ctx* c, int32_t which, const double* x, const double* y) {
  return guarded([&] {
    prep(c);
    upload(c, c->slot_x(which), x, c->n);
    upload(c, c->slot_y(which), y, c->m);
    if (which == FOLP_PT_CURRENT) refresh_kx(c);
    sync_transfers(c);
  });
}

int folp_gpu_get_point(folp_gpu_ctx* c, int32_t which, double* x, double* y) {
  return guarded([&] {
    prep(c);
    download(c, x, c->slot_x(which), c->n);
    download(c, y, c->slot_y(which), c->m);
    sync_transfers(c);
  });
}

int folp_gpu_get_reduced_point(folp_gpu_ctx* c, int32_t which, double* x, double* y) {
  return guarded([&] {
    prep(c);
    k_reduced_point<<<c->simple_grid(c->n + c->m), kBlock, 0, c->stream>>>(
        c->n, c->m, c->slot_x(which), c->slot_y(which), c->d1, c->d2, c->l0, c->u0, c->xr,
        c->yr);
    ++c->launches;
    CK(cudaGetLastError());
    download(c, x, c->xr, c->n);
    download(c, y, c->yr, c->m);
    sync_transfers(c);
  });
}

int folp_gpu_materialize_average(folp_gpu_ctx* c, double* weight) {
  return guarded([&] {
    prep(c);
    enqueue_average(c);
    CK(cudaStreamSynchronize(c->stream));
    if (weight) *weight = c->st_h->avg_weight;
  });
}

int folp_gpu_evaluate(folp_gpu_ctx* c, int32_t which, int32_t raw, folp_gpu_eval* out) {
  return guarded([&] {
    prep(c);
    enqueue_evaluate(c, which, raw, kResEval[0]);
    c->fetch_res(kResUsed);
    read_evaluate(c, kResEval[0], out);
  });
}

int folp_gpu_distance(folp_gpu_ctx* c, int32_t a, int32_t b, double* sx, double* sy) {
  return guarded([&] {
    prep(c);
    enqueue_distance(c, a, b, kResDist[0]);
    c->fetch_res(kResUsed);
    *sx = c->res_h[kResDist[0]];
    *sy = c->res_h[kResDist[0] + 1];
  });
}

int folp_gpu_ndg(folp_gpu_ctx* c, int32_t which, double radius, double omega, double* gap) {
  return guarded([&] {
    prep(c);
    check_ndg_args(radius, omega);
    enqueue_ndg_setup(c, which, 0, omega);
    enqueue_ndg_init(c, 0, -1, radius, omega);
    enqueue_ndg_solve(c, {true, false}, {omega, omega});
    CK(cudaStreamSynchronize(c->stream));
    finish_ndg(c, {true, false}, {omega, omega});
    *gap = c->ndg_h[0].result;
  });
}

int folp_gpu_evaluation_period(folp_gpu_ctx* c, double omega, int32_t want_gaps,
                               folp_gpu_period* out) {
  return guarded([&] {
    prep(c);
    if (want_gaps && !(omega > 0.0)) {
      throw EngineError(FOLP_E_NONPOSITIVE_WEIGHT, "normalized_duality_gap: omega must be > 0");
    }
    const int slots[2] = {FOLP_PT_CURRENT, FOLP_PT_AVERAGE};
    const int cur = c->st_h->cur;
    const bool graphable = !c->ordered && !c->sharded() && want_gaps && c->kx_valid &&
                           c->norms_ready;
    if (graphable && !c->eval_tried[cur]) build_eval_graph(c, cur);
    if (graphable && c->eval_exec[cur] != nullptr) {
      *c->eval_omega_h = omega;
      c->st_h->pending = 0.0;  // the graph clears the device copy after averaging
      CK(cudaGraphLaunch(c->eval_exec[cur], c->stream));
      c->launches += 16;
      CK(cudaStreamSynchronize(c->stream));
    } else {
      enqueue_average(c);
      for (int s = 0; s < 2; ++s) {
        enqueue_evaluate(c, slots[s], 0, kResEval[s], want_gaps ? c->kty_cache(s) : nullptr);
      }
      if (want_gaps) {
        for (int s = 0; s < 2; ++s) {
          enqueue_distance(c, slots[s], FOLP_PT_LAST, kResDist[s]);
          enqueue_ndg_setup(c, slots[s], s, omega, c->kty_cache(s));
          enqueue_ndg_init(c, s, kResDist[s], 0.0, omega);
        }
        enqueue_ndg_solve(c, {true, true}, {omega, omega});
      }
      c->fetch_res(kResUsed);
    }
    read_evaluate(c, kResEval[0], &out->current);
    read_evaluate(c, kResEval[1], &out->average);
    out->avg_weight = c->st_h->avg_weight;
    out->gaps_valid = 0;
    for (int s = 0; s < 2; ++s) {
      out->dist_x[s] = want_gaps ? c->res_h[kResDist[s]] : 0.0;
      out->dist_y[s] = want_gaps ? c->res_h[kResDist[s] + 1] : 0.0;
      out->gap[s] = 0.0;
    }
    // a non-finite or out-of-cone point ends the solve before any gap is used
    const bool bad = out->current.nonfinite || out->current.infinite_product ||
                     out->average.nonfinite || out->average.infinite_product;
    if (!want_gaps || bad) return;
    finish_ndg(c, {true, true}, {omega, omega});
    for (int s = 0; s < 2; ++s) {
      out->gap[s] = c->ndg_h[s].result;
      c->ndg_count += 1;
      c->ndg_passes += c->ndg_h[s].passes;
      c->ndg_grid_passes += c->ndg_h[s].grid_passes;
      c->ndg_levels += c->ndg_h[s].it;
    }
    out->gaps_valid = 1;
  });
}

int folp_gpu_restart_commit(folp_gpu_ctx* c, int32_t which, double radius, double omega,
                            double* reference_gap) {
  return guarded([&] {
    prep(c);
    const bool gap = radius > 0.0;
    if (gap) {
      check_ndg_args(radius, omega);
      enqueue_ndg_setup(c, which, 0, omega);
      enqueue_ndg_init(c, 0, -1, radius, omega);
      enqueue_ndg_solve(c, {true, false}, {omega, omega});
    }
    // the passes read only the scratch set, so the restart copies go behind them
    enqueue_restart(c, which, 1);
    CK(cudaStreamSynchronize(c->stream));
    if (gap) finish_ndg(c, {true, false}, {omega, omega});
    if (reference_gap) *reference_gap = gap ? c->ndg_h[0].result : 0.0;
  });
}

int folp_gpu_restart_to(folp_gpu_ctx* c, int32_t which, int32_t reset_average) {
  return guarded([&] {
    prep(c);
    enqueue_restart(c, which, reset_average);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int folp_gpu_mark_last(folp_gpu_ctx* c) {
  return guarded([&] {
    prep(c);
    copy_d2d(c, c->last_x, c->cur_x(), c->n);
    copy_d2d(c, c->last_y, c->cur_y(), c->m);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int folp_gpu_run_chunk(folp_gpu_ctx* c, folp_gpu_loop* loop) {
  return guarded([&] {
    set_device(c);
    if (loop->target < 1) throw std::invalid_argument("run_chunk: target must be >= 1");
    const int policy = loop->policy;
    if (policy != FOLP_STEP_ADAPTIVE && policy != FOLP_STEP_CONSTANT &&
        policy != FOLP_STEP_MALITSKY_POCK) {
      throw std::invalid_argument("run_chunk: unknown step policy");
    }
    if (policy != FOLP_STEP_MALITSKY_POCK && !c->kx_valid) refresh_kx(c);
    ensure_blocked(c);  // after rescaling: the working values are final
    if (!c->bounds_checked) check_uniform_bounds(c);
    if (c->sell && !c->sell_packed) {
      pack_sell(c, c->rows_sell);
      c->sell_packed = true;
    }
    if (loop->target > c->table_cap) {
      throw std::invalid_argument("run_chunk: target above the factor-table capacity");
    }
    if (loop->policy == FOLP_STEP_ADAPTIVE) {
      std::memcpy(c->red_h, loop->reduction, loop->target * sizeof(double));
      std::memcpy(c->grow_h, loop->growth, loop->target * sizeof(double));
      CK(cudaMemcpyAsync(c->red_d, c->red_h, loop->target * sizeof(double),
                         cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->grow_d, c->grow_h, loop->target * sizeof(double),
                         cudaMemcpyHostToDevice, c->stream));
    }
    DevState* st = c->st_h;
    st->running = 1;
    st->status = kRunning;
    st->policy = loop->policy;
    st->target = loop->target;
    st->accepted = 0;
    st->k_total = loop->k_total;
    st->k_chunk0 = loop->k_total;
    st->t_inner = loop->t_inner;
    st->trials_iter = 0;
    st->step_trials = loop->step_trials;
    st->violations = loop->violations;
    st->ledger_k = loop->ledger_k;
    st->ledger_kt = loop->ledger_kt;
    st->iteration_limit = loop->iteration_limit;
    st->kkt_pass_limit = loop->kkt_pass_limit;
    st->omega = loop->omega;
    st->eta = loop->eta;
    st->eta_hat = loop->eta;
    st->slots = 0;
    st->mp_theta = loop->theta;
    st->mp_break = loop->mp_breaking_factor;
    st->mp_down = loop->mp_downscaling_factor;
    st->mp_interp = loop->mp_interpolation_coefficient;
    c->push_state();
    if (c->sharded() && policy == FOLP_STEP_MALITSKY_POCK) {
      throw std::invalid_argument("sharded solve: the Malitsky-Pock policy runs on one GPU only");
    }
    if (!c->sharded() && !c->small_loop && !c->graph_tried[policy]) build_chunk_graph(c, policy);
    const int per_slot = policy == FOLP_STEP_MALITSKY_POCK ? 4 : 2;
    if (c->profiling) CK(cudaEventRecord(c->ev0, c->stream));
    if (c->small_loop && policy != FOLP_STEP_MALITSKY_POCK) {
      // small problem: the whole chunk in one cluster launch (k_chunk_cluster)
      const LoopBufs b = c->loop_bufs(cudaGraphConditionalHandle{}, 0);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kSmallCluster);
      cfg.blockDim = dim3(kSmallThreads);
      cfg.stream = c->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kSmallCluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_chunk_cluster<kSmallThreads>, b, c->rows.sp, c->cols.sp,
                            static_cast<const double*>(c->csr_work),
                            static_cast<const double*>(c->csc_work), c->small_multi));
      ++c->launches;
    } else if (c->sharded()) {
      if (!c->shard_values_ready) {  // K~ values of the local CSC, after rescaling
        k_gather_values<<<c->simple_grid(c->lnnz), kBlock, 0, c->stream>>>(
            c->lcsc_val, c->csc_work, c->lcsc_pos, c->lnnz);
        ++c->launches;
        CK(cudaGetLastError());
        c->shard_values_ready = true;
      }
      const LoopBufs b = c->loop_bufs(cudaGraphConditionalHandle{}, 0);
      int64_t remaining = loop->target;
      for (;;) {
        for (int64_t s = 0; s < remaining; ++s) launch_shard_slot(c, b);
        CK(cudaMemcpyAsync(st, c->st_d, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (!st->running) break;
        remaining = st->target - st->accepted;
      }
      c->rows_dirty = true;
    } else if (c->graph_ok[policy]) {
      CK(cudaGraphLaunch(c->chunk_exec[policy], c->stream));
    } else {
      // Plain stream launches: enough slots for the target plus a few
      // retries, then look at the state and continue if needed.
      const LoopBufs b = c->loop_bufs(cudaGraphConditionalHandle{}, 0);
      int64_t remaining = loop->target;
      for (;;) {
        for (int64_t s = 0; s < remaining + 2; ++s) launch_slot(c, policy, b);
        c->launches -= per_slot * (remaining + 2);
        CK(cudaMemcpyAsync(st, c->st_d, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (!st->running) break;
        remaining = st->target - st->accepted;
      }
    }
    if (c->profiling) CK(cudaEventRecord(c->ev1, c->stream));
    c->pull_state();
    if (!c->sharded() && !(c->small_loop && policy != FOLP_STEP_MALITSKY_POCK)) {
      // graph: whole body iterations (a stopped slot still launches, and exits)
      const int64_t bs = c->graph_ok[policy] ? c->body_slots[policy] : 1;
      c->launches += per_slot * ((st->slots + bs - 1) / bs) * bs;
    }
    if (policy == FOLP_STEP_MALITSKY_POCK) c->kx_valid = false;  // Kx cache not kept
    if (c->profiling) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      c->chunk_ms_total += ms;
      c->chunk_slots_total += st->slots;
    }
    loop->status = st->status;
    loop->accepted = st->accepted;
    loop->k_total = st->k_total;
    loop->t_inner = st->t_inner;
    loop->step_trials = st->step_trials;
    loop->violations = st->violations;
    loop->ledger_k = st->ledger_k;
    loop->ledger_kt = st->ledger_kt;
    loop->eta = st->policy == FOLP_STEP_ADAPTIVE ? st->eta_hat
              : st->policy == FOLP_STEP_MALITSKY_POCK ? st->eta
                                                      : loop->eta;
    loop->theta = st->mp_theta;
    loop->last_eta_used = st->last_eta_used;
    loop->avg_weight = st->avg_weight;
    loop->last_movement = st->movement;
    loop->last_cross = st->cross;
    loop->slots = st->slots;
  });
}

// Test / measurement entry of the exact parallel fold (exactfold.cuh): up to
// kFoldMaxJobs folds of host arrays in one cooperative launch; reps > 0
// times `reps` launches with CUDA events (ms = average per launch).
int folp_gpu_test_exact_fold(int32_t device, int32_t jobs, const double* const* terms,
                             const int64_t* counts, const double* inits, const int32_t* init_from,
                             const double* init_div, int32_t grid, int32_t reps, double* results,
                             double* ms) {
  return guarded([&] {
    if (jobs < 1 || jobs > kFoldMaxJobs) throw std::invalid_argument("test_exact_fold: 1..4 jobs");
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<void*> mem;
    auto dev = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      mem.push_back(p);
      return p;
    };
    FoldJobs fj{};
    fj.count = jobs;
    for (int j = 0; j < jobs; ++j) {
      double* d = static_cast<double*>(dev(counts[j] * sizeof(double)));
      if (counts[j] > 0) CK(cudaMemcpyAsync(d, terms[j], counts[j] * sizeof(double), cudaMemcpyHostToDevice, st));
      fj.job[j] = FoldJob{d, counts[j], inits[j], init_from ? init_from[j] : -1,
                          init_div ? init_div[j] : 1.0, nullptr, nullptr};
      if (fj.job[j].init_from >= j) throw std::invalid_argument("test_exact_fold: init_from must precede");
    }
    int dev_sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
    auto fn = k_exact_fold<FoldToMemory>;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(kFoldDynSmem)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFoldBlock, kFoldDynSmem));
    const int cap = dev_sms * per_sm;
    const int G = std::min(grid > 0 ? std::min(grid, cap) : cap, kFoldMaxCtas);
    FoldScratch sc{};
    sc.cap = G;
    sc.cta_sum = static_cast<double*>(dev(sizeof(double) * kFoldMaxJobs * G));
    sc.cta_abs = static_cast<double*>(dev(sizeof(double) * kFoldMaxJobs * G));
    sc.cta_ntot = static_cast<unsigned long long*>(dev(sizeof(unsigned long long) * kFoldMaxJobs * G));
    sc.cta_nbp = static_cast<int*>(dev(sizeof(int) * kFoldMaxJobs * G));
    sc.cta_bad = static_cast<int*>(dev(sizeof(int) * kFoldMaxJobs * G));
    sc.cta_flag = static_cast<int*>(dev(sizeof(int) * G));
    sc.cta_laste = static_cast<int*>(dev(sizeof(int) * kFoldMaxJobs * G));
    sc.cta_lastc = static_cast<unsigned long long*>(dev(sizeof(unsigned long long) * kFoldMaxJobs * G));
    sc.bps = static_cast<FoldBp*>(dev(sizeof(FoldBp) * kFoldMaxJobs * G * kFoldBpCap));
    sc.chain = static_cast<FoldEntry*>(dev(sizeof(FoldEntry) * kFoldMaxJobs * (static_cast<size_t>(G) * kFoldBpCap + 1)));
    sc.results = static_cast<double*>(dev(sizeof(double) * kFoldMaxJobs));
    sc.counter = static_cast<unsigned*>(dev(sizeof(unsigned)));
    CK(cudaMemsetAsync(sc.counter, 0, sizeof(unsigned), st));
    FoldToMemory fin{};
    void* args[] = {&fj, &sc, &fin};
    auto launch = [&] {
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(G), dim3(kFoldBlock), args,
                                     kFoldDynSmem, st));
    };
    launch();
    CK(cudaMemcpyAsync(results, sc.results, sizeof(double) * jobs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (reps > 0 && ms != nullptr) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < reps; ++r) launch();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, e0, e1));
      *ms = static_cast<double>(t) / reps;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    if (const char* env = std::getenv("FOLP_FOLD_TIMES")) {
      (void)env;
      unsigned long long tt[8];
      CK(cudaMemcpyFromSymbol(tt, g_fold_times, sizeof tt));
      std::fprintf(stderr, "[fold times us] phase1 %.2f sync %.2f phase2 %.2f ticket %.2f lists %.2f replay %.2f\n",
                   1e-3 * (tt[1] - tt[0]), 1e-3 * (tt[2] - tt[1]), 1e-3 * (tt[3] - tt[2]),
                   1e-3 * (double)(long long)(tt[4] - tt[3]), 1e-3 * (tt[5] - tt[4]), 1e-3 * (tt[6] - tt[5]));
    }
    for (void* p : mem) cudaFree(p);
    cudaStreamDestroy(st);
  });
}

int folp_gpu_spectral_norm(folp_gpu_ctx* c, const double* v0, double relative_tol,
                           int64_t max_iterations, double* norm, int64_t* multiplies) {
  return guarded([&] {
    prep(c);
    double* v = c->aux_x;
    double* w = c->aux_y;
    double* s = c->xr;
    upload(c, v, v0, c->n);
    sync_transfers(c);
    double lambda = 0.0;
    for (int64_t it = 0; it < max_iterations; ++it) {
      product(c, false, true, v, w);
      EpiStoreDotNorm e{w, v, s, c->res + 40};
      c->seg(c->cols, c->csc_work, e, 1);
      if (multiplies) *multiplies += 2;
      c->fetch_res(42);
      const double next = c->res_h[40];
      const double snorm = std::sqrt(c->res_h[41]);
      if (snorm == 0.0) {
        *norm = 0.0;
        return;
      }
      k_div_scalar<<<c->simple_grid(c->n), kBlock, 0, c->stream>>>(v, s, c->n, c->res + 41);
      ++c->launches;
      const bool converged = it > 0 && std::fabs(next - lambda) <= relative_tol * std::fabs(next);
      lambda = next;
      if (converged) break;
    }
    *norm = std::sqrt(std::max(lambda, 0.0));
  });
}

int folp_gpu_multiply(folp_gpu_ctx* c, int32_t working, const double* xh, double* out) {
  return guarded([&] {
    prep(c);
    upload(c, c->aux_x, xh, c->n);
    product(c, false, working != 0, c->aux_x, c->kx_aux);
    download(c, out, c->kx_aux, c->m);
    sync_transfers(c);
  });
}

int folp_gpu_multiply_transpose(folp_gpu_ctx* c, int32_t working, const double* yh, double* out) {
  return guarded([&] {
    prep(c);
    upload(c, c->aux_y, yh, c->m);
    product(c, true, working != 0, c->aux_y, c->xr);
    download(c, out, c->xr, c->n);
    sync_transfers(c);
  });
}

int folp_gpu_all_finite(folp_gpu_ctx* c, int32_t which, int32_t* finite) {
  return guarded([&] {
    prep(c);
    c->ew(c->n + c->m, OpCountNonFinite{c->n, c->slot_x(which), c->slot_y(which), c->res + 44}, 4);
    c->fetch_res(45);
    *finite = c->res_h[44] == 0.0 ? 1 : 0;
  });
}

int folp_gpu_axis_norms(folp_gpu_ctx* c, int32_t axis, double p, int32_t working, double* out) {
  return guarded([&] {
    prep(c);
    const bool rows = axis == 0;
    const int S = static_cast<int>(rows ? c->m : c->n);
    const int* ptr = rows ? c->csr_ptr : c->csc_ptr;
    const double* val = rows ? (working ? c->csr_work : c->csr_orig)
                             : (working ? c->csc_work : c->csc_orig);
    double* dst = rows ? c->yr : c->xr;
    (void)ptr;
    axis_pnorm(c, rows, val, p, dst);
    download(c, out, dst, S);
    sync_transfers(c);
  });
}

int folp_gpu_max_abs_entry(folp_gpu_ctx* c, int32_t working, double* out) {
  return guarded([&] {
    prep(c);
    const int nb = std::min<int64_t>(c->sms * 4, std::max<int64_t>(1, (c->nnz + kBlock - 1) / kBlock));
    k_absmax_blocks<<<nb, kBlock, 0, c->stream>>>(working ? c->csr_work : c->csr_orig, c->nnz,
                                                  c->partials);
    k_absmax_all<<<1, kBlock, 0, c->stream>>>(c->partials, nb, c->res + 46);
    c->launches += 2;
    c->fetch_res(47);
    *out = c->res_h[46];
  });
}

int64_t folp_gpu_launch_count(const folp_gpu_ctx* c) { return c->launches; }

int folp_gpu_debug_warp_times(folp_gpu_ctx* c, int32_t slot, uint64_t* out, int32_t max_warps) {
  return guarded([&] {
#ifdef FOLP_WARP_TIMES
    if (slot < 0 || slot > 1 || max_warps < 0) throw std::invalid_argument("debug_warp_times: slot");
    const int w = std::min(max_warps, kTraceWarps);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpyFromSymbol(out, g_warp_times, static_cast<size_t>(w) * 4 * sizeof(uint64_t),
                            static_cast<size_t>(slot) * kTraceWarps * 4 * sizeof(uint64_t)));
    if (max_warps > kTraceWarps) {  // + the last CTA's tail stamps
      CK(cudaMemcpyFromSymbol(out + 4 * kTraceWarps, g_tail_times, 3 * sizeof(uint64_t),
                              static_cast<size_t>(slot) * 4 * sizeof(uint64_t)));
    }
#else
    (void)c; (void)slot; (void)out; (void)max_warps;
    throw std::invalid_argument("debug_warp_times: build with -DFOLP_WARP_TIMES");
#endif
  });
}

void folp_gpu_set_default_reduction(int32_t ordered) { g_default_ordered = ordered != 0; }

int32_t folp_gpu_reduction_ordered(const folp_gpu_ctx* c) { return c->ordered ? 1 : 0; }

int32_t folp_gpu_default_reduction(void) {
  if (const char* env = std::getenv("FOLP_REDUCTION")) return std::strcmp(env, "ordered") == 0 ? 1 : 0;
  return g_default_ordered ? 1 : 0;
}


int folp_gpu_set_profiling(folp_gpu_ctx* c, int32_t enabled) {
  c->profiling = enabled != 0;
  c->chunk_ms_total = 0.0;
  c->chunk_slots_total = 0;
  return FOLP_OK;
}

int folp_gpu_chunk_timing(folp_gpu_ctx* c, double* chunk_ms, int64_t* slots) {
  if (chunk_ms) *chunk_ms = c->chunk_ms_total;
  if (slots) *slots = c->chunk_slots_total;
  return FOLP_OK;
}

int folp_gpu_timer_start(folp_gpu_ctx* c) {
  return guarded([&] {
    prep(c);
    CK(cudaEventRecord(c->tev0, c->stream));
  });
}

int folp_gpu_timer_stop(folp_gpu_ctx* c, double* ms) {
  return guarded([&] {
    prep(c);
    CK(cudaEventRecord(c->tev1, c->stream));
    CK(cudaEventSynchronize(c->tev1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    *ms = f;
  });
}

// ---------------------------------------------------------------------
// Row shards.
int folp_gpu_nccl_unique_id(unsigned char* out) {
  return guarded([&] {
    ncclUniqueId id;
    NCK(nccl_api().get_unique_id(&id));
    static_assert(sizeof(id) == FOLP_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
  });
}

int folp_gpu_loopback_create(int32_t world, void** out) {
  *out = nullptr;
  return guarded([&] {
    if (world < 1) throw std::invalid_argument("loopback group: world must be >= 1");
    *out = new LoopbackGroup(world);
  });
}

void folp_gpu_loopback_destroy(void* group) { delete static_cast<LoopbackGroup*>(group); }

int folp_gpu_shard_rows(int64_t m, const int64_t* row_start, int32_t world, int64_t* bounds) {
  return guarded([&] {
    if (world < 1 || m < 0) throw std::invalid_argument("shard_rows: bad arguments");
    const std::vector<int64_t> b = shard_rows(m, row_start, world);
    std::copy(b.begin(), b.end(), bounds);
  });
}

int folp_gpu_shard_local_csc(int64_t n, const int64_t* col_start, const int64_t* col_rows,
                             int64_t r0, int64_t r1, int64_t* lptr, int64_t* pos,
                             int64_t pos_capacity, int64_t* lnnz) {
  return guarded([&] {
    std::vector<int64_t> lp, ps;
    shard_local_csc(n, col_start, col_rows, r0, r1, lp, ps);
    *lnnz = static_cast<int64_t>(ps.size());
    std::copy(lp.begin(), lp.end(), lptr);
    if (pos != nullptr) {
      if (static_cast<int64_t>(ps.size()) > pos_capacity) {
        throw std::invalid_argument("shard_local_csc: pos capacity too small");
      }
      std::copy(ps.begin(), ps.end(), pos);
    }
  });
}

int folp_gpu_shard_local_csr(int64_t m, const int64_t* col_start, const int64_t* col_rows,
                             int64_t c0, int64_t c1, int64_t* lptr, int64_t* pos,
                             int64_t pos_capacity, int64_t* lnnz) {
  return guarded([&] {
    std::vector<int64_t> lp, ps;
    shard_local_csr(m, col_start, col_rows, c0, c1, lp, ps);
    *lnnz = static_cast<int64_t>(ps.size());
    std::copy(lp.begin(), lp.end(), lptr);
    if (pos != nullptr) {
      if (static_cast<int64_t>(ps.size()) > pos_capacity) {
        throw std::invalid_argument("shard_local_csr: pos capacity too small");
      }
      std::copy(ps.begin(), ps.end(), pos);
    }
  });
}

int folp_gpu_shard_attach(folp_gpu_ctx* c, const folp_gpu_shard* spec, const int64_t* row_start,
                          const int64_t* col_start, const int64_t* col_rows) {
  return guarded([&] {
    set_device(c);
    if (c->sharded()) throw std::invalid_argument("shard_attach: context already sharded");
    if (spec == nullptr || spec->world < 1 || spec->rank < 0 || spec->rank >= spec->world) {
      throw std::invalid_argument("shard_attach: bad rank / world");
    }
    if (c->ordered) {
      throw std::invalid_argument("shard_attach: the ordered reduction mode is single-GPU only");
    }
    if (row_start == nullptr || col_start == nullptr || col_rows == nullptr) {
      throw std::invalid_argument("shard_attach: CSR row starts and CSC arrays required");
    }
    if (spec->backend == FOLP_SHARD_NCCL) {
      c->comm = std::make_unique<NcclComm>(spec->nccl_id, spec->rank, spec->world);
    } else if (spec->backend == FOLP_SHARD_LOOPBACK) {
      auto* g = static_cast<LoopbackGroup*>(spec->loopback);
      if (g == nullptr || g->world != spec->world) {
        throw std::invalid_argument("shard_attach: loopback group missing or of another size");
      }
      c->comm = std::make_unique<LoopbackComm>(g, spec->rank);
    } else {
      throw std::invalid_argument("shard_attach: unknown backend");
    }
    const int64_t m = c->m, n = c->n;
    int part = spec->partition;
    if (part == FOLP_SHARD_AUTO) part = (m + 2 < n) ? FOLP_SHARD_COLS : FOLP_SHARD_ROWS;
    if (part != FOLP_SHARD_ROWS && part != FOLP_SHARD_COLS) {
      throw std::invalid_argument("shard_attach: unknown partition");
    }
    c->col_part = part == FOLP_SHARD_COLS;
    // Both partitions keep one plan over the full matrix restricted to the
    // own range (CSR rows, or CSC columns) and one over the local block in
    // the other orientation (lcsc_* arrays: entries of the block and their
    // full-CSC positions, for the value gather after rescaling).
    const int64_t axis = c->col_part ? n : m;
    c->shard_bounds = shard_rows(axis, c->col_part ? col_start : row_start, spec->world);
    c->r0 = c->shard_bounds[spec->rank];
    c->r1 = c->shard_bounds[spec->rank + 1];
    std::vector<int64_t> lptr, pos;
    if (c->col_part) {
      build_plan(c, col_start, c->r1, c->nnz, c->csc_ptr, c->csc_row, c->lcols, c->r0);
      shard_local_csr(m, col_start, col_rows, c->r0, c->r1, lptr, pos);
    } else {
      build_plan(c, row_start, c->r1, c->nnz, c->csr_ptr, c->csr_col, c->lrows, c->r0);
      shard_local_csc(n, col_start, col_rows, c->r0, c->r1, lptr, pos);
    }
    c->lnnz = static_cast<int64_t>(pos.size());
    const int64_t other = c->col_part ? m : n;
    std::vector<int> lptr32(lptr.begin(), lptr.end()), pos32(pos.size()), idx32(pos.size());
    for (size_t k = 0; k < pos.size(); ++k) pos32[k] = static_cast<int>(pos[k]);
    if (c->col_part) {  // the column of each local entry, from the CSC range it sits in
      const int64_t base = col_start[c->r0];
      std::vector<int> col_of(static_cast<size_t>(col_start[c->r1] - base));
      for (int64_t j = c->r0; j < c->r1; ++j) {
        for (int64_t k = col_start[j]; k < col_start[j + 1]; ++k) {
          col_of[static_cast<size_t>(k - base)] = static_cast<int>(j);
        }
      }
      for (size_t k = 0; k < pos.size(); ++k) idx32[k] = col_of[static_cast<size_t>(pos[k] - base)];
    } else {
      for (size_t k = 0; k < pos.size(); ++k) idx32[k] = static_cast<int>(col_rows[pos[k]]);
    }
    c->lcsc_ptr = c->alloc<int>(other + 1);
    c->lcsc_row = c->alloc<int>(c->lnnz + 8);
    c->lcsc_pos = c->alloc<int>(c->lnnz + 1);
    c->lcsc_val = c->alloc<double>(c->lnnz + 8);
    CK(cudaMemcpy(c->lcsc_ptr, lptr32.data(), (other + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (c->lnnz > 0) {
      CK(cudaMemcpy(c->lcsc_row, idx32.data(), c->lnnz * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->lcsc_pos, pos32.data(), c->lnnz * sizeof(int), cudaMemcpyHostToDevice));
    }
    build_plan(c, lptr.data(), other, c->lnnz, c->lcsc_ptr, c->lcsc_row,
               c->col_part ? c->lrows : c->lcols);
    // row partition: partial K'y [n]; column partition: partial Kx' [m] + sx, bad
    c->kty_part = c->alloc<double>(std::max<int64_t>(c->col_part ? m + 2 : n, 1));
    // FOLP_SHARD_EXCHANGE=peer|collective; default peer on the loopback
    // group, collective (NCCL all-reduce) on NCCL until the P2P path has run
    // on a multi-GPU node
    {
      const char* env = std::getenv("FOLP_SHARD_EXCHANGE");
      bool peer = spec->backend == FOLP_SHARD_LOOPBACK;
      if (env != nullptr && std::strcmp(env, "peer") == 0) peer = true;
      if (env != nullptr && std::strcmp(env, "collective") == 0) peer = false;
      // column partition over the peer exchange: the dual epilogue runs on
      // each rank's own rows (FOLP_SHARD_EPILOGUE=replicated keeps it on
      // every rank for all m rows)
      const char* epi = std::getenv("FOLP_SHARD_EPILOGUE");
      c->pdual = peer && spec->world > 1 && !(epi != nullptr && std::strcmp(epi, "replicated") == 0);
      // the epilogue's axis: rows (column partition) or columns (row partition)
      const int64_t ax = c->col_part ? m : n;
      if (peer) c->comm->peer_setup(c->col_part ? m + (c->pdual ? 8 : 2) : n + (c->pdual ? 8 : 0));
      if (c->pdual) {
        const int W = spec->world;
        c->pd_chunk = (ax + W - 1) / W;
        c->pd_bounds.assign(static_cast<size_t>(W) + 1, 0);
        for (int r = 0; r <= W; ++r) c->pd_bounds[r] = std::min<int64_t>(ax, r * c->pd_chunk);
        std::vector<double*> tab(2 * static_cast<size_t>(W));
        for (int par = 0; par < 2; ++par) {
          const std::vector<double*> ptrs = c->comm->exchange_pointers(c->col_part ? c->y[par] : c->x[par]);
          for (int r = 0; r < W; ++r) tab[par * W + r] = ptrs[r];
        }
        c->pd_vdst = c->alloc<double*>(tab.size());
        CK(cudaMemcpy(c->pd_vdst, tab.data(), tab.size() * sizeof(double*), cudaMemcpyHostToDevice));
        if (std::getenv("FOLP_TIMING") != nullptr) {
          std::fprintf(stderr, "[folp timing] shard %d/%d: partitioned %s epilogue, %s [%lld, %lld)\n",
                       spec->rank, W, c->col_part ? "dual" : "primal", c->col_part ? "rows" : "columns",
                       static_cast<long long>(c->pd_bounds[spec->rank]),
                       static_cast<long long>(c->pd_bounds[spec->rank + 1]));
        }
      }
    }
    c->shard_sums = c->alloc<double>(4);
    c->shard_values_ready = false;
    c->rows_dirty = false;
  });
}

int folp_gpu_shard_max(folp_gpu_ctx* c, double* value) {
  return guarded([&] {
    set_device(c);
    if (c->sharded()) *value = c->comm->max_scalar(*value, c->stream);
  });
}

int folp_gpu_shard_partition(folp_gpu_ctx* c, int32_t* partition) {
  return guarded([&] {
    *partition = c->sharded() && c->col_part ? FOLP_SHARD_COLS : FOLP_SHARD_ROWS;
  });
}

int folp_gpu_shard_info(folp_gpu_ctx* c, int32_t* rank, int32_t* world, int64_t* r0, int64_t* r1,
                        int64_t* local_nnz) {
  return guarded([&] {
    *rank = c->sharded() ? c->comm->rank : 0;
    *world = c->sharded() ? c->comm->world : 1;
    *r0 = c->sharded() ? c->r0 : 0;
    *r1 = c->sharded() ? c->r1 : (c->col_part ? c->n : c->m);
    *local_nnz = c->sharded() ? c->lnnz : c->nnz;
  });
}

}  // extern "C"
