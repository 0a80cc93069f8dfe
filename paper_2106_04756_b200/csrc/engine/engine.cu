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
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "folp_gpu.h"
#include "ops.cuh"

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

// ---------------------------------------------------------------------
// Collectives of the row-sharded loop.  One process (or, for
// the loopback group, one host thread) per shard; every shard calls the same
// collectives in the same order because every shard takes the same
// decisions.
struct ShardComm {
  int rank = 0, world = 1;
  virtual ~ShardComm() = default;
  // in-place sum over the shards, identical result on every shard
  virtual void allreduce_sum(double* buf, int64_t count, cudaStream_t s) = 0;
  // in-place: every shard receives root's buf[0..count)
  virtual void broadcast(double* buf, int64_t count, int root, cudaStream_t s) = 0;
  // host scalar max over the shards (wall-clock limit checks)
  virtual double max_scalar(double v, cudaStream_t s) = 0;
  // in-place: rows [bounds[r], bounds[r+1]) of buf from shard r, for every r
  virtual void gather_rows(double* buf, const std::vector<int64_t>& bounds, cudaStream_t s) = 0;
};

// NCCL, loaded at run time: the single-GPU path has no NCCL dependency, and
// a process that already loaded torch's libnccl.so.2 shares it.
struct NcclApi {
  void* handle = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    api.handle = h;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.bcast = reinterpret_cast<decltype(api.bcast)>(dlsym(h, "ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (api.handle == nullptr || api.comm_init_rank == nullptr || api.all_reduce == nullptr ||
      api.bcast == nullptr || api.get_unique_id == nullptr) {
    throw EngineError(FOLP_E_RUNTIME, "NCCL (libnccl.so.2) is not loadable");
  }
  return api;
}

#define NCK(call)                                                                  \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess) {                                                       \
      throw EngineError(FOLP_E_RUNTIME, std::string(#call) + ": " +                \
                                            nccl_api().error_string(r_));          \
    }                                                                              \
  } while (0)

struct NcclComm final : ShardComm {
  ncclComm_t comm = nullptr;
  double* scratch = nullptr;
  NcclComm(const unsigned char* id_bytes, int r, int w) {
    rank = r;
    world = w;
    const NcclApi& api = nccl_api();
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    NCK(api.comm_init_rank(&comm, w, id, r));
    CK(cudaMalloc(&scratch, sizeof(double)));
  }
  ~NcclComm() override {
    if (scratch) cudaFree(scratch);
    if (comm) nccl_api().comm_destroy(comm);
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t s) override {
    if (count > 0) NCK(nccl_api().all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm, s));
  }
  void broadcast(double* buf, int64_t count, int root, cudaStream_t s) override {
    if (count > 0) NCK(nccl_api().bcast(buf, buf, count, ncclFloat64, root, comm, s));
  }
  void gather_rows(double* buf, const std::vector<int64_t>& bounds, cudaStream_t s) override {
    const NcclApi& api = nccl_api();
    NCK(api.group_start());
    for (int r = 0; r < world; ++r) {
      const int64_t count = bounds[r + 1] - bounds[r];
      if (count > 0) {
        NCK(api.bcast(buf + bounds[r], buf + bounds[r], count, ncclFloat64, r, comm, s));
      }
    }
    NCK(api.group_end());
  }
  double max_scalar(double v, cudaStream_t s) override {
    CK(cudaMemcpyAsync(scratch, &v, sizeof(double), cudaMemcpyHostToDevice, s));
    NCK(nccl_api().all_reduce(scratch, scratch, 1, ncclFloat64, ncclMax, comm, s));
    CK(cudaMemcpyAsync(&v, scratch, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
  }
};

// In-process group: W shards driven by W host threads of one process, all
// on one device (parity tests of the sharded schedule on a single GPU).
// Every collective synchronizes the caller's stream first and exchanges
// through plain device copies, so no kernel ever waits on another shard.
__global__ void k_sum_shards(double* const* parts, int world, int64_t count, double* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = parts[0][i];
    for (int r = 1; r < world; ++r) s += parts[r][i];
    out[i] = s;
  }
}

struct LoopbackGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  bool poisoned = false;  // a shard left early (error): the others must not wait forever
  std::vector<double*> ptrs;
  std::vector<double> scalars;
  explicit LoopbackGroup(int w) : world(w), ptrs(w, nullptr), scalars(w, 0.0) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || poisoned; });
      if (generation == gen) {
        throw EngineError(FOLP_E_RUNTIME, "loopback shard group: another shard failed");
      }
    }
  }
  void poison() {
    std::lock_guard<std::mutex> lk(mu);
    poisoned = true;
    cv.notify_all();
  }
};

struct LoopbackComm final : ShardComm {
  LoopbackGroup* g;
  double** d_ptrs = nullptr;
  double* d_sum = nullptr;
  int64_t sum_cap = 0;
  LoopbackComm(LoopbackGroup* group, int r) : g(group) {
    rank = r;
    world = group->world;
  }
  ~LoopbackComm() override {
    // a shard that leaves releases anyone still waiting (after the last
    // collective nobody waits; before it, waiting would never end)
    g->poison();
    if (d_ptrs) cudaFree(d_ptrs);
    if (d_sum) cudaFree(d_sum);
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    g->ptrs[rank] = buf;
    g->barrier();
    if (rank == 0 && count > 0) {
      if (d_ptrs == nullptr) CK(cudaMalloc(&d_ptrs, world * sizeof(double*)));
      if (sum_cap < count) {
        if (d_sum) cudaFree(d_sum);
        CK(cudaMalloc(&d_sum, count * sizeof(double)));
        sum_cap = count;
      }
      CK(cudaMemcpyAsync(d_ptrs, g->ptrs.data(), world * sizeof(double*), cudaMemcpyHostToDevice, s));
      k_sum_shards<<<static_cast<int>(std::min<int64_t>((count + 255) / 256, 1184)), 256, 0, s>>>(
          d_ptrs, world, count, d_sum);
      CK(cudaGetLastError());
      for (int r = 0; r < world; ++r) {
        CK(cudaMemcpyAsync(g->ptrs[r], d_sum, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
      }
      CK(cudaStreamSynchronize(s));
    }
    g->barrier();
  }
  void broadcast(double* buf, int64_t count, int root, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    g->ptrs[rank] = buf;
    g->barrier();
    if (rank != root && count > 0) {
      CK(cudaMemcpyAsync(buf, g->ptrs[root], count * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
    }
    g->barrier();
  }
  void gather_rows(double* buf, const std::vector<int64_t>& bounds, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    g->ptrs[rank] = buf;
    g->barrier();
    for (int r = 0; r < world; ++r) {
      const int64_t count = bounds[r + 1] - bounds[r];
      if (r != rank && count > 0) {
        CK(cudaMemcpyAsync(buf + bounds[r], g->ptrs[r] + bounds[r], count * sizeof(double),
                           cudaMemcpyDeviceToDevice, s));
      }
    }
    CK(cudaStreamSynchronize(s));
    g->barrier();
  }
  double max_scalar(double v, cudaStream_t) override {
    g->scalars[rank] = v;
    g->barrier();
    double m = g->scalars[0];
    for (int r = 1; r < world; ++r) m = std::max(m, g->scalars[r]);
    g->barrier();
    return m;
  }
};


// Process-wide cache of device and pinned host blocks keyed by (device,
// bytes).  A solve context holds ~60 buffers; repeated solves of one size
// (bench e2e, batched solves, the session API) reuse them instead of paying
// cudaMalloc / cudaFree / cudaMallocHost every time (~100 ms per context on
// B200 for config 2).  Cached bytes are capped; beyond the cap blocks are
// released.  Blocks come back uninitialized, like cudaMalloc's.
struct BlockCache {
  std::mutex mu;
  std::unordered_multimap<uint64_t, void*> free_dev, free_host;
  std::unordered_map<void*, uint64_t> live;
  uint64_t cached_bytes = 0;
  static constexpr uint64_t kCap = uint64_t(16) << 30;
};
BlockCache& block_cache() {
  static BlockCache* bc = new BlockCache();  // process lifetime
  return *bc;
}
uint64_t block_key(size_t bytes, bool host) {
  int dev = 0;
  if (!host) cudaGetDevice(&dev);
  return static_cast<uint64_t>(bytes) | (static_cast<uint64_t>(dev) << 56);
}
void* block_alloc(size_t bytes, bool host) {
  BlockCache& bc = block_cache();
  const uint64_t key = block_key(bytes, host);
  auto& pool = host ? bc.free_host : bc.free_dev;
  {
    std::lock_guard<std::mutex> lk(bc.mu);
    auto it = pool.find(key);
    if (it != pool.end()) {
      void* p = it->second;
      pool.erase(it);
      bc.cached_bytes -= bytes;
      bc.live[p] = key | (host ? (uint64_t(1) << 55) : 0);
      return p;
    }
  }
  void* p = nullptr;
  if (host) {
    CK(cudaMallocHost(&p, bytes));
  } else {
    CK(cudaMalloc(&p, bytes));
  }
  std::lock_guard<std::mutex> lk(bc.mu);
  bc.live[p] = key | (host ? (uint64_t(1) << 55) : 0);
  return p;
}
void block_free(void* p) {
  if (p == nullptr) return;
  BlockCache& bc = block_cache();
  std::unique_lock<std::mutex> lk(bc.mu);
  auto it = bc.live.find(p);
  if (it == bc.live.end()) return;
  const bool host = (it->second >> 55) & 1;
  const uint64_t key = it->second & ~(uint64_t(1) << 55);
  const uint64_t bytes = key & ((uint64_t(1) << 55) - 1);
  bc.live.erase(it);
  if (bc.cached_bytes + bytes > BlockCache::kCap) {
    lk.unlock();
    if (host) {
      cudaFreeHost(p);
    } else {
      cudaFree(p);
    }
    return;
  }
  (host ? bc.free_host : bc.free_dev).emplace(key, p);
  bc.cached_bytes += bytes;
}

template <class T>
T* dalloc(size_t count) {
  if (count == 0) count = 1;
  return static_cast<T*>(block_alloc(count * sizeof(T), false));
}
template <class T>
void halloc(T** p, size_t count) {
  if (count == 0) count = 1;
  *p = static_cast<T*>(block_alloc(count * sizeof(T), true));
}

// ---------------------------------------------------------------------
// Scaling kernels (rescale_problem, scaling.cpp:48-96; axis_norms,
// sparse_matrix.cpp:156-186).
__global__ void k_axis_absmax(const int* __restrict__ ptr, const double* __restrict__ val,
                              int S, double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < S; s += nwarps) {
    if (ptr[s + 1] - ptr[s] > kWarpTile) {  // long: k_long_absmax takes it
      if (lane == 0) out[s] = 0.0;
      continue;
    }
    double a = 0.0;
    for (int k = ptr[s] + lane; k < ptr[s + 1]; k += 32) a = fmax(a, fabs(val[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) out[s] = a;  // max is order-independent: bit-exact
  }
}

// The long segments of an axis by the units of its plan (parts, or the
// ordered plan's single long units): warp maxima folded by an integer
// atomicMax on the bit pattern (non-negative doubles order like their bits),
// so the result is the exact maximum in any order.
__device__ __forceinline__ int long_unit_segment(const SegPlan& p, const int4& d) {
  if (d.x < 0) return p.multi_seg[-d.x - 1];
  return d.w - d.z > kWarpTile ? d.x : -1;
}

__global__ void k_long_absmax(SegPlan p, const double* __restrict__ val, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int u = warp; u < p.n_units; u += nwarps) {
    const int4 d = p.units[u];
    const int seg = long_unit_segment(p, d);
    if (seg < 0) continue;
    double a = 0.0;
    for (int k = d.z + lane; k < d.w; k += 32) a = fmax(a, fabs(val[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(out + seg),
                static_cast<unsigned long long>(__double_as_longlong(a)));
    }
  }
}

// Sequential per-segment p-norm in increasing index order: bit-identical to
// the reference's loop for p = 0, 1, 2 (pow for other p is CUDA's).
constexpr int kLongSeq = 1024;  // segments above this: k_axis_pnorm_long

template <int MODE>
__device__ __forceinline__ double pnorm_term(double v, double p) {
  const double a = fabs(v);
  if constexpr (MODE == 0) {
    return 1.0;
  } else if constexpr (MODE == 1) {
    return a;
  } else if constexpr (MODE == 2) {
    return a * a;
  } else {
    return pow(a, p);
  }
}
template <int MODE>
__device__ __forceinline__ double pnorm_finish(double acc, double p) {
  if constexpr (MODE == 2) {
    return sqrt(acc);
  } else if constexpr (MODE == 3) {
    return (isfinite(p) && p > 1.0) ? pow(acc, 1.0 / p) : acc;
  } else {
    return acc;
  }
}

// A long segment's norm, still one sequential sum in index order (the
// reference's rounding), but its terms are staged into shared memory by the
// whole warp (coalesced, double-buffered) so the single summing lane only
// waits on its add chain, not on a global load per term.
template <int MODE>
__global__ void __launch_bounds__(32) k_axis_pnorm_long(const int* __restrict__ ptr,
                                                        const double* __restrict__ val,
                                                        const int* __restrict__ segs, double p,
                                                        double* __restrict__ out) {
  constexpr int kChunk = 1024;
  __shared__ double buf[2][kChunk];
  const int s = segs[blockIdx.x];
  const int lane = threadIdx.x;
  const int b = ptr[s], e = ptr[s + 1];
  double acc = 0.0;
  int slot = 0;
  // a chunk's 32 loads per lane are issued back to back, then stored
  auto stage = [&](int c0, double* dst) {
    double v[kChunk / 32];
#pragma unroll
    for (int q = 0; q < kChunk / 32; ++q) {
      const int k = c0 + lane + 32 * q;
      v[q] = k < e ? val[k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kChunk / 32; ++q) {
      const int k = c0 + lane + 32 * q;
      if (k < e) dst[lane + 32 * q] = pnorm_term<MODE>(v[q], p);
    }
  };
  stage(b, buf[0]);
  __syncwarp();
  for (int c0 = b; c0 < e; c0 += kChunk, slot ^= 1) {
    const int c1 = min(c0 + kChunk, e);
    // stage the next chunk while lane 0 sums this one
    if (c1 < e) stage(c1, buf[slot ^ 1]);
    if (lane == 0) {
      const double* t = buf[slot];
      const int len = c1 - c0;
      int j = 0;
      for (; j + 16 <= len; j += 16) {  // loads hoisted ahead of the add chain
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = t[j + q];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += v[q];
      }
      for (; j < len; ++j) acc += t[j];
    }
    __syncwarp();
  }
  if (lane == 0) out[s] = pnorm_finish<MODE>(acc, p);
}

template <int MODE>  // 0: count, 1: sum |a|, 2: sqrt(sum a^2), 3: (sum |a|^p)^(1/p)
__global__ void k_axis_pnorm_seq(const int* __restrict__ ptr, const double* __restrict__ val,
                                 int S, double p, double* __restrict__ out) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int b = ptr[s], e = ptr[s + 1];
    if (e - b > kLongSeq) continue;  // k_axis_pnorm_long
    if constexpr (MODE == 0) {
      for (int k = b; k < e; ++k) acc += 1.0;
    } else {
#pragma unroll 8
      for (int k = b; k < e; ++k) {
        const double a = fabs(val[k]);
        if constexpr (MODE == 1) {
          acc += a;
        } else if constexpr (MODE == 2) {
          acc += a * a;
        } else {
          acc += pow(a, p);
        }
      }
    }
    if constexpr (MODE == 2) {
      acc = sqrt(acc);
    } else if constexpr (MODE == 3) {
      if (isfinite(p) && p > 1.0) acc = pow(acc, 1.0 / p);
    }
    out[s] = acc;
  }
}

__global__ void k_recip_sqrt_cum(double* __restrict__ v, double* __restrict__ cum, int S) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const double x = v[s];
    const double d = x > 0.0 ? 1.0 / sqrt(x) : 1.0;
    v[s] = d;
    cum[s] *= d;
  }
}

// SparseMatrix::scaled (sparse_matrix.cpp:222-242): out = src * (dseg*didx).
__global__ void k_scale_values(const int* __restrict__ ptr, const int* __restrict__ idx,
                               const double* __restrict__ src, double* __restrict__ dst,
                               int S, const double* __restrict__ dseg,
                               const double* __restrict__ didx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < S; s += nwarps) {
    if (ptr[s + 1] - ptr[s] > kWarpTile) continue;  // long: k_long_scale
    const double ds = dseg[s];
    for (int k = ptr[s] + lane; k < ptr[s + 1]; k += 32) dst[k] = src[k] * (ds * didx[idx[k]]);
  }
}

__global__ void k_long_scale(SegPlan p, const int* __restrict__ idx, const double* src,
                             double* dst, const double* __restrict__ dseg,
                             const double* __restrict__ didx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int u = warp; u < p.n_units; u += nwarps) {
    const int4 d = p.units[u];
    const int seg = long_unit_segment(p, d);
    if (seg < 0) continue;
    const double ds = dseg[seg];
    for (int k = d.z + lane; k < d.w; k += 32) dst[k] = src[k] * (ds * didx[idx[k]]);
  }
}

// Scaled vectors (scaling.cpp:82-94).
__global__ void k_scale_vectors(int64_t n, int64_t m, const double* c, const double* l,
                                const double* u, const double* q, const double* d1,
                                const double* d2, double* cw, double* lw, double* uw,
                                double* qw) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      const double s = d2[i];
      cw[i] = c[i] * s;
      lw[i] = l[i] / s;
      uw[i] = u[i] / s;
    } else {
      const int64_t j = i - n;
      qw[j] = q[j] * d1[j];
    }
  }
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_narrow(const int64_t* __restrict__ src, int* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = static_cast<int>(src[i]);
}

// Start point (solver.cpp:853-865): z/D then projected.
__global__ void k_start_point(int64_t n, int64_t m, int64_t m1, const double* x0,
                              const double* y0, const double* d1, const double* d2,
                              const double* lw, const double* uw, double* x, double* y,
                              double* lx, double* ly) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      const double v = ref_min(ref_max(x0[i] / d2[i], lw[i]), uw[i]);
      x[i] = v;
      lx[i] = v;
    } else {
      const int64_t j = i - n;
      double v = y0[j] / d1[j];
      if (j < m1) v = ref_max(v, 0.0);
      y[j] = v;
      ly[j] = v;
    }
  }
}

// reduced_point (solver.cpp:495-502).
__global__ void k_reduced_point(int64_t n, int64_t m, const double* xs, const double* ys,
                                const double* d1, const double* d2, const double* l,
                                const double* u, double* xr, double* yr) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      xr[i] = ref_min(ref_max(xs[i] * d2[i], l[i]), u[i]);
    } else {
      const int64_t j = i - n;
      yr[j] = ys[j] * d1[j];
    }
  }
}

__global__ void k_div_scalar(double* __restrict__ dst, const double* __restrict__ src,
                             int64_t n, const double* __restrict__ denom_sq) {
  const double snorm = sqrt(denom_sq[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] / snorm;  // sparse_matrix.cpp:213
}

// max |v|: grid-stride partial maxima into out_blocks, then one block folds
// them (max is order-independent, so exact).
__global__ void k_absmax_blocks(const double* __restrict__ v, int64_t n, double* out_blocks) {
  __shared__ double s[kWarps];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs(v[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kWarps; ++w) r = fmax(r, s[w]);
    out_blocks[blockIdx.x] = r;
  }
}

__global__ void k_absmax_all(const double* __restrict__ v, int64_t n, double* out) {
  __shared__ double s[kWarps];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fmax(a, fabs(v[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kWarps; ++w) r = fmax(r, s[w]);
    *out = r;
  }
}

struct OpCountNonFinite {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  int64_t n;
  const double* x;
  const double* y;
  double* result;
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    const double v = i < n ? x[i] : y[i - n];
    acc.add(0, i, isfinite(v) ? 0.0 : 1.0);
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
  __device__ void finalize_ordered(const double* t, int64_t cnt) const {
    result[0] = any_nonzero(t, cnt) ? 1.0 : 0.0;
  }
};

struct OpNormSq {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  const double* v;
  double* result;
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    acc.add(0, i, v[i] * v[i]);
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
  // linalg::norm2_squared order (linalg.hpp:31-35)
  __device__ void finalize_ordered(const double* t, int64_t cnt) const {
    result[0] = fold(0.0, t, cnt);
  }
};

// ---------------------------------------------------------------------
struct PlanDev {
  SegPlan sp{};
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
std::unordered_map<const void*, int> g_occ;

int occupancy(const void* fn, int smem = 0) {
  std::lock_guard<std::mutex> lk(g_occ_mu);
  auto it = g_occ.find(fn);
  if (it != g_occ.end()) return it->second;
  if (smem > 48 * 1024) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  int b = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kBlock, smem));
  if (b < 1) b = 1;
  g_occ[fn] = b;
  return b;
}

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
  bool coop_ok = true;            // cooperative launches available (else OpNdgPass passes)
  // evaluation period as a CUDA graph, one per CURRENT buffer parity
  cudaGraphExec_t eval_exec[2] = {nullptr, nullptr};
  bool eval_tried[2] = {false, false};
  bool capturing_eval = false;    // enqueue_*: read omega / weights on device
  double* eval_omega_h = nullptr;  // pinned: omega of the next graph launch
  double* eval_omega_d = nullptr;
  bool small_loop = false;        // k_chunk_cluster (tree mode, <= one unit per warp)
  double* small_multi = nullptr;  // its multi-part epilogue slots
  int64_t ndg_count = 0, ndg_passes = 0, ndg_levels = 0;  // FOLP_TIMING statistics
  void* loop_block = nullptr;  // K~ values + indices of CSR and CSC (one block)
  size_t loop_block_bytes = 0;

  // row shard: rows [r0, r1) of K~ are this shard's
  std::unique_ptr<ShardComm> comm;
  std::vector<int64_t> shard_bounds;  // [world + 1]
  int64_t r0 = 0, r1 = 0, lnnz = 0;
  PlanDev lrows, lcols;               // local rows of the CSR; local CSC
  BlockedAxis brows, bcols;           // window-blocked loop copies (large vectors)
  bool blocked_checked = false;
  int* lcsc_ptr = nullptr;
  int* lcsc_row = nullptr;
  int* lcsc_pos = nullptr;            // local CSC entry -> full CSC position
  double* lcsc_val = nullptr;
  double* kty_part = nullptr;
  double* shard_sums = nullptr;
  bool shard_values_ready = false;
  bool rows_dirty = false;            // y, Kx, avg_y outside [r0, r1) stale
  bool sharded() const { return comm != nullptr; }

  cudaGraphExec_t chunk_exec[3] = {nullptr, nullptr, nullptr};  // per step policy
  bool graph_tried[3] = {false, false, false};
  bool graph_ok[3] = {false, false, false};
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
  RedBuf red(int counter) { return RedBuf{partials, counters + counter, nullptr, 0}; }

  template <class Epi>
  void seg(const PlanDev& p, const double* val, const Epi& epi, int counter, int region = 1) {
    RedBuf rb = red(counter);
    const int64_t need = (static_cast<int64_t>(p.sp.n_units) + kWarps - 1) / kWarps;
    if (ordered) {
      rb.terms = terms[region];
      rb.nterm = p.sp.S;
      auto fn = segdot_kernel<Epi, true>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      fn<<<grid, kBlock, 0, stream>>>(p.sp, val, epi, rb);
    } else {
      auto fn = segdot_kernel<Epi, false>;
      const int64_t cap = static_cast<int64_t>(sms) * occupancy(reinterpret_cast<const void*>(fn));
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, std::min<int64_t>(cap, kMaxGrid))));
      fn<<<grid, kBlock, 0, stream>>>(p.sp, val, epi, rb);
    }
    ++launches;
    CK(cudaGetLastError());
  }

  template <class Op>
  void ew(int64_t count, const Op& op, int counter, int region = 1) {
    RedBuf rb = red(counter);
    if (ordered) {
      rb.terms = terms[region];
      rb.nterm = count;
      auto fn = elementwise_kernel<Op, true>;
      const int grid = ew_grid(count, reinterpret_cast<const void*>(fn));
      fn<<<grid, kBlock, 0, stream>>>(count, op, rb);
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
    return b;
  }

  ~folp_gpu_ctx() {
    if (ndg_count > 0 && std::getenv("FOLP_TIMING") != nullptr) {
      std::fprintf(stderr, "[folp timing] duality gaps %lld: %.1f passes, %.1f bisection levels each\n",
                   static_cast<long long>(ndg_count), static_cast<double>(ndg_passes) / ndg_count,
                   static_cast<double>(ndg_levels) / ndg_count);
    }
    if (device >= 0) cudaSetDevice(device);
    for (auto& e : chunk_exec)
      if (e) cudaGraphExecDestroy(e);
    for (auto& e : eval_exec)
      if (e) cudaGraphExecDestroy(e);
    block_free(eval_omega_h);
    if (stream) cudaStreamSynchronize(stream);  // cached blocks must be idle
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
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

// Warp units of one axis (see segdot.cuh): tiles of consecutive short
// segments (<= kWarpTile nonzeros, <= 256 segments each) and fixed parts of
// the longer ones, in index order.
void build_plan(folp_gpu_ctx* c, const int64_t* ptr, int64_t S, int64_t nnz,
                const int* d_ptr, const int* d_idx, PlanDev& out, int64_t s_begin = 0) {
  (void)nnz;
  const bool ordered = c->ordered;
  std::vector<int4> units;
  std::vector<int> multi_seg, multi_parts;
  int64_t seg0 = -1, tile_nnz = 0;
  auto close = [&](int64_t seg_end) {
    if (seg0 >= 0 && seg_end > seg0) {
      units.push_back(make_int4(static_cast<int>(seg0), static_cast<int>(seg_end),
                                static_cast<int>(ptr[seg0]), static_cast<int>(ptr[seg_end])));
    }
    seg0 = -1;
    tile_nnz = 0;
  };
  for (int64_t s = s_begin; s < S; ++s) {
    const int64_t len = ptr[s + 1] - ptr[s];
    if (len <= kWarpTile) {
      if (seg0 >= 0 && (tile_nnz + len > kWarpTile || s - seg0 >= kWarpTile)) close(s);
      if (seg0 < 0) seg0 = s;
      tile_nnz += len;
      continue;
    }
    close(s);
    if (ordered) {  // one lane sums the whole segment in index order
      units.push_back(make_int4(static_cast<int>(s), static_cast<int>(s + 1),
                                static_cast<int>(ptr[s]), static_cast<int>(ptr[s + 1])));
      continue;
    }
    const int multi = static_cast<int>(multi_seg.size());
    const int64_t part = len > kGiantMin ? kGiantPart : kWarpTile;
    const int first = static_cast<int>(units.size());
    for (int64_t b = ptr[s]; b < ptr[s + 1]; b += part) {
      units.push_back(make_int4(-(multi + 1), first, static_cast<int>(b),
                                static_cast<int>(std::min<int64_t>(b + part, ptr[s + 1]))));
    }
    multi_seg.push_back(static_cast<int>(s));
    multi_parts.push_back(static_cast<int>(units.size()) - first);
  }
  close(S);
  auto up = [&](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* d = dalloc<T>(v.size());
    out.owned.push_back(d);
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  };
  {
    std::vector<int> ls;
    for (int64_t sg = s_begin; sg < S; ++sg) {
      if (ptr[sg + 1] - ptr[sg] > kLongSeq) ls.push_back(static_cast<int>(sg));
    }
    out.n_long = static_cast<int>(ls.size());
    if (!ls.empty()) out.long_segs = up(ls);
  }
  SegPlan& p = out.sp;
  p.ptr = d_ptr;
  p.idx = d_idx;
  p.S = static_cast<int>(S);
  p.units = up(units);
  p.n_units = static_cast<int>(units.size());
  p.multi_seg = up(multi_seg);
  p.multi_parts = up(multi_parts);
  p.n_multi = static_cast<int>(multi_seg.size());
  p.part_sums = dalloc<double>(units.size());
  out.owned.push_back(p.part_sums);
  p.arrivals = dalloc<unsigned>(multi_seg.size());
  out.owned.push_back(p.arrivals);
  CK(cudaMemset(p.arrivals, 0, std::max<size_t>(1, multi_seg.size()) * sizeof(unsigned)));
  c->max_giant = std::max(c->max_giant, p.n_multi);
}

void upload_index(folp_gpu_ctx* c, const int64_t* src, int* dst, int64_t count, int64_t* stage,
                  int64_t stage_cap) {
  for (int64_t off = 0; off < count; off += stage_cap) {
    const int64_t len = std::min(stage_cap, count - off);
    CK(cudaMemcpyAsync(stage, src + off, len * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    k_narrow<<<c->simple_grid(len), kBlock, 0, c->stream>>>(stage, dst + off, len);
    ++c->launches;
    CK(cudaGetLastError());
  }
}

void upload(folp_gpu_ctx* c, double* dst, const double* src, int64_t count) {
  if (count <= 0) return;
  if (src == nullptr) {
    CK(cudaMemsetAsync(dst, 0, count * sizeof(double), c->stream));
  } else {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
}
void download(folp_gpu_ctx* c, double* dst, const double* src, int64_t count) {
  if (count > 0 && dst != nullptr) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  }
}
void copy_d2d(folp_gpu_ctx* c, double* dst, const double* src, int64_t count) {
  if (count > 0 && dst != src) {
    CK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
}

// CSR -> CSC on the device (the reference's counting
// pass, sparse_matrix.cpp:82-102): a stable radix sort of the entries by
// column keeps each column in increasing row order, i.e. exactly the
// reference's layout.  Fills csc_ptr / csc_row / csc_orig and returns the
// column starts on the host (for the unit plan).
// Segment id of every entry: a mark at each segment start (empty segments
// stack their marks), then an inclusive scan -- no thread walks a whole
// segment (config 3's dense row has 2M entries).
__global__ void k_segment_marks(const int* ptr, int64_t S, int64_t nnz, int* marks) {
  for (int64_t r = 1 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < S;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = ptr[r];
    if (k < nnz) atomicAdd(&marks[k], 1);  // integer counts: order-free
  }
}
__global__ void k_iota(int* v, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    v[i] = static_cast<int>(i);
  }
}
void segment_ids(folp_gpu_ctx* c, const int* ptr, int64_t S, int64_t nnz, int* out,
                 std::vector<void*>& tmp);

__global__ void k_col_counts(const int* col, int64_t nnz, int* counts) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&counts[col[i] + 1], 1);  // integer counts: order-free
  }
}
__global__ void k_csc_fill(const int* order, const int* rowid, const double* vals, int64_t nnz,
                           int* csc_row, double* csc_val) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = order[i];
    csc_row[i] = rowid[k];
    csc_val[i] = vals[k];
  }
}

void segment_ids(folp_gpu_ctx* c, const int* ptr, int64_t S, int64_t nnz, int* out,
                 std::vector<void*>& tmp) {
  cudaStream_t st = c->stream;
  int* marks = static_cast<int*>(block_alloc(std::max<size_t>(nnz * sizeof(int), 16), false));
  tmp.push_back(marks);
  CK(cudaMemsetAsync(marks, 0, nnz * sizeof(int), st));
  k_segment_marks<<<c->simple_grid(S), kBlock, 0, st>>>(ptr, S, nnz, marks);
  ++c->launches;
  CK(cudaGetLastError());
  size_t bytes = 0;
  CK(cub::DeviceScan::InclusiveSum(nullptr, bytes, marks, out, static_cast<int>(nnz), st));
  void* t = block_alloc(std::max<size_t>(bytes, 16), false);
  tmp.push_back(t);
  CK(cub::DeviceScan::InclusiveSum(t, bytes, marks, out, static_cast<int>(nnz), st));
}

void device_transpose(folp_gpu_ctx* c, std::vector<int64_t>& col_start) {
  const int64_t m = c->m, n = c->n, nnz = c->nnz;
  cudaStream_t s = c->stream;
  std::vector<void*> tmp;
  auto scratch = [&](size_t bytes) {
    void* p = block_alloc(std::max<size_t>(bytes, 16), false);
    tmp.push_back(p);
    return p;
  };
  try {
    int* rowid = static_cast<int*>(scratch(nnz * sizeof(int)));
    int* keys = static_cast<int*>(scratch(nnz * sizeof(int)));
    int* order_in = static_cast<int*>(scratch(nnz * sizeof(int)));
    int* order = static_cast<int*>(scratch(nnz * sizeof(int)));
    int* counts = static_cast<int*>(scratch((n + 1) * sizeof(int)));
    const int grid = c->simple_grid(std::max<int64_t>(m, nnz));
    segment_ids(c, c->csr_ptr, m, nnz, rowid, tmp);
    k_iota<<<grid, kBlock, 0, s>>>(order_in, nnz);
    CK(cudaMemsetAsync(counts, 0, (n + 1) * sizeof(int), s));
    k_col_counts<<<grid, kBlock, 0, s>>>(c->csr_col, nnz, counts);
    c->launches += 2;
    CK(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 31 && (int64_t(1) << end_bit) < n) ++end_bit;
    size_t sort_bytes = 0, scan_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, c->csr_col, keys, order_in, order,
                                       static_cast<int>(nnz), 0, end_bit, s));
    CK(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, counts, c->csc_ptr,
                                     static_cast<int>(n + 1), s));
    void* sort_tmp = scratch(sort_bytes);
    void* scan_tmp = scratch(scan_bytes);
    CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, c->csr_col, keys, order_in, order,
                                       static_cast<int>(nnz), 0, end_bit, s));
    CK(cub::DeviceScan::InclusiveSum(scan_tmp, scan_bytes, counts, c->csc_ptr,
                                     static_cast<int>(n + 1), s));
    k_csc_fill<<<grid, kBlock, 0, s>>>(order, rowid, c->csr_orig, nnz, c->csc_row, c->csc_orig);
    c->launches += 3;  // + the two cub passes' kernels, not counted
    CK(cudaGetLastError());
    std::vector<int> cs32(static_cast<size_t>(n) + 1);
    CK(cudaMemcpyAsync(cs32.data(), c->csc_ptr, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    col_start.assign(cs32.begin(), cs32.end());
  } catch (...) {
    cudaStreamSynchronize(s);
    for (void* p : tmp) block_free(p);
    throw;
  }
  for (void* p : tmp) block_free(p);
}

int pick_device(int device) {
  if (device >= 0) return device;
  const char* env = std::getenv("FOLP_DEVICE");
  return env ? std::atoi(env) : 0;
}

void set_device(folp_gpu_ctx* c) { CK(cudaSetDevice(c->device)); }

// ---------------------------------------------------------------------
// Window-blocked loop copies (tree mode).  When the vector an axis gathers
// from is larger than about half the L2 (config 4: x is 320 MB), its random
// gathers become HBM sector reads (55 G gathers/s instead of ~270 G/s from
// L2 -- tools/microbench/spmv_ceiling.cu on config 4).  The axis' entries
// are then split by gather index into windows of kGatherWindow elements
// and stored window-major; the product runs one phase per window,
// so every phase gathers from an L2-resident slice (ops.cuh EpiCarry).
constexpr int64_t kGatherWindow = int64_t(1) << 22;  // 32 MB: measured best on config 4 (2M: 13.2, 4M: 7.6, 8M: 8.1 ms per trial)
constexpr int64_t kBlockedMinVector = int64_t(12) << 20;  // elements (96 MB)

__global__ void k_window_keys(const int* idx, int64_t nnz, int64_t window, int* keys) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    keys[i] = static_cast<int>(idx[i] / window);
  }
}
__global__ void k_window_counts(const int* keys_sorted, const int* segid, const int* perm,
                                int64_t nnz, int64_t segs, int* counts) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&counts[static_cast<int64_t>(keys_sorted[i]) * (segs + 1) + segid[perm[i]] + 1], 1);
  }
}
__global__ void k_permute(const int* perm, const int* idx_in, const double* val_in, int64_t nnz,
                          int* idx_out, double* val_out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = perm[i];
    idx_out[i] = idx_in[k];
    val_out[i] = val_in[k];
  }
}

void build_blocked(folp_gpu_ctx* c, bool rows_axis) {
  BlockedAxis& ax = rows_axis ? c->brows : c->bcols;
  const int64_t S = rows_axis ? c->m : c->n;      // segments
  const int64_t X = rows_axis ? c->n : c->m;      // gathered vector length
  const int64_t nnz = c->nnz;
  const char* env = std::getenv("FOLP_GATHER_WINDOW");
  const int64_t window = env ? std::max<int64_t>(1024, std::atoll(env)) : kGatherWindow;
  const char* thr = std::getenv("FOLP_BLOCKED_MIN");
  const int64_t min_vec = thr ? std::atoll(thr) : kBlockedMinVector;
  if (c->ordered || c->sharded() || X < min_vec || nnz == 0 || X <= window) return;
  const int* ptr = rows_axis ? c->csr_ptr : c->csc_ptr;
  const int* idx = rows_axis ? c->csr_col : c->csc_row;
  const double* val = rows_axis ? c->csr_work : c->csc_work;
  const int windows = static_cast<int>((X + window - 1) / window);
  cudaStream_t st = c->stream;
  std::vector<void*> tmp;
  auto scratch = [&](size_t bytes) {
    void* p = block_alloc(std::max<size_t>(bytes, 16), false);
    tmp.push_back(p);
    return p;
  };
  auto keep = [&](size_t bytes) {
    void* p = block_alloc(std::max<size_t>(bytes, 16), false);
    ax.owned.push_back(p);
    return p;
  };
  int* segid = static_cast<int*>(scratch(nnz * sizeof(int)));
  int* keys = static_cast<int*>(scratch(nnz * sizeof(int)));
  int* keys_sorted = static_cast<int*>(scratch(nnz * sizeof(int)));
  int* iota = static_cast<int*>(scratch(nnz * sizeof(int)));
  int* perm = static_cast<int*>(scratch(nnz * sizeof(int)));
  int* counts = static_cast<int*>(scratch(static_cast<size_t>(windows) * (S + 1) * sizeof(int)));
  const int grid = c->simple_grid(nnz);
  segment_ids(c, ptr, S, nnz, segid, tmp);
  k_window_keys<<<grid, kBlock, 0, st>>>(idx, nnz, window, keys);
  k_iota<<<grid, kBlock, 0, st>>>(iota, nnz);
  c->launches += 2;
  CK(cudaGetLastError());
  int end_bit = 1;
  while ((1 << end_bit) < windows) ++end_bit;
  size_t sort_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys_sorted, iota, perm,
                                     static_cast<int>(nnz), 0, end_bit, st));
  void* sort_tmp = scratch(sort_bytes);
  CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, keys, keys_sorted, iota, perm,
                                     static_cast<int>(nnz), 0, end_bit, st));
  ax.idx = static_cast<int*>(keep((nnz + 8) * sizeof(int)));
  ax.val = static_cast<double*>(keep((nnz + 8) * sizeof(double)));
  ax.val_orig = static_cast<double*>(keep((nnz + 8) * sizeof(double)));
  ax.carry = static_cast<double*>(keep(S * sizeof(double)));
  int* idx_scratch = static_cast<int*>(scratch((nnz + 8) * sizeof(int)));
  k_permute<<<grid, kBlock, 0, st>>>(perm, idx, val, nnz, ax.idx, ax.val);
  k_permute<<<grid, kBlock, 0, st>>>(perm, idx, rows_axis ? c->csr_orig : c->csc_orig, nnz,
                                     idx_scratch, ax.val_orig);
  CK(cudaMemsetAsync(counts, 0, static_cast<size_t>(windows) * (S + 1) * sizeof(int), st));
  k_window_counts<<<grid, kBlock, 0, st>>>(keys_sorted, segid, perm, nnz, S, counts);
  c->launches += 2;
  CK(cudaGetLastError());
  std::vector<int> cnt(static_cast<size_t>(windows) * (S + 1));
  CK(cudaMemcpyAsync(cnt.data(), counts, cnt.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (void* p : tmp) block_free(p);
  // absolute window-major segment starts, one unit plan per window
  ax.plans.resize(windows);
  std::vector<int64_t> ptr_abs(static_cast<size_t>(S) + 1);
  std::vector<int> ptr32(static_cast<size_t>(S) + 1);
  int64_t base = 0;
  for (int w = 0; w < windows; ++w) {
    const int* cw = cnt.data() + static_cast<size_t>(w) * (S + 1);
    ptr_abs[0] = base;
    for (int64_t sg = 0; sg < S; ++sg) ptr_abs[sg + 1] = ptr_abs[sg] + cw[sg + 1];
    for (int64_t sg = 0; sg <= S; ++sg) ptr32[sg] = static_cast<int>(ptr_abs[sg]);
    int* dptr = static_cast<int*>(keep((S + 1) * sizeof(int)));
    CK(cudaMemcpy(dptr, ptr32.data(), (S + 1) * sizeof(int), cudaMemcpyHostToDevice));
    build_plan(c, ptr_abs.data(), S, nnz, dptr, ax.idx, ax.plans[w]);
    base = ptr_abs[S];
  }
  ax.window = window;
  ax.windows = windows;
}

void ensure_blocked(folp_gpu_ctx* c) {
  if (c->blocked_checked) return;
  c->blocked_checked = true;
  build_blocked(c, true);
  build_blocked(c, false);
}

// One product of the loop over a blocked axis: windows-1 carry phases, then
// the epilogue phase.
template <class Epi>
void phased(folp_gpu_ctx* c, BlockedAxis& ax, const double* val, const Epi& epi, int counter,
            int region) {
  for (int w = 0; w + 1 < ax.windows; ++w) {
    c->seg(ax.plans[w], val, EpiCarry<Epi>{epi, w == 0 ? nullptr : ax.carry, ax.carry}, counter,
           region);
  }
  c->seg(ax.plans[ax.windows - 1], val, EpiCarryIn<Epi>{epi, ax.carry}, counter, region);
}

// A product over the rows (K v) or the columns (K' v) of the working or the
// original values, window-blocked when that axis is.
template <class Epi>
void axis_product(folp_gpu_ctx* c, bool rows_axis, bool working, const Epi& epi, int counter,
                  int region = 1) {
  BlockedAxis& ax = rows_axis ? c->brows : c->bcols;
  if (ax.windows > 0) {
    phased(c, ax, working ? ax.val : ax.val_orig, epi, counter, region);
  } else if (rows_axis) {
    c->seg(c->rows, working ? c->csr_work : c->csr_orig, epi, counter, region);
  } else {
    c->seg(c->cols, working ? c->csc_work : c->csc_orig, epi, counter, region);
  }
}

// Per-axis scaling primitives (SparseMatrix::axis_norms, ::scaled): short
// segments one warp each, long ones by their plan's units (no warp walks
// config 3's 2M-entry row alone).
void axis_absmax(folp_gpu_ctx* c, bool rows_axis, const double* val, double* out) {
  const int S = static_cast<int>(rows_axis ? c->m : c->n);
  const PlanDev& plan = rows_axis ? c->rows : c->cols;
  k_axis_absmax<<<c->simple_grid(static_cast<int64_t>(S) * 32), kBlock, 0, c->stream>>>(
      rows_axis ? c->csr_ptr : c->csc_ptr, val, S, out);
  k_long_absmax<<<c->simple_grid(static_cast<int64_t>(plan.sp.n_units) * 32), kBlock, 0,
                  c->stream>>>(plan.sp, val, out);
  c->launches += 2;
  CK(cudaGetLastError());
}

void axis_scale(folp_gpu_ctx* c, bool rows_axis, const double* src, double* dst,
                const double* dseg, const double* didx) {
  const int S = static_cast<int>(rows_axis ? c->m : c->n);
  const PlanDev& plan = rows_axis ? c->rows : c->cols;
  const int* idx = rows_axis ? c->csr_col : c->csc_row;
  k_scale_values<<<c->simple_grid(static_cast<int64_t>(S) * 32), kBlock, 0, c->stream>>>(
      rows_axis ? c->csr_ptr : c->csc_ptr, idx, src, dst, S, dseg, didx);
  k_long_scale<<<c->simple_grid(static_cast<int64_t>(plan.sp.n_units) * 32), kBlock, 0,
                 c->stream>>>(plan.sp, idx, src, dst, dseg, didx);
  c->launches += 2;
  CK(cudaGetLastError());
}

// p-norms in each segment's index order (bit-identical to the reference for
// p = 0, 1, 2); p = inf goes to axis_absmax.
void axis_pnorm(folp_gpu_ctx* c, bool rows_axis, const double* val, double p, double* out) {
  if (std::isinf(p)) {
    axis_absmax(c, rows_axis, val, out);
    return;
  }
  const int S = static_cast<int>(rows_axis ? c->m : c->n);
  const int* ptr = rows_axis ? c->csr_ptr : c->csc_ptr;
  const int grid = c->simple_grid(S);
  const PlanDev& plan = rows_axis ? c->rows : c->cols;
  auto run = [&](auto mode) {
    constexpr int M = decltype(mode)::value;
    k_axis_pnorm_seq<M><<<grid, kBlock, 0, c->stream>>>(ptr, val, S, p, out);
    if (plan.n_long > 0) {
      k_axis_pnorm_long<M><<<plan.n_long, 32, 0, c->stream>>>(ptr, val, plan.long_segs, p, out);
    }
  };
  if (p == 0.0) {
    run(std::integral_constant<int, 0>{});
  } else if (p == 1.0) {
    run(std::integral_constant<int, 1>{});
  } else if (p == 2.0) {
    run(std::integral_constant<int, 2>{});
  } else {
    run(std::integral_constant<int, 3>{});
  }
  c->launches += plan.n_long > 0 ? 2 : 1;
  CK(cudaGetLastError());
}

// K x of the CURRENT point into kx[cur] (after a start or a restart).
void refresh_kx(folp_gpu_ctx* c) {
  EpiStore e{c->cur_x(), c->kx[c->st_h->cur]};
  axis_product(c, true, true, e, 0);
  c->kx_valid = true;
}

// Product with the context matrix into device memory.
void product(folp_gpu_ctx* c, bool transpose, bool working, const double* v, double* out) {
  EpiStore e{v, out};
  if (transpose) {
    c->seg(c->cols, working ? c->csc_work : c->csc_orig, e, 1);
  } else {
    c->seg(c->rows, working ? c->csr_work : c->csr_orig, e, 1);
  }
}

void zero_average(folp_gpu_ctx* c) {
  if (c->n) CK(cudaMemsetAsync(c->avg_x, 0, c->n * sizeof(double), c->stream));
  if (c->m) CK(cudaMemsetAsync(c->avg_y, 0, c->m * sizeof(double), c->stream));
  c->st_h->avg_weight = 0.0;
  c->st_h->pending = 0.0;
}

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
constexpr int kBisectThreads = 512;
// ||d||_w^2 and g'd per midpoint, then the bracket sums of the analytic
// finish: elements with a breakpoint inside, Q, H, S (ndg_finish_analytic)
constexpr int kBisectVals = 2 * kNuCands + 4;

struct BisectArgs {
  int64_t n, total;
  const double* g[2];
  const double* lo[2];
  const double* hi[2];
  NdgState* ns[2];
  int active[2];
  double* partials;  // [2 parity][2 sets][kBisectVals][grid]
};

__global__ void __launch_bounds__(kBisectThreads) k_ndg_bisect(BisectArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ NdgState st[2];
  __shared__ double wsum[kBisectThreads / 32][2][kBisectVals];
  __shared__ double tot[2][kBisectVals];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = gridDim.x;
  if (tid < 2) {
    st[tid] = *a.ns[tid];
    if (!a.active[tid]) st[tid].done = 1;
  }
  __syncthreads();
  for (int parity = 0;; parity ^= 1) {
    const bool run[2] = {st[0].done == 0, st[1].done == 0};
    if (!run[0] && !run[1]) break;  // same state in every block
    double acc[2][kBisectVals];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int k = 0; k < kBisectVals; ++k) acc[s][k] = 0.0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (!run[s]) continue;
      const double* g = a.g[s];
      const double* lo = a.lo[s];
      const double* hi = a.hi[s];
      const double omega = st[s].omega, winv = st[s].winv;
      for (int64_t i = static_cast<int64_t>(blockIdx.x) * kBisectThreads + tid; i < a.total;
           i += static_cast<int64_t>(nb) * kBisectThreads) {
        const double gs = g[i];
        const bool primal = i < a.n;
        const double w = primal ? omega : winv;
        const double los = lo[i];
        const double his = primal ? hi[i] : INFINITY;
        const double* rcp = primal ? st[s].rcp_primal : st[s].rcp_dual;
#pragma unroll
        for (int p = 0; p < kNuCands; ++p) {
          const double d = ref_min(ref_max(gs * rcp[p], los), his);
          acc[s][2 * p] += w * d * d;
          acc[s][2 * p + 1] += gs * d;
        }
        if (gs != 0.0) {
          const int side = primal ? 0 : 1;
          const double ulo = gs * st[s].rcp_lo[side];  // |u| largest at nu_lo
          const double uhi = gs * st[s].rcp_hi[side];
          const bool clamped_lo = ulo < los || ulo > his;
          const bool clamped_hi = uhi < los || uhi > his;
          if (clamped_lo && !clamped_hi) acc[s][2 * kNuCands] += 1.0;
          if (clamped_hi) {  // clamped over the whole bracket
            const double cv = uhi > his ? his : los;
            acc[s][2 * kNuCands + 1] += w * cv * cv;
            acc[s][2 * kNuCands + 2] += gs * cv;
          }
          if (!clamped_lo) acc[s][2 * kNuCands + 3] += gs * gs * (primal ? winv : omega);
        }
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int k = 0; k < kBisectVals; ++k) {
        double v = acc[s][k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) wsum[warp][s][k] = v;
      }
    __syncthreads();
    double* part = a.partials + static_cast<size_t>(parity) * 2 * kBisectVals * nb;
    if (tid < 2 * kBisectVals) {
      const int s = tid / kBisectVals, k = tid % kBisectVals;
      double v = 0.0;
      for (int w = 0; w < kBisectThreads / 32; ++w) v += wsum[w][s][k];
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
    __syncthreads();
    if (tid < 2 && run[tid]) {
      double nsq[kNuCands], gd[kNuCands];
      for (int p = 0; p < kNuCands; ++p) {
        nsq[p] = tot[tid][2 * p];
        gd[p] = tot[tid][2 * p + 1];
      }
      ndg_replay(&st[tid], nsq, gd, kNuLevels);
      // no breakpoint inside this pass's bracket: none inside the narrower one
      if (!st[tid].done && tot[tid][2 * kNuCands] == 0.0) {
        ndg_finish_analytic(&st[tid], tot[tid][2 * kNuCands + 1], tot[tid][2 * kNuCands + 2],
                            tot[tid][2 * kNuCands + 3]);
      }
    }
    __syncthreads();
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
void enqueue_evaluate(folp_gpu_ctx* c, int which, int raw, int base) {
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
void enqueue_ndg_setup(folp_gpu_ctx* c, int which, int s, double omega) {
  const int64_t n = c->n, m = c->m;
  double* px = c->slot_x(which);
  double* py = c->slot_y(which);
  double* sums = c->res + kResNdg[s];
  EpiNdgPrimal ep{py, px, c->cw, c->lw, c->uw, omega, c->g[s], c->lo[s], c->hi[s], sums};
  if (c->capturing_eval) ep.omega_dev = c->eval_omega_d;
  axis_product(c, false, true, ep, 13, 0);
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

void ensure_gathered(folp_gpu_ctx* c) {
  if (!c->sharded() || !c->rows_dirty) return;
  const int cur = c->st_h->cur;
  c->comm->gather_rows(c->y[cur], c->shard_bounds, c->stream);
  c->comm->gather_rows(c->kx[cur], c->shard_bounds, c->stream);
  c->comm->gather_rows(c->avg_y, c->shard_bounds, c->stream);
  c->rows_dirty = false;
}

// Entry of every engine call that reads the iterate: a sharded context
// first reassembles the row-space vectors the loop kept local.
void prep(folp_gpu_ctx* c) {
  set_device(c);
  ensure_gathered(c);
}

// One sharded trial slot (see ops.cuh, "Row-sharded trial").
void launch_shard_slot(folp_gpu_ctx* c, const LoopBufs& b) {
  c->seg(c->lcols, c->lcsc_val, EpiShardKty{b, c->kty_part, nullptr}, 1);
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
    axis_product(c, false, true, EpiPrimal{b}, 2, 0);
    axis_product(c, true, true, EpiDual{b}, 3, 1);
  }
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
        launch_slot(c, policy, b);
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
    for (int s = 0; s < 2; ++s) enqueue_evaluate(c, slots[s], 0, kResEval[s]);
    for (int s = 0; s < 2; ++s) {
      enqueue_distance(c, slots[s], FOLP_PT_LAST, kResDist[s]);
      enqueue_ndg_setup(c, slots[s], s, 1.0);
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

}  // namespace

// =====================================================================
extern "C" {

const char* folp_gpu_last_error(void) { return g_err.c_str(); }

int folp_gpu_create(const folp_gpu_problem* p, int device, folp_gpu_ctx** out) {
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
    c->ordered = g_default_ordered;
    if (const char* env = std::getenv("FOLP_REDUCTION")) {
      c->ordered = std::strcmp(env, "ordered") == 0;
    }
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
    const bool device_csc = col_start == nullptr || col_rows == nullptr || col_values == nullptr;

    // value / index streams padded by 8 entries: bulk tiles are staged in
    // 16-byte-aligned windows that may run up to 3 entries past the end
    c->csr_ptr = c->alloc<int>(m + 1);
    c->csc_ptr = c->alloc<int>(n + 1);
    c->csr_orig = c->alloc<double>(nnz + 8);
    c->csc_orig = c->alloc<double>(nnz + 8);
    {
      // The loop's streams -- working values and indices of both layouts --
      // in ONE block, so a single L2 access-policy window can cover them.
      const size_t vb = static_cast<size_t>(nnz + 8) * sizeof(double);
      const size_t ib = (static_cast<size_t>(nnz + 8) * sizeof(int) + 255) / 256 * 256;
      char* blk = c->alloc<char>(2 * vb + 2 * ib);
      c->csr_work = reinterpret_cast<double*>(blk);
      c->csc_work = reinterpret_cast<double*>(blk + vb);
      c->csr_col = reinterpret_cast<int*>(blk + 2 * vb);
      c->csc_row = reinterpret_cast<int*>(blk + 2 * vb + ib);
      c->loop_block = blk;
      c->loop_block_bytes = 2 * vb + 2 * ib;
    }
    {
      const int64_t cap = std::min<int64_t>(std::max<int64_t>({m + 1, n + 1, nnz}), int64_t(1) << 26);
      int64_t* stage = dalloc<int64_t>(cap);
      try {
        upload_index(c.get(), p->row_start, c->csr_ptr, m + 1, stage, cap);
        upload_index(c.get(), p->row_cols, c->csr_col, nnz, stage, cap);
        if (!device_csc) {
          upload_index(c.get(), col_start, c->csc_ptr, n + 1, stage, cap);
          upload_index(c.get(), col_rows, c->csc_row, nnz, stage, cap);
        }
        CK(cudaStreamSynchronize(c->stream));
      } catch (...) {
        block_free(stage);
        throw;
      }
      block_free(stage);
    }
    mark("indices");
    upload(c.get(), c->csr_orig, p->row_values, nnz);
    if (device_csc) {
      device_transpose(c.get(), cs);
      col_start = cs.data();
    } else {
      upload(c.get(), c->csc_orig, col_values, nnz);
    }
    copy_d2d(c.get(), c->csr_work, c->csr_orig, nnz);
    copy_d2d(c.get(), c->csc_work, c->csc_orig, nnz);

    mark("values");
    build_plan(c.get(), p->row_start, m, nnz, c->csr_ptr, c->csr_col, c->rows);
    build_plan(c.get(), col_start, n, nnz, c->csc_ptr, c->csc_row, c->cols);

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
    c->partials = c->alloc<double>(static_cast<size_t>(kMaxGrid + c->max_giant + 8) * kMaxAcc);
    if (c->ordered) {
      c->terms[0] = c->alloc<double>(5 * std::max(n, m) + 8);
      c->terms[1] = c->alloc<double>(5 * (n + m) + 8);
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
    CK(cudaStreamSynchronize(c->stream));
    const char* l2env = std::getenv("FOLP_L2_PERSIST");
    if (l2env == nullptr || std::atoi(l2env) > 0) {
      // keep the loop's streams in L2 (persisting lines) across trials
      int max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
      if (max_persist > 0 && max_window > 0) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(max_persist));
        cudaStreamAttrValue attr{};
        const size_t bytes = std::min(c->loop_block_bytes, static_cast<size_t>(max_window));
        attr.accessPolicyWindow.base_ptr = c->loop_block;
        attr.accessPolicyWindow.num_bytes = bytes;
        attr.accessPolicyWindow.hitRatio =
            static_cast<float>(std::min(1.0, static_cast<double>(max_persist) / bytes));
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
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
    CK(cudaStreamSynchronize(c->stream));
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
    CK(cudaStreamSynchronize(c->stream));
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
    CK(cudaStreamSynchronize(c->stream));
  });
}

int folp_gpu_set_point(folp_gpu_ctx* c, int32_t which, const double* x, const double* y) {
  return guarded([&] {
    prep(c);
    upload(c, c->slot_x(which), x, c->n);
    upload(c, c->slot_y(which), y, c->m);
    if (which == FOLP_PT_CURRENT) refresh_kx(c);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int folp_gpu_get_point(folp_gpu_ctx* c, int32_t which, double* x, double* y) {
  return guarded([&] {
    prep(c);
    download(c, x, c->slot_x(which), c->n);
    download(c, y, c->slot_y(which), c->m);
    CK(cudaStreamSynchronize(c->stream));
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
    CK(cudaStreamSynchronize(c->stream));
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
      for (int s = 0; s < 2; ++s) enqueue_evaluate(c, slots[s], 0, kResEval[s]);
      if (want_gaps) {
        for (int s = 0; s < 2; ++s) {
          enqueue_distance(c, slots[s], FOLP_PT_LAST, kResDist[s]);
          enqueue_ndg_setup(c, slots[s], s, omega);
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
      c->launches += per_slot * st->slots;
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

int folp_gpu_spectral_norm(folp_gpu_ctx* c, const double* v0, double relative_tol,
                           int64_t max_iterations, double* norm, int64_t* multiplies) {
  return guarded([&] {
    prep(c);
    double* v = c->aux_x;
    double* w = c->aux_y;
    double* s = c->xr;
    upload(c, v, v0, c->n);
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
    CK(cudaStreamSynchronize(c->stream));
  });
}

int folp_gpu_multiply_transpose(folp_gpu_ctx* c, int32_t working, const double* yh, double* out) {
  return guarded([&] {
    prep(c);
    upload(c, c->aux_y, yh, c->m);
    product(c, true, working != 0, c->aux_y, c->xr);
    download(c, out, c->xr, c->n);
    CK(cudaStreamSynchronize(c->stream));
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
    CK(cudaStreamSynchronize(c->stream));
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

void folp_gpu_set_default_reduction(int32_t ordered) { g_default_ordered = ordered != 0; }

int32_t folp_gpu_reduction_ordered(const folp_gpu_ctx* c) { return c->ordered ? 1 : 0; }


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
    c->shard_bounds = shard_rows(m, row_start, spec->world);
    c->r0 = c->shard_bounds[spec->rank];
    c->r1 = c->shard_bounds[spec->rank + 1];
    build_plan(c, row_start, c->r1, c->nnz, c->csr_ptr, c->csr_col, c->lrows, c->r0);
    std::vector<int64_t> lptr, pos;
    shard_local_csc(n, col_start, col_rows, c->r0, c->r1, lptr, pos);
    c->lnnz = static_cast<int64_t>(pos.size());
    std::vector<int> lptr32(lptr.begin(), lptr.end()), pos32(pos.size()), row32(pos.size());
    for (size_t k = 0; k < pos.size(); ++k) {
      pos32[k] = static_cast<int>(pos[k]);
      row32[k] = static_cast<int>(col_rows[pos[k]]);
    }
    c->lcsc_ptr = c->alloc<int>(n + 1);
    c->lcsc_row = c->alloc<int>(c->lnnz + 8);
    c->lcsc_pos = c->alloc<int>(c->lnnz + 1);
    c->lcsc_val = c->alloc<double>(c->lnnz + 8);
    CK(cudaMemcpy(c->lcsc_ptr, lptr32.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
    if (c->lnnz > 0) {
      CK(cudaMemcpy(c->lcsc_row, row32.data(), c->lnnz * sizeof(int), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->lcsc_pos, pos32.data(), c->lnnz * sizeof(int), cudaMemcpyHostToDevice));
    }
    build_plan(c, lptr.data(), n, c->lnnz, c->lcsc_ptr, c->lcsc_row, c->lcols);
    c->kty_part = c->alloc<double>(std::max<int64_t>(n, 1));
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

int folp_gpu_shard_info(folp_gpu_ctx* c, int32_t* rank, int32_t* world, int64_t* r0, int64_t* r1,
                        int64_t* local_nnz) {
  return guarded([&] {
    *rank = c->sharded() ? c->comm->rank : 0;
    *world = c->sharded() ? c->comm->world : 1;
    *r0 = c->sharded() ? c->r0 : 0;
    *r1 = c->sharded() ? c->r1 : c->m;
    *local_nnz = c->sharded() ? c->lnnz : c->nnz;
  });
}

}  // extern "C"
