// comm.cuh -- collectives of the row-sharded loop (NCCL, in-process loopback).
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

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

  // Peer exchange -- the all-reduce of a trial's partial product fused into
  // the product's epilogue: rank p's producer stores its partial straight
  // into slot p of every rank's receive area (NVLink P2P stores on a
  // multi-GPU node), peer_fence() waits until every rank's stores have
  // landed, and each rank sums its W slots in rank order (so every rank
  // holds bit-identical sums without a collective on the data).  Receive
  // areas are double-buffered by exchange parity: a rank can run at most one
  // exchange ahead of another (each fence waits for all producers).
  bool peer = false;        // exchange through peer slots (peer_setup done)
  int64_t peer_cap = 0;     // doubles per slot
  double** peer_dst_d = nullptr;  // [2][W] device: slot `rank` of every rank's area
  double** peer_src_d = nullptr;  // [2][W] device: this rank's W slots
  virtual void peer_setup(int64_t count) { (void)count; }
  virtual void peer_fence(cudaStream_t s) { (void)s; }
  // Every rank's `mine` (a cudaMalloc base pointer of this rank's buffer)
  // as addressable from this rank: [W] (CUDA IPC on NCCL ranks, plain
  // pointers on the loopback group).  Collective: every rank calls it.
  virtual std::vector<double*> exchange_pointers(double* mine) = 0;
  double* const* peer_dst(int parity) const { return peer_dst_d + parity * world; }
  const double* const* peer_src(int parity) const { return peer_src_d + parity * world; }
  // device pointer tables from host vectors ([2][W] each)
  void upload_tables(const std::vector<double*>& dst, const std::vector<double*>& src) {
    CK(cudaMalloc(&peer_dst_d, 2 * world * sizeof(double*)));
    CK(cudaMalloc(&peer_src_d, 2 * world * sizeof(double*)));
    CK(cudaMemcpy(peer_dst_d, dst.data(), 2 * world * sizeof(double*), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(peer_src_d, src.data(), 2 * world * sizeof(double*), cudaMemcpyHostToDevice));
  }
  void free_tables() {
    if (peer_dst_d) cudaFree(peer_dst_d);
    if (peer_src_d) cudaFree(peer_src_d);
    peer_dst_d = peer_src_d = nullptr;
  }
};

// NCCL, loaded at run time: the single-GPU path has no NCCL dependency, and
// a process that already loaded torch's libnccl.so.2 shares it.
struct NcclApi {
  void* handle = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
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
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
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
    CK(cudaMemset(scratch, 0, sizeof(double)));
  }
  double* area = nullptr;             // own receive area [2][W][cap]
  std::vector<double*> peer_areas;    // mapped areas of the other ranks (IPC)
  ~NcclComm() override {
    for (size_t r = 0; r < peer_areas.size(); ++r) {
      if (peer_areas[r] && static_cast<int>(r) != rank) cudaIpcCloseMemHandle(peer_areas[r]);
    }
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    free_tables();
    if (area) cudaFree(area);
    if (scratch) cudaFree(scratch);
    if (comm) nccl_api().comm_destroy(comm);
  }
  std::vector<void*> opened;  // IPC mappings of exchange_pointers, closed at exit
  std::vector<double*> exchange_pointers(double* mine_ptr) override {
    const NcclApi& api = nccl_api();
    if (api.all_gather == nullptr) throw EngineError(FOLP_E_RUNTIME, "ncclAllGather missing");
    cudaIpcMemHandle_t mine;
    CK(cudaIpcGetMemHandle(&mine, mine_ptr));
    std::vector<cudaIpcMemHandle_t> all(world);
    char* dev = nullptr;
    CK(cudaMalloc(&dev, world * sizeof(cudaIpcMemHandle_t)));
    CK(cudaMemcpy(dev + rank * sizeof(cudaIpcMemHandle_t), &mine, sizeof(mine), cudaMemcpyHostToDevice));
    NCK(api.all_gather(dev + rank * sizeof(cudaIpcMemHandle_t), dev, sizeof(cudaIpcMemHandle_t),
                       ncclUint8, comm, nullptr));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(all.data(), dev, world * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost));
    cudaFree(dev);
    std::vector<double*> out(world, nullptr);
    for (int r = 0; r < world; ++r) {
      if (r == rank) {
        out[r] = mine_ptr;
      } else {
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
        opened.push_back(ptr);
        out[r] = static_cast<double*>(ptr);
      }
    }
    return out;
  }
  // Receive areas: allocated here, exported as CUDA IPC handles, the handles
  // all-gathered through NCCL, the peers' areas opened with peer access.
  void peer_setup(int64_t count) override {
    const NcclApi& api = nccl_api();
    if (api.all_gather == nullptr) throw EngineError(FOLP_E_RUNTIME, "ncclAllGather missing");
    peer_cap = std::max<int64_t>(count, 1);
    CK(cudaMalloc(&area, 2 * world * peer_cap * sizeof(double)));
    cudaIpcMemHandle_t mine;
    CK(cudaIpcGetMemHandle(&mine, area));
    std::vector<cudaIpcMemHandle_t> all(world);
    char* dev = nullptr;
    CK(cudaMalloc(&dev, world * sizeof(cudaIpcMemHandle_t)));
    CK(cudaMemcpy(dev + rank * sizeof(cudaIpcMemHandle_t), &mine, sizeof(mine), cudaMemcpyHostToDevice));
    NCK(api.all_gather(dev + rank * sizeof(cudaIpcMemHandle_t), dev, sizeof(cudaIpcMemHandle_t),
                       ncclUint8, comm, nullptr));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(all.data(), dev, world * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost));
    cudaFree(dev);
    peer_areas.assign(world, nullptr);
    for (int r = 0; r < world; ++r) {
      if (r == rank) {
        peer_areas[r] = area;
      } else {
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, all[r], cudaIpcMemLazyEnablePeerAccess));
        peer_areas[r] = static_cast<double*>(ptr);
      }
    }
    std::vector<double*> dst(2 * world), src(2 * world);
    for (int par = 0; par < 2; ++par) {
      for (int r = 0; r < world; ++r) {
        dst[par * world + r] = peer_areas[r] + (par * world + rank) * peer_cap;
        src[par * world + r] = area + (par * world + r) * peer_cap;
      }
    }
    upload_tables(dst, src);
    peer = true;
  }
  // Every rank's producer has completed (and its P2P stores with it) once
  // this one-element all-reduce completes on the stream.
  void peer_fence(cudaStream_t s) override {
    // ncclMax of the same value on every rank: the scratch never changes
    if (world > 1) NCK(nccl_api().all_reduce(scratch, scratch, 1, ncclFloat64, ncclMax, comm, s));
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
  int live = 0;           // attached comms; the first of a new set resets the group
  std::vector<double*> ptrs;
  std::vector<double> scalars;
  explicit LoopbackGroup(int w) : world(w), ptrs(w, nullptr), scalars(w, 0.0) {}
  // A group is reusable for consecutive solves: when a new set of shards
  // attaches after every comm of the previous set has left, the poison of
  // their departure and any half-counted barrier are cleared.
  void attach() {
    std::lock_guard<std::mutex> lk(mu);
    if (live == 0) {
      poisoned = false;
      arrived = 0;
      ++generation;
    }
    ++live;
  }
  void detach() {
    std::lock_guard<std::mutex> lk(mu);
    --live;
    poisoned = true;
    cv.notify_all();
  }
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
    g->attach();
  }
  double* area = nullptr;  // own receive area [2][W][cap]
  ~LoopbackComm() override {
    // a shard that leaves releases anyone still waiting (after the last
    // collective nobody waits; before it, waiting would never end)
    g->detach();
    free_tables();
    if (area) cudaFree(area);
    if (d_ptrs) cudaFree(d_ptrs);
    if (d_sum) cudaFree(d_sum);
  }
  // Same layout as the NCCL/IPC areas; on one GPU the peers' areas are
  // plain device pointers published through the group.
  void peer_setup(int64_t count) override {
    peer_cap = std::max<int64_t>(count, 1);
    CK(cudaMalloc(&area, 2 * world * peer_cap * sizeof(double)));
    g->ptrs[rank] = area;
    g->barrier();
    std::vector<double*> dst(2 * world), src(2 * world);
    for (int par = 0; par < 2; ++par) {
      for (int r = 0; r < world; ++r) {
        dst[par * world + r] = g->ptrs[r] + (par * world + rank) * peer_cap;
        src[par * world + r] = area + (par * world + r) * peer_cap;
      }
    }
    g->barrier();
    upload_tables(dst, src);
    peer = true;
  }
  std::vector<double*> exchange_pointers(double* mine) override {
    g->ptrs[rank] = mine;
    g->barrier();
    std::vector<double*> out(g->ptrs.begin(), g->ptrs.end());
    g->barrier();
    return out;
  }
  // The producers of every shard have finished: no kernel ever waits on
  // another shard's kernel (they share one GPU).
  void peer_fence(cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));
    g->barrier();
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
