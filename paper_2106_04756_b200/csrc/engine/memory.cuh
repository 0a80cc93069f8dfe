// memory.cuh -- process-wide device / pinned host block cache.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

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
