// parallel.hpp -- host-side data-parallel helpers for the ingest path
// (copying, validating and counting 10^8-10^9 entries is seconds of
// single-threaded host time on config 4).  Results never depend on the
// thread count: every helper either writes disjoint ranges or merges
// integer counts.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <type_traits>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace folp::host {

inline int host_threads(int64_t work) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int64_t by_work = std::max<int64_t>(1, work / (int64_t(1) << 17));  // >= 128K items each
  return static_cast<int>(std::min<int64_t>({hw, by_work, 32}));
}

// Persistent workers for parallel_for.  Starting and joining up to 32
// std::threads per call cost ~0.5 ms each on the B200 hosts, and config 2's
// end-to-end solve makes a dozen such calls (ingest, histogram, staging);
// the workers are started once per process and sleep between calls.  Any
// number of host threads may submit batches at once; the submitting thread
// takes chunks itself, so a batch completes even when every worker is busy
// (or when it is submitted from inside another batch).
class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool* pool = new WorkerPool();  // process lifetime: never joined at exit
    return *pool;
  }
  // job(i) for every chunk i in [0, chunks); returns when all have run and
  // rethrows the first exception a chunk raised.
  void run(int chunks, const std::function<void(int)>& job) {
    Batch batch;
    batch.job = &job;
    batch.chunks = chunks;
    batch.left = chunks;
    {
      std::lock_guard<std::mutex> lk(mu_);
      queue_.push_back(&batch);
    }
    cv_.notify_all();
    for (;;) {  // the submitter works too
      int i = -1;
      {
        std::lock_guard<std::mutex> lk(mu_);
        i = claim(&batch);
      }
      if (i < 0) break;
      execute(&batch, i);
    }
    std::unique_lock<std::mutex> lk(batch.mu);
    batch.cv.wait(lk, [&] { return batch.left == 0; });
    if (batch.err) std::rethrow_exception(batch.err);
  }

 private:
  struct Batch {
    const std::function<void(int)>* job = nullptr;
    int chunks = 0;
    int next = 0;   // guarded by the pool mutex
    int left = 0;   // guarded by mu
    std::mutex mu;
    std::condition_variable cv;
    std::exception_ptr err;
  };
  WorkerPool() {
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int workers = std::min(hw, 32) - 1;
    for (int w = 0; w < workers; ++w) {
      std::thread([this] { work(); }).detach();
    }
  }
  // pool mutex held: the next chunk of `only` (or of the oldest open batch)
  int claim(Batch* only, Batch** from = nullptr) {
    for (auto it = queue_.begin(); it != queue_.end(); ++it) {
      Batch* b = *it;
      if (only != nullptr && b != only) continue;
      const int i = b->next++;
      if (b->next >= b->chunks) queue_.erase(it);
      if (from != nullptr) *from = b;
      return i;
    }
    return -1;
  }
  static void execute(Batch* b, int i) {
    std::exception_ptr err;
    try {
      (*b->job)(i);
    } catch (...) {
      err = std::current_exception();
    }
    // the last touch of *b: the submitter may return once left reaches 0
    std::lock_guard<std::mutex> lk(b->mu);
    if (err && !b->err) b->err = err;
    if (--b->left == 0) b->cv.notify_one();
  }
  void work() {
    for (;;) {
      Batch* b = nullptr;
      int i = -1;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !queue_.empty(); });
        i = claim(nullptr, &b);
      }
      if (i >= 0) execute(b, i);
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Batch*> queue_;
};

// f(begin, end, chunk) over [0, n) split into contiguous chunks; `work`
// (default n) sizes the chunk count (a row loop passes its nonzeros).
template <class F>
void parallel_for(int64_t n, F&& f, int64_t work = -1) {
  const int t = static_cast<int>(std::min<int64_t>(host_threads(work < 0 ? n : work), std::max<int64_t>(n, 1)));
  if (t <= 1) {
    f(int64_t(0), n, 0);
    return;
  }
  const std::function<void(int)> job = [&f, n, t](int i) {
    f(n * i / t, n * (i + 1) / t, i);
  };
  WorkerPool::get().run(t, job);
}

// A vector of n trivially-copyable elements WITHOUT the value-initializing
// pass: std::vector<T>(n) zero-fills on one thread, and that fill is also the
// first touch of every fresh page (config 2's CSR: 84 MB, 5-30 ms before any
// copy starts).  The elements are left for the caller to overwrite in
// parallel.  The standard containers offer no such constructor; this sets
// the end pointer of a reserved vector through the three-pointer layout
// libstdc++ and libc++ share, and falls back to resize() when the layout
// check fails.
template <class T>
std::vector<T> uninitialized_vector(int64_t n) {
  static_assert(std::is_trivially_copyable_v<T> && std::is_trivially_destructible_v<T>);
  std::vector<T> v;
  if (n <= 0) return v;
  v.reserve(static_cast<std::size_t>(n));
  struct Raw { T* begin; T* end; T* cap; };
  if constexpr (sizeof(Raw) == sizeof(std::vector<T>)) {
    Raw raw;
    std::memcpy(&raw, static_cast<const void*>(&v), sizeof raw);
    if (raw.begin == v.data() && raw.end == raw.begin && raw.cap >= raw.begin + n) {
      raw.end = raw.begin + n;
      std::memcpy(static_cast<void*>(&v), &raw, sizeof raw);
      if (v.size() == static_cast<std::size_t>(n)) return v;
      raw.end = raw.begin;  // unexpected layout: undo
      std::memcpy(static_cast<void*>(&v), &raw, sizeof raw);
    }
  }
  v.resize(static_cast<std::size_t>(n));
  return v;
}

template <class T>
std::vector<T> parallel_copy(const T* src, int64_t n) {
  std::vector<T> out = uninitialized_vector<T>(n);
  parallel_for(n, [&](int64_t b, int64_t e, int) { std::copy(src + b, src + e, out.data() + b); });
  return out;
}

// counts[v] += 1 for every v in keys[0, n) (0 <= v < bins).  Per-thread
// 32-bit histograms merged by bin range when they fit (config 2: 400k bins;
// no contention on the power law's hot bins), relaxed atomics on the shared
// array otherwise (config 4's 4*10^7 columns x threads would not fit).
inline void parallel_histogram(const int64_t* keys, int64_t n, int64_t bins, int64_t* counts) {
  const int t = host_threads(n);
  if (t > 1 && bins * t * 4 <= (int64_t(256) << 20) && bins < (int64_t(1) << 31) && n < (int64_t(1) << 31)) {
    std::vector<std::vector<int32_t>> local(static_cast<std::size_t>(t));
    parallel_for(n, [&](int64_t b, int64_t e, int i) {
      std::vector<int32_t>& h = local[static_cast<std::size_t>(i)];
      h.assign(static_cast<std::size_t>(bins), 0);
      for (int64_t k = b; k < e; ++k) ++h[static_cast<std::size_t>(keys[k])];
    });
    parallel_for(bins, [&](int64_t b, int64_t e, int) {
      for (const auto& h : local) {
        if (h.empty()) continue;
        for (int64_t v = b; v < e; ++v) counts[v] += h[static_cast<std::size_t>(v)];
      }
    }, bins * t);
    return;
  }
  parallel_for(n, [&](int64_t b, int64_t e, int) {
    for (int64_t k = b; k < e; ++k) {
      std::atomic_ref<int64_t>(counts[keys[k]]).fetch_add(1, std::memory_order_relaxed);
    }
  });
}

}  // namespace folp::host
