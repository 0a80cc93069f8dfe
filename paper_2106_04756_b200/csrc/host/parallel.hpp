// parallel.hpp -- host-side data-parallel helpers for the ingest path
// (copying, validating and counting 10^8-10^9 entries is seconds of
// single-threaded host time on config 4).  Results never depend on the
// thread count: every helper either writes disjoint ranges or merges
// integer counts.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <thread>
#include <vector>

namespace folp::host {

inline int host_threads(int64_t work) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int64_t by_work = std::max<int64_t>(1, work / (int64_t(1) << 20));  // >= 1M items each
  return static_cast<int>(std::min<int64_t>({hw, by_work, 32}));
}

// f(begin, end, thread) over [0, n) split into contiguous chunks.
template <class F>
void parallel_for(int64_t n, F&& f) {
  const int t = host_threads(n);
  if (t <= 1) {
    f(int64_t(0), n, 0);
    return;
  }
  // joins on every exit path: a failed thread start must not leave joinable
  // threads behind (std::terminate in ~thread)
  struct Pool {
    std::vector<std::thread> v;
    ~Pool() {
      for (auto& th : v)
        if (th.joinable()) th.join();
    }
  } pool;
  pool.v.reserve(t);
  for (int i = 0; i < t; ++i) {
    const int64_t b = n * i / t, e = n * (i + 1) / t;
    pool.v.emplace_back([&f, b, e, i] { f(b, e, i); });
  }
}

template <class T>
std::vector<T> parallel_copy(const T* src, int64_t n) {
  std::vector<T> out(static_cast<std::size_t>(n));
  parallel_for(n, [&](int64_t b, int64_t e, int) { std::copy(src + b, src + e, out.data() + b); });
  return out;
}

// counts[v] += 1 for every v in keys[0, n) (0 <= v < bins); relaxed atomic
// increments on the shared array (per-thread histograms would cost bins x
// threads of memory for config 4's 4*10^7 columns).
inline void parallel_histogram(const int64_t* keys, int64_t n, int64_t bins, int64_t* counts) {
  (void)bins;
  parallel_for(n, [&](int64_t b, int64_t e, int) {
    for (int64_t k = b; k < e; ++k) {
      std::atomic_ref<int64_t>(counts[keys[k]]).fetch_add(1, std::memory_order_relaxed);
    }
  });
}

}  // namespace folp::host
