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
#include <thread>
#include <vector>

namespace folp::host {

inline int host_threads(int64_t work) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int64_t by_work = std::max<int64_t>(1, work / (int64_t(1) << 17));  // >= 128K items each
  return static_cast<int>(std::min<int64_t>({hw, by_work, 32}));
}

// f(begin, end, thread) over [0, n) split into contiguous chunks; `work`
// (default n) sizes the thread count (a row loop passes its nonzeros).
template <class F>
void parallel_for(int64_t n, F&& f, int64_t work = -1) {
  const int t = static_cast<int>(std::min<int64_t>(host_threads(work < 0 ? n : work), std::max<int64_t>(n, 1)));
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
