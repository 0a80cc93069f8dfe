// Host-side helpers of the ingest path (paper_2106_04756_b200/csrc/host/parallel.hpp):
// the persistent worker pool behind parallel_for, the histogram and the
// uninitialized vector.  Built and run by tests/test_host_parallel.py.
#include <atomic>
#include <cstdio>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <vector>

#include "parallel.hpp"

using namespace folp::host;

#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAILED %s (line %d)\n", #cond, __LINE__);            \
      return 1;                                                         \
    }                                                                   \
  } while (0)

int main() {
  const int64_t n = int64_t(1) << 22;
  // every index visited exactly once, chunks contiguous and disjoint
  {
    std::vector<int> hits(static_cast<size_t>(n), 0);
    parallel_for(n, [&](int64_t b, int64_t e, int) {
      for (int64_t i = b; i < e; ++i) ++hits[static_cast<size_t>(i)];
    });
    CHECK(std::all_of(hits.begin(), hits.end(), [](int v) { return v == 1; }));
  }
  // chunk ids are 0 .. t-1, each used once
  {
    std::vector<std::atomic<int>> seen(64);
    for (auto& s : seen) s = 0;
    parallel_for(n, [&](int64_t, int64_t, int t) { ++seen[static_cast<size_t>(t)]; });
    int used = 0;
    for (auto& s : seen) {
      CHECK(s <= 1);
      used += s;
    }
    CHECK(used == host_threads(n));
  }
  // a batch submitted from inside a batch completes (the submitter works)
  {
    std::atomic<int64_t> total{0};
    parallel_for(8, [&](int64_t b, int64_t e, int) {
      for (int64_t i = b; i < e; ++i) {
        parallel_for(n / 8, [&](int64_t bb, int64_t ee, int) { total += ee - bb; });
      }
    }, n);
    CHECK(total == n);
  }
  // batches from several host threads at once
  {
    std::vector<int64_t> sums(6, 0);
    std::vector<std::thread> callers;
    for (int c = 0; c < 6; ++c) {
      callers.emplace_back([&, c] {
        for (int rep = 0; rep < 20; ++rep) {
          std::atomic<int64_t> s{0};
          parallel_for(n / 4, [&](int64_t b, int64_t e, int) { s += e - b; });
          sums[static_cast<size_t>(c)] += s;
        }
      });
    }
    for (auto& t : callers) t.join();
    for (int64_t s : sums) CHECK(s == 20 * (n / 4));
  }
  // the first exception of a chunk reaches the caller, the pool stays usable
  {
    bool thrown = false;
    try {
      parallel_for(n, [&](int64_t b, int64_t, int) {
        if (b == 0) throw std::runtime_error("chunk failed");
      });
    } catch (const std::runtime_error&) {
      thrown = true;
    }
    CHECK(thrown);
    std::atomic<int64_t> s{0};
    parallel_for(n, [&](int64_t b, int64_t e, int) { s += e - b; });
    CHECK(s == n);
  }
  // histogram equals the sequential count (per-thread and atomic paths)
  for (const int64_t bins : {int64_t(1000), int64_t(1) << 25}) {
    const int64_t keys_n = int64_t(1) << 21;
    std::vector<int64_t> keys(static_cast<size_t>(keys_n));
    uint64_t x = 88172645463325252ull;
    for (auto& k : keys) {
      x ^= x << 13, x ^= x >> 7, x ^= x << 17;
      k = static_cast<int64_t>(x % static_cast<uint64_t>(std::min<int64_t>(bins, 5000)));
    }
    std::vector<int64_t> want(static_cast<size_t>(std::min<int64_t>(bins, 5000)), 0);
    for (int64_t k : keys) ++want[static_cast<size_t>(k)];
    std::vector<int64_t> got(static_cast<size_t>(bins), 0);
    parallel_histogram(keys.data(), keys_n, bins, got.data());
    for (size_t v = 0; v < want.size(); ++v) CHECK(got[v] == want[v]);
  }
  // uninitialized_vector: size, capacity, writable, copyable, destructible
  {
    std::vector<double> v = uninitialized_vector<double>(n);
    CHECK(static_cast<int64_t>(v.size()) == n && v.capacity() >= v.size());
    parallel_for(n, [&](int64_t b, int64_t e, int) {
      for (int64_t i = b; i < e; ++i) v[static_cast<size_t>(i)] = static_cast<double>(i);
    });
    std::vector<double> w = v;
    CHECK(w[123456] == 123456.0 && w.back() == static_cast<double>(n - 1));
    v.push_back(1.0);
    CHECK(static_cast<int64_t>(v.size()) == n + 1);
    CHECK(uninitialized_vector<int>(0).empty());
    const std::vector<int64_t> src(100000, 7);
    CHECK(parallel_copy(src.data(), 100000) == src);
  }
  std::printf("ok\n");
  return 0;
}
