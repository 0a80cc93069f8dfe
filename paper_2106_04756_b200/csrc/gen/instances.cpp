// instances.cpp -- seeded generators for the BASELINE.json configurations
// (SURVEY.md section 8d).  Harness code: it builds inputs, it is not the
// solver.  Only raw std::mt19937_64 draws are used (the reference's own rule,
// /root/reference/proj/src/instance_gen.cpp:25-40), so every platform sees
// the same instance.  Draw order is documented per family below.
#include "folp_gen.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t seed) : g(seed) {}
  double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }  // U[0,1)
  int64_t index(int64_t n) {  // unbiased, instance_gen.cpp:31-40
    const uint64_t bound = static_cast<uint64_t>(n);
    const uint64_t limit = std::numeric_limits<uint64_t>::max() / bound * bound;
    uint64_t d;
    do {
      d = g();
    } while (d >= limit);
    return static_cast<int64_t>(d % bound);
  }
  double normal() {  // Box-Muller, cosine branch only
    const double u1 = unit(), u2 = unit();
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
  }
};

struct Holder {
  folp_gen_lp view{};
  std::vector<int64_t> rs, rc, cs, cr;
  std::vector<double> rv, cv, c, q, l, u;

  void publish(int64_t m, int64_t n, int64_t m1) {
    view.num_rows = m;
    view.num_cols = n;
    view.num_inequality_rows = m1;
    view.nnz = static_cast<int64_t>(rv.size());
    view.row_start = rs.data();
    view.row_cols = rc.data();
    view.row_values = rv.data();
    view.col_start = cs.data();
    view.col_rows = cr.data();
    view.col_values = cv.data();
    view.objective = c.data();
    view.right_hand_side = q.data();
    view.variable_lower = l.data();
    view.variable_upper = u.data();
    view.objective_constant = 0.0;
    view.max_row_len = 0;
    view.max_col_len = 0;
    for (int64_t i = 0; i < m; ++i) view.max_row_len = std::max(view.max_row_len, rs[i + 1] - rs[i]);
    for (int64_t j = 0; j < n; ++j) view.max_col_len = std::max(view.max_col_len, cs[j + 1] - cs[j]);
  }
};

// CSR from CSC by a counting pass (columns come out increasing per row).
void csr_from_csc(Holder& h, int64_t m, int64_t n) {
  const int64_t nnz = static_cast<int64_t>(h.cv.size());
  h.rs.assign(static_cast<size_t>(m) + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) ++h.rs[h.cr[e] + 1];
  for (int64_t i = 0; i < m; ++i) h.rs[i + 1] += h.rs[i];
  h.rc.resize(static_cast<size_t>(nnz));
  h.rv.resize(static_cast<size_t>(nnz));
  std::vector<int64_t> fill(h.rs.begin(), h.rs.end() - 1);
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t e = h.cs[j]; e < h.cs[j + 1]; ++e) {
      const int64_t slot = fill[h.cr[e]]++;
      h.rc[slot] = j;
      h.rv[slot] = h.cv[e];
    }
  }
}

// CSC from CSR (rows come out increasing per column).
void csc_from_csr(Holder& h, int64_t m, int64_t n) {
  const int64_t nnz = static_cast<int64_t>(h.rv.size());
  h.cs.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) ++h.cs[h.rc[e] + 1];
  for (int64_t j = 0; j < n; ++j) h.cs[j + 1] += h.cs[j];
  h.cr.resize(static_cast<size_t>(nnz));
  h.cv.resize(static_cast<size_t>(nnz));
  std::vector<int64_t> fill(h.cs.begin(), h.cs.end() - 1);
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t e = h.rs[i]; e < h.rs[i + 1]; ++e) {
      const int64_t slot = fill[h.rc[e]]++;
      h.cr[slot] = i;
      h.cv[slot] = h.rv[e];
    }
  }
}

// Configs 1, 2, 4: random sparse LP, feasible by construction.
// Draw order: per column j: degree d_j (cfg 2 only), d_j distinct rows
// (rejection), d_j values; then x0 (n, U[0,5]), y0 (m, N(0,1), |.| on the
// >= rows), slack s (m1, U[0,1]), z0 (n, U[0,1]).  q = K x0 - (s; 0),
// c = K'y0 + z0, bounds [0, 10].  The >= rows are rows 0..m1-1.
template <class Degree, class Value>
Holder random_sparse(uint64_t seed, int64_t m, int64_t m1, int64_t n, Degree degree,
                     Value value) {
  Rng rng(seed);
  Holder h;
  h.cs.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<std::pair<int64_t, double>> col;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t d = std::min<int64_t>(degree(rng), m);
    col.clear();
    while (static_cast<int64_t>(col.size()) < d) {
      const int64_t r = rng.index(m);
      bool dup = false;
      for (const auto& e : col) dup = dup || e.first == r;
      if (!dup) col.emplace_back(r, 0.0);
    }
    for (auto& e : col) e.second = value(rng);
    std::sort(col.begin(), col.end());
    for (const auto& e : col) {
      h.cr.push_back(e.first);
      h.cv.push_back(e.second);
    }
    h.cs[j + 1] = static_cast<int64_t>(h.cr.size());
  }
  csr_from_csc(h, m, n);
  std::vector<double> x0(static_cast<size_t>(n)), y0(static_cast<size_t>(m)),
      s(static_cast<size_t>(m1)), z0(static_cast<size_t>(n));
  for (double& v : x0) v = 5.0 * rng.unit();
  for (int64_t i = 0; i < m; ++i) {
    const double v = rng.normal();
    y0[i] = i < m1 ? std::fabs(v) : v;
  }
  for (double& v : s) v = rng.unit();
  for (double& v : z0) v = rng.unit();
  h.q.assign(static_cast<size_t>(m), 0.0);
  for (int64_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int64_t e = h.rs[i]; e < h.rs[i + 1]; ++e) acc += h.rv[e] * x0[h.rc[e]];
    h.q[i] = i < m1 ? acc - s[i] : acc;
  }
  h.c.assign(static_cast<size_t>(n), 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t e = h.cs[j]; e < h.cs[j + 1]; ++e) acc += h.cv[e] * y0[h.cr[e]];
    h.c[j] = acc + z0[j];
  }
  h.l.assign(static_cast<size_t>(n), 0.0);
  h.u.assign(static_cast<size_t>(n), 10.0);
  h.publish(m, n, m1);
  return h;
}

// Config 3: PageRank LP on a directed preferential-attachment graph.
// Nodes 0..8 form a complete digraph (no dangling node: every node has
// out-degree 8, recorded as the dangling-node choice in DESIGN.md); node
// v >= 9 draws 8 distinct targets with probability proportional to
// (in-degree + 1) by uniform picks from a multiset list.  P_ij = 1/outdeg(j)
// for j -> i.  Rows: x_i - lambda (P x)_i >= (1 - lambda)/N (N rows), then
// 1'x = 1; c = 0, x >= 0, lambda = 0.99.
Holder pagerank(uint64_t seed, int64_t N) {
  constexpr int64_t kOut = 8;
  constexpr double kLambda = 0.99;
  Rng rng(seed);
  std::vector<int64_t> src, dst;  // edges src -> dst
  src.reserve(static_cast<size_t>(N * kOut));
  dst.reserve(static_cast<size_t>(N * kOut));
  std::vector<int64_t> pool;  // node i appears (in-degree(i) + 1) times
  pool.reserve(static_cast<size_t>(N * (kOut + 1)));
  const int64_t seeds = std::min<int64_t>(kOut + 1, N);
  for (int64_t v = 0; v < seeds; ++v) pool.push_back(v);
  for (int64_t v = 0; v < seeds; ++v) {
    for (int64_t t = 0; t < seeds; ++t) {
      if (t == v) continue;
      src.push_back(v);
      dst.push_back(t);
      pool.push_back(t);
    }
  }
  int64_t picked[kOut];
  for (int64_t v = seeds; v < N; ++v) {
    int64_t k = 0;
    while (k < kOut) {
      const int64_t t = pool[rng.index(static_cast<int64_t>(pool.size()))];
      bool dup = false;
      for (int64_t a = 0; a < k; ++a) dup = dup || picked[a] == t;
      if (!dup) picked[k++] = t;
    }
    for (int64_t a = 0; a < kOut; ++a) {
      src.push_back(v);
      dst.push_back(picked[a]);
      pool.push_back(picked[a]);
    }
    pool.push_back(v);
  }
  std::vector<int64_t> outdeg(static_cast<size_t>(N), 0), indeg(static_cast<size_t>(N), 0);
  for (size_t e = 0; e < src.size(); ++e) {
    ++outdeg[src[e]];
    ++indeg[dst[e]];
  }
  const int64_t m = N + 1;
  Holder h;
  // rows: node rows (diag + in-edges, columns increasing), then the sum row
  h.rs.assign(static_cast<size_t>(m) + 1, 0);
  for (int64_t i = 0; i < N; ++i) h.rs[i + 1] = 1 + indeg[i];
  h.rs[N + 1] = N;
  for (int64_t i = 0; i < m; ++i) h.rs[i + 1] += h.rs[i];
  const int64_t nnz = h.rs[m];
  h.rc.resize(static_cast<size_t>(nnz));
  h.rv.resize(static_cast<size_t>(nnz));
  std::vector<int64_t> fill(h.rs.begin(), h.rs.end() - 1);
  // in-edges grouped by destination, sources increasing
  std::vector<int64_t> order(src.size());
  for (size_t e = 0; e < order.size(); ++e) order[e] = static_cast<int64_t>(e);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return dst[a] != dst[b] ? dst[a] < dst[b] : src[a] < src[b];
  });
  size_t pos = 0;
  for (int64_t i = 0; i < N; ++i) {
    bool diag_done = false;
    while (pos < order.size() && dst[order[pos]] == i) {
      const int64_t j = src[order[pos]];
      if (!diag_done && j > i) {
        h.rc[fill[i]] = i;
        h.rv[fill[i]++] = 1.0;
        diag_done = true;
      }
      h.rc[fill[i]] = j;
      h.rv[fill[i]++] = -kLambda / static_cast<double>(outdeg[j]);
      ++pos;
    }
    if (!diag_done) {
      h.rc[fill[i]] = i;
      h.rv[fill[i]++] = 1.0;
    }
  }
  for (int64_t j = 0; j < N; ++j) {
    h.rc[fill[N]] = j;
    h.rv[fill[N]++] = 1.0;
  }
  csc_from_csr(h, m, N);
  h.q.assign(static_cast<size_t>(m), (1.0 - kLambda) / static_cast<double>(N));
  h.q[N] = 1.0;
  h.c.assign(static_cast<size_t>(N), 0.0);
  h.l.assign(static_cast<size_t>(N), 0.0);
  h.u.assign(static_cast<size_t>(N), std::numeric_limits<double>::infinity());
  h.publish(m, N, N);
  return h;
}

// Config 5: transportation LP.  Draw order: supply points (S x 2),
// demand points (D x 2), demands d (D, U[10,40]), supplies s (S, U[50,150]),
// then s scaled so sum s = 1.1 sum d.  Variable s*D + d costs the Euclidean
// distance.  Rows: -sum_d x_sd >= -s_s (S rows), then sum_s x_sd = d_d.
Holder transportation(uint64_t seed, int64_t S, int64_t D) {
  Rng rng(seed);
  std::vector<double> spx(S), spy(S), dpx(D), dpy(D), dem(D), sup(S);
  for (int64_t s = 0; s < S; ++s) {
    spx[s] = rng.unit();
    spy[s] = rng.unit();
  }
  for (int64_t d = 0; d < D; ++d) {
    dpx[d] = rng.unit();
    dpy[d] = rng.unit();
  }
  double total_d = 0.0, total_s = 0.0;
  for (double& v : dem) {
    v = 10.0 + 30.0 * rng.unit();
    total_d += v;
  }
  for (double& v : sup) {
    v = 50.0 + 100.0 * rng.unit();
    total_s += v;
  }
  const double factor = 1.1 * total_d / total_s;
  for (double& v : sup) v *= factor;
  const int64_t n = S * D, m = S + D;
  Holder h;
  h.rs.assign(static_cast<size_t>(m) + 1, 0);
  for (int64_t s = 0; s < S; ++s) h.rs[s + 1] = h.rs[s] + D;
  for (int64_t d = 0; d < D; ++d) h.rs[S + d + 1] = h.rs[S + d] + S;
  h.rc.resize(static_cast<size_t>(2 * n));
  h.rv.resize(static_cast<size_t>(2 * n));
  for (int64_t s = 0; s < S; ++s) {
    for (int64_t d = 0; d < D; ++d) {
      h.rc[s * D + d] = s * D + d;
      h.rv[s * D + d] = -1.0;
    }
  }
  for (int64_t d = 0; d < D; ++d) {
    const int64_t base = h.rs[S + d];
    for (int64_t s = 0; s < S; ++s) {
      h.rc[base + s] = s * D + d;
      h.rv[base + s] = 1.0;
    }
  }
  csc_from_csr(h, m, n);
  h.q.resize(static_cast<size_t>(m));
  for (int64_t s = 0; s < S; ++s) h.q[s] = -sup[s];
  for (int64_t d = 0; d < D; ++d) h.q[S + d] = dem[d];
  h.c.resize(static_cast<size_t>(n));
  for (int64_t s = 0; s < S; ++s) {
    for (int64_t d = 0; d < D; ++d) {
      const double dx = spx[s] - dpx[d], dy = spy[s] - dpy[d];
      h.c[s * D + d] = std::sqrt(dx * dx + dy * dy);
    }
  }
  h.l.assign(static_cast<size_t>(n), 0.0);
  h.u.assign(static_cast<size_t>(n), std::numeric_limits<double>::infinity());
  h.publish(m, n, S);
  return h;
}

// Degree pmf p(k) ~ k^-2.1 on {2..2000} by inverse CDF (config 2).
struct PowerLawDegree {
  std::vector<double> cdf;
  PowerLawDegree() {
    double total = 0.0;
    for (int k = 2; k <= 2000; ++k) total += std::pow(static_cast<double>(k), -2.1);
    double acc = 0.0;
    for (int k = 2; k <= 2000; ++k) {
      acc += std::pow(static_cast<double>(k), -2.1) / total;
      cdf.push_back(acc);
    }
    cdf.back() = 1.0;
  }
  int64_t operator()(Rng& rng) const {
    const double u = rng.unit();
    const auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
    return 2 + static_cast<int64_t>(it - cdf.begin());
  }
};

int64_t scaled(double full, double scale, int64_t floor_) {
  return std::max<int64_t>(floor_, static_cast<int64_t>(std::llround(full * scale)));
}

}  // namespace

extern "C" {

folp_gen_lp* folp_gen_config(int32_t cfg, uint64_t seed, double scale) {
  try {
    if (!(scale > 0.0 && scale <= 1.0)) throw std::invalid_argument("scale must be in (0, 1]");
    std::unique_ptr<Holder> h;
    auto normal = [](Rng& r) { return r.normal(); };
    switch (cfg) {
      case 1: {
        const int64_t m = 2 * scaled(500, scale, 5), n = scaled(2000, scale, 10);
        h = std::make_unique<Holder>(random_sparse(
            seed, m, m / 2, n, [](Rng&) { return int64_t(5); }, normal));
        break;
      }
      case 2: {
        const int64_t m = 2 * scaled(100000, scale, 50), n = scaled(400000, scale, 100);
        const PowerLawDegree deg;
        h = std::make_unique<Holder>(random_sparse(
            seed, m, m / 2, n, [&](Rng& r) { return deg(r); },
            [](Rng& r) {
              const double sign = r.unit() < 0.5 ? -1.0 : 1.0;
              return sign * std::pow(10.0, 6.0 * r.unit() - 3.0);
            }));
        break;
      }
      case 3:
        h = std::make_unique<Holder>(pagerank(seed, scaled(2000000, scale, 20)));
        break;
      case 4: {
        const int64_t m = 2 * scaled(10000000, scale, 50), n = scaled(40000000, scale, 100);
        h = std::make_unique<Holder>(random_sparse(
            seed, m, m / 2, n, [](Rng&) { return int64_t(10); }, normal));
        break;
      }
      case 5:
        h = std::make_unique<Holder>(
            transportation(seed, scaled(2000, scale, 4), scaled(8000, scale, 8)));
        break;
      default:
        throw std::invalid_argument("cfg must be 1..5");
    }
    Holder* raw = h.release();
    return &raw->view;  // view is the first member
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void folp_gen_free(folp_gen_lp* lp) { delete reinterpret_cast<Holder*>(lp); }

const char* folp_gen_last_error(void) { return g_err.c_str(); }

}  // extern "C"
