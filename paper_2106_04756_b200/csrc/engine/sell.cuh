// sell.cuh -- lane-per-segment (SELL-32) groups for the loop's row products.
// Fragment of engine.cu: included inside its anonymous namespace, after
// plans.cuh (one translation unit; see engine.cu for the order).
//
// K x' over rows gathers x'[col] entry by entry.  A warp walking one row's
// entries is coalesced when the row's columns are contiguous (config 5's
// supply rows) but touches one sector per entry when they are strided --
// config 5's demand rows: entry s of demand row d is column s*D + d, so one
// row strides by D = 8,000 and every gather is its own 32-byte sector of a
// 128 MB vector (profiles/r2_launches_cfg5.txt: the window-blocked row
// product at ~41 % of the HBM roofline).  The SAME gathers taken across 32
// neighbouring demand rows at one entry index are 32 consecutive columns:
// 8 sectors.  So 32 consecutive equal-length rows whose interleaved gathers
// touch at most half the sectors of their own rows' are stored interleaved
// (segdot.cuh SellPlan), one lane per row, each lane summing its row in entry
// order; the other rows keep their CSR units.  The reference's op is
// SparseMatrix::multiply (proj/src/sparse_matrix.cpp:106-119).
//
// Tree mode only (part sums in part order: deterministic, not the sequential
// fold), the loop's K x' (EpiDual) only; evaluations keep the CSR plan.
// FOLP_SELL=0 disables, FOLP_SELL_MIN_LEN sets the shortest row length
// considered (default 64).
#pragma once

struct SellHost {
  std::vector<int> row0, len;  // groups: first row, row length
  int64_t nnz = 0;             // entries in groups
  bool gathers_coalesced = false;  // SELL + contiguous CSR rows cover the axis
};

// Distinct 32-byte sectors among 32 gather indices.
inline int sectors32(const int64_t* v) {
  int64_t s[32];
  for (int i = 0; i < 32; ++i) s[i] = v[i] >> 2;
  std::sort(s, s + 32);
  return static_cast<int>(std::unique(s, s + 32) - s);
}

SellHost detect_sell(const int64_t* rs, const int64_t* rc, int64_t m, int64_t nnz) {
  SellHost h;
  const char* env = std::getenv("FOLP_SELL");
  if (env != nullptr && std::atoi(env) == 0) return h;
  const char* mlen = std::getenv("FOLP_SELL_MIN_LEN");
  const int64_t min_len = mlen ? std::max<int64_t>(1, std::atoll(mlen)) : 64;
  int64_t r = 0;
  while (r < m) {
    const int64_t L = rs[r + 1] - rs[r];
    int64_t e = r + 1;
    while (e < m && rs[e + 1] - rs[e] == L) ++e;
    if (L >= min_len && L <= (int64_t(1) << 24)) {
      for (int64_t g0 = r; g0 + 32 <= e; g0 += 32) {
        // sample a few entry positions: interleaved vs per-row sectors
        int sell = 0, csr = 0;
        const int64_t js[4] = {0, L / 3, (2 * L) / 3, L - 1};
        for (int64_t j : js) {
          int64_t v[32];
          for (int l = 0; l < 32; ++l) v[l] = rc[rs[g0 + l] + j];
          sell += sectors32(v);
          const int64_t j0 = std::min<int64_t>(j, std::max<int64_t>(0, L - 32));
          for (int l = 0; l < 32; ++l) v[l] = rc[rs[g0] + std::min<int64_t>(j0 + l, L - 1)];
          csr += sectors32(v);
        }
        if (2 * sell <= csr) {
          h.row0.push_back(static_cast<int>(g0));
          h.len.push_back(static_cast<int>(L));
          h.nnz += 32 * L;
        }
      }
    }
    r = e;
  }
  if (h.row0.empty()) return h;
  // the remaining rows: contiguous columns gather coalesced as they are
  std::vector<char> in(static_cast<size_t>(m), 0);
  for (size_t g = 0; g < h.row0.size(); ++g)
    for (int l = 0; l < 32; ++l) in[static_cast<size_t>(h.row0[g] + l)] = 1;
  int64_t contiguous = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (in[static_cast<size_t>(i)]) continue;
    for (int64_t k = rs[i] + 1; k < rs[i + 1]; ++k) contiguous += rc[k] == rc[k - 1] + 1 ? 1 : 0;
  }
  h.gathers_coalesced = static_cast<double>(h.nnz + contiguous) >= 0.9 * static_cast<double>(nnz);
  return h;
}

// The SELL plan of the rows axis: CSR units for the other rows, SELL parts
// for the groups (interleaved arrays filled by pack_sell after rescaling).
void build_sell_plan(folp_gpu_ctx* c, const int64_t* rs, int64_t m, int64_t nnz, const SellHost& h,
                     PlanDev& out) {
  const int G = static_cast<int>(h.row0.size());
  std::vector<char> skip(static_cast<size_t>(m), 0);
  std::vector<int> base(G), nparts(G), slot0(G);
  std::vector<int4> extra;
  int64_t b = 0;
  int slots = 0;
  const char* penv = std::getenv("FOLP_SELL_PART");  // entries per lane per unit
  const int part = penv != nullptr ? std::max(8, std::atoi(penv)) : kSellPart;
  static_assert(kSellGiantMin >= kWarpTile, "giant parts start above a tile");
  for (int g = 0; g < G; ++g) {
    for (int l = 0; l < 32; ++l) skip[static_cast<size_t>(h.row0[g] + l)] = 1;
    base[g] = static_cast<int>(b);
    const int L = h.len[g];
    nparts[g] = (L + part - 1) / part;
    slot0[g] = slots;
    for (int q = 0; q < nparts[g]; ++q) {
      extra.push_back(make_int4(-(kSellTag + g), q, q * part, std::min(L, (q + 1) * part)));
    }
    slots += nparts[g];
    b += 32 * static_cast<int64_t>(L);
  }
  // the rows left to CSR units here are the contiguous ones (gathers
  // coalesced): 2048-entry parts above 4096 entries halve their part sums,
  // fences and arrival atomics (config 5's 8,000-entry supply rows: with
  // 128-entry SELL parts, trial 515 -> 478 us)
  build_plan(c, rs, m, nnz, c->csr_ptr, c->csr_col, out, 0, &skip, &extra, kSellGiantMin);
  auto up = [&](const std::vector<int>& v) {
    int* d = dalloc<int>(v.size());
    out.owned.push_back(d);
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    return d;
  };
  SellPlan& q = out.sp.sell;
  q.base = up(base);
  q.row0 = up(h.row0);
  q.nparts = up(nparts);
  q.slot0 = up(slot0);
  q.part_sums = dalloc<double>(static_cast<size_t>(slots) * 32);
  out.owned.push_back(q.part_sums);
  q.arrivals = dalloc<unsigned>(G);
  out.owned.push_back(q.arrivals);
  CK(cudaMemset(q.arrivals, 0, G * sizeof(unsigned)));
  int* idx = dalloc<int>(static_cast<size_t>(b));
  double* val = dalloc<double>(static_cast<size_t>(b));
  out.owned.push_back(idx);
  out.owned.push_back(val);
  q.idx = idx;
  q.val = val;
  q.n_groups = G;
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    c->max_giant = std::max(c->max_giant, out.sp.n_multi + G);
  }
}

// interleave: entry j of row row0[g] + lane -> base[g] + 32 j + lane
__global__ void k_sell_pack(const int* __restrict__ ptr, const int* __restrict__ col,
                            const double* __restrict__ val, const int* __restrict__ base,
                            const int* __restrict__ row0, int n_groups, int* idx_out,
                            double* val_out) {
  for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
    const int b = base[g];
    const int r0 = row0[g];
    const int len = ptr[r0 + 1] - ptr[r0];
    for (int t = threadIdx.x; t < 32 * len; t += blockDim.x) {
      const int j = t >> 5, lane = t & 31;
      const int k = ptr[r0 + lane] + j;
      idx_out[b + t] = col[k];
      val_out[b + t] = val[k];
    }
  }
}

void pack_sell(folp_gpu_ctx* c, PlanDev& p) {
  SellPlan& q = p.sp.sell;
  if (q.n_groups == 0) return;
  k_sell_pack<<<std::min(q.n_groups, c->sms * 8), 256, 0, c->stream>>>(
      c->csr_ptr, c->csr_col, c->csr_work, q.base, q.row0, q.n_groups, const_cast<int*>(q.idx),
      const_cast<double*>(q.val));
  ++c->launches;
  CK(cudaGetLastError());
}

// ---------------------------------------------------------------------
// Uniform working bounds (ops.cuh LoopBufs l_uni / u_uni): one pass per
// vector comparing bit patterns with the first entry; FOLP_UNIFORM_BOUNDS=0
// keeps the arrays.
__global__ void k_uniform_check(const double* __restrict__ v, int64_t n, int* differs) {
  const long long v0 = __double_as_longlong(v[0]);
  int d = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    d |= __double_as_longlong(v[i]) != v0;
  }
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(differs, 1);
}

void check_uniform_bounds(folp_gpu_ctx* c) {
  c->bounds_checked = true;
  const char* env = std::getenv("FOLP_UNIFORM_BOUNDS");
  if ((env != nullptr && std::atoi(env) == 0) || c->n == 0) return;
  int* flags = dalloc<int>(2);
  CK(cudaMemsetAsync(flags, 0, 2 * sizeof(int), c->stream));
  k_uniform_check<<<c->simple_grid(c->n), kBlock, 0, c->stream>>>(c->lw, c->n, flags);
  k_uniform_check<<<c->simple_grid(c->n), kBlock, 0, c->stream>>>(c->uw, c->n, flags + 1);
  c->launches += 2;
  int h[2] = {1, 1};
  double v[2] = {0.0, 0.0};
  CK(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&v[0], c->lw, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&v[1], c->uw, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  block_free(flags);
  c->l_uni = h[0] == 0 ? 1 : 0;
  c->u_uni = h[1] == 0 ? 1 : 0;
  c->l_const = v[0];
  c->u_const = v[1];
}
