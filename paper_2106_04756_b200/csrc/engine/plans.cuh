// plans.cuh -- unit plans, uploads and the device CSR->CSC transpose.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

double tile_segs_cutoff() {
  const char* env = std::getenv("FOLP_TILE_CUTOFF");
  return env ? std::atof(env) : 0.0;  // mean segment length below which tiles hold <= 64 segments
}

// Warp units of one axis (see segdot.cuh): tiles of consecutive short
// segments (<= kWarpTile nonzeros, <= 256 segments each) and fixed parts of
// the longer ones, in index order.
// `skip` (optional): segments left out of the tiles and parts (the SELL
// groups' rows); `extra`: units appended to every build (their SELL parts).
void build_plan(folp_gpu_ctx* c, const int64_t* ptr, int64_t S, int64_t nnz,
                const int* d_ptr, const int* d_idx, PlanDev& out, int64_t s_begin = 0,
                const std::vector<char>* skip = nullptr, const std::vector<int4>* extra = nullptr,
                int64_t giant_min_plan = kGiantMin) {
  const bool ordered = c->ordered;
  // segments per tile: tree mode caps it when segments are very short (a
  // lane then owns several segments, and every extra round waits behind the
  // gather queue for its operands); FOLP_TILE_SEGS overrides
  int64_t max_segs = kWarpTile;
  if (!ordered && S > s_begin) {
    const double mean = static_cast<double>(ptr[S] - ptr[s_begin]) / static_cast<double>(S - s_begin);
    if (const char* env = std::getenv("FOLP_TILE_SEGS")) {
      max_segs = std::max(1, std::atoi(env));
    } else if (mean < tile_segs_cutoff()) {
      max_segs = 64;
    }
  }
  // tree mode, large axes: segments longer than the serial cap are summed by
  // a warp (one "single part" unit, epilogue into the warp's accumulators)
  // instead of by one lane -- a lane walking up to 256 products in sequence
  // made the slowest warp of a power-law axis 40 % slower than the median
  // (tools/warp_timeline.py).  FOLP_SERIAL_CAP overrides (256 = off; default
  // kSerialCap).  Not
  // for small axes, whose plans may run in k_chunk_cluster.
  int64_t serial_cap = kWarpTile;
  // ... and segments up to single_max entries are one warp unit each (no
  // parts: no arrival atomics, fences or slots; the balanced order below
  // spreads their cost).  FOLP_SINGLE_MAX overrides.
  int64_t single_max = kWarpTile;
  if (!ordered && nnz > (int64_t(1) << 20)) {
    const char* env = std::getenv("FOLP_SERIAL_CAP");
    serial_cap = std::min<int64_t>(kWarpTile, std::max<int64_t>(1, env ? std::atoi(env) : kSerialCap));
    const char* smax = std::getenv("FOLP_SINGLE_MAX");
    single_max = std::max<int64_t>(kWarpTile, smax ? std::atoll(smax) : kSingleMax);
    if (single_max > kWarpTile) serial_cap = std::min<int64_t>(serial_cap, kWarpTile);
  }
  std::vector<int4> units;
  std::vector<int> multi_seg, multi_parts, multi_first;
  // segments above giant_min entries are cut in kGiantPart-entry parts
  // (fewer part sums, fences and arrival atomics); FOLP_GIANT_MIN overrides
  const char* genv = std::getenv("FOLP_GIANT_MIN");
  const int64_t giant_min = genv != nullptr ? std::max<int64_t>(kWarpTile, std::atoll(genv)) : giant_min_plan;
  // One pass over the segments with tiles of at most `target` nonzeros.
  auto build = [&](int64_t target) {
    units.clear();
    multi_seg.clear();
    multi_parts.clear();
    multi_first.clear();
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
      if (skip != nullptr && (*skip)[static_cast<size_t>(s)]) {
        close(s);
        continue;
      }
      const int64_t len = ptr[s + 1] - ptr[s];
      if (len > serial_cap && (len <= kWarpTile || len <= single_max)) {
        close(s);
        units.push_back(make_int4(-1, -static_cast<int>(s) - 2, static_cast<int>(ptr[s]),
                                  static_cast<int>(ptr[s + 1])));
        continue;
      }
      if (len <= kWarpTile) {
        if (seg0 >= 0 && (tile_nnz + len > target || s - seg0 >= max_segs)) close(s);
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
      // parts: d.y = the part's own slot (its index in this original order)
      const int multi = static_cast<int>(multi_seg.size());
      const int64_t part = len > giant_min ? kGiantPart : kWarpTile;
      multi_first.push_back(static_cast<int>(units.size()));
      for (int64_t b = ptr[s]; b < ptr[s + 1]; b += part) {
        units.push_back(make_int4(-(multi + 1), static_cast<int>(units.size()), static_cast<int>(b),
                                  static_cast<int>(std::min<int64_t>(b + part, ptr[s + 1]))));
      }
      multi_seg.push_back(static_cast<int>(s));
      multi_parts.push_back(static_cast<int>(units.size()) - multi_first.back());
    }
    close(S);
    if (extra != nullptr) units.insert(units.end(), extra->begin(), extra->end());
  };
  // The number of units build(target) makes, without making them (the tile
  // retargeting below probes many targets; pure, so probes run concurrently).
  auto count_units = [&](int64_t target) -> int64_t {
    int64_t made = 0, seg0 = -1, tile_nnz = 0;
    auto close = [&](int64_t seg_end) {
      if (seg0 >= 0 && seg_end > seg0) ++made;
      seg0 = -1;
      tile_nnz = 0;
    };
    for (int64_t s = s_begin; s < S; ++s) {
      if (skip != nullptr && (*skip)[static_cast<size_t>(s)]) {
        close(s);
        continue;
      }
      const int64_t len = ptr[s + 1] - ptr[s];
      if (len > serial_cap && (len <= kWarpTile || len <= single_max)) {
        close(s);
        ++made;
        continue;
      }
      if (len <= kWarpTile) {
        if (seg0 >= 0 && (tile_nnz + len > target || s - seg0 >= max_segs)) close(s);
        if (seg0 < 0) seg0 = s;
        tile_nnz += len;
        continue;
      }
      close(s);
      if (ordered) {
        ++made;
        continue;
      }
      const int64_t part = len > giant_min ? kGiantPart : kWarpTile;
      made += (len + part - 1) / part;
    }
    close(S);
    return made + (extra != nullptr ? static_cast<int64_t>(extra->size()) : 0);
  };
  build(kWarpTile);
  // Tree mode, large axes: balance the persistent grid's warps.  A warp's
  // units run back to back behind its SM's gather queue, so a kernel ends
  // with its most loaded SM (tools/warp_timeline.py: per-warp work spread
  // 1.7x on config 2's power-law columns).  (1) Tile size retargeted so the
  // unit count is a whole number of rounds of the grid's warps; (2) per
  // round, the round's units (contiguous in memory) go to the warps with the
  // least work so far, largest first (LPT).  FOLP_BALANCE=0 disables.
  const char* benv = std::getenv("FOLP_BALANCE");
  const int nw = c->sms * kPlanCtasPerSm * kWarps;
  // modelled unit cost: entries + kCostSeg per segment + kCostUnit per unit
  // (FOLP_COST_SEG / FOLP_COST_UNIT override, for tuning)
  const char* cs_env = std::getenv("FOLP_COST_SEG");
  const char* cu_env = std::getenv("FOLP_COST_UNIT");
  const int64_t cost_seg = cs_env != nullptr ? std::atoll(cs_env) : 2;
  const int64_t cost_unit = cu_env != nullptr ? std::atoll(cu_env) : 24;
  auto cost = [cost_seg, cost_unit](const int4& d) -> int64_t {
    if (d.x <= -kSellTag) return 32 * static_cast<int64_t>(d.w - d.z) + 64 + cost_unit;
    const int64_t segs = d.x >= 0 ? d.y - d.x : 1;
    return (d.w - d.z) + cost_seg * segs + cost_unit;
  };
  // max / mean CTA load of the plain round-robin order: even plans (config
  // 5's equal parts and tiles) are left alone -- reordering them measured
  // 14 % slower there, while skewed ones gain (config 3: 11 %)
  auto rr_imbalance = [&]() {
    const int nc = nw / kWarps;
    std::vector<int64_t> ld(nc, 0);
    int64_t tot = 0;
    for (size_t u = 0; u < units.size(); ++u) {
      ld[(u % nw) / kWarps] += cost(units[u]);
      tot += cost(units[u]);
    }
    const int64_t mx = *std::max_element(ld.begin(), ld.end());
    return tot > 0 ? static_cast<double>(mx) * nc / static_cast<double>(tot) : 1.0;
  };
  const double imb0 = units.size() > static_cast<size_t>(nw) ? rr_imbalance() : 1.0;
  // (ordered plans stay in index order: balancing them measured 188 -> 165
  // us per trial on config 2 but broke config 3's full-size ordered solve --
  // NumericalError at the first restart -- for a reason not yet found)
  const bool may = !ordered;
  const bool balance = may && nnz > (int64_t(1) << 20) && (benv == nullptr || std::atoi(benv) > 0) &&
                       static_cast<int64_t>(units.size()) > nw && imb0 > kBalanceMin;
  if (std::getenv("FOLP_TIMING") != nullptr && units.size() > static_cast<size_t>(nw)) {
    std::fprintf(stderr, "[folp timing] plan S=%lld units=%zu round-robin CTA imbalance %.3f%s\n",
                 static_cast<long long>(S - s_begin), units.size(), imb0, balance ? " -> balanced" : "");
  }
  if (balance) {
    int64_t tile_units = 0, tile_nnz_total = 0;
    for (const int4& d : units) {
      if (d.x >= 0) {
        ++tile_units;
        tile_nnz_total += d.w - d.z;
      }
    }
    const int64_t other = static_cast<int64_t>(units.size()) - tile_units;
    const int64_t rounds = (static_cast<int64_t>(units.size()) + nw - 1) / nw;
    const int64_t want_tiles = rounds * nw - other;
    if (want_tiles > tile_units && tile_units > 0) {
      // the smallest tile target whose plan still fits the rounds (greedy
      // packing leaves gaps, so search rather than divide)
      const int64_t cap_units = rounds * nw;
      int64_t lo = std::max<int64_t>(32, tile_nnz_total / want_tiles), hi = kWarpTile;
      // the same bisection as probing one target after the other, with the
      // next three levels of its probe tree counted concurrently (a probe is
      // a pass over all segments: 8 sequential ones were 4 ms of config 2's
      // end-to-end solve)
      std::map<int64_t, int64_t> made;
      std::function<void(int64_t, int64_t, int, std::vector<int64_t>&)> probes =
          [&](int64_t a, int64_t b, int depth, std::vector<int64_t>& out_targets) {
            if (a >= b || depth == 0) return;
            const int64_t mid = (a + b) / 2;
            if (made.find(mid) == made.end()) out_targets.push_back(mid);
            probes(a, mid, depth - 1, out_targets);
            probes(mid + 1, b, depth - 1, out_targets);
          };
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (made.find(mid) == made.end()) {
          std::vector<int64_t> targets;
          probes(lo, hi, 3, targets);
          std::vector<int64_t> counts(targets.size(), 0);
          folp::host::parallel_for(static_cast<int64_t>(targets.size()), [&](int64_t b, int64_t e, int) {
            for (int64_t i = b; i < e; ++i) counts[static_cast<size_t>(i)] = count_units(targets[static_cast<size_t>(i)]);
          }, static_cast<int64_t>(targets.size()) << 17);
          for (size_t i = 0; i < targets.size(); ++i) made[targets[i]] = counts[i];
        }
        if (made[mid] <= cap_units) hi = mid; else lo = mid + 1;
      }
      build(lo);
      if (made.find(lo) != made.end() && made[lo] != static_cast<int64_t>(units.size())) {
        throw std::logic_error("build_plan: unit count and unit list disagree");
      }
    }
    // Balanced at CTA granularity: the 8 consecutive units a CTA's warps
    // take in one round stay together and in order (neighbouring segments
    // share gathered lines in L1); per round, the round's chunks go to the
    // CTAs with the least work so far, largest first.  A short last round
    // lands on the least loaded CTAs (CTA indices relabelled).
    const int64_t nu = static_cast<int64_t>(units.size());
    const int nc = nw / kWarps;                      // CTAs of the persistent grid
    const int64_t nchunks = (nu + kWarps - 1) / kWarps;
    auto chunk_cost = [&](int64_t ch) {
      int64_t t = 0;
      for (int64_t u = ch * kWarps; u < std::min<int64_t>(nu, (ch + 1) * kWarps); ++u) t += cost(units[u]);
      return t;
    };
    const int64_t full = nchunks / nc;
    std::vector<int64_t> assign(static_cast<size_t>(full) * nc);
    std::vector<int64_t> load(nc, 0);
    std::vector<int> co(nc);
    std::vector<int64_t> ko(nc);
    for (int64_t r = 0; r < full; ++r) {
      for (int i = 0; i < nc; ++i) ko[i] = r * nc + i;
      std::stable_sort(ko.begin(), ko.end(),
                       [&](int64_t a, int64_t b) { return chunk_cost(a) > chunk_cost(b); });
      for (int b = 0; b < nc; ++b) co[b] = b;
      std::stable_sort(co.begin(), co.end(), [&](int a, int b) { return load[a] < load[b]; });
      for (int i = 0; i < nc; ++i) {
        assign[r * nc + co[i]] = ko[i];
        load[co[i]] += chunk_cost(ko[i]);
      }
    }
    for (int b = 0; b < nc; ++b) co[b] = b;
    std::stable_sort(co.begin(), co.end(), [&](int a, int b) { return load[a] < load[b]; });
    std::vector<int> label(nc);
    for (int i = 0; i < nc; ++i) label[co[i]] = i;
    // unit u runs on warp u mod nw = CTA (u mod nw) / 8; round r of CTA b is
    // units r * nw + 8 b .. + 7
    // slots the balanced order leaves empty (a partial chunk not in the
    // last position) hold empty tiles {0, 0, 0, 0}: no segment, no entry
    const int64_t rest_chunks = nchunks - full * nc;
    std::vector<int4> perm(static_cast<size_t>(full * nw + rest_chunks * kWarps), make_int4(0, 0, 0, 0));
    auto put_chunk = [&](int64_t r, int b, int64_t ch) {
      for (int j = 0; j < kWarps; ++j) {
        const int64_t src = ch * kWarps + j, dst = r * nw + static_cast<int64_t>(b) * kWarps + j;
        if (src < nu) perm[dst] = units[src];
      }
    };
    for (int64_t r = 0; r < full; ++r) {
      for (int b = 0; b < nc; ++b) put_chunk(r, label[b], assign[r * nc + b]);
    }
    const int64_t rest = nchunks - full * nc;
    if (rest > 0) {  // CTAs 0..rest-1 are the least loaded: largest chunks first
      std::vector<int64_t> ro(rest);
      for (int64_t i = 0; i < rest; ++i) ro[i] = full * nc + i;
      std::stable_sort(ro.begin(), ro.end(),
                       [&](int64_t a, int64_t b) { return chunk_cost(a) > chunk_cost(b); });
      // the last round's slots are the first nu - full * nw; a partial chunk
      // must take the highest slots so no slot inside the range stays empty
      const int64_t last = nchunks - 1;
      const bool partial = nu % kWarps != 0;
      int64_t slot = 0;
      for (int64_t i = 0; i < rest; ++i) {
        if (partial && ro[i] == last) continue;
        put_chunk(full, static_cast<int>(slot++), ro[i]);
      }
      if (partial) put_chunk(full, static_cast<int>(slot), last);
    }
    while (!perm.empty() && perm.back().x == 0 && perm.back().y == 0 && perm.back().w == 0) perm.pop_back();
    if (std::getenv("FOLP_TIMING") != nullptr) {
      units.swap(perm);
      std::fprintf(stderr, "[folp timing] plan S=%lld balanced: units=%zu imbalance %.3f\n",
                   static_cast<long long>(S - s_begin), units.size(), rr_imbalance());
      units.swap(perm);
    }
    units.swap(perm);
  }
  auto up = [&](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* d = dalloc<T>(v.size());
    out.owned.push_back(d);
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  };
  {
    std::vector<int> ls;
    bool pairs = s_begin == 0 && S > 0 && skip == nullptr && ptr[0] == 0;
    for (int64_t sg = s_begin; sg < S; ++sg) {
      const int64_t len = ptr[sg + 1] - ptr[sg];
      if (len > kLongSeq) ls.push_back(static_cast<int>(sg));
      pairs = pairs && len == 2;
    }
    out.pair_len = pairs ? 2 : 0;  // every segment s is entries 2s, 2s+1 (pair_kernel)
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
  p.multi_first = up(multi_first);
  p.n_multi = static_cast<int>(multi_seg.size());
  p.part_sums = dalloc<double>(units.size());
  out.owned.push_back(p.part_sums);
  p.arrivals = dalloc<unsigned>(multi_seg.size());
  out.owned.push_back(p.arrivals);
  CK(cudaMemset(p.arrivals, 0, std::max<size_t>(1, multi_seg.size()) * sizeof(unsigned)));
  {
    static std::mutex mu;  // plans of one context may be built on two host threads
    std::lock_guard<std::mutex> lk(mu);
    c->max_giant = std::max(c->max_giant, p.n_multi);
  }
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

// Host <-> device vector copies.  Vectors of at least kStageMin doubles go
// through a cached pinned block: pageable cudaMemcpyAsync ran at 2-3 GB/s on
// the B200 hosts (the final point of config 2, 4.8 MB, took 1.8 ms), a DMA
// from / to pinned memory plus a memcpy on all host cores a fifth of that.
// A staged copy completes in sync_transfers(), which every entry point that
// uploads or downloads calls in place of its stream synchronize.
constexpr int64_t kStageMin = int64_t(1) << 15;
void upload(folp_gpu_ctx* c, double* dst, const double* src, int64_t count) {
  if (count <= 0) return;
  const size_t bytes = static_cast<size_t>(count) * sizeof(double);
  if (src == nullptr) {
    CK(cudaMemsetAsync(dst, 0, bytes, c->stream));
  } else if (count >= kStageMin) {
    double* h = static_cast<double*>(block_alloc(bytes, true));
    c->staged.push_back({h, nullptr, bytes});
    folp::host::parallel_for(count, [&](int64_t b, int64_t e, int) {
      std::memcpy(h + b, src + b, static_cast<size_t>(e - b) * sizeof(double));
    });
    CK(cudaMemcpyAsync(dst, h, bytes, cudaMemcpyHostToDevice, c->stream));
  } else {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
  }
}
void download(folp_gpu_ctx* c, double* dst, const double* src, int64_t count) {
  if (count <= 0 || dst == nullptr) return;
  const size_t bytes = static_cast<size_t>(count) * sizeof(double);
  if (count >= kStageMin) {
    double* h = static_cast<double*>(block_alloc(bytes, true));
    c->staged.push_back({h, dst, bytes});
    CK(cudaMemcpyAsync(h, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  } else {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
  }
}
// Stream synchronize + the host half of the staged copies.
void sync_transfers(folp_gpu_ctx* c) {
  const cudaError_t err = cudaStreamSynchronize(c->stream);
  for (const auto& s : c->staged) {
    if (err == cudaSuccess && s.host_dst != nullptr) {
      const int64_t count = static_cast<int64_t>(s.bytes / sizeof(double));
      const double* h = static_cast<const double*>(s.pinned);
      double* d = s.host_dst;
      folp::host::parallel_for(count, [&](int64_t b, int64_t e, int) {
        std::memcpy(d + b, h + b, static_cast<size_t>(e - b) * sizeof(double));
      });
    }
    block_free(s.pinned);
  }
  c->staged.clear();
  CK(err);
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
