// blocked.cuh -- window-blocked products and per-axis scaling primitives.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

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
  // rows whose gathers are coalesced already (SELL-32 groups + contiguous
  // rows, sell.cuh) read x as streams: no windows needed
  if (rows_axis && c->sell && c->sell_coalesced) return;
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
