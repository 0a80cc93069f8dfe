// setup_kernels.cuh -- scaling, start-point, reduced-point and small utility kernels.
// Fragment of engine.cu: included inside its anonymous namespace, after
// the pieces it uses (one translation unit; see engine.cu for the order).
#pragma once

// ---------------------------------------------------------------------
// Scaling kernels (rescale_problem, scaling.cpp:48-96; axis_norms,
// sparse_matrix.cpp:156-186).
__global__ void k_axis_absmax(const int* __restrict__ ptr, const double* __restrict__ val,
                              int S, double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < S; s += nwarps) {
    if (ptr[s + 1] - ptr[s] > kWarpTile) {  // long: k_long_absmax takes it
      if (lane == 0) out[s] = 0.0;
      continue;
    }
    double a = 0.0;
    for (int k = ptr[s] + lane; k < ptr[s + 1]; k += 32) a = fmax(a, fabs(val[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) out[s] = a;  // max is order-independent: bit-exact
  }
}

// The long segments of an axis by the units of its plan (parts, or the
// ordered plan's single long units): warp maxima folded by an integer
// atomicMax on the bit pattern (non-negative doubles order like their bits),
// so the result is the exact maximum in any order.
__device__ __forceinline__ int long_unit_segment(const SegPlan& p, const int4& d) {
  if (d.x < 0) {  // single units: the long ones are this axis' long segments too
    if (d.y < 0) return d.w - d.z > kWarpTile ? -d.y - 2 : -1;
    return p.multi_seg[-d.x - 1];
  }
  return d.w - d.z > kWarpTile ? d.x : -1;
}

__global__ void k_long_absmax(SegPlan p, const double* __restrict__ val, double* out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int u = warp; u < p.n_units; u += nwarps) {
    const int4 d = p.units[u];
    const int seg = long_unit_segment(p, d);
    if (seg < 0) continue;
    double a = 0.0;
    for (int k = d.z + lane; k < d.w; k += 32) a = fmax(a, fabs(val[k]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
    if (lane == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(out + seg),
                static_cast<unsigned long long>(__double_as_longlong(a)));
    }
  }
}

// Sequential per-segment p-norm in increasing index order: bit-identical to
// the reference's loop for p = 0, 1, 2 (pow for other p is CUDA's).
constexpr int kLongSeq = 1024;  // segments above this: k_axis_pnorm_long

template <int MODE>
__device__ __forceinline__ double pnorm_term(double v, double p) {
  const double a = fabs(v);
  if constexpr (MODE == 0) {
    return 1.0;
  } else if constexpr (MODE == 1) {
    return a;
  } else if constexpr (MODE == 2) {
    return a * a;
  } else {
    return pow(a, p);
  }
}
template <int MODE>
__device__ __forceinline__ double pnorm_finish(double acc, double p) {
  if constexpr (MODE == 2) {
    return sqrt(acc);
  } else if constexpr (MODE == 3) {
    return (isfinite(p) && p > 1.0) ? pow(acc, 1.0 / p) : acc;
  } else {
    return acc;
  }
}

// A long segment's norm, still one sequential sum in index order (the
// reference's rounding), but its terms are staged into shared memory by the
// whole warp (coalesced, double-buffered) so the single summing lane only
// waits on its add chain, not on a global load per term.
template <int MODE>
__global__ void __launch_bounds__(32) k_axis_pnorm_long(const int* __restrict__ ptr,
                                                        const double* __restrict__ val,
                                                        const int* __restrict__ segs, double p,
                                                        double* __restrict__ out) {
  constexpr int kChunk = 1024;
  __shared__ double buf[2][kChunk];
  const int s = segs[blockIdx.x];
  const int lane = threadIdx.x;
  const int b = ptr[s], e = ptr[s + 1];
  double acc = 0.0;
  int slot = 0;
  // a chunk's 32 loads per lane are issued back to back, then stored
  auto stage = [&](int c0, double* dst) {
    double v[kChunk / 32];
#pragma unroll
    for (int q = 0; q < kChunk / 32; ++q) {
      const int k = c0 + lane + 32 * q;
      v[q] = k < e ? val[k] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kChunk / 32; ++q) {
      const int k = c0 + lane + 32 * q;
      if (k < e) dst[lane + 32 * q] = pnorm_term<MODE>(v[q], p);
    }
  };
  stage(b, buf[0]);
  __syncwarp();
  for (int c0 = b; c0 < e; c0 += kChunk, slot ^= 1) {
    const int c1 = min(c0 + kChunk, e);
    // stage the next chunk while lane 0 sums this one
    if (c1 < e) stage(c1, buf[slot ^ 1]);
    if (lane == 0) {
      const double* t = buf[slot];
      const int len = c1 - c0;
      int j = 0;
      for (; j + 16 <= len; j += 16) {  // loads hoisted ahead of the add chain
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = t[j + q];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += v[q];
      }
      for (; j < len; ++j) acc += t[j];
    }
    __syncwarp();
  }
  if (lane == 0) out[s] = pnorm_finish<MODE>(acc, p);
}

template <int MODE>  // 0: count, 1: sum |a|, 2: sqrt(sum a^2), 3: (sum |a|^p)^(1/p)
__global__ void k_axis_pnorm_seq(const int* __restrict__ ptr, const double* __restrict__ val,
                                 int S, double p, double* __restrict__ out) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    double acc = 0.0;
    const int b = ptr[s], e = ptr[s + 1];
    if (e - b > kLongSeq) continue;  // k_axis_pnorm_long
    if constexpr (MODE == 0) {
      for (int k = b; k < e; ++k) acc += 1.0;
    } else {
#pragma unroll 8
      for (int k = b; k < e; ++k) {
        const double a = fabs(val[k]);
        if constexpr (MODE == 1) {
          acc += a;
        } else if constexpr (MODE == 2) {
          acc += a * a;
        } else {
          acc += pow(a, p);
        }
      }
    }
    if constexpr (MODE == 2) {
      acc = sqrt(acc);
    } else if constexpr (MODE == 3) {
      if (isfinite(p) && p > 1.0) acc = pow(acc, 1.0 / p);
    }
    out[s] = acc;
  }
}

__global__ void k_recip_sqrt_cum(double* __restrict__ v, double* __restrict__ cum, int S) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const double x = v[s];
    const double d = x > 0.0 ? 1.0 / sqrt(x) : 1.0;
    v[s] = d;
    cum[s] *= d;
  }
}

// SparseMatrix::scaled (sparse_matrix.cpp:222-242): out = src * (dseg*didx).
__global__ void k_scale_values(const int* __restrict__ ptr, const int* __restrict__ idx,
                               const double* __restrict__ src, double* __restrict__ dst,
                               int S, const double* __restrict__ dseg,
                               const double* __restrict__ didx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < S; s += nwarps) {
    if (ptr[s + 1] - ptr[s] > kWarpTile) continue;  // long: k_long_scale
    const double ds = dseg[s];
    for (int k = ptr[s] + lane; k < ptr[s + 1]; k += 32) dst[k] = src[k] * (ds * didx[idx[k]]);
  }
}

__global__ void k_long_scale(SegPlan p, const int* __restrict__ idx, const double* src,
                             double* dst, const double* __restrict__ dseg,
                             const double* __restrict__ didx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int u = warp; u < p.n_units; u += nwarps) {
    const int4 d = p.units[u];
    const int seg = long_unit_segment(p, d);
    if (seg < 0) continue;
    const double ds = dseg[seg];
    for (int k = d.z + lane; k < d.w; k += 32) dst[k] = src[k] * (ds * didx[idx[k]]);
  }
}

// Scaled vectors (scaling.cpp:82-94).
__global__ void k_scale_vectors(int64_t n, int64_t m, const double* c, const double* l,
                                const double* u, const double* q, const double* d1,
                                const double* d2, double* cw, double* lw, double* uw,
                                double* qw) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      const double s = d2[i];
      cw[i] = c[i] * s;
      lw[i] = l[i] / s;
      uw[i] = u[i] / s;
    } else {
      const int64_t j = i - n;
      qw[j] = q[j] * d1[j];
    }
  }
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_narrow(const int64_t* __restrict__ src, int* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = static_cast<int>(src[i]);
}

// Working column numbering (folp_gpu_create_ordered): column indices
// through rank[], n-vectors gathered through order[].
__global__ void k_renumber(int* __restrict__ idx, const int* __restrict__ rank, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = rank[idx[i]];
}
__global__ void k_gather_order(const double* __restrict__ src, const int* __restrict__ order,
                               double* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[order[i]];
}

// Start point (solver.cpp:853-865): z/D then projected.
__global__ void k_start_point(int64_t n, int64_t m, int64_t m1, const double* x0,
                              const double* y0, const double* d1, const double* d2,
                              const double* lw, const double* uw, double* x, double* y,
                              double* lx, double* ly) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      const double v = ref_min(ref_max(x0[i] / d2[i], lw[i]), uw[i]);
      x[i] = v;
      lx[i] = v;
    } else {
      const int64_t j = i - n;
      double v = y0[j] / d1[j];
      if (j < m1) v = ref_max(v, 0.0);
      y[j] = v;
      ly[j] = v;
    }
  }
}

// reduced_point (solver.cpp:495-502).
__global__ void k_reduced_point(int64_t n, int64_t m, const double* xs, const double* ys,
                                const double* d1, const double* d2, const double* l,
                                const double* u, double* xr, double* yr) {
  const int64_t total = n + m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      xr[i] = ref_min(ref_max(xs[i] * d2[i], l[i]), u[i]);
    } else {
      const int64_t j = i - n;
      yr[j] = ys[j] * d1[j];
    }
  }
}

__global__ void k_div_scalar(double* __restrict__ dst, const double* __restrict__ src,
                             int64_t n, const double* __restrict__ denom_sq) {
  const double snorm = sqrt(denom_sq[0]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] / snorm;  // sparse_matrix.cpp:213
}

// max |v|: grid-stride partial maxima into out_blocks, then one block folds
// them (max is order-independent, so exact).
__global__ void k_absmax_blocks(const double* __restrict__ v, int64_t n, double* out_blocks) {
  __shared__ double s[kWarps];
  double a = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs(v[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kWarps; ++w) r = fmax(r, s[w]);
    out_blocks[blockIdx.x] = r;
  }
}

__global__ void k_absmax_all(const double* __restrict__ v, int64_t n, double* out) {
  __shared__ double s[kWarps];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fmax(a, fabs(v[i]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kWarps; ++w) r = fmax(r, s[w]);
    *out = r;
  }
}

struct OpCountNonFinite {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  int64_t n;
  const double* x;
  const double* y;
  double* result;
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    const double v = i < n ? x[i] : y[i - n];
    acc.add(0, i, isfinite(v) ? 0.0 : 1.0);
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
  __device__ void finalize_ordered(const double* t, int64_t cnt) const {
    result[0] = any_nonzero(t, cnt) ? 1.0 : 0.0;
  }
};

struct OpNormSq {
  static constexpr int K = 1;
  static constexpr bool kReduce = true;
  const double* v;
  double* result;
  __device__ bool prepare() { return true; }
  template <class Acc>
  __device__ void apply(int64_t i, Acc& acc) const {
    acc.add(0, i, v[i] * v[i]);
  }
  __device__ void finalize(const double (&tot)[K]) const { result[0] = tot[0]; }
  // linalg::norm2_squared order (linalg.hpp:31-35)
  __device__ void finalize_ordered(const double* t, int64_t cnt) const {
    result[0] = fold(0.0, t, cnt);
  }
  // ordered mode through the exact parallel fold (one thread walking 400k
  // terms took 13 ms per norm)
  __host__ void fold_plan(const double* t, int64_t cnt, FoldJobs& f) const {
    f.count = 1;
    f.job[0] = FoldJob{t, cnt, 0.0, -1, 1.0, nullptr, nullptr};
  }
  __device__ void finalize_exact(const double* r, unsigned) const { result[0] = r[0]; }
};
