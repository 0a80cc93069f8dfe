// segdot.cuh -- the one sparse-product kernel family of the engine.
//
// Every K-application of the PDLP loop is a "segmented dot": for each
// segment s (a CSR row for K x, a CSC column = row of K' for K'y),
//     dot_s = sum_{k in seg s} val[k] * vec[idx[k]]
// followed by a per-segment *epilogue* that consumes dot_s in registers
// (the fused primal / dual projected step, a residual, ...) and feeds
// per-thread reduction accumulators.  The reductions are deterministic:
// a fixed block->work mapping, fixed shuffle trees, per-block partials and a
// last-block-done final pass in index order -- no floating-point atomics, so
// a rerun is bit-identical (the reference pins that in
// proj/tests/acceptance_main.cpp:653-682).
//
// Load balancing for skewed segment lengths (power-law columns of config 2,
// the 2M-entry sum row of config 3, 8000-long rows of config 5) uses four
// work classes built once on the host (SegPlan):
//   bulk  : segments in natural order, L lanes each (L = 1..32 from the mean
//           length), len <= bulk_max       -> coalesced epilogue accesses
//   long  : warp per segment, len <= kLongMax
//   huge  : CTA per segment,  len <= kHugeMax
//   giant : several CTAs per segment (fixed parts); the last part to arrive
//           sums the parts in part order and runs the epilogue; its
//           reduction contribution goes to a per-segment slot so the final
//           order does not depend on arrival order.
// Tiles of all classes are distributed round-robin over a persistent grid
// (a few CTAs per SM), so the partial count stays ~1e3 at every size.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace folpgpu {

constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr int kLongMax = 2048;     // warp-per-segment up to this length
constexpr int kHugeMax = 65536;    // CTA-per-segment up to this length
constexpr int kGiantPart = 16384;  // nnz per part of a giant segment
constexpr int kMaxAcc = 30;        // widest reduction (bisection pass)

// std::max / std::min semantics (NaN in `a` propagates), which the
// reference's projections rely on for its NonFiniteIterate detection.
__device__ __forceinline__ double ref_max(double a, double b) {
  return (a < b) ? b : a;
}
__device__ __forceinline__ double ref_min(double a, double b) {
  return (b < a) ? b : a;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

struct SegPlan {
  const int* ptr;   // [S+1]
  const int* idx;   // [nnz] gather index of each entry
  int S;
  int bulk_max;     // bulk class handles len <= bulk_max
  int n_bulk_tiles; // ceil(S / (kBlock / L))
  const int* long_ids;
  int n_long;
  int n_long_tiles;  // ceil(n_long / kWarps)
  const int* huge_ids;
  int n_huge;
  const int* giant_ids;   // [n_giant]
  const int* giant_first; // [n_giant + 1] first part of each giant segment
  int n_giant;
  const int* part_giant;  // [n_parts] owning giant index
  const int* part_beg;    // [n_parts]
  const int* part_end;    // [n_parts]
  int n_parts;
  double* part_sums;        // [n_parts]
  unsigned* giant_arrivals; // [n_giant]
  int total_tiles;
};

struct RedBuf {
  double* partials;   // [(gridDim.x + n_giant) * K]
  unsigned* counter;  // zero between launches (reset by the last block)
};

// Sum over the CTA; result valid in thread 0.  Ends with a barrier so the
// scratch can be reused immediately.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += scratch[w];
  }
  __syncthreads();
  return s;
}

template <int K>
__device__ __forceinline__ void block_sum_vec(double (&acc)[K],
                                              double (*scratch)[K],
                                              double (&out)[K]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) scratch[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += scratch[w][k];
      out[k] = s;
    }
  }
  __syncthreads();
}

// Per-block partial + last-block-done final reduction, then epi.finalize().
template <class Epi>
__device__ __forceinline__ void reduce_tail(const Epi& epi, double (&acc)[Epi::K],
                                            RedBuf rb, int n_extra) {
  constexpr int K = Epi::K;
  __shared__ double s_vec[kWarps][K];
  __shared__ int s_last;
  double tot[K];
  block_sum_vec<K>(acc, s_vec, tot);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) rb.partials[blockIdx.x * K + k] = tot[k];
    __threadfence();
    const unsigned ticket = atomicAdd(rb.counter, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int np = static_cast<int>(gridDim.x) + n_extra;
  double part[K];
#pragma unroll
  for (int k = 0; k < K; ++k) part[k] = 0.0;
  for (int i = threadIdx.x; i < np; i += kBlock) {
#pragma unroll
    for (int k = 0; k < K; ++k) part[k] += ld_cg(&rb.partials[i * K + k]);
  }
  block_sum_vec<K>(part, s_vec, tot);
  if (threadIdx.x == 0) {
    epi.finalize(tot);
    *rb.counter = 0u;
  }
}

// The segmented-dot kernel.  L = lanes per bulk segment.
// Epi must provide:  static constexpr int K (>= 1); static constexpr bool
//   kReduce (run the reduction tail); __device__ bool prepare();
//   __device__ const double* vec() const;
//   __device__ void apply(int seg, double dot, double (&acc)[K]) const;
//   __device__ void finalize(const double (&tot)[K]) const;
template <int L, class Epi>
__global__ void __launch_bounds__(kBlock)
segdot_kernel(SegPlan p, const double* __restrict__ val, Epi epi, RedBuf rb) {
  constexpr int K = Epi::K;
  if (!epi.prepare()) return;  // loop slot disabled: every CTA agrees
  const double* __restrict__ vec = epi.vec();
  const int* __restrict__ idx = p.idx;
  __shared__ double s_cta[kWarps];
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t_huge0 = p.n_parts;
  const int t_long0 = t_huge0 + p.n_huge;
  const int t_bulk0 = t_long0 + p.n_long_tiles;

  for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
    if (t >= t_bulk0) {
      // ---- bulk: kBlock/L consecutive segments, L lanes each ----
      const int seg = (t - t_bulk0) * (kBlock / L) + tid / L;
      const int sub = tid % L;
      double s = 0.0;
      bool mine = false;
      if (seg < p.S) {
        const int beg = p.ptr[seg], end = p.ptr[seg + 1];
        mine = (end - beg) <= p.bulk_max;
        if (mine) {
#pragma unroll 4
          for (int k = beg + sub; k < end; k += L) s += val[k] * __ldg(&vec[idx[k]]);
        }
      }
      if (L > 1) {
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off, L);
      }
      if (mine && sub == 0) epi.apply(seg, s, acc);
    } else if (t >= t_long0) {
      // ---- long: one warp per segment ----
      const int i = (t - t_long0) * kWarps + warp;
      if (i < p.n_long) {
        const int seg = p.long_ids[i];
        const int beg = p.ptr[seg], end = p.ptr[seg + 1];
        double s = 0.0;
#pragma unroll 4
        for (int k = beg + lane; k < end; k += 32) s += val[k] * __ldg(&vec[idx[k]]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
        if (lane == 0) epi.apply(seg, s, acc);
      }
    } else if (t >= t_huge0) {
      // ---- huge: one CTA per segment ----
      const int seg = p.huge_ids[t - t_huge0];
      const int beg = p.ptr[seg], end = p.ptr[seg + 1];
      double s = 0.0;
#pragma unroll 4
      for (int k = beg + tid; k < end; k += kBlock) s += val[k] * __ldg(&vec[idx[k]]);
      s = block_sum(s, s_cta);
      if (tid == 0) epi.apply(seg, s, acc);
    } else {
      // ---- giant: one fixed part of a segment ----
      const int beg = p.part_beg[t], end = p.part_end[t];
      double s = 0.0;
#pragma unroll 4
      for (int k = beg + tid; k < end; k += kBlock) s += val[k] * __ldg(&vec[idx[k]]);
      s = block_sum(s, s_cta);
      if (tid == 0) {
        p.part_sums[t] = s;
        __threadfence();
        const int g = p.part_giant[t];
        const int first = p.giant_first[g];
        const int np = p.giant_first[g + 1] - first;
        const unsigned arrived = atomicAdd(&p.giant_arrivals[g], 1u);
        if (arrived == static_cast<unsigned>(np - 1)) {
          __threadfence();
          double total = 0.0;
          for (int q = 0; q < np; ++q) total += ld_cg(&p.part_sums[first + q]);
          double gacc[K];
#pragma unroll
          for (int k = 0; k < K; ++k) gacc[k] = 0.0;
          epi.apply(p.giant_ids[g], total, gacc);
          if constexpr (Epi::kReduce) {
#pragma unroll
            for (int k = 0; k < K; ++k) rb.partials[(gridDim.x + g) * K + k] = gacc[k];
          }
          p.giant_arrivals[g] = 0u;
        }
      }
    }
  }
  if constexpr (Epi::kReduce) reduce_tail(epi, acc, rb, p.n_giant);
}

// Elementwise kernel with the same deterministic reduction tail.
// Op must provide K (>= 1), kReduce, prepare(), apply(i, acc), finalize(tot).
template <class Op>
__global__ void __launch_bounds__(kBlock) elementwise_kernel(int64_t n, Op op, RedBuf rb) {
  constexpr int K = Op::K;
  if (!op.prepare()) return;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kBlock;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; i < n; i += stride) {
    op.apply(i, acc);
  }
  if constexpr (Op::kReduce) reduce_tail(op, acc, rb, 0);
}

}  // namespace folpgpu
