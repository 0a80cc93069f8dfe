// tma_gather.cu -- can the TMA unit add random-gather throughput on top of
// the L1tex (LSU) path?  The step kernels are bound by the L1tex data pipe:
// one wavefront per gathered 8-byte element, ~242 G gathers/s on B200
// (spmv_ceiling).  A TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4)
// fetches four 16-byte rows of a [X/2][2] fp64 view into shared memory without
// LSU wavefronts; the consumer then reads them with 2 smem wavefronts per warp.
// Variants (same index stream: the config matrix's CSR column indices):
//   lsu     : s += x[idx[k]]                                   (baseline)
//   tma     : every gather through gather4, summed from smem
//   mixed F : gathers of chunk slots < F*256 via TMA, the rest via LSU
// Prints us and G gathers/s (CUDA events, 20 reps after warm-up).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>

#include "folp_gen.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int kChunk = 256;  // gathers per chunk = threads per CTA
constexpr int kStages = 4;

__device__ __forceinline__ void block_add(double v, double* out) {
  __shared__ double ws[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    atomicAdd(out, t);
  }
}

__global__ void k_lsu(const int* __restrict__ idx, const double* __restrict__ x, int64_t nnz,
                      double* out) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
#pragma unroll 8
  for (; k < nnz; k += stride) s += __ldg(&x[idx[k]]);
  block_add(s, out);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap* map, void* dst, uint64_t* bar, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
      "r"(smem_u32(bar))
      : "memory");
}

// Chunks c = blockIdx.x + i * gridDim.x of kChunk gathers.  Slots below
// n_tma (multiple of 4) are fetched by gather4 (one op per 4 slots, issued by
// threads 0 .. n_tma/4-1), the rest by the consuming thread through the LSU.
__global__ void __launch_bounds__(kChunk) k_tma(const __grid_constant__ CUtensorMap map,
                                                const int* __restrict__ idx,
                                                const double* __restrict__ x, int64_t nnz,
                                                int n_tma, double* out) {
  __shared__ alignas(128) double buf[kStages][kChunk * 4];  // 128-B slot per gather4
  __shared__ uint64_t bar[kStages];
  const int t = threadIdx.x;
  const int64_t n_chunks = nnz / kChunk;
  const int n_issue = n_tma / 4;
  if (t == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t c, int s) {
    if (c >= n_chunks) return;
    if (t == 0) mbar_expect(&bar[s], n_tma * 16);
    if (t < n_issue) {
      int4 r = *reinterpret_cast<const int4*>(idx + c * kChunk + 4 * t);
      r.x >>= 1; r.y >>= 1; r.z >>= 1; r.w >>= 1;
      tma_gather4(&map, &buf[s][t * 16], &bar[s], r);
    }
  };
  int64_t c = blockIdx.x;
  for (int s = 0; s < kStages; ++s) issue(c + (int64_t)s * gridDim.x, s);
  double acc = 0.0;
  unsigned phase = 0;
  for (int i = 0; c < n_chunks; ++i, c += gridDim.x) {
    const int s = i % kStages;
    const int j = idx[c * kChunk + t];
    double lsu = 0.0;
    if (t >= n_tma) lsu = __ldg(&x[j]);
    if (n_tma > 0) mbar_wait(&bar[s], phase);
    acc += t < n_tma ? buf[s][(t >> 2) * 16 + (t & 3) * 2 + (j & 1)] : lsu;
    if (s == kStages - 1) phase ^= 1u;
    __syncthreads();
    if (t < n_issue) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(c + (int64_t)kStages * gridDim.x, s);
  }
  block_add(acc, out);
}


// Fair additivity test: warps [0, 8-T) gather [0, nL) through the LSU in
// k_lsu's pattern; warps [8-T, 8) gather [nL, nnz) through gather4 with a
// per-warp ring of kRing 128-entry stages (lane l issues entries 4l..4l+3 of
// a stage, then the warp consumes the oldest stage: 4 values per lane).
constexpr int kRing = 5;
template <int T>
__global__ void __launch_bounds__(256) k_mix(const __grid_constant__ CUtensorMap map,
                                             const int* __restrict__ idx,
                                             const double* __restrict__ x, int64_t nL, int64_t nnz,
                                             double* out) {
  __shared__ alignas(128) double ring[T][kRing][32 * 16];  // 32 gather4 slots of 128 B
  __shared__ uint64_t bar[T][kRing];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < T; ++w)
      for (int s = 0; s < kRing; ++s) mbar_init(&bar[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp < 8 - T) {
    const int64_t stride = (int64_t)gridDim.x * (8 - T) * 32;
    int64_t k = (int64_t)blockIdx.x * (8 - T) * 32 + threadIdx.x;
#pragma unroll 8
    for (; k < nL; k += stride) acc += __ldg(&x[idx[k]]);
  } else {
    const int tw = warp - (8 - T);
    const int64_t n_st = (nnz - nL) / 128;
    const int64_t gw = (int64_t)gridDim.x * T;
    const int64_t me = (int64_t)blockIdx.x * T + tw;
    auto issue = [&](int64_t c, int s) {
      if (c >= n_st) return;
      if (lane == 0) mbar_expect(&bar[tw][s], 128 * 16);
      __syncwarp();
      int4 r = *reinterpret_cast<const int4*>(idx + nL + c * 128 + 4 * lane);
      r.x >>= 1; r.y >>= 1; r.z >>= 1; r.w >>= 1;
      tma_gather4(&map, &ring[tw][s][lane * 16], &bar[tw][s], r);
    };
    for (int s = 0; s < kRing; ++s) issue(me + s * gw, s);
    unsigned phase = 0;
    int s = 0;
    for (int64_t c = me; c < n_st; c += gw) {
      const int4 j = *reinterpret_cast<const int4*>(idx + nL + c * 128 + 4 * lane);
      mbar_wait(&bar[tw][s], phase);
      const double* b = &ring[tw][s][lane * 16];
      acc += b[0 + (j.x & 1)] + b[2 + (j.y & 1)] + b[4 + (j.z & 1)] + b[6 + (j.w & 1)];
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + kRing * gw, s);
      if (++s == kRing) { s = 0; phase ^= 1u; }
    }
    // tail entries [nL + n_st*128, nnz) through the LSU
    for (int64_t k = nL + n_st * 128 + me * 32 + lane; k < nnz; k += gw * 32) acc += __ldg(&x[idx[k]]);
  }
  block_add(acc, out);
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int cfg = argc > 1 ? atoi(argv[1]) : 2;
  folp_gen_lp* lp = folp_gen_config(cfg, 1, 1.0);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeTiled encode = reinterpret_cast<EncodeTiled>(fn);
  for (int axis = 0; axis < 2; ++axis) {
    const int64_t X = axis == 0 ? lp->num_cols : lp->num_rows;
    const int64_t nnz = (lp->nnz / kChunk) * kChunk;
    const int64_t* i64 = axis == 0 ? lp->row_cols : lp->col_rows;
    std::vector<int> i32(nnz);
    for (int64_t i = 0; i < nnz; ++i) i32[i] = (int)i64[i];
    const int64_t Xp = (X + 1) & ~int64_t(1);
    std::vector<double> xh(Xp);
    double expect = 0.0;
    for (int64_t i = 0; i < Xp; ++i) xh[i] = (double)(i % 1024);
    for (int64_t i = 0; i < nnz; ++i) expect += xh[i32[i]];
    int* di;
    double *dx, *dout;
    CK(cudaMalloc(&di, nnz * 4));
    CK(cudaMalloc(&dx, Xp * 8));
    CK(cudaMalloc(&dout, 64));
    CK(cudaMemcpy(di, i32.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, xh.data(), Xp * 8, cudaMemcpyHostToDevice));
    CUtensorMap map;
    memset(&map, 0, sizeof map);
    cuuint64_t dims[2] = {2, (cuuint64_t)(Xp / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, (cuuint32_t)(argc > 2 ? atoi(argv[2]) : 1)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dx, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("cfg %d axis %s: X=%lld nnz=%lld encode=%d\n", cfg, axis ? "cols(K'y)" : "rows(Kx)",
           (long long)X, (long long)nnz, (int)r);
    auto report = [&](const char* name, float ms) {
      printf("  %-12s %8.2f us  %6.1f Ggather/s\n", name, ms * 1e3, nnz / ms / 1e6);
    };
    auto verify = [&](auto launch, const char* name) {
      CK(cudaMemset(dout, 0, 8));
      launch();
      double got = 0.0;
      CK(cudaMemcpy(&got, dout, 8, cudaMemcpyDeviceToHost));
      if (got != expect) printf("  %s: MISMATCH got %.1f expect %.1f\n", name, got, expect);
    };
    verify([&] { k_lsu<<<sms * 8, 256>>>(di, dx, nnz, dout); }, "lsu");
    for (int n_tma : {64, 256}) verify([&] { k_tma<<<sms * 8, kChunk>>>(map, di, dx, nnz, n_tma, dout); }, "tma");
    report("lsu", timeit([&] { k_lsu<<<sms * 8, 256>>>(di, dx, nnz, dout); }));
    {
      // hot-first renumbering: vector entries ordered by how often they are
      // gathered (descending), indices remapped -- the locality a degree
      // ordering of the gathered axis would give
      std::vector<int64_t> cnt(Xp, 0);
      for (int64_t i = 0; i < nnz; ++i) ++cnt[i32[i]];
      std::vector<int> order(Xp), rank(Xp);
      for (int64_t i = 0; i < Xp; ++i) order[i] = (int)i;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cnt[a] > cnt[b]; });
      for (int64_t i = 0; i < Xp; ++i) rank[order[i]] = (int)i;
      std::vector<int> ih(nnz);
      for (int64_t i = 0; i < nnz; ++i) ih[i] = rank[i32[i]];
      int* dh;
      CK(cudaMalloc(&dh, nnz * 4));
      CK(cudaMemcpy(dh, ih.data(), nnz * 4, cudaMemcpyHostToDevice));
      report("lsu_hot", timeit([&] { k_lsu<<<sms * 8, 256>>>(dh, dx, nnz, dout); }));
      for (int64_t win : {int64_t(4096), int64_t(32768), int64_t(262144)}) {
        for (int64_t i = 0; i < nnz; ++i) ih[i] = (int)(i32[i] % win);
        CK(cudaMemcpy(dh, ih.data(), nnz * 4, cudaMemcpyHostToDevice));
        char name[32];
        snprintf(name, sizeof name, "lsu_win%lldk", (long long)(win * 8 / 1024));
        report(name, timeit([&] { k_lsu<<<sms * 8, 256>>>(dh, dx, nnz, dout); }));
      }
      cudaFree(dh);
      // hot share: fraction of gathers landing in the first 4k / 32k entries
      int64_t h1 = 0, h2 = 0;
      for (int64_t i = 0; i < nnz; ++i) { h1 += rank[i32[i]] < 4096; h2 += rank[i32[i]] < 32768; }
      printf("  gathers into the 4k / 32k hottest entries: %.1f %% / %.1f %%\n", 100.0 * h1 / nnz, 100.0 * h2 / nnz);
    }
    for (double f : {0.0}) {
      const int64_t nL = ((int64_t)((1.0 - f) * nnz) / 128) * 128;
      char name[32];
      verify([&] { k_mix<1><<<sms * 4, 256>>>(map, di, dx, nL, nnz, dout); }, "mix1");
      snprintf(name, sizeof name, "mix1 f%.1f", f);
      report(name, timeit([&] { k_mix<1><<<sms * 4, 256>>>(map, di, dx, nL, nnz, dout); }));
      verify([&] { k_mix<2><<<sms * 4, 256>>>(map, di, dx, nL, nnz, dout); }, "mix2");
      snprintf(name, sizeof name, "mix2 f%.1f", f);
      report(name, timeit([&] { k_mix<2><<<sms * 4, 256>>>(map, di, dx, nL, nnz, dout); }));
    }
    for (int ctas : {4}) {
      for (int n_tma : {256}) {
        char name[32];
        snprintf(name, sizeof name, "tma%d/c%d", n_tma, ctas);
        report(name, timeit([&] { k_tma<<<sms * ctas, kChunk>>>(map, di, dx, nnz, n_tma, dout); }));
        CK(cudaGetLastError());
      }
    }
    CK(cudaDeviceSynchronize());
    cudaFree(di);
    cudaFree(dx);
    cudaFree(dout);
  }
  folp_gen_free(lp);
  return 0;
}
