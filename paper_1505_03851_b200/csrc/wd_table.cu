// wd_table.cu -- the reference's split table / search API on the device.
//
// The draw kernels never materialise the butterfly table: they fuse build
// and search per token (wd_draw.cuh).  The reference also exports the two
// halves separately, and its sampler bench, CLI and tests call them that
// way:
//   build_block_tables(products, config) -> (warp, p, sums)   kernels.py:580-600
//     = build_butterfly_table over theta_local := products     kernels.py:170-225
//   butterfly_search(warp, p, sums, stop) -> index per lane   kernels.py:317-362
//     (+ _butterfly_block_walk, kernels.py:268-314)
// These kernels compute exactly those tables and indices, lane for lane: one
// thread per emulated lane, W threads per warp group (W = 2..64), the
// shuffle / shuffle_xor of the emulator as a shared-memory exchange inside
// the CTA (so W = 64 works across two hardware warps).
//
// Layouts (the reference's LocalArray layout, contiguous):
//   products [G][W][K], p [K][G][W], sums / stops / index [G][W].
#include <cuda_runtime.h>

#include <cstdint>

#include "warpdraw_b200.h"
#include "wd_device.cuh"

namespace wd {

int device_sm_count();
void set_last_cuda_error(cudaError_t e);

constexpr int kTableThreads = 128;

template <typename T>
struct Xchg {
  T* buf;  // kTableThreads values
  // value of lane `src` of this thread's group (every thread of the CTA calls it)
  __device__ __forceinline__ T from(T v, int group_base, int src) {
    buf[threadIdx.x] = v;
    __syncthreads();
    const T r = buf[group_base + src];
    __syncthreads();
    return r;
  }
};

// build_butterfly_table (kernels.py:170-225) with theta_local := products
// (fill_theta_local_transposed, kernels.py:561-577) and phi := 1.
template <typename T, int W>
__global__ void __launch_bounds__(kTableThreads) table_build_kernel(const T* __restrict__ prods, int K, int64_t G,
                                                                    T* __restrict__ p, T* __restrict__ sums) {
  __shared__ T sbuf[kTableThreads];
  Xchg<T> x{sbuf};
  constexpr int GPB = kTableThreads / W;  // groups per CTA
  const int lane = threadIdx.x % W;
  const int gib = threadIdx.x / W;
  const int base = gib * W;
  for (int64_t g0 = (int64_t)blockIdx.x * GPB; g0 < G; g0 += (int64_t)gridDim.x * GPB) {
    const int64_t g = g0 + gib;
    const bool live = g < G;  // tail groups run the exchanges on dummy data
    const T* pr = prods + (live ? g : 0) * W * K;
    auto P = [&](int k) -> T& { return p[((int64_t)k * G + g) * W + lane]; };
    T s = T(0);
    const int rem = K % W;
    int j = 0;
    for (; j < rem; ++j) {  // remnant: lane-own running sums (kernels.py:199-205)
      s = add_rn(s, mul_rn(pr[lane * K + j], T(1)));
      if (live) P(j) = s;
    }
    for (; j < K; j += W) {
      T a[W];
#pragma unroll
      for (int k = 0; k < W; ++k) a[k] = mul_rn(pr[k * K + j + lane], T(1));  // theta_local[j+k] * phi
#pragma unroll
      for (int bit = 1; bit < W; bit <<= 1) {
        const bool hi = (lane & bit) != 0;
#pragma unroll
        for (int t = 0; t < W / (2 * bit); ++t) {
          const int d = 2 * bit * t + (bit - 1);
          const T h = hi ? a[d] : a[d + bit];
          const T v = x.from(h, base, lane ^ bit);
          if (hi) a[d] = a[d + bit];
          a[d + bit] = add_rn(a[d], v);
          if (live) P(j + d) = a[d];
        }
      }
      s = add_rn(s, a[W - 1]);
      if (live) P(j + W - 1) = s;
    }
    if (live) sums[g * W + lane] = s;
  }
}

// butterfly_search (kernels.py:317-362) + _butterfly_block_walk (kernels.py:268-314)
template <typename T, int W>
__global__ void __launch_bounds__(kTableThreads) table_search_kernel(const T* __restrict__ p, const T* __restrict__ sums,
                                                                     const T* __restrict__ stops, int K, int64_t G,
                                                                     int64_t* __restrict__ out,
                                                                     unsigned long long* err) {
  __shared__ int64_t ibuf[kTableThreads];
  __shared__ T vbuf[kTableThreads];
  Xchg<int64_t> xi{ibuf};
  Xchg<T> xv{vbuf};
  constexpr int GPB = kTableThreads / W;
  constexpr int LOG2W = W == 2 ? 1 : W == 4 ? 2 : W == 8 ? 3 : W == 16 ? 4 : W == 32 ? 5 : 6;
  const int lane = threadIdx.x % W;
  const int gib = threadIdx.x / W;
  const int base = gib * W;
  for (int64_t g0 = (int64_t)blockIdx.x * GPB; g0 < G; g0 += (int64_t)gridDim.x * GPB) {
    const int64_t g = g0 + gib;
    const bool live_g = g < G;
    const int64_t gg = live_g ? g : 0;
    auto P = [&](int64_t k) -> T { return p[(k * G + gg) * W + lane]; };
    const T stop = stops[gg * W + lane];
    const T sm = sums[gg * W + lane];
    const bool live = sm > T(0);
    if (live_g && (stop < T(0) || (live && stop >= sm) || (!live && stop > T(0)))) atomicAnd(err + 1, 0ull);
    // block bisection over the blocks' final rows
    const int rem = K % W;
    const int nb = K / W;
    const int64_t search_base = rem + (W - 1);
    int64_t jj = 0, kk = nb - 1;
    while (jj < kk) {
      const int64_t mid = (jj + kk) >> 1;
      if (stop < P(mid * W + search_base)) kk = mid; else jj = mid + 1;
    }
    const int64_t block_base = rem + jj * W;
    int64_t result = 0;
    if (K >= W) {
      const bool has_prev = block_base > 0;
      T low = has_prev ? P(block_base - 1) : T(0);
      T high = P(block_base + (W - 1));
      int64_t flip = 0;
#pragma unroll
      for (int b = 0; b < LOG2W; ++b) {
        const int bit = 1 << (LOG2W - 1 - b);
        const int mask = ((W - 1) * (2 * bit)) & (W - 1);
        T y = T(0);
        for (int t = 0; t < W / (2 * bit); ++t) {
          const int d = (bit - 1) + 2 * bit * t;
          const int him = (d & mask) + (lane & ~mask);
          const int64_t his_base = xi.from(block_base, base, him);
          const T fetched = P(his_base + d);
          const T tval = xv.from(fetched, base, (int)(lane ^ flip));
          if (((lane ^ d) & mask) == 0) y = tval;
        }
        const bool hi_half = (lane & bit) != 0;
        const T compare = hi_half ? sub_rn(high, y) : add_rn(low, y);
        const bool less = stop < compare;
        if (less) high = compare; else low = compare;
        flip = less ? (flip ^ (bit & lane)) : (flip ^ (bit & ~lane));
      }
      result = block_base + (flip ^ lane);
    }
    // linear fallback over the remnant (kernels.py:354-361)
    if (block_base > 0 && live && stop < P(block_base - 1)) {
      for (int t = 0; t < rem; ++t)
        if (stop < P(t)) { result = t; break; }
    }
    if (live_g) out[g * W + lane] = result;
  }
}

template <typename T, int W>
static int launch_build(const void* prods, int K, int64_t G, void* p, void* sums, cudaStream_t st) {
  constexpr int GPB = kTableThreads / W;
  int64_t grid = (G + GPB - 1) / GPB;
  const int64_t cap = (int64_t)device_sm_count() * 16;
  if (grid > cap) grid = cap;
  table_build_kernel<T, W><<<(int)grid, kTableThreads, 0, st>>>((const T*)prods, K, G, (T*)p, (T*)sums);
  return WD_OK;
}
template <typename T, int W>
static int launch_search(const void* p, const void* sums, const void* stops, int K, int64_t G, int64_t* out,
                         uint64_t* err, cudaStream_t st) {
  constexpr int GPB = kTableThreads / W;
  int64_t grid = (G + GPB - 1) / GPB;
  const int64_t cap = (int64_t)device_sm_count() * 16;
  if (grid > cap) grid = cap;
  table_search_kernel<T, W><<<(int)grid, kTableThreads, 0, st>>>((const T*)p, (const T*)sums, (const T*)stops, K, G,
                                                                   out, (unsigned long long*)err);
  return WD_OK;
}

template <typename T>
static int build_w(int W, const void* prods, int K, int64_t G, void* p, void* sums, cudaStream_t st) {
  switch (W) {
    case 2: return launch_build<T, 2>(prods, K, G, p, sums, st);
    case 4: return launch_build<T, 4>(prods, K, G, p, sums, st);
    case 8: return launch_build<T, 8>(prods, K, G, p, sums, st);
    case 16: return launch_build<T, 16>(prods, K, G, p, sums, st);
    case 32: return launch_build<T, 32>(prods, K, G, p, sums, st);
    case 64: return launch_build<T, 64>(prods, K, G, p, sums, st);
    default: return WD_ERR_INVALID_ARGUMENT;
  }
}
template <typename T>
static int search_w(int W, const void* p, const void* sums, const void* stops, int K, int64_t G, int64_t* out,
                    uint64_t* err, cudaStream_t st) {
  switch (W) {
    case 2: return launch_search<T, 2>(p, sums, stops, K, G, out, err, st);
    case 4: return launch_search<T, 4>(p, sums, stops, K, G, out, err, st);
    case 8: return launch_search<T, 8>(p, sums, stops, K, G, out, err, st);
    case 16: return launch_search<T, 16>(p, sums, stops, K, G, out, err, st);
    case 32: return launch_search<T, 32>(p, sums, stops, K, G, out, err, st);
    case 64: return launch_search<T, 64>(p, sums, stops, K, G, out, err, st);
    default: return WD_ERR_INVALID_ARGUMENT;
  }
}

static int finish() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

}  // namespace wd

extern "C" {

int wd_build_block_tables(int dtype, int lanes, const void* products, int32_t n_topics, int64_t n_groups, void* p,
                          void* sums, void* stream) {
  if ((dtype != WD_FLOAT32 && dtype != WD_FLOAT64) || n_topics <= 0 || n_groups < 0) return WD_ERR_INVALID_ARGUMENT;
  if (n_groups == 0) return WD_OK;
  if (!products || !p || !sums) return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = dtype == WD_FLOAT32 ? wd::build_w<float>(lanes, products, n_topics, n_groups, p, sums, st)
                                     : wd::build_w<double>(lanes, products, n_topics, n_groups, p, sums, st);
  return rc != WD_OK ? rc : wd::finish();
}

int wd_butterfly_search(int dtype, int lanes, const void* p, const void* sums, const void* stops, int32_t n_topics,
                        int64_t n_groups, int64_t* out, uint64_t* err, void* stream) {
  if ((dtype != WD_FLOAT32 && dtype != WD_FLOAT64) || n_topics <= 0 || n_groups < 0 || !err)
    return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(err, 0xFF, 2 * sizeof(uint64_t), st) != cudaSuccess) return wd::finish();
  if (n_groups == 0) return WD_OK;
  if (!p || !sums || !stops || !out) return WD_ERR_INVALID_ARGUMENT;
  const int rc = dtype == WD_FLOAT32 ? wd::search_w<float>(lanes, p, sums, stops, n_topics, n_groups, out, err, st)
                                     : wd::search_w<double>(lanes, p, sums, stops, n_topics, n_groups, out, err, st);
  return rc != WD_OK ? rc : wd::finish();
}

}  // extern "C"
