// wd_resample.cu -- throughput-mode Dirichlet resample and log-likelihood on
// the device.
//
// Reference: lda.py:185-208 resample_params
//     theta[m]   ~ Dir(alpha + doc_topic[m])   (row-normalised Gammas)
//     phi[:, k]  ~ Dir(beta  + word_topic[:, k]) (column-normalised Gammas)
// and lda.py:289-305 log_likelihood.
//
// Statistical (not bitwise) parity: the reference draws its Gammas from
// numpy's PCG64 stream, which has no device equivalent.  Here every Gamma
// attempt is one Philox4x32-10 block: counter (global row lo, row hi, topic,
// attempt), key = the 64-bit iteration seed -- a bijection of the full
// 128-bit counter, so no two (row, topic, attempt) cells of one iteration
// share their words at any corpus size, and the result is independent of
// launch geometry and of the number of GPUs.  Marsaglia-Tsang
// (shape < 1 boosted by U^(1/a)) is evaluated in LOG space, so the tiny
// Gammas of alpha = 0.1 / beta = 0.01 shapes never underflow before
// normalisation.  Reductions use a fixed order, so a given (seed, counts)
// always gives the same bits.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "warpdraw_b200.h"
#include "wd_device.cuh"

namespace wd {

int device_sm_count();
void set_last_cuda_error(cudaError_t e);

// The Gamma stream: attempt `ctr` of Gamma (row, k) is the Philox4x32-10
// block of counter (row lo, row hi, k, ctr) under the iteration seed (128-bit
// counter, 64-bit key: distinct cells never share words).  The previous
// stream folded (row, topic) into one 32-bit hash, so at 1e9 cells per
// iteration ~21% of the cells shared their uniforms with another cell.
struct GammaRow {
  uint32_t r0, r1, k0, k1;
};
__device__ __forceinline__ GammaRow gamma_row(uint64_t seed, uint64_t row) {
  return {(uint32_t)row, (uint32_t)(row >> 32), (uint32_t)seed, (uint32_t)(seed >> 32)};
}
__device__ __forceinline__ uint4 rand4(const GammaRow& g, uint32_t k, uint32_t ctr) {
  return philox4x32_10(g.r0, g.r1, k, ctr, g.k0, g.k1);
}

// uniform in (0, 1) from all 32 bits: (x + 1/2) 2^-32, never 0 (rounded to
// float: the resolution near 0 is 2^-33, so log U reaches -22.9)
__device__ __forceinline__ float u01(uint32_t x) { return fmaf((float)x, 0x1p-32f, 0x1p-33f); }

// __logf (lg2.approx.ftz times ln2, the same two instructions and bits) as
// volatile asm, which the compiler may not hoist out of a branch
__device__ __forceinline__ float logf_unspeculated(float x) {
  float y;
  asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y * 0.693147182464599609375f;
}

// One Marsaglia-Tsang attempt (2000) for log Gamma(a, 1) from the counter
// block (row key, topic, attempt); shapes a < 1 use the boost Gamma(a) = Gamma(a + 1)
// * U^(1/a) (numpy's construction) with U taken from the same block -- its
// acceptance depends only on the other three words, so U stays independent.
// Evaluated in LOG space so alpha = 0.1 / beta = 0.01 shapes never underflow.
// SFU approximations (__logf, __cosf, rsqrtf, __fdividef; this file is
// compiled with FMA contraction and flush-to-zero): statistical, not bitwise.
__device__ __forceinline__ bool log_gamma_attempt(float a, const GammaRow& g, uint32_t k, uint32_t ctr, float& out) {
  const uint4 r = rand4(g, k, ctr);
  float boost = 0.f;
  if (a < 1.f) {
    boost = __fdividef(__logf(u01(r.w)), a);
    a += 1.f;
  }
  const float d = a - (1.f / 3.f);
  const float c = rsqrtf(9.f * d);
  const float m2l = -2.f * __logf(u01(r.x));  // Box-Muller normal from (x, y)
  const float x = m2l * rsqrtf(m2l) * __cosf(6.28318530718f * (u01(r.y) - 0.5f));
  float v = 1.f + c * x;
  if (v <= 0.f) return false;
  v = v * v * v;
  const float u = u01(r.z);
  const float x2 = x * x;
  // the squeeze accepts ~98% of attempts; the exact test's two logs run only
  // when it fails (volatile: ptxas would otherwise evaluate them for every
  // attempt -- the same values, so the same decisions, either way)
  bool ok = u < 1.f - 0.0331f * x2 * x2;
  if (!ok) ok = logf_unspeculated(u) < 0.5f * x2 + d * (1.f - v + logf_unspeculated(v));
  if (ok) out = __logf(d * v) + boost;
  return ok;
}

// Shapes below kSmallShape (the zero-count cells of theta: alpha = 0.1):
// the small-shape sampler of Liu, Martin & Syring (2017), exact, one
// Philox block per attempt, no normal variate.  Z = -a log X has density
// proportional to exp(-z - e^(-z/a)); the envelope is e^(-z) on z >= 0 (mass 1)
// and e^(lambda z - 1) on z < 0 (mass w), lambda = 1/a - 1, w = a / (e (1 - a)).
// In y = -z/a = log X:
//   with probability 1/(1+w): y = log(U (1+w)) / a  (y <= 0), accepted when log V < -e^y;
//   otherwise:                y = -log(U') / (1 - a) (y > 0), accepted when log V < 1 + y - e^y.
// Acceptance at a = 0.1: Gamma(1.1) / (1 + w) = 0.91.
constexpr float kSmallShape = 0.5f;
__device__ __forceinline__ bool log_gamma_small_attempt(float a, const GammaRow& g, uint32_t k, uint32_t ctr,
                                                        float& out) {
  const uint4 r = rand4(g, k, ctr);
  const float w = __fdividef(a, 2.718281828459045f * (1.f - a));
  const float one_w = 1.f + w;
  const float u = u01(r.x);
  float y;
  if (u * one_w <= 1.f) y = __fdividef(__logf(u * one_w), a);
  else y = __fdividef(-__logf(u01(r.y)), 1.f - a);
  const float ey = __expf(y);
  const float lv = __logf(u01(r.z));
  if (y <= 0.f ? lv < -ey : lv < 1.f + y - ey) {
    out = y;
    return true;
  }
  return false;
}
// one attempt for any shape (the per-cell entry point of wd_log_gamma_draws)
__device__ __forceinline__ bool log_gamma_any(float a, const GammaRow& g, uint32_t k, uint32_t ctr, float& out) {
  return a < kSmallShape ? log_gamma_small_attempt(a, g, k, ctr, out) : log_gamma_attempt(a, g, k, ctr, out);
}

// Warp-level queue of the cells of one document that need the general
// (Marsaglia-Tsang) sampler: shape >= kSmallShape, i.e. the topics the
// document's tokens hit (need_of(k), evaluated by lane k mod 32).  They are a minority (e.g. ~17% at K = 1024 with
// 200 tokens); gathering them 32 at a time keeps every lane busy on one.
template <typename Need, typename Shape, typename Store>
__device__ __forceinline__ void warp_general_cells(int K, int lane, int* q, const GammaRow& rkey, Need need_of,
                                                   Shape shape, Store store) {
  int qn = 0;
  const unsigned lt = (1u << lane) - 1u;
  auto drain = [&](int n) {  // lanes < n take q[lane]
    if (lane < n) {
      const int k = q[lane];
      const float a = shape(k);
      float v;
      uint32_t ctr = 0;
      while (!log_gamma_attempt(a, rkey, (uint32_t)k, ctr, v)) ++ctr;
      store(k, v);
    }
    __syncwarp();
  };
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    const bool need = k < K && need_of(k);  // evaluated by the lane that owns topic k
    const unsigned m = __ballot_sync(FULL, need);
    if (need) q[qn + __popc(m & lt)] = k;
    qn += __popc(m);
    __syncwarp();
    if (qn >= 32) {
      drain(32);
      if (lane < qn - 32) q[lane] = q[32 + lane];
      __syncwarp();
      qn -= 32;
    }
  }
  drain(qn);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// theta[m, :] ~ Dir(alpha + hist(z of doc m)); one warp per document; the
// doc-topic histogram never touches HBM (it lives in the warp's smem slice).
template <typename T>
__global__ void __launch_bounds__(256) theta_kernel(const int32_t* __restrict__ z, const int64_t* __restrict__ off,
                                                    int64_t n_docs, int32_t K, float alpha, uint64_t seed,
                                                    int64_t doc_base, T* __restrict__ theta, int64_t ld) {
  extern __shared__ float tsm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* lg = tsm + (size_t)wib * K;
  int* hist = reinterpret_cast<int*>(lg);
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t m = (int64_t)blockIdx.x * wpb + wib; m < n_docs; m += (int64_t)gridDim.x * wpb) {
    for (int k = lane; k < K; k += 32) hist[k] = 0;
    __syncwarp();
    const int64_t a = off[m], b = off[m + 1];
    for (int64_t t = a + lane; t < b; t += 32) atomicAdd(hist + z[t], 1);
    __syncwarp();
    const uint64_t row = (uint64_t)(doc_base + m);
    float mx = -INFINITY;
    const GammaRow rkey = gamma_row(seed, row);
    // per-lane progress: a rejection costs that lane one more attempt instead
    // of stalling the whole warp at every topic (divergence only at the
    // tail).  (The two-phase small-shape + queued general sampling of the
    // wide kernel measured slower here: K = 200 / 1024 / 2048 resample
    // 1.67 / 4.37 / 12.6 -> 2.26 / 5.88 / 14.0 ms.)
    uint32_t ctr = 0;
    for (int k = lane; k < K;) {
      float v;
      if (log_gamma_attempt(alpha + (float)hist[k], rkey, (uint32_t)k, ctr, v)) {
        lg[k] = v;
        mx = fmaxf(mx, v);
        k += 32;
        ctr = 0;
      } else {
        ++ctr;
      }
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int k = lane; k < K; k += 32) {
      const float e = __expf(lg[k] - mx);
      lg[k] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
    T* out = theta + m * ld;
    for (int k = lane; k < K; k += 32) out[k] = (T)(lg[k] * inv);
    __syncwarp();
  }
}

// Large K (float): the same draw as theta_kernel, but only the doc-topic
// counts live in shared memory (two 16-bit counters per word), and the
// log-Gammas go to the document's output row, normalised there in two more
// coalesced passes.  4 B/topic of shared memory per warp became 2 B/topic:
// at K = 4096 the plain kernel fit 8 warps per SM and was latency-bound.
// Used above K = 2048.  Sampling in two phases: the topics the document's
// tokens did not hit (shape alpha < 1/2) with the small-shape sampler,
// per-lane progress, then the hit topics gathered 32 at a time for
// Marsaglia-Tsang (warp_general_cells): configs[4] shard resample 45.2 ->
// 41.1 ms (at K <= 2048 the same scheme was slower; theta_kernel keeps the
// single loop).
__global__ void __launch_bounds__(256) theta_kernel_wide(const int32_t* __restrict__ z,
                                                         const int64_t* __restrict__ off, int64_t n_docs, int32_t K,
                                                         float alpha, uint64_t seed, int64_t doc_base,
                                                         float* __restrict__ theta, int64_t ld) {
  extern __shared__ uint32_t hsm[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int KW = (K + 1) >> 1;
  uint32_t* h2 = hsm + (size_t)wib * (KW + 64);
  int* q = reinterpret_cast<int*>(h2 + KW);  // the general-sampler queue (64)
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t m = (int64_t)blockIdx.x * wpb + wib; m < n_docs; m += (int64_t)gridDim.x * wpb) {
    float* out = theta + m * ld;
    const int64_t a = off[m], b = off[m + 1];
    // documents of 65536+ tokens could overflow a 16-bit counter: their
    // counts go to the output row (int32, global atomics) instead
    const bool big = b - a > 65535;
    int* gh = reinterpret_cast<int*>(out);
    if (big) {
      for (int k = lane; k < K; k += 32) gh[k] = 0;
      __syncwarp();
      for (int64_t t = a + lane; t < b; t += 32) atomicAdd(gh + z[t], 1);
      __threadfence_block();
    } else {
      for (int w = lane; w < KW; w += 32) h2[w] = 0u;
      __syncwarp();
      for (int64_t t = a + lane; t < b; t += 32) {
        const int k = z[t];
        atomicAdd(h2 + (k >> 1), 1u << ((k & 1) * 16));
      }
    }
    __syncwarp();
    const GammaRow rkey = gamma_row(seed, (uint64_t)(doc_base + m));
    float mx = -INFINITY;
    if (big) {  // counts in the output row itself: one pass, one sampler per cell
      uint32_t ctr = 0;
      for (int k = lane; k < K;) {
        const int cnt = __ldcg(gh + k);
        float v;
        if (log_gamma_any(alpha + (float)cnt, rkey, (uint32_t)k, ctr, v)) {
          out[k] = v;  // (the count at k is read above, then replaced)
          mx = fmaxf(mx, v);
          k += 32;
          ctr = 0;
        } else {
          ++ctr;
        }
      }
    } else {
      auto shape = [&](int k) { return alpha + (float)((h2[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu); };
      uint32_t ctr = 0;
      for (int k = lane; k < K;) {  // (1) small shapes, per-lane progress
        const float a = shape(k);
        if (!(a < kSmallShape)) {
          k += 32;
          continue;
        }
        float v;
        if (log_gamma_small_attempt(a, rkey, (uint32_t)k, ctr, v)) {
          out[k] = v;
          mx = fmaxf(mx, v);
          k += 32;
          ctr = 0;
        } else {
          ++ctr;
        }
      }
      __syncwarp();
      // (2) the rest, 32 at a time
      warp_general_cells(K, lane, q, rkey, [&](int k) { return !(shape(k) < kSmallShape); }, shape,
                         [&](int k, float v) { out[k] = v; mx = fmaxf(mx, v); });
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int k = lane; k < K; k += 32) {
      const float e = __expf(out[k] - mx);
      out[k] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
    for (int k = lane; k < K; k += 32) out[k] = out[k] * inv;
    __syncwarp();
  }
}

// wd_log_gamma_draws: the per-cell attempt loop of the resample kernels.
__global__ void log_gamma_cells(uint64_t seed, const int64_t* __restrict__ rows, const int32_t* __restrict__ topics,
                                const float* __restrict__ shapes, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const GammaRow g = gamma_row(seed, (uint64_t)rows[i]);
    float v;
    uint32_t ctr = 0;
    while (!log_gamma_any(shapes[i], g, (uint32_t)topics[i], ctr, v)) ++ctr;
    out[i] = v;
  }
}

// phi[:, k] ~ Dir(beta + word_topic[:, k]): three passes over V x K with
// per-CTA column partials reduced in a fixed order (deterministic).
constexpr int kPhiThreads = 256;

// The V rows are cut into n_chunks fixed row chunks (ceil(V / n_chunks)
// rows each); CTA i of a launch handles chunk chunk0 + i and writes that
// chunk's column partials.  The whole matrix is chunk0 = 0 with n_chunks
// CTAs; a rank of a sharded resample runs its own chunk range -- the same
// chunks, the same Gamma counters, the same partials, so the result is
// bit-identical for any number of ranks.
template <typename T>
__global__ void __launch_bounds__(kPhiThreads) phi_pass(int pass, const int32_t* __restrict__ wt, int64_t V,
                                                        int32_t K, float beta, uint64_t seed, T* __restrict__ phi,
                                                        int64_t ld, float* __restrict__ part,
                                                        const float* __restrict__ colstat, int chunk0, int n_chunks) {
  const int64_t g = (int64_t)chunk0 + blockIdx.x;
  const int64_t rows_per = (V + n_chunks - 1) / n_chunks;
  const int64_t v0 = g * rows_per < V ? g * rows_per : V;
  const int64_t v1 = v0 + rows_per < V ? v0 + rows_per : V;
  // gridDim.y column blocks split a chunk's columns (each column, and so its
  // partial, is still computed by exactly one thread: the same bits)
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < K; k += gridDim.y * blockDim.x) {
    float acc = pass == 0 ? -INFINITY : 0.f;
    const float cs = pass == 0 ? 0.f : colstat[k];
    if (pass == 0) {
      uint32_t ctr = 0;
      GammaRow rkey = gamma_row(seed, (uint64_t)v0);
      for (int64_t v = v0; v < v1;) {
        float lgv;
        if (log_gamma_attempt(beta + (float)wt[v * (int64_t)K + k], rkey, (uint32_t)k, ctr, lgv)) {
          phi[v * ld + k] = (T)lgv;
          acc = fmaxf(acc, lgv);
          ++v;
          ctr = 0;
          rkey = gamma_row(seed, (uint64_t)v);
        } else {
          ++ctr;
        }
      }
    }
    if (pass > 0) {
      // four rows' loads in flight before their arithmetic (the column sum
      // keeps its row order: the same bits as one row at a time)
      int64_t v = v0;
      for (; v + 4 <= v1; v += 4) {
        T* p = phi + v * ld + k;
        float x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = (float)p[i * ld];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (pass == 1) {
            const float e = __expf(x[i] - cs);
            p[i * ld] = (T)e;
            acc += e;
          } else {
            p[i * ld] = (T)(x[i] / cs);
          }
        }
      }
      for (; v < v1; ++v) {
        T* p = phi + v * ld + k;
        if (pass == 1) {
          const float e = __expf((float)*p - cs);
          *p = (T)e;
          acc += e;
        } else {
          *p = (T)((float)*p / cs);
        }
      }
    }
    if (pass < 2) part[g * K + k] = acc;
  }
}

__global__ void col_reduce(int pass, const float* __restrict__ part, int G, int32_t K, float* __restrict__ colstat) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float acc = pass == 0 ? -INFINITY : 0.f;
  for (int g = 0; g < G; ++g) {
    const float v = part[(int64_t)g * K + k];
    acc = pass == 0 ? fmaxf(acc, v) : acc + v;
  }
  colstat[k] = acc;
}

// log-likelihood: sum over tokens of log(theta_hat[m] . phi_hat[w]) where
// theta_hat = theta / rowsum, phi_hat = phi / colsum (lda.py:289-305).
// One warp per 32-token chunk; per token a K-dot over coalesced rows.
template <typename T>
__global__ void __launch_bounds__(256) ll_kernel(const T* __restrict__ theta, int64_t ldt, const T* __restrict__ phi,
                                                 int64_t ldp, const int32_t* __restrict__ words,
                                                 const int32_t* __restrict__ td, int64_t n, int32_t K,
                                                 const double* __restrict__ inv_rows,
                                                 const double* __restrict__ inv_cols, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t t = gw; t < n; t += nw) {
    const int32_t m = td[t], w = words[t];
    const T* th = theta + (int64_t)m * ldt;
    const T* ph = phi + (int64_t)w * ldp;
    double dot = 0.0;
    for (int k = lane; k < K; k += 32) dot += (double)th[k] * (double)ph[k] * inv_cols[k];
    dot = warp_sum_d(dot) * inv_rows[m];
    if (lane == 0) acc += log(dot);
  }
  if (lane == 0) atomicAdd(out, acc);
}

template <typename T>
__global__ void row_inv_sums(const T* __restrict__ theta, int64_t ld, int64_t n_docs, int32_t K, double* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t m = gw; m < n_docs; m += nw) {
    double s = 0.0;
    for (int k = lane; k < K; k += 32) s += (double)theta[m * ld + k];
    s = warp_sum_d(s);
    if (lane == 0) inv[m] = 1.0 / s;
  }
}

template <typename T>
__global__ void col_inv_sums(const T* __restrict__ phi, int64_t ld, int64_t V, int32_t K, double* __restrict__ inv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  double s = 0.0;
  for (int64_t v = 0; v < V; ++v) s += (double)phi[v * ld + k];
  inv[k] = 1.0 / s;
}

static int ck() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

static int phi_grid() { return device_sm_count() * 4; }

template <typename T>
static int resample_theta_t(const int32_t* z, const int64_t* off, int64_t n_docs, int32_t K, float alpha, uint64_t seed,
                            int64_t doc_base, T* theta, int64_t ld, cudaStream_t st) {
  const int threads = 256;
  if constexpr (std::is_same<T, float>::value) {
    // measured (1M docs): K = 4096 44.4 -> 31.1 ms; K = 2048 10.7 -> 12.2 (kept plain);
    // WD_THETA_WIDE_MIN_K overrides the threshold (A/B)
    static const int wide_min = [] {
      const char* e = getenv("WD_THETA_WIDE_MIN_K");
      return (e && e[0]) ? atoi(e) : 2049;
    }();
    if (K >= wide_min) {
      const size_t smem_w = (size_t)(threads / 32) * ((K + 1) / 2 + 64) * sizeof(uint32_t);
      if (smem_w > 48 * 1024)
        cudaFuncSetAttribute((const void*)theta_kernel_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_w);
      if (smem_w <= 227 * 1024) {
        int64_t want = (n_docs + 7) / 8;
        int64_t cap = (int64_t)device_sm_count() * 64;
        int grid = (int)(want < cap ? want : cap);
        if (grid < 1) return WD_OK;
        theta_kernel_wide<<<grid, threads, smem_w, st>>>(z, off, n_docs, K, alpha, seed, doc_base, theta, ld);
        return ck();
      }
    }
  }
  size_t smem = (size_t)(threads / 32) * K * sizeof(float);
  int wpb = threads / 32;
  int th = threads;
  while (smem > 200 * 1024 && wpb > 1) {
    wpb /= 2;
    th = wpb * 32;
    smem = (size_t)wpb * K * sizeof(float);
  }
  if (smem > 227 * 1024) return WD_ERR_UNSUPPORTED;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute((const void*)theta_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t want = (n_docs + wpb - 1) / wpb;
  int64_t cap = (int64_t)device_sm_count() * 64;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) return WD_OK;
  theta_kernel<T><<<grid, th, smem, st>>>(z, off, n_docs, K, alpha, seed, doc_base, theta, ld);
  return ck();
}

template <typename T>
static int resample_phi_t(const int32_t* wt, int64_t V, int32_t K, float beta, uint64_t seed, T* phi, int64_t ld,
                          void* ws, size_t ws_bytes, cudaStream_t st) {
  const int G = phi_grid();
  size_t need = ((size_t)G * K + 2 * (size_t)K) * sizeof(float);
  if (!ws || ws_bytes < need) return WD_ERR_WORKSPACE;
  float* part = (float*)ws;
  float* colstat = part + (size_t)G * K;
  int cb = (K + 255) / 256;
  phi_pass<T><<<G, kPhiThreads, 0, st>>>(0, wt, V, K, beta, seed, phi, ld, part, nullptr, 0, G);
  col_reduce<<<cb, 256, 0, st>>>(0, part, G, K, colstat);
  phi_pass<T><<<G, kPhiThreads, 0, st>>>(1, wt, V, K, beta, seed, phi, ld, part, colstat, 0, G);
  col_reduce<<<cb, 256, 0, st>>>(1, part, G, K, colstat + K);
  phi_pass<T><<<G, kPhiThreads, 0, st>>>(2, wt, V, K, beta, seed, phi, ld, part, colstat + K, 0, G);
  return ck();
}

template <typename T>
static int ll_t(const T* theta, int64_t ldt, const T* phi, int64_t ldp, const int32_t* words, const int32_t* td,
                int64_t n_docs, int64_t n_tokens, int64_t V, int32_t K, double* out, void* ws, size_t ws_bytes,
                cudaStream_t st) {
  size_t need = ((size_t)n_docs + (size_t)K) * sizeof(double);
  if (!ws || ws_bytes < need) return WD_ERR_WORKSPACE;
  double* inv_rows = (double*)ws;
  double* inv_cols = inv_rows + n_docs;
  cudaMemsetAsync(out, 0, sizeof(double), st);
  int g = device_sm_count() * 8;
  if (n_docs > 0) row_inv_sums<T><<<g, 256, 0, st>>>(theta, ldt, n_docs, K, inv_rows);
  col_inv_sums<T><<<(K + 127) / 128, 128, 0, st>>>(phi, ldp, V, K, inv_cols);
  if (n_tokens > 0) ll_kernel<T><<<g, 256, 0, st>>>(theta, ldt, phi, ldp, words, td, n_tokens, K, inv_rows, inv_cols, out);
  return ck();
}

}  // namespace wd

using namespace wd;

extern "C" {

int wd_resample_theta(int dtype, const int32_t* z, const int64_t* doc_offsets, int64_t n_docs, int32_t n_topics,
                      double alpha, uint64_t seed, int64_t doc_base, void* theta, int64_t ld_theta, void* stream) {
  if (n_docs < 0 || n_topics <= 0 || !doc_offsets || !theta || ld_theta < n_topics || alpha <= 0)
    return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == WD_FLOAT32)
    return resample_theta_t<float>(z, doc_offsets, n_docs, n_topics, (float)alpha, seed, doc_base, (float*)theta,
                                   ld_theta, st);
  if (dtype == WD_FLOAT64)
    return resample_theta_t<double>(z, doc_offsets, n_docs, n_topics, (float)alpha, seed, doc_base, (double*)theta,
                                    ld_theta, st);
  return WD_ERR_INVALID_ARGUMENT;
}

int wd_log_gamma_draws(uint64_t seed, const int64_t* rows, const int32_t* topics, const float* shapes, int64_t n,
                       float* out, void* stream) {
  if (n < 0 || (n > 0 && (!rows || !topics || !shapes || !out))) return WD_ERR_INVALID_ARGUMENT;
  if (n == 0) return WD_OK;
  int64_t want = (n + 255) / 256, cap = (int64_t)device_sm_count() * 16;
  log_gamma_cells<<<(int)(want < cap ? want : cap), 256, 0, (cudaStream_t)stream>>>(seed, rows, topics, shapes, n, out);
  return ck();
}

size_t wd_resample_phi_workspace_bytes(int32_t n_topics) {
  return ((size_t)phi_grid() * n_topics + 2 * (size_t)n_topics) * sizeof(float);
}

int wd_resample_phi(int dtype, const int32_t* word_topic, int64_t vocab_size, int32_t n_topics, double beta,
                    uint64_t seed, void* phi, int64_t ld_phi, void* workspace, size_t workspace_bytes, void* stream) {
  if (vocab_size <= 0 || n_topics <= 0 || !word_topic || !phi || ld_phi < n_topics || beta <= 0)
    return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == WD_FLOAT32)
    return resample_phi_t<float>(word_topic, vocab_size, n_topics, (float)beta, seed, (float*)phi, ld_phi, workspace,
                                 workspace_bytes, st);
  if (dtype == WD_FLOAT64)
    return resample_phi_t<double>(word_topic, vocab_size, n_topics, (float)beta, seed, (double*)phi, ld_phi,
                                  workspace, workspace_bytes, st);
  return WD_ERR_INVALID_ARGUMENT;
}

int wd_resample_phi_chunks(void) { return phi_grid(); }

int wd_resample_phi_pass(int dtype, int pass, const int32_t* word_topic, int64_t vocab_size, int32_t n_topics,
                         double beta, uint64_t seed, void* phi, int64_t ld_phi, int chunk0, int chunk1, int n_chunks,
                         float* partials, const float* colstat, void* stream) {
  if (pass < 0 || pass > 2 || vocab_size <= 0 || n_topics <= 0 || !word_topic || !phi || ld_phi < n_topics ||
      beta <= 0 || n_chunks <= 0 || chunk0 < 0 || chunk1 > n_chunks || chunk0 > chunk1 || !partials ||
      (pass > 0 && !colstat))
    return WD_ERR_INVALID_ARGUMENT;
  if (chunk1 == chunk0) return WD_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // pass 1 reads the column maxima (colstat[0, K)), pass 2 the sums (colstat[K, 2K))
  const float* cs = pass == 0 ? nullptr : (pass == 1 ? colstat : colstat + n_topics);
  // a rank's share of the chunks alone would leave SMs idle: its columns
  // are split over enough CTAs to cover the GPU
  int cols = (n_topics + wd::kPhiThreads - 1) / wd::kPhiThreads;
  const int want = wd::phi_grid();
  int ysplit = 1;
  while (ysplit < cols && (chunk1 - chunk0) * ysplit < want) ysplit *= 2;
  if (ysplit > cols) ysplit = cols;
  const dim3 grid(chunk1 - chunk0, ysplit);
  if (dtype == WD_FLOAT32)
    wd::phi_pass<float><<<grid, wd::kPhiThreads, 0, st>>>(pass, word_topic, vocab_size, n_topics, (float)beta, seed,
                                                          (float*)phi, ld_phi, partials, cs, chunk0, n_chunks);
  else if (dtype == WD_FLOAT64)
    wd::phi_pass<double><<<grid, wd::kPhiThreads, 0, st>>>(pass, word_topic, vocab_size, n_topics, (float)beta, seed,
                                                           (double*)phi, ld_phi, partials, cs, chunk0, n_chunks);
  else
    return WD_ERR_INVALID_ARGUMENT;
  return wd::ck();
}

int wd_resample_phi_reduce(int pass, const float* partials, int n_chunks, int32_t n_topics, float* colstat,
                           void* stream) {
  if ((pass != 0 && pass != 1) || !partials || !colstat || n_chunks <= 0 || n_topics <= 0)
    return WD_ERR_INVALID_ARGUMENT;
  wd::col_reduce<<<(n_topics + 255) / 256, 256, 0, (cudaStream_t)stream>>>(pass, partials, n_chunks, n_topics,
                                                                          colstat + (pass == 0 ? 0 : n_topics));
  return wd::ck();
}

int wd_log_likelihood(int dtype, const void* theta, int64_t ld_theta, const void* phi, int64_t ld_phi,
                      const int32_t* words, const int32_t* token_doc, int64_t n_docs, int64_t n_tokens,
                      int64_t vocab_size, int32_t n_topics, double* out, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (n_topics <= 0 || !theta || !phi || !out || n_docs < 0 || n_tokens < 0) return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == WD_FLOAT32)
    return ll_t<float>((const float*)theta, ld_theta, (const float*)phi, ld_phi, words, token_doc, n_docs, n_tokens,
                       vocab_size, n_topics, out, workspace, workspace_bytes, st);
  if (dtype == WD_FLOAT64)
    return ll_t<double>((const double*)theta, ld_theta, (const double*)phi, ld_phi, words, token_doc, n_docs,
                        n_tokens, vocab_size, n_topics, out, workspace, workspace_bytes, st);
  return WD_ERR_INVALID_ARGUMENT;
}

}  // extern "C"
