// wd_stream.cu -- the reference's sequential-stream samplers on the device:
// SAMPLERS["binary"] and SAMPLERS["alias"] (bench.py:118-126; SURVEY.md
// section 8(f) rank 4, the paper's related-work comparator).
//
// The reference takes draw i from positions i (binary) or 2i, 2i+1 (alias)
// of ONE xoshiro256** stream (rng.py:47-77).  xoshiro's state transition is
// linear over GF(2), so the state after s steps is T^s * state0 for a 256x256
// bit matrix T.  One small kernel builds J[k] = T^(R * 2^k) (R = the draws one
// thread takes times the outputs per draw) by square-and-multiply in shared
// memory; each draw thread then jumps to its first position with popcount(t)
// matrix-vector products and walks its contiguous range sequentially, so the
// n results are exactly the reference's n sequential draws.
#include <cuda_runtime.h>

#include <cstdint>

#include "warpdraw_b200.h"
#include "wd_device.cuh"

namespace wd {

int device_sm_count();
void set_last_cuda_error(cudaError_t e);

namespace {

constexpr int kMaxJumps = 32;                          // thread index < 2^32
constexpr size_t kMatBytes = 256 * 4 * sizeof(uint64_t);  // one GF(2) 256x256 matrix, column-major
constexpr int kSub = 32;                               // draws per lane between coalesced stores

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Xo {
  uint64_t s0, s1, s2, s3;
  // rng.py:63-74
  __device__ __forceinline__ uint64_t next() {
    const uint64_t r = rotl64(s1 * 5ull, 7) * 9ull;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return r;
  }
};

// out = M * x over GF(2); M column-major, column i = M * e_i (4 words).
template <bool SHARED>
__device__ __forceinline__ void matvec(const uint64_t* __restrict__ M, const uint64_t x[4], uint64_t out[4]) {
  uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = x[w];
    while (bits) {
      const int b = __ffsll((long long)bits) - 1;
      bits &= bits - 1;
      const uint64_t* c = M + (size_t)(w * 64 + b) * 4;
      if (SHARED) {
        o0 ^= c[0]; o1 ^= c[1]; o2 ^= c[2]; o3 ^= c[3];
      } else {
        const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(c));
        const ulonglong2 d = __ldg(reinterpret_cast<const ulonglong2*>(c + 2));
        o0 ^= a.x; o1 ^= a.y; o2 ^= d.x; o3 ^= d.y;
      }
    }
  }
  out[0] = o0; out[1] = o1; out[2] = o2; out[3] = o3;
}

// J[k] = T^(R * 2^k), k < n_jumps.  One block of 256 threads; thread j owns
// column j of every matrix.  Powers of T commute, so A*B = B*A throughout.
__global__ void __launch_bounds__(256) jump_build_kernel(uint64_t R, int n_jumps, uint64_t* __restrict__ J) {
  __shared__ uint64_t A[256 * 4], P[256 * 4];
  const int j = threadIdx.x;
  Xo e{0, 0, 0, 0};
  uint64_t col[4] = {0, 0, 0, 0};
  col[j >> 6] = 1ull << (j & 63);
  e.s0 = col[0]; e.s1 = col[1]; e.s2 = col[2]; e.s3 = col[3];
  e.next();  // T e_j
  A[j * 4 + 0] = e.s0; A[j * 4 + 1] = e.s1; A[j * 4 + 2] = e.s2; A[j * 4 + 3] = e.s3;
  P[j * 4 + 0] = col[0]; P[j * 4 + 1] = col[1]; P[j * 4 + 2] = col[2]; P[j * 4 + 3] = col[3];  // identity
  __syncthreads();
  uint64_t v[4], x[4];
  while (R) {
    if (R & 1) {  // P = A * P
      for (int w = 0; w < 4; ++w) x[w] = P[j * 4 + w];
      matvec<true>(A, x, v);
      __syncthreads();
      for (int w = 0; w < 4; ++w) P[j * 4 + w] = v[w];
      __syncthreads();
    }
    R >>= 1;
    if (R) {  // A = A * A
      for (int w = 0; w < 4; ++w) x[w] = A[j * 4 + w];
      matvec<true>(A, x, v);
      __syncthreads();
      for (int w = 0; w < 4; ++w) A[j * 4 + w] = v[w];
      __syncthreads();
    }
  }
  for (int k = 0; k < n_jumps; ++k) {
    for (int w = 0; w < 4; ++w) J[(size_t)k * 1024 + j * 4 + w] = x[w] = P[j * 4 + w];
    if (k + 1 == n_jumps) break;
    matvec<true>(P, x, v);  // P = P * P
    __syncthreads();
    for (int w = 0; w < 4; ++w) P[j * 4 + w] = v[w];
    __syncthreads();
  }
}

// Thread t takes draws [t*D, min(n, (t+1)*D)), D a multiple of kSub.  Each
// lane stages kSub results in shared memory; the warp then stores every
// lane's run as one 128-byte row.
template <int METHOD>
__global__ void __launch_bounds__(256) stream_draw_kernel(const double* __restrict__ table,
                                                         const uint64_t* __restrict__ thresh,
                                                         const int32_t* __restrict__ alias, int64_t K,
                                                         uint64_t seed, int64_t n, int64_t D,
                                                         const uint64_t* __restrict__ J, int32_t* __restrict__ out) {
  __shared__ int32_t stage[8][32][kSub + 1];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t first = (int64_t)t * D;
  // SplitMix64 seeding (rng.py:54-61), then the jump to position t*D*U
  uint64_t s[4];
  for (int i = 0; i < 4; ++i) s[i] = fin64(seed + (uint64_t)(i + 1) * GAMMA);
  if (first < n) {
    uint64_t bits = t;
    for (int k = 0; bits; ++k, bits >>= 1) {
      if (bits & 1) {
        uint64_t o[4];
        matvec<false>(J + (size_t)k * 1024, s, o);
        s[0] = o[0]; s[1] = o[1]; s[2] = o[2]; s[3] = o[3];
      }
    }
  }
  Xo g{s[0], s[1], s[2], s[3]};
  double total = 0.0;
  if (METHOD == WD_STREAM_BINARY) total = __ldg(table + K - 1);
  const double dK = (double)K;
  const int64_t warp_first = first - (int64_t)lane * D;
  for (int64_t sub = 0; sub < D; sub += kSub) {
#pragma unroll 4
    for (int i = 0; i < kSub; ++i) {
      const int64_t d = first + sub + i;
      if (d >= n) break;
      int32_t r;
      if (METHOD == WD_STREAM_BINARY) {
        // sampling.py:86-92: stop = total * u; binary_search (sampling.py:65-76)
        const double u = __dmul_rn(__ull2double_rn(g.next() >> 11), 0x1p-53);
        const double stop = __dmul_rn(total, u);
        int64_t lo = 0, hi = K - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (stop < __ldg(table + mid)) hi = mid;
          else lo = mid + 1;
        }
        r = (int32_t)lo;
      } else {
        // sampling.py:134-138: k = int(u1 * n); k if u2 < F[k] else A[k]
        const double u1 = __dmul_rn(__ull2double_rn(g.next() >> 11), 0x1p-53);
        int64_t k = __double2ll_rz(__dmul_rn(u1, dK));
        k = k < K ? k : K - 1;  // u1 * K rounds below K for every 53-bit u1 < 1
        const uint64_t b2 = g.next() >> 11;
        r = b2 < __ldg(thresh + k) ? (int32_t)k : __ldg(alias + k);
      }
      stage[wib][lane][i] = r;
    }
    __syncwarp();
#pragma unroll 4
    for (int row = 0; row < 32; ++row) {
      const int64_t d = warp_first + (int64_t)row * D + sub + lane;
      if (d < n && d < warp_first + (int64_t)(row + 1) * D) out[d] = stage[wib][row][lane];
    }
    __syncwarp();
  }
}

}  // namespace

// wd_prefix_f64: sequential float64 running sums (sampling.py:46-52:
// np.cumsum in float64 is a left-to-right loop), one thread.
__global__ void prefix_f64_kernel(const double* __restrict__ w, int64_t K, double* __restrict__ p) {
  double s = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    s = __dadd_rn(s, w[k]);
    p[k] = s;
  }
}

static int check_launch_stream() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

}  // namespace wd

extern "C" {

int wd_prefix_f64(const double* weights, int64_t n_weights, double* table, void* stream) {
  if (n_weights <= 0 || !weights || !table) return WD_ERR_INVALID_ARGUMENT;
  wd::prefix_f64_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(weights, n_weights, table);
  return wd::check_launch_stream();
}

size_t wd_stream_workspace_bytes(int64_t n_draws) {
  (void)n_draws;
  return (size_t)wd::kMaxJumps * wd::kMatBytes;
}

int wd_stream_draws(int method, const double* table, const uint64_t* thresh, const int32_t* alias,
                    int64_t n_weights, uint64_t seed, int64_t n_draws, int32_t* out, void* workspace,
                    size_t workspace_bytes, void* stream) {
  if (n_draws < 0 || n_weights <= 0 || n_weights > INT32_MAX) return WD_ERR_INVALID_ARGUMENT;
  if (method == WD_STREAM_BINARY ? !table : (method == WD_STREAM_ALIAS ? (!thresh || !alias) : true))
    return WD_ERR_INVALID_ARGUMENT;
  if (n_draws == 0) return WD_OK;
  if (!out) return WD_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < wd_stream_workspace_bytes(n_draws)) return WD_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  // threads: enough to fill the GPU, but at least ~256 draws each so the
  // jump (popcount(t) 256-bit matrix-vector products) stays a small share
  const int64_t cap = (int64_t)wd::device_sm_count() * 1024;
  int64_t threads = (n_draws + 255) / 256;
  threads = threads < 1 ? 1 : (threads > cap ? cap : threads);
  int64_t D = (n_draws + threads - 1) / threads;
  D = (D + wd::kSub - 1) / wd::kSub * wd::kSub;
  threads = (n_draws + D - 1) / D;
  int n_jumps = 1;
  while (n_jumps < wd::kMaxJumps && (1ll << n_jumps) < threads) ++n_jumps;
  const uint64_t U = method == WD_STREAM_ALIAS ? 2 : 1;
  uint64_t* J = static_cast<uint64_t*>(workspace);
  wd::jump_build_kernel<<<1, 256, 0, st>>>((uint64_t)D * U, n_jumps, J);
  const int blocks = (int)((threads + 255) / 256);
  if (method == WD_STREAM_BINARY)
    wd::stream_draw_kernel<WD_STREAM_BINARY><<<blocks, 256, 0, st>>>(table, thresh, alias, n_weights, seed, n_draws,
                                                                      D, J, out);
  else
    wd::stream_draw_kernel<WD_STREAM_ALIAS><<<blocks, 256, 0, st>>>(table, thresh, alias, n_weights, seed, n_draws,
                                                                     D, J, out);
  return wd::check_launch_stream();
}

}  // extern "C"
