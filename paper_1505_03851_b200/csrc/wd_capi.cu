// wd_capi.cu -- the extern "C" boundary (include/warpdraw_b200.h) and the
// small auxiliary kernels (corpus preparation, units KAT, topic counts).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "warpdraw_b200.h"
#include "wd_launch.cuh"

namespace wd {

template <typename T>
int launch_draw(int variant, int W, int vec, int mode, const DrawParams<T>& p, void* ws,
                size_t ws_bytes, cudaStream_t st);
int launch_draw_mixed(int variant, int W, const DrawParams<float>& p, cudaStream_t st);
extern template int launch_draw<float>(int, int, int, int, const DrawParams<float>&, void*, size_t,
                                       cudaStream_t);
extern template int launch_draw<double>(int, int, int, int, const DrawParams<double>&, void*, size_t,
                                        cudaStream_t);

static thread_local char g_last_err[256] = "";

void set_last_cuda_error(cudaError_t e) {
  snprintf(g_last_err, sizeof(g_last_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

int device_sm_count() {
  // queried once per device (cudaGetDevice is a cheap thread-local read)
  constexpr int kMaxDev = 64;
  static int cache[kMaxDev] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < kMaxDev && cache[dev] > 0) return cache[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  n = n > 0 ? n : 1;
  if (dev >= 0 && dev < kMaxDev) cache[dev] = n;
  return n;
}

// --------------------------------------------------------- aux kernels
// token -> local doc (one warp per document, grid-stride)
__global__ void token_doc_kernel(const int64_t* __restrict__ off, int64_t n_docs, int32_t* __restrict__ td) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t m = wid; m < n_docs; m += nw) {
    const int64_t a = off[m], b = off[m + 1];
    for (int64_t t = a + lane; t < b; t += 32) td[t] = (int32_t)m;
  }
}

// last_key[m] = G_q - 1, G_q = max length over the lanes-doc group of m
// (kernels.py:520-536: the final redraw of a short document's last word
// happens at master step G_q - 1 and its value wins).
__global__ void last_key_kernel(const int64_t* __restrict__ off, int64_t n_docs, int64_t doc_base, int W,
                                int32_t* __restrict__ lk) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n_docs;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gm = doc_base + m;
    const int64_t q0 = (gm / W) * W - doc_base;
    int64_t g = 0;
    for (int64_t d = q0; d < q0 + W; ++d) {
      if (d < 0 || d >= n_docs) continue;
      const int64_t len = off[d + 1] - off[d];
      g = len > g ? len : g;
    }
    lk[m] = (int32_t)(g - 1);
  }
}

__global__ void units_kernel(uint64_t seed, int n_keys, const int64_t* __restrict__ k0,
                             const int64_t* __restrict__ k1, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = seed;
    if (n_keys > 0) h = mix64(h ^ (uint64_t)k0[i]);
    if (n_keys > 1) h = mix64(h ^ (uint64_t)k1[i]);
    out[i] = __dmul_rn(__ull2double_rn(unit_bits(h)), 0x1p-53);
  }
}

__global__ void counts_kernel(const int32_t* __restrict__ words, const int32_t* __restrict__ td,
                              const int32_t* __restrict__ z, int64_t n, int32_t K, int32_t* __restrict__ dt,
                              int32_t* __restrict__ wt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = z[t];
    if (wt) atomicAdd(wt + (int64_t)words[t] * K + k, 1);
    if (dt) atomicAdd(dt + (int64_t)td[t] * K + k, 1);
  }
}

static int grid_1d(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)device_sm_count() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

static int check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

static bool valid_lanes(int W) { return W == 2 || W == 4 || W == 8 || W == 16 || W == 32 || W == 64; }

// 16-byte-vector eligibility of a row-major operand for block width Weff.
static bool vec_ok(const void* ptr, int64_t ld, int K, int Weff, size_t esz) {
  if (ptr == nullptr) return true;
  const int E = Weff >= 4 ? 4 : Weff;
  size_t vb = (size_t)E * esz;  // fp32: 16 B segments; fp64: 32 B (one 256-bit load)
  if (vb > 32) vb = 32;
  const int64_t ve = (int64_t)(vb / esz);
  return ((uintptr_t)ptr % vb) == 0 && (ld % ve) == 0 && ((K % Weff) % ve) == 0;
}

template <typename T>
static int draw_common(int variant, int lanes, int mode, DrawParams<T>& p, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  // rows are addressed as 32-bit row index x 32-bit byte stride (RowSet)
  if ((uint64_t)p.ld_phi * sizeof(T) >= (1ull << 32) || (uint64_t)p.ld_theta * sizeof(T) >= (1ull << 32) ||
      (mode == MODE_ROWS && (uint64_t)p.n_tokens >= (1ull << 32)))
    return WD_ERR_UNSUPPORTED;
  const int Weff = variant == WD_BUTTERFLY ? lanes : 32;
  int vec = vec_ok(p.phi, p.ld_phi, p.K, Weff, sizeof(T)) &&
            (mode == MODE_ROWS || vec_ok(p.theta, p.ld_theta, p.K, Weff, sizeof(T)));
  // LDA, fp32, W = 32: 256-bit lane segments when every block start of phi and
  // theta is 32-byte aligned (block_aligned_rows layouts)
  auto a32 = [&](const void* ptr, int64_t ld) {
    return ptr != nullptr && ((uintptr_t)ptr % 32) == 0 && (ld % 8) == 0 && ((p.K % Weff) % 8) == 0;
  };
  if (vec && variant == WD_BUTTERFLY && sizeof(T) == 4 && lanes == 32 && a32(p.phi, p.ld_phi) &&
      (mode == MODE_ROWS || a32(p.theta, p.ld_theta)))
    vec = 2;
  return launch_draw<T>(variant, lanes, vec, mode, p, ws, ws_bytes, st);
}

static int reset_err(uint64_t* err, cudaStream_t st) {
  if (err == nullptr) return WD_ERR_INVALID_ARGUMENT;
  // both words start at all-ones: one memset (one launch) per call
  if (cudaMemsetAsync(err, 0xFF, 2 * sizeof(uint64_t), st) != cudaSuccess) return check_launch();
  return WD_OK;
}

template <typename T>
static DrawParams<T> make_params() {
  DrawParams<T> p;
  memset(&p, 0, sizeof(p));
  return p;
}

}  // namespace wd

using namespace wd;

extern "C" {

int wd_abi_version(void) { return 1; }

const char* wd_status_string(int status) {
  switch (status) {
    case WD_OK: return "ok";
    case WD_ERR_INVALID_ARGUMENT: return "invalid argument";
    case WD_ERR_CUDA: return "CUDA error";
    case WD_ERR_UNSUPPORTED: return "unsupported configuration";
    case WD_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

const char* wd_last_cuda_error(void) { return g_last_err; }

int wd_corpus_prepare(const int64_t* doc_offsets, int64_t n_docs, int64_t n_tokens, int64_t doc_base, int lanes,
                      int32_t* token_doc, int32_t* last_key, void* stream) {
  if (!doc_offsets || n_docs < 0 || n_tokens < 0 || !valid_lanes(lanes) || doc_base < 0) return WD_ERR_INVALID_ARGUMENT;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_docs == 0) return WD_OK;
  if (token_doc && n_tokens > 0) token_doc_kernel<<<grid_1d(n_docs * 32, 256), 256, 0, st>>>(doc_offsets, n_docs, token_doc);
  if (last_key) last_key_kernel<<<grid_1d(n_docs, 256), 256, 0, st>>>(doc_offsets, n_docs, doc_base, lanes, last_key);
  return check_launch();
}

size_t wd_workspace_bytes(int variant, int dtype, int lanes, int32_t n_topics) {
  if (n_topics <= 0) return 0;
  size_t esz = dtype == WD_FLOAT64 ? 8 : 4;
  // butterfly: the shared-vector search table (wd_sample_rows with ld = 0)
  if (variant == WD_BUTTERFLY) return valid_lanes(lanes) ? shared_table_elems(lanes, n_topics) * esz : 0;
  if (variant != WD_PREFIX) return 0;
  return (size_t)prefix_table_cols() * (size_t)n_topics * esz;
}

int wd_draw_z(int variant, int dtype, int lanes, const void* theta, int64_t ld_theta, const void* phi,
              int64_t ld_phi, int32_t n_topics, const int64_t* doc_offsets, const int32_t* words,
              const int32_t* token_doc, const int32_t* token_pos, const int32_t* last_key, int64_t n_docs,
              int64_t n_tokens, int64_t doc_base, int stop_mode, int key_rule, uint64_t seed, const double* units,
              const void* stops, int32_t* z, int32_t* word_topic, int32_t* doc_topic, uint64_t* err,
              void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!valid_lanes(lanes) || (dtype != WD_FLOAT32 && dtype != WD_FLOAT64 && dtype != WD_FLOAT32_PHI64) ||
      n_topics <= 0 || n_tokens < 0 || n_docs < 0 || doc_base < 0 ||
      (variant != WD_BUTTERFLY && variant != WD_PREFIX))
    return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode < WD_STOPS_SEEDED || stop_mode > WD_STOPS_PHILOX) return WD_ERR_INVALID_ARGUMENT;
  if (key_rule != WD_KEYS_MASTER && key_rule != WD_KEYS_POSITION) return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode == WD_STOPS_UNITS && !units) return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode == WD_STOPS_EXPLICIT && !stops) return WD_ERR_INVALID_ARGUMENT;
  int rc = reset_err(err, st);
  if (rc != WD_OK) return rc;
  if (n_tokens == 0) return WD_OK;
  if (!theta || !phi || !doc_offsets || !words || !token_doc || !z) return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode == WD_STOPS_SEEDED && key_rule == WD_KEYS_MASTER && !last_key) return WD_ERR_INVALID_ARGUMENT;
  auto fill = [&](auto& p) {
    using TT = typename std::remove_pointer<decltype(p.phi)>::type;
    using T = typename std::remove_const<TT>::type;
    p.theta = (const T*)theta;
    p.ld_theta = ld_theta;
    p.phi = (const T*)phi;
    p.ld_phi = ld_phi;
    p.K = n_topics;
    p.offsets = doc_offsets;
    p.words = words;
    p.token_doc = token_doc;
    p.token_pos = token_pos;
    p.last_key = last_key;
    p.n_tokens = n_tokens;
    p.doc_base = doc_base;
    p.stop_mode = stop_mode;
    p.key_rule = key_rule;
    p.lanes = lanes;
    p.seed = seed;
    p.units = units;
    p.stops = (const T*)stops;
    p.z = z;
    p.word_topic = word_topic;
    p.doc_topic = doc_topic;
    p.err = (unsigned long long*)err;
  };
  if (dtype == WD_FLOAT32) {
    auto p = make_params<float>();
    fill(p);
    return draw_common<float>(variant, lanes, MODE_LDA, p, workspace, workspace_bytes, st);
  }
  if (dtype == WD_FLOAT32_PHI64) {  // p.phi carries the float64 rows (wd_mixed.cu)
    auto p = make_params<float>();
    fill(p);
    const int rc = launch_draw_mixed(variant, lanes, p, st);
    return rc;
  }
  auto p = make_params<double>();
  fill(p);
  return draw_common<double>(variant, lanes, MODE_LDA, p, workspace, workspace_bytes, st);
}

int wd_sample_rows(int variant, int dtype, int lanes, const void* weights, int64_t ld, int64_t n_rows,
                   int32_t n_topics, int64_t row_base, int stop_mode, uint64_t seed, const double* units,
                   const void* stops, int32_t* out, uint64_t* err, void* workspace, size_t workspace_bytes,
                   void* stream) {
  return wd_sample_rows_ex(variant, dtype, lanes, weights, ld, n_rows, n_topics, row_base, stop_mode, seed, units,
                           stops, out, err, workspace, workspace_bytes, 0, stream);
}

int wd_sample_rows_ex(int variant, int dtype, int lanes, const void* weights, int64_t ld, int64_t n_rows,
                      int32_t n_topics, int64_t row_base, int stop_mode, uint64_t seed, const double* units,
                      const void* stops, int32_t* out, uint64_t* err, void* workspace, size_t workspace_bytes,
                      int flags, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!valid_lanes(lanes) || (dtype != WD_FLOAT32 && dtype != WD_FLOAT64) || n_topics <= 0 || n_rows < 0 ||
      ld < 0 || (variant != WD_BUTTERFLY && variant != WD_PREFIX))
    return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode < WD_STOPS_SEEDED || stop_mode > WD_STOPS_PHILOX) return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode == WD_STOPS_UNITS && !units) return WD_ERR_INVALID_ARGUMENT;
  if (stop_mode == WD_STOPS_EXPLICIT && !stops) return WD_ERR_INVALID_ARGUMENT;
  if (!err) return WD_ERR_INVALID_ARGUMENT;
  int rc = (flags & WD_ERR_ACCUMULATE) ? WD_OK : reset_err(err, st);
  if (rc != WD_OK) return rc;
  if (n_rows == 0) return WD_OK;
  if (!weights || !out) return WD_ERR_INVALID_ARGUMENT;
  auto fill = [&](auto& p) {
    using TT = typename std::remove_pointer<decltype(p.phi)>::type;
    using T = typename std::remove_const<TT>::type;
    p.phi = (const T*)weights;
    p.ld_phi = ld;
    p.K = n_topics;
    p.n_tokens = n_rows;
    p.doc_base = row_base;
    p.stop_mode = stop_mode;
    p.key_rule = WD_KEYS_POSITION;
    p.lanes = lanes;
    p.seed = seed;
    p.units = units;
    p.stops = (const T*)stops;
    p.z = out;
    p.err = (unsigned long long*)err;
  };
  if (dtype == WD_FLOAT32) {
    auto p = make_params<float>();
    fill(p);
    return draw_common<float>(variant, lanes, MODE_ROWS, p, workspace, workspace_bytes, st);
  }
  auto p = make_params<double>();
  fill(p);
  return draw_common<double>(variant, lanes, MODE_ROWS, p, workspace, workspace_bytes, st);
}

int wd_units(uint64_t seed, int n_keys, const int64_t* k0, const int64_t* k1, int64_t n, double* out, void* stream) {
  if (n_keys < 0 || n_keys > 2 || n < 0 || (n > 0 && !out) || (n_keys > 0 && !k0) || (n_keys > 1 && !k1))
    return WD_ERR_INVALID_ARGUMENT;
  if (n == 0) return WD_OK;
  units_kernel<<<grid_1d(n, 256), 256, 0, (cudaStream_t)stream>>>(seed, n_keys, k0, k1, n, out);
  return check_launch();
}

int wd_topic_counts(const int32_t* words, const int32_t* token_doc, const int32_t* z, int64_t n_tokens,
                    int32_t n_topics, int32_t* doc_topic, int32_t* word_topic, void* stream) {
  if (n_tokens < 0 || n_topics <= 0 || !z || (word_topic && !words) || (doc_topic && !token_doc))
    return WD_ERR_INVALID_ARGUMENT;
  if (n_tokens == 0 || (!doc_topic && !word_topic)) return WD_OK;
  counts_kernel<<<grid_1d(n_tokens, 256), 256, 0, (cudaStream_t)stream>>>(words, token_doc, z, n_tokens, n_topics,
                                                                         doc_topic, word_topic);
  return check_launch();
}

}  // extern "C"
