// wd_launch.cuh -- host-side instantiation and launch of the draw kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <type_traits>
#include <mutex>
#include <tuple>
#include <utility>

#include "wd_draw.cuh"
#include "wd_lean.cuh"
#include "wd_rows_lane.cuh"
#include "wd_small.cuh"
#include "wd_shared.cuh"

namespace wd {

// bit 0: K = 32 through the double-buffered stash kernel; bit 1: K = 64 too
#ifndef WD_STASH2
#define WD_STASH2 1
#endif
#ifndef WD_ROWS_V8
#define WD_ROWS_V8 1
#endif
constexpr int kThreads = 128;          // 4 warps per CTA
constexpr int kPrefixBlocksPerSM = 8;  // persistent grid of the prefix baseline

int device_sm_count();
void set_last_cuda_error(cudaError_t e);

inline int occupancy_blocks(const void* fn, size_t smem, int threads = kThreads) {
  static std::mutex mu;
  // keyed by (device, function): cudaFuncSetAttribute applies to the current
  // device only, and occupancy may differ between devices of one process
  static std::map<std::tuple<int, const void*, size_t>, int> cache;
  static std::map<std::pair<int, const void*>, size_t> smem_attr;  // largest opt-in set so far
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  // the opt-in dynamic shared memory limit is per function: only ever raise it
  // (a smaller request after a larger one must not lower it under a cached launch)
  auto fkey = std::make_pair(dev, fn);
  if (smem > 48 * 1024 && smem > smem_attr[fkey]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_attr[fkey] = smem;
  }
  auto key = std::make_tuple(dev, fn, smem * 1024 + (size_t)threads);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int nb = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem);
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    nb = 0;
  }
  cache[key] = nb;
  return nb;
}

// shared memory of one warp: running block sums S[b][lane] (sized for the
// cooperative reload tile when that aliases S) + remnant tile + cp.async ring
template <typename T>
inline size_t bfly_smem_per_warp(int W, int K, int mode, int pipe, bool vec, int kv) {
  int nb = K / W;
  int G = (kv == KV_COARSE && nb > 32) ? (nb + 31) / 32 : 1;  // coarse running sums (bfly_kernel)
  int nbc = nb > 0 ? (nb + G - 1) / G : 1;
  const int TS = vec ? W + 4 : W + 1;
  const bool coop = mode == MODE_LDA && vec && kv == KV_SMALL;
  size_t b = (size_t)bfly_s_elems(nbc, K % W, TS, coop) * sizeof(T);
  if (K % W || pipe >= 5) b += (size_t)32 * TS * sizeof(T);  // remnant tile (the ring sits after it)
  if (pipe >= 5) b += (size_t)(pipe == 6 ? 4 : 3) * ((W >= 4 ? W / 4 : 1) + 2) * 32 * 16;  // cp.async ring
  return b;
}
template <typename T>
inline size_t prefix_smem() {
  return (size_t)(kThreads / 32) * 32 * 33 * sizeof(T);
}
inline int64_t prefix_table_cols() { return (int64_t)device_sm_count() * kPrefixBlocksPerSM * kThreads; }

// Block-loop variant (see bfly_blocks) per mode; WD_PIPE_ROWS / WD_PIPE_LDA
// override the defaults for experiments.
inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && e[0]) ? atoi(e) : dflt;
}
inline int pipe_variant(int mode, int nb) {
  // measured (profiles/): standalone rows -> one block in flight with the
  // most warps (1) for <= 4 blocks per row, software pipelining (2) for 5-7,
  // the cp.async ring (5) from 8 (K = 384 / 480 / 4096: 5894 / 5864 / 5751
  // -> 6276 / 6374 / 6126 GB/s against pipelining); LDA -> one
  // block of register loads in flight (1): its gathers need the warps
  static int rows = env_int("WD_PIPE_ROWS", 0);
  static int lda = env_int("WD_PIPE_LDA", 1);
  if (mode == MODE_ROWS) return rows ? rows : (nb <= 4 ? 1 : (nb <= 7 ? 2 : 5));
  return lda >= 5 ? 1 : lda;  // the ring does not pay for the LDA gathers (occupancy)
}
// L2 policies (0 normal, 1 evict_last, 2 evict_first); WD_L2_X / WD_L2_T override
inline void l2_policies(int mode, int& px, int& pt) {
  static int lx = env_int("WD_L2_X", -1), lt = env_int("WD_L2_T", -1);
  px = lx >= 0 ? lx : (mode == MODE_LDA ? 0 : 0);
  pt = lt >= 0 ? lt : 0;
}

template <typename T, int W, int VEC, int MODE, int PIPE, int KV>
int launch_bfly_pc(const DrawParams<T>& p, cudaStream_t st) {
  const void* fn = (const void*)bfly_kernel<T, W, VEC, MODE, PIPE, KV>;
  const size_t per_warp = bfly_smem_per_warp<T>(W, p.K, MODE, PIPE, VEC, KV);
  int wpb = kThreads / 32;  // fewer warps per CTA when the block sums are large
  while (wpb > 1 && (size_t)wpb * per_warp > 227 * 1024) wpb >>= 1;
  const size_t smem = (size_t)wpb * per_warp;
  if (smem > 227 * 1024) return WD_ERR_UNSUPPORTED;
  const int threads = wpb * 32;
  int per_sm = occupancy_blocks(fn, smem, threads);
  if (per_sm <= 0) return WD_ERR_CUDA;
  int64_t chunks = (p.n_tokens + 31) / 32;
  int64_t want = (chunks + wpb - 1) / wpb;
  int64_t cap = (int64_t)per_sm * device_sm_count();
  int grid = (int)(want < cap ? want : cap);
  if (grid <= 0) return WD_OK;
  bfly_kernel<T, W, VEC, MODE, PIPE, KV><<<grid, threads, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}

// K variant: more than 32 blocks per row -> coarse running sums; LDA vector
// path with at most 16 blocks -> the cooperative pass-2 reload (measured:
// K = 200 draw -3.5%; at K = 1024 it cost +6%, so larger K keep the per-lane
// reload)
#ifndef WD_SMALL_MAX_BLOCKS
#define WD_SMALL_MAX_BLOCKS 16
#endif
constexpr int kSmallMaxBlocks = WD_SMALL_MAX_BLOCKS;
constexpr int kSmallMinBlocks = 4;
template <typename T, int W, int VEC, int MODE, int PIPE>
int launch_bfly_pipe(const DrawParams<T>& p, cudaStream_t st) {
  const int nb = p.K / W;
  if (nb > 32) return launch_bfly_pc<T, W, VEC, MODE, PIPE, KV_COARSE>(p, st);
  if constexpr (MODE == MODE_LDA && VEC && PIPE == 1) {
    // measured: it pays on (document, word)-ordered tiles (DeviceLDA, K = 200:
    // -3%) but not on a CSR-order draw (K = 16..240: +2..15%), nor below 4 blocks
    if (nb >= kSmallMinBlocks && nb <= kSmallMaxBlocks && p.token_pos != nullptr)
      return launch_bfly_pc<T, W, VEC, MODE, PIPE, KV_SMALL>(p, st);
  }
  return launch_bfly_pc<T, W, VEC, MODE, PIPE, KV_FINE>(p, st);
}

template <typename T, int W, int VEC, int MODE>
int launch_bfly_inst(const DrawParams<T>& p0, cudaStream_t st) {
  DrawParams<T> p = p0;
  l2_policies(MODE, p.l2_policy_x, p.l2_policy_t);
  // the multi-block variants are instantiated for the fp32 W=32 vector paths
  // (the cp.async ring and the experimental 3/4 for 128-bit segments only)
  if constexpr (std::is_same<T, float>::value && W == 32 && VEC == 2) {
    if (pipe_variant(MODE, p.K / W) == 2) return launch_bfly_pipe<T, W, VEC, MODE, 2>(p, st);
  }
  if constexpr (std::is_same<T, float>::value && W == 32 && VEC == 1) {
    const int v = pipe_variant(MODE, p.K / W);
    if (v == 2) return launch_bfly_pipe<T, W, VEC, MODE, 2>(p, st);
    if (v == 3) return launch_bfly_pipe<T, W, VEC, MODE, 3>(p, st);
    if (v == 4) return launch_bfly_pipe<T, W, VEC, MODE, 4>(p, st);
    if (v == 5) return launch_bfly_pipe<T, W, VEC, MODE, 5>(p, st);
    if (v == 6) return launch_bfly_pipe<T, W, VEC, MODE, 6>(p, st);
  }
  return launch_bfly_pipe<T, W, VEC, MODE, 1>(p, st);
}

template <typename T, bool VEC, int MODE>
int launch_prefix_inst(const DrawParams<T>& p, void* ws, size_t ws_bytes, cudaStream_t st) {
  const void* fn = (const void*)prefix_kernel<T, VEC, MODE>;
  size_t smem = prefix_smem<T>();
  int64_t cols = prefix_table_cols();
  size_t need = (size_t)cols * (size_t)p.K * sizeof(T);
  if (ws == nullptr || ws_bytes < need) return WD_ERR_WORKSPACE;
  if (occupancy_blocks(fn, smem) <= 0) return WD_ERR_CUDA;
  int grid = (int)(cols / kThreads);
  prefix_kernel<T, VEC, MODE><<<grid, kThreads, smem, st>>>(p, reinterpret_cast<T*>(ws), cols);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}

template <typename T, bool VEC, int MODE>
int launch_bfly_w(int W, const DrawParams<T>& p, cudaStream_t st) {
  switch (W) {
    case 2: return launch_bfly_inst<T, 2, VEC, MODE>(p, st);
    case 4: return launch_bfly_inst<T, 4, VEC, MODE>(p, st);
    case 8: return launch_bfly_inst<T, 8, VEC, MODE>(p, st);
    case 16: return launch_bfly_inst<T, 16, VEC, MODE>(p, st);
    case 32: return launch_bfly_inst<T, 32, VEC, MODE>(p, st);
    case 64: return launch_bfly_inst<T, 64, VEC, MODE>(p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}

// one shared weight vector (ld = 0): table once, then one search per draw
template <typename T, int W>
int launch_shared_inst(const DrawParams<T>& p, void* ws, cudaStream_t st) {
  T* tab = reinterpret_cast<T*>(ws);
  shared_build_kernel<T, W><<<1, 256, 0, st>>>(p.phi, p.K, tab);
  int64_t grid = (p.n_tokens + 255) / 256;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  grid = grid > cap ? cap : grid;
  shared_draw_kernel<T, W><<<(int)grid, 256, 0, st>>>(p, tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}

template <typename T>
int launch_shared(int W, const DrawParams<T>& p, void* ws, cudaStream_t st) {
  switch (W) {
    case 2: return launch_shared_inst<T, 2>(p, ws, st);
    case 4: return launch_shared_inst<T, 4>(p, ws, st);
    case 8: return launch_shared_inst<T, 8>(p, ws, st);
    case 16: return launch_shared_inst<T, 16>(p, ws, st);
    case 32: return launch_shared_inst<T, 32>(p, ws, st);
    case 64: return launch_shared_inst<T, 64>(p, ws, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}

template <typename T, int W, int NB, int NS = 1>
int launch_rows_stash(const DrawParams<T>& p0, cudaStream_t st) {
  DrawParams<T> p = p0;
  int px = 0, pt = 0;
  l2_policies(MODE_ROWS, px, pt);
  p.l2_policy_x = px;
  const void* fn = NS == 2 ? (const void*)rows_stash2_kernel<T, W, NB> : (const void*)rows_stash_kernel<T, W, NB>;
  const int wpb = kThreads / 32;
  const size_t smem = (size_t)NS * wpb * NB * 32 * (W + 4) * sizeof(T);
  const int per_sm = occupancy_blocks(fn, smem, kThreads);
  if (per_sm <= 0) return WD_ERR_CUDA;
  const int64_t chunks = (p.n_tokens + 31) / 32;
  const int64_t want = (chunks + wpb - 1) / wpb;
  const int64_t cap = (int64_t)per_sm * device_sm_count();
  const int grid = (int)(want < cap ? want : cap);
  if (grid <= 0) return WD_OK;
  if constexpr (NS == 2) rows_stash2_kernel<T, W, NB><<<grid, kThreads, smem, st>>>(p);
  else rows_stash_kernel<T, W, NB><<<grid, kThreads, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}

// The register-lean LDA draw (wd_lean.cuh): fp32, W = 32, 256-bit segments,
// K % 32 == 0 with at least WD_LEAN_MIN_NB blocks.  WD_LEAN=0 disables it
// (A/B against bfly_kernel).  Measured (tools/configs.py, draw ms, old ->
// lean): K = 2048 145.2 -> 118.9, configs[4] shard (K = 4096) 363.6 -> 304.4;
// at K = 1024 the general kernel is already at the L2 -> SM read ceiling
// (ncu: 17.96 TB/s xbar -> L1) and lean is 1-2% slower, so it starts at 64
// blocks.
inline bool lean_eligible(const DrawParams<float>& p) {
  static int on = env_int("WD_LEAN", 1);
  static int min_nb = env_int("WD_LEAN_MIN_NB", 64);
  return on && p.K % 32 == 0 && p.K / 32 >= min_nb;
}
inline int launch_lean(const DrawParams<float>& p0, cudaStream_t st) {
  DrawParams<float> p = p0;
  // theta streams from HBM once per vocabulary tile (evict_first) while the
  // tile's phi slice should stay in L2 (evict_last): cfg5 shard 318 -> 304 ms
  static int lx = env_int("WD_L2_X", 1), lt = env_int("WD_L2_T", 2);
  p.l2_policy_x = lx;
  p.l2_policy_t = lt;
  static int pf = env_int("WD_LEAN_PF", 0);
  // the warp-cooperative pass 2 moved fewer L1 wavefronts but measured
  // slower (cfg5 shard 318 vs 335 ms, K = 2048 123 vs 127): off by default
  static int coop = env_int("WD_LEAN_COOP", 0);
  p.theta_prefetch = pf;
  const void* fn = coop ? (const void*)lda_lean_kernel<WD_LEAN_MIN_BLOCKS, true>
                        : (const void*)lda_lean_kernel<WD_LEAN_MIN_BLOCKS, false>;
  const int wpb = kThreads / 32;
  const size_t smem = (size_t)wpb * kLeanWarpFloats * sizeof(float);
  const int per_sm = occupancy_blocks(fn, smem, kThreads);
  if (per_sm <= 0) return WD_ERR_CUDA;
  const int64_t chunks = (p.n_tokens + 31) / 32;
  const int64_t want = (chunks + wpb - 1) / wpb;
  const int64_t cap = (int64_t)per_sm * device_sm_count();
  const int grid = (int)(want < cap ? want : cap);
  if (grid <= 0) return WD_OK;
  if (coop) lda_lean_kernel<WD_LEAN_MIN_BLOCKS, true><<<grid, kThreads, smem, st>>>(p);
  else lda_lean_kernel<WD_LEAN_MIN_BLOCKS, false><<<grid, kThreads, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}

// Standalone rows with K = 8 * RM + 32 * NB, NB <= 4 (fp32, W = 32, 32-byte
// aligned rows): one row per thread (wd_rows_lane.cuh).  WD_ROWS_LANE=0
// disables it; WD_ROWS_LANE_MAX_NB caps the block count it takes.
template <int NB, int RM>
int launch_rows_lane_inst(const DrawParams<float>& p, cudaStream_t st) {
  const void* fn = (const void*)rows_lane_kernel<NB, RM>;
  const int per_sm = occupancy_blocks(fn, 0, kThreads);
  if (per_sm <= 0) return WD_ERR_CUDA;
  const int64_t want = (p.n_tokens + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)per_sm * device_sm_count();
  const int grid = (int)(want < cap ? want : cap);
  if (grid <= 0) return WD_OK;
  rows_lane_kernel<NB, RM><<<grid, kThreads, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}
template <int NB>
int launch_rows_lane_nb(int rm, const DrawParams<float>& p, cudaStream_t st) {
  switch (rm) {
    case 0: if constexpr (NB > 0) return launch_rows_lane_inst<NB, 0>(p, st); else return WD_ERR_UNSUPPORTED;
    case 1: return launch_rows_lane_inst<NB, 1>(p, st);
    case 2: return launch_rows_lane_inst<NB, 2>(p, st);
    case 3: return launch_rows_lane_inst<NB, 3>(p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}
// Measured against the warp-cooperative kernels (tools/sweep.py, 2^20 rows;
// 2^24-row steady state in brackets, fraction of HBM): K = 8 / 16 / 24
// 0.25 / 0.36 / 0.39 -> 0.40 / 0.52 / 0.60 (0.37 / 0.52 / 0.58 -> 0.90 /
// 1.02 / 1.02); K = 40-56 and 136-152 (a remnant next to 1 or 4 blocks)
// +5-11%; K = 32, 64-128 (whole blocks, 2-3 blocks) are as fast or faster
// on the cooperative kernels (K = 64: 0.72 vs 0.58), which keep them.
inline bool rows_lane_eligible(const DrawParams<float>& p) {
  static int on = env_int("WD_ROWS_LANE", 1);  // 2: every shape it supports (A/B)
  const int nb = p.K / 32, rm = (p.K % 32) / 8;
  if (!on || p.ld_phi == 0 || (p.K % 32) % 8 != 0 || nb > 4) return false;
  return on == 2 || nb == 0 || (rm > 0 && (nb == 1 || nb == 4));
}
inline int launch_rows_lane(const DrawParams<float>& p, cudaStream_t st) {
  const int nb = p.K / 32, rm = (p.K % 32) / 8;
  switch (nb) {
    case 0: return launch_rows_lane_nb<0>(rm, p, st);
    case 1: return launch_rows_lane_nb<1>(rm, p, st);
    case 2: return launch_rows_lane_nb<2>(rm, p, st);
    case 3: return launch_rows_lane_nb<3>(rm, p, st);
    case 4: return launch_rows_lane_nb<4>(rm, p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}

// The small-K LDA draw (wd_small.cuh): K = 8 * RM + 32 * NB, 2 <= NB <= 8,
// fp32, W = 32, 256-bit aligned rows.  WD_SMALL_LDA: 0 off, 1 (default) on
// vocabulary tiles (DeviceLDA's run-padded token order) and on CSR-order
// draws up to K = 256, 2 on every eligible draw.  CSR order, 1M documents,
// general kernel -> small (ms): K = 64 9.91 -> 5.75, 128 12.54 -> 8.55,
// 200 16.62 -> 12.82, 256 17.35 -> 13.61, 280 22.65 -> 22.61; at 20 tokens
// per document K = 280 loses (10.1 -> 11.9), hence the cap.
template <int NB, int RM>
int launch_small_inst(const DrawParams<float>& p, cudaStream_t st) {
  const void* fn = (const void*)lda_small_kernel<NB, RM>;
  const int wpb = kThreads / 32;
  const size_t smem = (size_t)wpb * NB * 4 * 40 * sizeof(float);
  const int per_sm = occupancy_blocks(fn, smem, kThreads);
  if (per_sm <= 0) return WD_ERR_CUDA;
  const int64_t chunks = (p.n_tokens + 31) / 32;
  const int64_t want = (chunks + wpb - 1) / wpb;
  const int64_t cap = (int64_t)per_sm * device_sm_count();
  const int grid = (int)(want < cap ? want : cap);
  if (grid <= 0) return WD_OK;
  lda_small_kernel<NB, RM><<<grid, kThreads, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_last_cuda_error(e); return WD_ERR_CUDA; }
  return WD_OK;
}
template <int NB>
int launch_small_nb(int rm, const DrawParams<float>& p, cudaStream_t st) {
  switch (rm) {
    case 0: return launch_small_inst<NB, 0>(p, st);
    case 1: return launch_small_inst<NB, 1>(p, st);
    case 2: return launch_small_inst<NB, 2>(p, st);
    case 3: return launch_small_inst<NB, 3>(p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}
inline bool small_lda_eligible(const DrawParams<float>& p) {
  static int on = env_int("WD_SMALL_LDA", 1);
  const int nb = p.K / 32;
  if (!on || (p.K % 32) % 8 != 0 || nb < 2 || nb > 8) return false;
  return on == 2 || p.token_pos != nullptr || p.K <= 256;
}
inline int launch_small_lda(const DrawParams<float>& p0, cudaStream_t st) {
  DrawParams<float> p = p0;
  l2_policies(MODE_LDA, p.l2_policy_x, p.l2_policy_t);
  const int rm = (p.K % 32) / 8;
  switch (p.K / 32) {
    case 2: return launch_small_nb<2>(rm, p, st);
    case 3: return launch_small_nb<3>(rm, p, st);
    case 4: return launch_small_nb<4>(rm, p, st);
    case 5: return launch_small_nb<5>(rm, p, st);
    case 6: return launch_small_nb<6>(rm, p, st);
    case 7: return launch_small_nb<7>(rm, p, st);
    case 8: return launch_small_nb<8>(rm, p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}

// Dispatch on (variant, W, VEC, MODE); explicit instantiations live in
// wd_draw_f32.cu / wd_draw_f64.cu so the two element types compile in parallel.
template <typename T>
int launch_draw(int variant, int W, int vec, int mode, const DrawParams<T>& p, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  if (variant == WD_BUTTERFLY) {
    // shared vector with a table workspace: build once, search per draw
    // (without one, every row runs the full per-row kernel: same results)
    if (mode == MODE_ROWS && p.ld_phi == 0 && ws != nullptr &&
        ws_bytes >= shared_table_elems(W, p.K) * sizeof(T))
      return launch_shared<T>(W, p, ws, st);
    if (mode == MODE_LDA) {
      if constexpr (std::is_same<T, float>::value) {
        // 256-bit lane segments (vec 2: 32-byte aligned fp32 blocks, W = 32)
        if (vec == 2 && W == 32 && lean_eligible(p)) return launch_lean(p, st);
        if (vec == 2 && W == 32 && small_lda_eligible(p)) return launch_small_lda(p, st);
        if (vec == 2 && W == 32) return launch_bfly_inst<T, 32, 2, MODE_LDA>(p, st);
      }
      return vec ? launch_bfly_w<T, true, MODE_LDA>(W, p, st) : launch_bfly_w<T, false, MODE_LDA>(W, p, st);
    }
    if constexpr (std::is_same<T, float>::value) {
      // K = W (fp32, W = 32): the single block staged in shared memory
      // (rows_stash_kernel; measured K = 32: 21.3 -> 27.4 G draws/s; staging
      // two blocks at K = 64 was slower than the per-row kernel, 15.9 vs 18.5)
      // K = 32: the double-buffered own-row variant (rows_stash2_kernel,
      // measured 26.5 -> 31.1 G draws/s; at K = 64, two blocks per stage,
      // 20.4 -> 19.5: not used)
      // one row per thread at small K (256-bit aligned rows)
      if (vec == 2 && W == 32 && rows_lane_eligible(p)) return launch_rows_lane(p, st);
      if (vec && W == 32 && p.K == 32) {
        if (WD_STASH2 & 1) return launch_rows_stash<T, 32, 1, 2>(p, st);
        return launch_rows_stash<T, 32, 1>(p, st);
      }
#if WD_STASH2 & 2
      if (vec && W == 32 && p.K == 64) return launch_rows_stash<T, 32, 2, 2>(p, st);
#endif
      // 256-bit segments while the block loop is register-resident (the
      // cp.async ring from 8 blocks keeps 128-bit segments)
      if (vec == 2 && W == 32 && p.K / 32 < 8 && WD_ROWS_V8) return launch_bfly_inst<T, 32, 2, MODE_ROWS>(p, st);
    }
    return vec ? launch_bfly_w<T, true, MODE_ROWS>(W, p, st) : launch_bfly_w<T, false, MODE_ROWS>(W, p, st);
  }
  if (variant == WD_PREFIX) {
    if (mode == MODE_LDA)
      return vec ? launch_prefix_inst<T, true, MODE_LDA>(p, ws, ws_bytes, st)
                 : launch_prefix_inst<T, false, MODE_LDA>(p, ws, ws_bytes, st);
    return vec ? launch_prefix_inst<T, true, MODE_ROWS>(p, ws, ws_bytes, st)
               : launch_prefix_inst<T, false, MODE_ROWS>(p, ws, ws_bytes, st);
  }
  return WD_ERR_INVALID_ARGUMENT;
}

}  // namespace wd
