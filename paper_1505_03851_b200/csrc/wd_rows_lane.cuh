// wd_rows_lane.cuh -- standalone rows at small K: one row per thread.
//
// For K <= rem + 4 * W (W = 32, fp32) the draw of a row is mostly fixed
// per-row work -- the 64-bit u hash, the stop, the block bisection and the
// walk -- next to only 64-640 bytes of weights.  The warp-cooperative kernels
// (transposed 256-bit loads + shuffle transpose-reduce, shared running sums,
// cooperative or staged pass-2 reloads) spend ~430-500 warp instructions per
// 32-row chunk on that (ncu) and issue-bind at K <= 64.
// Here every thread owns one row outright:
//
//   * its weights arrive with 256-bit loads (rows 32-byte aligned, rem % 8 ==
//     0); the warp's 32 rows are contiguous, so every fetched sector is used;
//   * remnant (kernels.py:199-205): sequential running sums in registers
//     (re-read and re-summed for the rare fallback scan);
//   * each W-topic block: the pairwise Tree<32> of the row in registers --
//     the same sums the reference's shuffle_xor sets produce
//     (kernels.py:206-224), so the same bits as the transposed kernels --
//     and the running block sums S_b in registers (NB <= 4);
//   * stop = fl(total * fl(u)) (kernels.py:95-101), the first block whose
//     running sum exceeds it (== the reference's bisection, S nondecreasing),
//     the selected block re-read (an L1 hit: the row was just read) and the
//     add-or-subtract walk (Walk<float, 16>, kernels.py:268-314), or the
//     linear remnant fallback (kernels.py:354-361);
//   * no shuffles, no shared memory, no warp-uniform control flow.
#pragma once

#include "wd_draw.cuh"

namespace wd {

#ifndef WD_ROWS_LANE_MIN_BLOCKS
#define WD_ROWS_LANE_MIN_BLOCKS 8
#endif

__device__ __forceinline__ void ld8(float (&a)[8], const float* p) {
  asm("ld.global.nc.L1::evict_last.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7])
      : "l"(p));
}

// the 32 weights of one block (4 x 256-bit)
__device__ __forceinline__ void ld_block32(float (&c)[32], const float* p) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float a[8];
    ld8(a, p + g * 8);
#pragma unroll
    for (int e = 0; e < 8; ++e) c[g * 8 + e] = a[e];
  }
}

// NB: blocks per row (K = rem + NB * 32), RM: remnant segments of 8 (rem = 8 * RM)
// The weights of one row held in registers: RM remnant segments of 8 and NB
// blocks of 32 (loaded together, so all of a row's bytes are in flight at once).
template <int NB, int RM> struct LaneRow {
  float rem[RM > 0 ? RM * 8 : 1];
  float blk[NB > 0 ? NB : 1][32];
  __device__ __forceinline__ void load(const float* x) {
#pragma unroll
    for (int g = 0; g < RM; ++g) {
      float a[8];
      ld8(a, x + g * 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) rem[g * 8 + e] = a[e];
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) ld_block32(blk[b], x + RM * 8 + b * 32);
  }
};

// One row's draw from its weights (x: the row in global memory, re-read for
// the selected block / the remnant fallback -- L1 hits).
template <int NB, int RM>
__device__ __forceinline__ void lane_row_draw(const DrawParams<float>& p, int64_t row, const float* x,
                                              const LaneRow<NB, RM>& w) {
  constexpr int W = 32;
  constexpr int REM = 8 * RM;
  // remnant: sequential running sums
  float acc = 0.f;
#pragma unroll
  for (int t = 0; t < REM; ++t) acc = add_rn(acc, w.rem[t]);
  const float prem = acc;
  float S[NB > 0 ? NB : 1];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    acc = add_rn(acc, Tree<float, 32>::sum(w.blk[b]));
    S[b] = acc;
  }
  const float total = acc;
  uint64_t ka, kb;
  unsigned long long ekey;
  int r;
  int64_t zidx;
  token_keys<float, MODE_ROWS>(p, row, 0, W, ka, kb, ekey, r, zidx);
  const float stop = make_stop<float>(p, zidx, total, ka, kb, true);
  const bool live = total > 0.f;
  if (!live) atomicMin(p.err, ekey);
  // first block whose running sum exceeds stop (nb - 1 if none)
  int j = 0;
#pragma unroll
  for (int b = 0; b + 1 < NB; ++b) j += (S[b] <= stop) ? 1 : 0;
  float prev = prem, high = 0.f;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b == j) high = S[b];
    if (b + 1 == j) prev = S[b];
  }
  const int bb = REM + j * W;
  if (bb == 0) prev = 0.f;
  const bool fallback = bb > 0 && stop < prev && live;
  int result = 0;
  if (NB > 0 && !fallback) {
    float c[32];
    if constexpr (NB == 1) {
#pragma unroll
      for (int e = 0; e < 32; ++e) c[e] = w.blk[0][e];
    } else {
      ld_block32(c, x + bb);  // re-read: L1 hit
    }
    float low = prev;
    int lo = 0;
    Walk<float, W / 2>::run(c, low, high, stop, r, lo);
    result = bb + lo;
  }
  if (fallback) {
    // first remnant index whose running sum exceeds stop (same additions)
    float a2 = 0.f;
    int t = 0;
#pragma unroll
    for (int u = 0; u < REM; ++u) {
      a2 = add_rn(a2, w.rem[u]);
      t += (a2 <= stop) ? 1 : 0;
    }
    if (t < REM) result = t;
  }
  p.z[zidx] = result;
}

// RPT rows per thread in flight (their loads issued together) when a row is
// small enough; register-heavy shapes run 6 CTAs per SM instead of 8.
template <int NB, int RM> struct LaneShape {
  static constexpr int FLOATS = NB * 32 + RM * 8;
#ifndef WD_ROWS_LANE_RPT32  // rows per thread for 17-32 floats (A/B)
#define WD_ROWS_LANE_RPT32 1
#endif
#ifndef WD_ROWS_LANE_RPT8
#define WD_ROWS_LANE_RPT8 4
#endif
#ifndef WD_ROWS_LANE_RPT16
#define WD_ROWS_LANE_RPT16 2
#endif
  static constexpr int RPT = FLOATS <= 8 ? WD_ROWS_LANE_RPT8
                                         : (FLOATS <= 16 ? WD_ROWS_LANE_RPT16 : (FLOATS <= 32 ? WD_ROWS_LANE_RPT32 : 1));
  static constexpr int MINB = FLOATS * RPT > 40 ? 6 : WD_ROWS_LANE_MIN_BLOCKS;
};

template <int NB, int RM>
__global__ void __launch_bounds__(128, (LaneShape<NB, RM>::MINB)) rows_lane_kernel(DrawParams<float> p) {
  constexpr int RPT = LaneShape<NB, RM>::RPT;
  const int64_t n = p.n_tokens;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t row0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row0 < n; row0 += stride * RPT) {
    LaneRow<NB, RM> w[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t row = row0 + i * stride;
      if (row < n) w[i].load(p.phi + row * p.ld_phi);
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t row = row0 + i * stride;
      if (row < n) lane_row_draw<NB, RM>(p, row, p.phi + row * p.ld_phi, w[i]);
    }
  }
}

}  // namespace wd
