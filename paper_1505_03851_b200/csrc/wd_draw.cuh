// wd_draw.cuh -- the draw kernels (butterfly and prefix-table) for sm_100a.
//
// Reference behaviour (paths under /root/reference/pkg/src/warpdraw/):
//   kernels.py:170-225  build_butterfly_table   -> bfly_kernel pass 1
//   kernels.py:268-362  butterfly_search / walk -> bfly_kernel pass 2
//   kernels.py:95-101   _stops_from_units       -> make_stop
//   kernels.py:487-539  draw_z_butterfly        -> bfly_kernel<..., LDA>
//   kernels.py:580-600  build_block_tables      -> bfly_kernel<..., ROWS>
//   kernels.py:380-484  draw_z_basic/transposed -> prefix_kernel
//
// Layout and mapping (DESIGN.md sections 3-4):
//   * one warp owns a CHUNK of 32 consecutive tokens (a vocabulary tile's
//     (document, word) order, or CSR order) or rows; in LDA mode each lane
//     group loads consecutive chunk rows, so its theta segments are shared;
//   * the block loop walks W-topic blocks; per block every lane issues L
//     vector loads, each covering E consecutive topics of one row, so a warp
//     instruction reads R full contiguous row segments of W*sizeof(T) bytes
//     (128 B for fp32, W=32): coalesced and 128-bit vectorised;
//   * the first log2(E) levels of each block's pairwise tree are summed in
//     registers, the remaining log2(L) levels by a transpose-reduce over
//     __shfl_xor_sync (L-1 exchanges per lane per block) -- the paper's
//     butterfly exchange, widened by the vector loads; it leaves every lane
//     holding the block total of ONE row (its "own" token);
//   * only the running block sums S_b are kept (shared memory, [b][lane]);
//     the full K-entry table the reference stores (kernels.py:198-224) is
//     never written: after the block bisection the selected block is
//     re-read (per lane, or warp-cooperatively through a shared tile in the
//     small-K variant) and its tree rebuilt in registers for the walk,
//     which performs the same IEEE operations as the reference's
//     cross-lane fetch walk;
//   * variants by K (KV): fine (<= 32 blocks per row), coarse (every G-th
//     running sum), small (cooperative reload); rows_stash_kernel stages a
//     single-block row (K = W) in shared memory during the load.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "wd_device.cuh"

namespace wd {

enum { MODE_LDA = 0, MODE_ROWS = 1 };

// Minimum resident CTAs per SM requested for the LDA draw (caps registers so
// that enough warps are resident to cover L2 gather latency).
#ifndef WD_LDA_MIN_BLOCKS
#define WD_LDA_MIN_BLOCKS 6
#endif
#ifndef WD_LDA_MIN_BLOCKS_F64  // float64 LDA draw (unbounded: 237 registers, 8 warps/SM)
#define WD_LDA_MIN_BLOCKS_F64 4  // measured (cfg4 fp64 draw): unbounded 419 ms, 3 -> 156, 4 -> 153, 5 -> 155, 6 -> 236
#endif
#ifndef WD_MIN_BLOCKS_OTHER  // vector path, W != 32 or float64 rows
#define WD_MIN_BLOCKS_OTHER 4
#endif
#ifndef WD_BLOCK_UNROLL  // unroll of the one-block-in-flight loop (address math amortised)
#define WD_BLOCK_UNROLL 2  // measured: 1 -> 2 cfg4 draw -3.7%, cfg3 -3.9%; 4 is slower
#endif
constexpr int kBlockUnroll = WD_BLOCK_UNROLL;
#ifndef WD_PHI_L1NA  // LDA phi rows with L1::no_allocate (each read once per
#define WD_PHI_L1NA 0  // chunk): uniform cfg3 -1.8%, cfg4 -1.1%, but Zipf cfg4 +30% (repeated words lose their L1 hits)
#endif
#ifndef WD_LDA_MIN_BLOCKS_SMALL  // small-K variant with 256-bit segments
#define WD_LDA_MIN_BLOCKS_SMALL 7  // measured cfg3: 6 -> 16.3 ms, 7 -> 15.6, 8 -> 19.6 (spills)
#endif
#ifndef WD_LDA_MIN_BLOCKS_COARSE  // K > 32 * W: the group recompute needs more registers
                                   // (measured at K = 4096: 4 -> 463 ms, 5 -> 415, 6 -> 468 per cfg5 draw)
#define WD_LDA_MIN_BLOCKS_COARSE 5
#endif

template <typename T> struct DrawParams {
  const T* theta;  // LDA: doc rows (ld_theta); ROWS: unused
  int64_t ld_theta;
  const T* phi;  // LDA: word rows; ROWS: weight rows (ld_phi, 0 = shared)
  int64_t ld_phi;
  int32_t K;
  const int64_t* offsets;   // LDA CSR offsets [n_docs + 1]
  const int32_t* words;     // LDA [n_tokens]
  const int32_t* token_doc; // LDA [n_tokens]
  const int32_t* last_key;  // LDA master rule [n_docs]
  const int32_t* token_pos; // LDA, optional: the token list is a permutation (vocabulary
                            // tiles); token j is word token_pos[j] of doc token_doc[j] and its
                            // original CSR index offsets[doc] + pos indexes z / units / stops
  int64_t n_tokens;         // LDA tokens / ROWS rows
  int64_t doc_base;         // LDA global doc id of local doc 0 / ROWS row_base
  int stop_mode;
  int key_rule;
  int lanes;  // reference W (prefix kernel: r and master groups only)
  uint64_t seed;
  const double* units;
  const T* stops;
  int32_t* z;
  int32_t* word_topic;
  int32_t* doc_topic;
  unsigned long long* err;  // [0] AllZero key (min), [1] stop range flag (0 = bad)
  int l2_policy_x;          // L2 policy of the phi / weights loads (see make_l2_policy)
  int l2_policy_t;          // L2 policy of the theta loads
  uint32_t opaque_zero;     // always 0; the compiler cannot prove it (see BlockRegs::join)
  int theta_prefetch;       // lean LDA draw: L2 prefetch distance (blocks) of the theta segments, 0 = off
};

// Identity of the token/row a lane owns: global doc id (or row id), its hash
// keys, and the error ordering key.
template <typename T, int MODE>
__device__ __forceinline__ void token_keys(const DrawParams<T>& p, int64_t tok, int32_t doc, int W,
                                           uint64_t& ka, uint64_t& kb, unsigned long long& ekey,
                                           int& r, int64_t& zidx) {
  if (MODE == MODE_ROWS) {
    int64_t id = p.doc_base + tok;
    ka = (uint64_t)id;
    kb = 0;
    ekey = (unsigned long long)id;
    r = (int)(((id % W) + W) % W);
    zidx = tok;
  } else {
    int64_t gm = p.doc_base + doc;
    int64_t o0 = p.offsets[doc];
    int64_t i = p.token_pos ? (int64_t)p.token_pos[tok] : tok - o0;
    zidx = o0 + i;
    int64_t key = i;
    if (p.key_rule == WD_KEYS_MASTER) {
      int64_t n = p.offsets[doc + 1] - o0;
      if (i == n - 1 && p.stop_mode == WD_STOPS_SEEDED) key = p.last_key[doc];
      ekey = ((unsigned long long)(gm / W) << 40) | ((unsigned long long)i << 8) |
             (unsigned long long)(gm % W);
    } else {
      ekey = ((unsigned long long)gm << 32) | (unsigned long long)i;
    }
    ka = (uint64_t)gm;
    kb = (uint64_t)key;
    r = (int)(gm % W);
  }
}

// kernels.py:95-101 (stop = fl(total * fl(u)), kept strictly below total)
// plus the StopOutOfRangeError check of kernels.py:329-331 for explicit stops.
template <typename T>
__device__ __forceinline__ T make_stop(const DrawParams<T>& p, int64_t tok, T total, uint64_t ka,
                                       uint64_t kb, bool rows) {
  T stop;
  if (p.stop_mode == WD_STOPS_EXPLICIT) {
    stop = p.stops[tok];
    bool live = total > T(0);
    if (stop < T(0) || (live && stop >= total) || (!live && stop > T(0))) atomicAnd(p.err + 1, 0ull);
    return stop;
  }
  T uf;
  if (p.stop_mode == WD_STOPS_UNITS) {
    uf = from_double<T>(p.units[tok]);
  } else if (p.stop_mode == WD_STOPS_PHILOX) {
    uf = unit_to<T>(philox_bits(p.seed, ka, kb));
  } else {
    uf = unit_to<T>(rows ? unit_bits1(p.seed, ka) : unit_bits2(p.seed, ka, kb));
  }
  stop = mul_rn(total, uf);
  if (!(total > T(0))) return T(0);
  if (stop >= total) stop = next_below(total);
  return stop;
}

// make_stop in two halves, so the 64-bit u hash can run before pass 1 (its
// keys do not depend on the products) and overlap the block loads:
// stop_pre = fl_T(u) (or the explicit stop), stop_finish(pre, total) = the
// same value make_stop returns.
template <typename T>
__device__ __forceinline__ T stop_pre(const DrawParams<T>& p, int64_t tok, uint64_t ka, uint64_t kb, bool rows) {
  if (p.stop_mode == WD_STOPS_EXPLICIT) return p.stops[tok];
  if (p.stop_mode == WD_STOPS_UNITS) return from_double<T>(p.units[tok]);
  if (p.stop_mode == WD_STOPS_PHILOX) return unit_to<T>(philox_bits(p.seed, ka, kb));
  return unit_to<T>(rows ? unit_bits1(p.seed, ka) : unit_bits2(p.seed, ka, kb));
}
template <typename T>
__device__ __forceinline__ T stop_finish(const DrawParams<T>& p, T pre, T total) {
  if (p.stop_mode == WD_STOPS_EXPLICIT) {
    const T stop = pre;
    bool live = total > T(0);
    if (stop < T(0) || (live && stop >= total) || (!live && stop > T(0))) atomicAnd(p.err + 1, 0ull);
    return stop;
  }
  T stop = mul_rn(total, pre);
  if (!(total > T(0))) return T(0);
  if (stop >= total) stop = next_below(total);
  return stop;
}

// ============================================================== butterfly
// cp.async (LDGSTS): 16-byte global -> shared copies that hold no registers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// 128-bit shared-memory moves of one E-element segment (16-byte aligned)
__device__ __forceinline__ void store_seg(float* p, const float (&a)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(a[0], a[1], a[2], a[3]);
}
__device__ __forceinline__ void store_seg(double* p, const double (&a)[4]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(a[0], a[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(a[2], a[3]);
}
__device__ __forceinline__ void store_seg(float* p, const float (&a)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(a[0], a[1], a[2], a[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(a[4], a[5], a[6], a[7]);
}
template <typename T, int E>
__device__ __forceinline__ void store_seg(T* p, const T (&a)[E]) {
#pragma unroll
  for (int e = 0; e < E; ++e) p[e] = a[e];
}
__device__ __forceinline__ void load_seg_smem(float (&a)[4], const float* p) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
}
__device__ __forceinline__ void load_seg_smem(double (&a)[4], const double* p) {
  const double2 v0 = reinterpret_cast<const double2*>(p)[0], v1 = reinterpret_cast<const double2*>(p)[1];
  a[0] = v0.x; a[1] = v0.y; a[2] = v1.x; a[3] = v1.y;
}
__device__ __forceinline__ void load_seg_smem(float (&a)[8], const float* p) {
  const float4 v0 = reinterpret_cast<const float4*>(p)[0], v1 = reinterpret_cast<const float4*>(p)[1];
  a[0] = v0.x; a[1] = v0.y; a[2] = v0.z; a[3] = v0.w;
  a[4] = v1.x; a[5] = v1.y; a[6] = v1.z; a[7] = v1.w;
}
template <typename T, int E>
__device__ __forceinline__ void load_seg_smem(T (&a)[E], const T* p) {
#pragma unroll
  for (int e = 0; e < E; ++e) a[e] = p[e];
}

// the first n (< E) elements of a segment, scalar loads (tail of the remnant)
template <typename T, int E>
__device__ __forceinline__ void load_first(T (&v)[E], const T* __restrict__ p, int n) {
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = e < n ? __ldg(p + e) : T(0);
}

// 256-bit read-only global load (sm_100: LDG.E.256), 32-byte aligned address
__device__ __forceinline__ void ld_v8(float (&a)[8], const float* p) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7])
      : "l"(p));
}
template <typename T>
__device__ __forceinline__ void ld_v8(T (&)[8], const T*) {}  // (float only; never instantiated for T != float)

// Levels log2(E)+1 .. log2(W) of the block trees: transpose-reduce of the L
// per-lane partial sums q over lanes s ^ 1, s ^ 2, ... (the paper's butterfly
// exchange).  Afterwards the lane holds the block total of row s*R + lane/L.
template <typename T, int L>
__device__ __forceinline__ T xreduce(T (&q)[L], int s) {
#pragma unroll
  for (int bit = 1, n = L; bit < L; bit <<= 1, n >>= 1) {
    const bool hi = (s & bit) != 0;
#pragma unroll
    for (int t = 0; t < n / 2; ++t) {
      const T x0 = q[2 * t], x1 = q[2 * t + 1];
      const T send = hi ? x0 : x1;
      const T keep = hi ? x1 : x0;
      q[t] = add_rn(keep, __shfl_xor_sync(FULL, send, bit));
    }
  }
  return q[0];
}

__device__ __forceinline__ uint32_t lo_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t lo_bits(double v) { return (uint32_t)__double_as_longlong(v); }
__device__ __forceinline__ void or_bits(float& v, uint32_t d) { v = __uint_as_float(__float_as_uint(v) | d); }
__device__ __forceinline__ void or_bits(double& v, uint32_t d) {
  v = __longlong_as_double(__double_as_longlong(v) | (long long)d);
}

// N row addresses kept as 32-bit row indices over one 64-bit column base
// (row stride in bytes < 2^32): 1 register per row instead of 2, and one
// IMAD.WIDE per load.
template <typename T, int N> struct RowSet {
  uint32_t idx[N];
  const char* base;  // column base of row 0 (bytes)
  uint32_t ldb;      // row stride in bytes
  __device__ __forceinline__ const T* ptr(int i, int64_t off) const {
    return reinterpret_cast<const T*>(base + (uint64_t)idx[i] * ldb) + off;
  }
};

// One W-topic block of the 32-row chunk held in registers: L vector segments
// of phi (or weights) per lane, plus theta segments: ND = 1 when every row of
// the chunk belongs to one document, ND = 2 when to two (rows pick theirs by
// the bit mask dsel), ND = 0 one theta segment per row.
template <typename T, int W, int VEC, int MODE, int ND> struct BlockRegs {
  static constexpr int E = GeoV<W, VEC>::E, L = GeoV<W, VEC>::L;
  static constexpr int NT = MODE == MODE_LDA ? (ND == 0 ? L : ND) : 1;
  static constexpr int LT = L < 2 ? 2 : L;  // theta pointer slots (>= 2 for ND == 2)
  Seg<T, E, (VEC != 0)> x[L];
  Seg<T, E, (VEC != 0)> th[NT];
  // every load is unconditional (invalid rows point at a valid row) so all
  // of them are in flight before the first use
  __device__ __forceinline__ void load(const RowSet<T, L>& P, const RowSet<T, LT>& Q, int64_t off,
                                       uint64_t pol_x, uint64_t pol_t) {
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      if (MODE == MODE_LDA && WD_PHI_L1NA) x[kk].load_na(P.ptr(kk, off), pol_x);
      else x[kk].load(P.ptr(kk, off), pol_x);
    }
    if (MODE == MODE_LDA) {
#pragma unroll
      for (int i = 0; i < NT; ++i) th[i].load(Q.ptr(i, off), pol_t);
    }
  }
  // Make every consumer depend on EVERY load of the block (through an
  // opaque runtime zero), so ptxas cannot interleave consumers between the
  // loads to save registers: all of the block's loads stay in flight together.
  __device__ __forceinline__ void join(uint32_t opaque_zero) {
    uint32_t d = 0;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) d ^= lo_bits(x[kk].v[0]);
    if (MODE == MODE_LDA) {
#pragma unroll
      for (int i = 0; i < NT; ++i) d ^= lo_bits(th[i].v[0]);
    }
    d &= opaque_zero;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) or_bits(x[kk].v[0], d);
    if (MODE == MODE_LDA) {
#pragma unroll
      for (int i = 0; i < NT; ++i) or_bits(th[i].v[0], d);
    }
  }
  // block total of this lane's own row: first log2(E) tree levels in
  // registers, remaining log2(L) by the shuffle transpose-reduce
  __device__ __forceinline__ T reduce(const bool (&rvalid)[L], int s, uint32_t dsel) const {
    T q[L];
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      T a[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        T t = T(0);
        if (MODE == MODE_LDA) {
          if (ND == 1) t = th[0].v[e];
          else if (ND == 2) t = ((dsel >> kk) & 1u) ? th[NT - 1].v[e] : th[0].v[e];
          else t = th[kk].v[e];
        }
        a[e] = MODE == MODE_LDA ? mul_rn(t, x[kk].v[e]) : x[kk].v[e];
      }
      // rows of invalid tokens (padding, chunk tail) are summed too: they
      // load valid rows, and a row's partials only ever reach its own
      // (invalid, discarded) owner lane in the transpose-reduce
      q[kk] = Tree<T, E>::sum(a);
    }
    return xreduce<T, L>(q, s);
  }
};

// Rows from more than two documents (LDA, ND = 0): theta is loaded per row,
// in two half batches so at most L/2 (phi, theta) pairs are live at once.
template <typename T, int W, int VEC>
__device__ __forceinline__ T block_total_nd0(const RowSet<T, GeoV<W, VEC>::L>& P,
                                             const RowSet<T, (GeoV<W, VEC>::L < 2 ? 2 : GeoV<W, VEC>::L)>& Q,
                                             int64_t off, const bool (&rvalid)[GeoV<W, VEC>::L], int s, uint64_t px,
                                             uint64_t pt) {
  constexpr int E = GeoV<W, VEC>::E, L = GeoV<W, VEC>::L;
  constexpr int H = L >= 4 ? L / 2 : L;
  T q[L];
#pragma unroll
  for (int h = 0; h < L; h += H) {
    Seg<T, E, (VEC != 0)> x[H], th[H];
#pragma unroll
    for (int j = 0; j < H; ++j) {
      x[j].load(P.ptr(h + j, off), px);
      th[j].load(Q.ptr(h + j, off), pt);
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      T a[E];
#pragma unroll
      for (int e = 0; e < E; ++e) a[e] = mul_rn(th[j].v[e], x[j].v[e]);
      q[h + j] = Tree<T, E>::sum(a);  // invalid rows: see BlockRegs::reduce
    }
  }
  return xreduce<T, L>(q, s);
}

// Running sums are kept for every G-th block only (G = ceil(nb / 32)), so a
// warp's S array stays <= 32 entries per lane for any K; the exact S_b of
// the selected group are recomputed after the search (same IEEE operations).
template <typename T>
__device__ __forceinline__ void store_s(T* __restrict__ S, int b, int nb, int G, int lane, T v) {
  if (G == 1) S[b * 32 + lane] = v;
  else if ((b + 1) % G == 0 || b == nb - 1) S[(b / G) * 32 + lane] = v;
}

// Pass 1 over all blocks: running block sums S_b of the own row
// (sequential over blocks, kernels.py:221-223).  Memory-level parallelism:
//   PIPE = 1  one block's loads in flight, then its arithmetic;
//   PIPE = 2  block b+1's loads issued before block b's arithmetic;
//   PIPE = 3  two blocks' loads issued together, then both reduced.
template <typename T, int W, int VEC, int MODE, int ND, int PIPE>
__device__ __forceinline__ T bfly_blocks(const RowSet<T, GeoV<W, VEC>::L>& prow,
                                         const RowSet<T, (GeoV<W, VEC>::L < 2 ? 2 : GeoV<W, VEC>::L)>& trow,
                                         const bool (&rvalid)[GeoV<W, VEC>::L], int nb, int s, T acc,
                                         T* __restrict__ S, int lane, uint64_t px, uint64_t pt,
                                         uint32_t opaque_zero, uint32_t dsel, bool raw, int G) {
  // raw: store the block totals T_b themselves (the running sums are formed
  // after the remnant prefix is known); else S_b = S_{b-1} + T_b directly
  using R = BlockRegs<T, W, VEC, MODE, ND>;
  if (MODE == MODE_LDA && ND == 0 && PIPE != 4) {
    for (int b = 0; b < nb; ++b) {
      const T t = block_total_nd0<T, W, VEC>(prow, trow, (int64_t)b * W, rvalid, s, px, pt);
      acc = raw ? t : add_rn(acc, t);
      store_s(S, b, nb, G, lane, acc);
    }
  } else if (PIPE == 1 || PIPE == 4) {
#pragma unroll (MODE == MODE_LDA ? kBlockUnroll : 1)  // rows: unrolling cost 3-5% at K = 64-128
    for (int b = 0; b < nb; ++b) {
      R cur;
      cur.load(prow, trow, (int64_t)b * W, px, pt);
      if (PIPE == 4) cur.join(opaque_zero);
      const T t = cur.reduce(rvalid, s, dsel);
      acc = raw ? t : add_rn(acc, t);
      store_s(S, b, nb, G, lane, acc);
    }
  } else if (PIPE == 2) {
    R cur;
    if (nb > 0) cur.load(prow, trow, 0, px, pt);
    for (int b = 0; b < nb; ++b) {
      R nxt;
      if (b + 1 < nb) nxt.load(prow, trow, (int64_t)(b + 1) * W, px, pt);
      const T t = cur.reduce(rvalid, s, dsel);
      acc = raw ? t : add_rn(acc, t);
      store_s(S, b, nb, G, lane, acc);
      cur = nxt;
    }
  } else {
    int b = 0;
    for (; b + 1 < nb; b += 2) {
      R c0, c1;
      c0.load(prow, trow, (int64_t)b * W, px, pt);
      c1.load(prow, trow, (int64_t)(b + 1) * W, px, pt);
      const T t0 = c0.reduce(rvalid, s, dsel);
      acc = raw ? t0 : add_rn(acc, t0);
      store_s(S, b, nb, G, lane, acc);
      const T t1 = c1.reduce(rvalid, s, dsel);
      acc = raw ? t1 : add_rn(acc, t1);
      store_s(S, b + 1, nb, G, lane, acc);
    }
    if (b < nb) {
      R c0;
      c0.load(prow, trow, (int64_t)b * W, px, pt);
      const T t0 = c0.reduce(rvalid, s, dsel);
      acc = raw ? t0 : add_rn(acc, t0);
      store_s(S, b, nb, G, lane, acc);
    }
  }
  return acc;
}

// Ring depth of the cp.async block pipeline (PIPE 5 -> 3 stages, 6 -> 4).
template <int PIPE> struct RingDepth { static constexpr int NS = PIPE == 6 ? 4 : 3; };
// cp.async wait with a compile-time group count
template <int N> __device__ __forceinline__ void cp_async_wait_n() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// bytes of one ring stage: L phi segments + up to 2 theta segments, 16 B per lane
template <int W> struct RingStage { static constexpr int BYTES = (Geo<W>::L + 2) * 32 * 16; };

// Pass 1 with the block loads staged through a per-warp shared-memory ring by
// cp.async (fp32, 16-byte segments): block b+NS-1 is in flight while block b
// is reduced, and in-flight data occupies shared memory instead of
// registers.  Each lane reads back only the segments it copied itself, so the
// per-thread wait_group is the only synchronisation needed.
template <typename T, int W, int MODE, int ND, int NS>
__device__ __forceinline__ T bfly_blocks_ring(const RowSet<T, Geo<W>::L>& prow,
                                              const RowSet<T, (Geo<W>::L < 2 ? 2 : Geo<W>::L)>& trow,
                                              const bool (&rvalid)[Geo<W>::L], int nb, int s, T acc,
                                              T* __restrict__ S, int lane, uint32_t dsel, bool raw,
                                              char* __restrict__ ring, int G) {
  static_assert(sizeof(T) * Geo<W>::E == 16, "ring path needs 16-byte segments");
  constexpr int L = Geo<W>::L;
  constexpr int NT = MODE == MODE_LDA ? ND : 0;
  constexpr int STAGE = RingStage<W>::BYTES;
  using R = BlockRegs<T, W, true, MODE, (MODE == MODE_LDA ? ND : 1)>;
  auto issue = [&](int b) {
    char* st = ring + (b % NS) * STAGE + lane * 16;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) cp_async16(st + kk * 512, prow.ptr(kk, (int64_t)b * W));
#pragma unroll
    for (int i = 0; i < NT; ++i) cp_async16(st + (L + i) * 512, trow.ptr(i, (int64_t)b * W));
  };
#pragma unroll
  for (int b = 0; b < NS - 1; ++b) {
    if (b < nb) issue(b);
    cp_async_commit();
  }
  for (int b = 0; b < nb; ++b) {
    if (b + NS - 1 < nb) issue(b + NS - 1);
    cp_async_commit();
    cp_async_wait_n<NS - 1>();  // block b's group has landed
    const char* st = ring + (b % NS) * STAGE + lane * 16;
    R cur;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const float4 v = *reinterpret_cast<const float4*>(st + kk * 512);
      cur.x[kk].v[0] = v.x; cur.x[kk].v[1] = v.y; cur.x[kk].v[2] = v.z; cur.x[kk].v[3] = v.w;
    }
    if (MODE == MODE_LDA) {
#pragma unroll
      for (int i = 0; i < R::NT; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(st + (L + i) * 512);
        cur.th[i].v[0] = v.x; cur.th[i].v[1] = v.y; cur.th[i].v[2] = v.z; cur.th[i].v[3] = v.w;
      }
    }
    const T t = cur.reduce(rvalid, s, dsel);
    acc = raw ? t : add_rn(acc, t);
    store_s(S, b, nb, G, lane, acc);
  }
  cp_async_wait_n<0>();
  return acc;
}

// In-block walk (kernels.py:268-314).  Per level the reference compares stop
// with low + node(lo, lo+bit-1) or with high - node(lo+bit, lo+2bit-1), picked
// by bit `bit` of r = doc mod W; the nodes are the block's pairwise-tree nodes
// (what its cross-lane fetch of the butterfly table returns).  cur[0, 2*BIT)
// holds the products of the live range; the range halves every level.
template <typename T, int BIT> struct Walk {
  static __device__ __forceinline__ void run(T* cur, T& low, T& high, T stop, int r, int& lo) {
    const T cmp = (r & BIT) ? sub_rn(high, Tree<T, BIT>::sum(cur + BIT)) : add_rn(low, Tree<T, BIT>::sum(cur));
    const bool less = stop < cmp;
    if (less) high = cmp;
    else { low = cmp; lo += BIT; }
#pragma unroll
    for (int t = 0; t < BIT; ++t) cur[t] = less ? cur[t] : cur[t + BIT];
    Walk<T, BIT / 2>::run(cur, low, high, stop, r, lo);
  }
};
template <typename T> struct Walk<T, 0> {
  static __device__ __forceinline__ void run(T*, T&, T&, T, int, int&) {}
};

// Elements of the per-warp running-sum array S: nbc blocks x 32 lanes, at
// least a [32][TS] tile when the cooperative pass-2 reload uses S as its tile
// (no remnant tile).  Shared by the kernel and the launcher.
__host__ __device__ constexpr int bfly_s_elems(int nbc, int rem, int TS, bool coop) {
  return (coop && rem == 0 && nbc * 32 < 32 * TS) ? 32 * TS : nbc * 32;
}

// Minimum resident CTAs per SM (register cap) of each bfly_kernel instantiation.
// KV (K variant) of a bfly_kernel instantiation: which block-sum storage and
// pass-2 reload it compiles (chosen per launch from nb = K / W).
enum { KV_FINE = 0, KV_COARSE = 1, KV_SMALL = 2 };

template <typename T, int W, int VEC, int MODE, int PIPE, int KV>
constexpr int bfly_min_blocks() {
  constexpr bool COARSE = KV == KV_COARSE;
  if (sizeof(T) == 4 && W == 32 && VEC)
    return PIPE == 2 ? 4
                     : (MODE == MODE_LDA ? (COARSE ? WD_LDA_MIN_BLOCKS_COARSE
                                                   : (KV == KV_SMALL && VEC == 2 ? WD_LDA_MIN_BLOCKS_SMALL
                                                                                 : WD_LDA_MIN_BLOCKS))
                                         : 8);
  if (sizeof(T) == 8 && W == 32 && VEC && MODE == MODE_LDA) return WD_LDA_MIN_BLOCKS_F64;
  // other lane counts: uncapped they take 150-250 registers (float64 W = 64
  // would spill at 4 CTAs)
  if (VEC) return (sizeof(T) == 8 && W == 64) ? 2 : WD_MIN_BLOCKS_OTHER;
  return 1;
}

template <typename T, int W, int VEC, int MODE, int PIPE, int KV>
__global__ void __launch_bounds__(128, (bfly_min_blocks<T, W, VEC, MODE, PIPE, KV>()))
    bfly_kernel(DrawParams<T> p) {
  // KV_COARSE: more than 32 blocks per row, every G-th running sum kept;
  // KV_SMALL (LDA, vector, at most 16 blocks): warp-cooperative pass-2 reload
  constexpr bool COARSE = KV == KV_COARSE;
  using GW = GeoV<W, VEC>;
  constexpr int E = GW::E, L = GW::L, R = GW::R;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int K = p.K;
  const int nb = K / W, rem = K % W;
  // coarse running sums beyond 32 blocks (COARSE instantiation only)
  const int G = COARSE ? (nb > 32 ? (nb + 31) / 32 : 1) : 1;
  const int nbc = nb > 0 ? (nb + G - 1) / G : 1;
  const int wpb_i = blockDim.x >> 5;
  // remnant tile [32 rows][TS] per warp (after every warp's S).  Vector path:
  // stride W + 4 keeps rows 16-byte aligned and the 128-bit segment stores /
  // row scans conflict-free; scalar path: odd stride W + 1.
  constexpr int TS = VEC ? W + 4 : W + 1;
  // warp-cooperative pass-2 reload (LDA, vector, fine): with no remnant tile
  // the reload tile aliases S, which is then sized for it
  constexpr bool COOP = MODE == MODE_LDA && VEC && KV == KV_SMALL;
  // rows with pipelined block loads: the remnant prefix is stored for a
  // vector fallback scan (measured: K = 176-240 +5%; the PIPE 1 variant, K <= 144,
  // lost 13% at K = 16 and keeps the re-adding scan)
  constexpr bool kPrefixScan = MODE == MODE_ROWS && PIPE >= 2;
  const size_t SW = (size_t)bfly_s_elems(nbc, rem, TS, COOP);  // S elements per warp
  T* S = reinterpret_cast<T*>(smem_raw) + (size_t)wib * SW;
  T* RT = reinterpret_cast<T*>(smem_raw) + (size_t)wpb_i * SW + (size_t)wib * 32 * TS;
  // cp.async ring (PIPE 5/6), after every warp's S and remnant tile
  constexpr bool RING = PIPE >= 5;
  char* ring = reinterpret_cast<char*>(reinterpret_cast<T*>(smem_raw) + (size_t)wpb_i * SW +
                                       (size_t)wpb_i * 32 * TS) +
               (size_t)wib * RingDepth<PIPE>::NS * RingStage<W>::BYTES;
  const int s = lane % L;
  const int rg = lane / L;
  // Chunk row of the lane's kk-th load.  LDA: each lane group rg loads L
  // CONSECUTIVE rows (a warp instruction still reads R full row segments),
  // so a lane's rows span few documents and their theta segments are shared
  // (per-lane ND = 2 below); rows: interleaved.  The transpose-reduce leaves
  // lane (s, rg) with the total of its kk = s row.
  constexpr bool CONTIG = MODE == MODE_LDA;
  auto row_of = [&](int kk) { return CONTIG ? rg * L + kk : kk * R + rg; };
  const int own = row_of(s);  // chunk row this lane ends up owning
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t wpb = blockDim.x >> 5;
  const uint64_t pol_x = make_l2_policy(p.l2_policy_x);
  const uint64_t pol_t = make_l2_policy(p.l2_policy_t);
  for (int64_t c = (int64_t)blockIdx.x * wpb + wib; c < n_chunks; c += (int64_t)gridDim.x * wpb) {
    const int64_t tok0 = c << 5;
    bool my_valid = tok0 + lane < n;
    int32_t my_doc = 0, my_word = 0;
    if (MODE == MODE_LDA && my_valid) {
      my_doc = p.token_doc[tok0 + lane];
      my_word = p.words[tok0 + lane];
      // padding slot of a run-padded vocabulary tile (token_pos < 0): it
      // carries its run's document and a word of it (valid loads, so the
      // lane group stays single-document) but draws nothing
      if (p.token_pos != nullptr) my_valid = p.token_pos[tok0 + lane] >= 0;
    }
    const uint32_t vmask = __ballot_sync(FULL, my_valid);
    constexpr int LT = L < 2 ? 2 : L;
    RowSet<T, L> prow;  // the L rows this lane loads (phi / weights)
    RowSet<T, LT> trow;  // their theta rows (LDA)
    prow.base = reinterpret_cast<const char*>(p.phi + rem + s * E);
    prow.ldb = (uint32_t)(p.ld_phi * sizeof(T));
    trow.base = MODE == MODE_LDA ? reinterpret_cast<const char*>(p.theta + rem + s * E) : nullptr;
    trow.ldb = (uint32_t)(p.ld_theta * sizeof(T));
    bool rvalid[L];
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const int k = row_of(kk);
      rvalid[kk] = (vmask >> k) & 1u;
      if (MODE == MODE_LDA) {
        // an invalid row (run padding, chunk tail) reads the phi row of a
        // valid row of the SAME load instruction (rows k ^ j*L), so the
        // coalescer merges it and it costs no extra L1/L2 traffic; its theta
        // stays its own run's document (the lane group's); sums discarded
        int src = k;
        if (!COARSE && !rvalid[kk]) {
#pragma unroll
          for (int j = R - 1; j >= 1; --j)
            if ((vmask >> (k ^ (j * L))) & 1u) src = k ^ (j * L);
        }
        prow.idx[kk] = (uint32_t)__shfl_sync(FULL, my_word, src);
        trow.idx[kk] = (uint32_t)__shfl_sync(FULL, my_doc, k);
      } else {
        prow.idx[kk] = (uint32_t)(rvalid[kk] ? tok0 + k : tok0);
        trow.idx[kk] = 0;
      }
    }
    if (L < 2) trow.idx[LT - 1] = trow.idx[0];
    const int64_t own_tok = tok0 + own;
    const bool own_valid = (vmask >> own) & 1u;
    const int32_t own_doc = __shfl_sync(FULL, my_doc, own);
    const int32_t own_word = __shfl_sync(FULL, my_word, own);
    const T* pown = p.phi + (MODE == MODE_LDA ? (int64_t)own_word : own_tok) * p.ld_phi;
    const T* town = MODE == MODE_LDA ? p.theta + (int64_t)own_doc * p.ld_theta : nullptr;

    // remnant (topics [0, rem)), loaded cooperatively like a block into the
    // warp's shared tiles and summed sequentially along the own row
    // (kernels.py:199-205).  Vector path: cp.async copies issued now, consumed
    // after the block loop, so the remnant costs no extra memory round trip;
    // the block loop then stores raw block totals and the running sums are
    // formed once the remnant prefix is known (same IEEE additions).
    T acc = T(0);
    const bool async_rem = VEC && rem > 0 && rem % E == 0 && (E * sizeof(T)) % 16 == 0 && G == 1;
    const bool raw = async_rem;  // block totals stored raw, running sums formed after the loop
    T prem = T(0);
    if (async_rem) {
#pragma unroll
      for (int kk = 0; kk < L; ++kk) {
        if (s * E < rem) {
          const int k = row_of(kk);
#pragma unroll
          for (int c = 0; c < (int)(E * sizeof(T) / 16); ++c)
            cp_async16(RT + k * TS + s * E + c * (16 / sizeof(T)), prow.ptr(kk, -rem + c * (16 / (int)sizeof(T))));
        }
      }
      cp_async_commit();
    } else if (rem > 0) {
      // half batches of rows keep the live loads (and the kernel's register
      // budget) at the level of the block loop
      constexpr int HB = L >= 4 ? L / 2 : L;
#pragma unroll
      for (int h = 0; h < L; h += HB) {
#pragma unroll
        for (int kk = h; kk < h + HB; ++kk) {
          if (s * E < rem) {
            const int k = row_of(kk);
            const bool full = s * E + E <= rem;  // else: partial segment, scalar loads
            Seg<T, E, (VEC != 0)> x;
            if (full) x.load(prow.ptr(kk, -rem)); else load_first(x.v, prow.ptr(kk, -rem), rem - s * E);
            T a[E];
            if (MODE == MODE_LDA) {
              Seg<T, E, (VEC != 0)> th;
              if (full) th.load(trow.ptr(kk, -rem)); else load_first(th.v, trow.ptr(kk, -rem), rem - s * E);
#pragma unroll
              for (int e = 0; e < E; ++e) a[e] = mul_rn(th.v[e], x.v[e]);
            } else {
#pragma unroll
              for (int e = 0; e < E; ++e) a[e] = x.v[e];
            }
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (s * E + e < rem) RT[k * TS + s * E + e] = a[e];
          }
        }
      }
      __syncwarp();
      for (int t = 0; t < rem; ++t) prem = add_rn(prem, RT[own * TS + t]);  // sequential
      acc = prem;
    }
    // theta rows: one document for the whole chunk (ND = 1), else ND = 2
    // with the first and last document of the LANE's rows (its L rows are
    // consecutive; each lane loads its own pair of theta segments, a warp
    // instruction still covering R row segments), the rows of the second
    // flagged in dsel; ND = 0 (per-row theta loads) only when some lane's
    // rows touch three documents.
    int nd = 1;
    uint32_t dsel = 0;
    RowSet<T, LT> trow_nd = trow;
    if (MODE == MODE_LDA) {
      const int32_t d0 = __shfl_sync(FULL, my_doc, 0);
      const int32_t d1 = __reduce_max_sync(FULL, my_valid ? my_doc : d0);
      if (d1 != d0) {
        const uint32_t da = trow.idx[0];
        uint32_t db = da;
#pragma unroll
        for (int kk = 0; kk < L; ++kk)
          if (rvalid[kk]) db = trow.idx[kk];
        bool ok = true;
#pragma unroll
        for (int kk = 0; kk < L; ++kk) {
          ok = ok && (!rvalid[kk] || trow.idx[kk] == da || trow.idx[kk] == db);
          if (rvalid[kk] && trow.idx[kk] != da) dsel |= 1u << kk;
        }
        nd = __all_sync(FULL, ok) ? 2 : 0;
        if (!COARSE && nd == 2 && __all_sync(FULL, dsel == 0u)) {
          // every lane's rows are one document (per lane group; always so
          // on run-padded tiles): one theta segment per lane, no per-row
          // selection.  Fine instantiation only: in the coarse one the extra
          // path costs more (register allocation) than it saves unpadded
          // (measured at K = 4096: 420 vs 443 ms)
          nd = 1;
          trow_nd.idx[0] = da;
        } else if (nd == 2) {
          trow_nd.idx[0] = da;
          trow_nd.idx[1] = db;
        } else {
          dsel = 0;
        }
      } else {
        trow_nd.idx[0] = (uint32_t)d0;
      }
    }
    if constexpr (RING) {
      if (MODE == MODE_ROWS || nd == 1)
        acc = bfly_blocks_ring<T, W, MODE, 1, RingDepth<PIPE>::NS>(prow, trow_nd, rvalid, nb, s, acc, S, lane, 0u,
                                                                   raw, ring, G);
      else if (nd == 2)
        acc = bfly_blocks_ring<T, W, MODE, 2, RingDepth<PIPE>::NS>(prow, trow_nd, rvalid, nb, s, acc, S, lane, dsel,
                                                                   raw, ring, G);
      else  // >2 documents: per-row theta segments, register path
        acc = bfly_blocks<T, W, VEC, MODE, 0, 1>(prow, trow_nd, rvalid, nb, s, acc, S, lane, pol_x, pol_t,
                                                 p.opaque_zero, 0u, raw, G);
    } else if constexpr (MODE == MODE_ROWS) {
      acc = bfly_blocks<T, W, VEC, MODE, 1, PIPE>(prow, trow_nd, rvalid, nb, s, acc, S, lane, pol_x, pol_t,
                                                  p.opaque_zero, 0u, raw, G);
    } else {
      if (nd == 1)
        acc = bfly_blocks<T, W, VEC, MODE, 1, PIPE>(prow, trow_nd, rvalid, nb, s, acc, S, lane, pol_x, pol_t,
                                                    p.opaque_zero, 0u, raw, G);
      else if (nd == 2)
        acc = bfly_blocks<T, W, VEC, MODE, 2, PIPE>(prow, trow_nd, rvalid, nb, s, acc, S, lane, pol_x, pol_t,
                                                    p.opaque_zero, dsel, raw, G);
      else  // >2 documents: per-row theta segments
        acc = bfly_blocks<T, W, VEC, MODE, 0, (PIPE != 4 ? 1 : PIPE)>(prow, trow_nd, rvalid, nb, s, acc, S, lane,
                                                                      pol_x, pol_t, p.opaque_zero, 0u, raw, G);
    }
    if (raw) {
      cp_async_wait_all();
      __syncwarp();
      // sequential remnant prefix of the own row (products formed here on the
      // asynchronous path, already in the tile on the synchronous one)
      if (async_rem) {
        for (int t = 0; t < rem; t += E) {
          T a[E];
          load_seg_smem(a, RT + own * TS + t);
          if (MODE == MODE_LDA) {  // the own document's theta remnant (L1-resident)
            Seg<T, E, (VEC != 0)> th;
            th.load(town + t);
#pragma unroll
            for (int e = 0; e < E; ++e) a[e] = mul_rn(th.v[e], a[e]);
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            prem = add_rn(prem, a[e]);
            a[e] = prem;
          }
          // rows: the own row's remnant prefix P[t] replaces its products, so
          // the remnant fallback scans it without re-adding (a chain of
          // dependent shared loads and adds before; LDA keeps the products:
          // its tuned register allocation spills with the store)
          if constexpr (kPrefixScan) store_seg(RT + own * TS + t, a);
        }
      }
      acc = prem;
      for (int b = 0; b < nb; ++b) {  // S_b = S_{b-1} + T_b from the raw totals
        acc = add_rn(acc, S[b * 32 + lane]);
        S[b * 32 + lane] = acc;
      }
    }
    __syncwarp();
    const T total = acc;

    if constexpr (!COOP) {
      // per-lane pass 2 (kept verbatim for the fine and coarse variants:
      // their register allocation is tuned)
      if (own_valid) {
        uint64_t ka, kb;
        unsigned long long ekey;
        int r;
        int64_t zidx;
        token_keys<T, MODE>(p, own_tok, own_doc, W, ka, kb, ekey, r, zidx);
        const T stop = make_stop<T>(p, zidx, total, ka, kb, MODE == MODE_ROWS);
        if (!(total > T(0))) atomicMin(p.err, ekey);
        // block bisection over S (kernels.py:337-346): the first block whose
        // running sum exceeds stop (S is nondecreasing, so any search that finds
        // that block is the reference's bisection)
        T cur[W];
        int j;
        T prev, high;
        auto load_block = [&](int64_t base) {  // own row's products of one block
          constexpr int NG = W / E;
          constexpr int HG = NG >= 4 ? NG / 2 : NG;
          if constexpr (sizeof(T) == 4 && VEC && E == 4 && W % 16 == 0) {
            // 256-bit loads when the block is 32-byte aligned (block_aligned_rows
            // layouts): each lane's 32 B are one whole sector, where a 128-bit
            // load touches a sector per lane for half of its bytes
            const T* xp = pown + base;
            const T* tp = MODE == MODE_LDA ? town + base : xp;
            if (((reinterpret_cast<uintptr_t>(xp) | reinterpret_cast<uintptr_t>(tp)) & 31) == 0) {
              constexpr int N8 = W / 8;
              constexpr int H8 = N8 >= 4 ? N8 / 2 : N8;
#pragma unroll
              for (int h = 0; h < N8; h += H8) {
#pragma unroll
                for (int g = h; g < h + H8; ++g) {
                  float x8[8];
                  ld_v8(x8, xp + g * 8);
                  if (MODE == MODE_LDA) {
                    float t8[8];
                    ld_v8(t8, tp + g * 8);
#pragma unroll
                    for (int e = 0; e < 8; ++e) cur[g * 8 + e] = mul_rn(t8[e], x8[e]);
                  } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) cur[g * 8 + e] = x8[e];
                  }
                }
              }
              return;
            }
          }
#pragma unroll
          for (int h = 0; h < NG; h += HG) {
#pragma unroll
            for (int g = h; g < h + HG; ++g) {
              Seg<T, E, (VEC != 0)> x;
              x.load(pown + base + g * E);
              if (MODE == MODE_LDA) {
                Seg<T, E, (VEC != 0)> th;
                th.load(town + base + g * E);
#pragma unroll
                for (int e = 0; e < E; ++e) cur[g * E + e] = mul_rn(th.v[e], x.v[e]);
              } else {
#pragma unroll
                for (int e = 0; e < E; ++e) cur[g * E + e] = x.v[e];
              }
            }
          }
        };
        {
          int lo2 = 0, hi2 = nbc - 1;
          while (lo2 < hi2) {
            const int mid = (lo2 + hi2) >> 1;
            if (stop < S[mid * 32 + lane]) hi2 = mid; else lo2 = mid + 1;
          }
          if (!COARSE || G == 1) {
            j = lo2;
            prev = j > 0 ? S[(j - 1) * 32 + lane] : prem;
            high = nb > 0 ? S[j * 32 + lane] : T(0);
          } else {
            // recompute the selected group's block totals and running sums
            T run = lo2 > 0 ? S[(lo2 - 1) * 32 + lane] : prem;
            const int b0 = lo2 * G, b1 = min(b0 + G, nb);
            j = b1 - 1;
            prev = run;
            high = run;
            for (int bj = b0; bj < b1; ++bj) {
              load_block((int64_t)rem + (int64_t)bj * W);
              const T sb = add_rn(run, Tree<T, W>::sum(cur));
              if (stop < sb || bj == b1 - 1) {
                j = bj;
                prev = run;
                high = sb;
                break;
              }
              run = sb;
            }
          }
        }
        const int64_t bb = (int64_t)rem + (int64_t)j * W;
        if (bb == 0) prev = T(0);
        const bool fallback = bb > 0 && stop < prev && total > T(0);
        int result = 0;
        if (nb > 0 && !fallback) {
          // rebuild the selected block's products (own row) and walk it
          load_block(bb);  // coarse: reloaded (L1 hit) rather than kept live, which
                           // lets the coarse kernel fit 5 CTAs per SM
          T low = prev;
          int lo = 0;
          Walk<T, W / 2>::run(cur, low, high, stop, r, lo);
          result = (int)bb + lo;
        }
        if (kPrefixScan && fallback && async_rem) {
          // linear remnant fallback (kernels.py:354-361) over the prefix P[t]
          // the raw pass stored (the same sequential sums): first t with
          // stop < P[t], one vector shared load per E topics
          int found = -1;
          for (int t = 0; t < rem && found < 0; t += E) {
            T pv[E];
            load_seg_smem(pv, RT + own * TS + t);
#pragma unroll
            for (int e = E - 1; e >= 0; --e)
              if (stop < pv[e]) found = t + e;
          }
          if (found >= 0) result = found;
        } else if (fallback) {
          // linear remnant fallback (kernels.py:354-361), products from the tile(s)
          T a2 = T(0);
          for (int t = 0; t < rem; ++t) {
            const T a = (MODE == MODE_LDA && async_rem) ? mul_rn(__ldg(town + t), RT[own * TS + t]) : RT[own * TS + t];
            a2 = add_rn(a2, a);
            if (stop < a2) { result = t; break; }
          }
        }
        p.z[zidx] = result;
        if (MODE == MODE_LDA) {
          if (p.word_topic) atomicAdd(p.word_topic + (int64_t)own_word * K + result, 1);
          if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)own_doc * K + result, 1);
        }
      }
    } else {
      // ---- pass 2a (per lane): keys, stop, block bisection over S
      uint64_t ka = 0, kb = 0;
      unsigned long long ekey = 0;
      int r = 0;
      int64_t zidx = 0;
      T stop = T(0), prev = T(0), high = T(0);
      int j = 0;
      T cur[W];
      auto load_block = [&](int64_t base) {  // own row's products of one block
        constexpr int NG = W / E;
        constexpr int HG = NG >= 4 ? NG / 2 : NG;
#pragma unroll
        for (int h = 0; h < NG; h += HG) {
#pragma unroll
          for (int g = h; g < h + HG; ++g) {
            Seg<T, E, (VEC != 0)> x;
            x.load(pown + base + g * E);
            if (MODE == MODE_LDA) {
              Seg<T, E, (VEC != 0)> th;
              th.load(town + base + g * E);
#pragma unroll
              for (int e = 0; e < E; ++e) cur[g * E + e] = mul_rn(th.v[e], x.v[e]);
            } else {
#pragma unroll
              for (int e = 0; e < E; ++e) cur[g * E + e] = x.v[e];
            }
          }
        }
      };
      if (own_valid) {
        token_keys<T, MODE>(p, own_tok, own_doc, W, ka, kb, ekey, r, zidx);
        stop = make_stop<T>(p, zidx, total, ka, kb, MODE == MODE_ROWS);
        if (!(total > T(0))) atomicMin(p.err, ekey);
        // block bisection over S (kernels.py:337-346): the first block whose
        // running sum exceeds stop (S is nondecreasing, so any search that finds
        // that block is the reference's bisection)
        int lo2 = 0, hi2 = nbc - 1;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (stop < S[mid * 32 + lane]) hi2 = mid; else lo2 = mid + 1;
        }
        if (!COARSE || G == 1) {
          j = lo2;
          prev = j > 0 ? S[(j - 1) * 32 + lane] : prem;
          high = nb > 0 ? S[j * 32 + lane] : T(0);
        } else {
          // recompute the selected group's block totals and running sums
          T run = lo2 > 0 ? S[(lo2 - 1) * 32 + lane] : prem;
          const int b0 = lo2 * G, b1 = min(b0 + G, nb);
          j = b1 - 1;
          prev = run;
          high = run;
          for (int bj = b0; bj < b1; ++bj) {
            load_block((int64_t)rem + (int64_t)bj * W);
            const T sb = add_rn(run, Tree<T, W>::sum(cur));
            if (stop < sb || bj == b1 - 1) {
              j = bj;
              prev = run;
              high = sb;
              break;
            }
            run = sb;
          }
        }
      }
      const int64_t bb = (int64_t)rem + (int64_t)j * W;
      if (bb == 0) prev = T(0);
      const bool fallback = own_valid && bb > 0 && stop < prev && total > T(0);
      const bool walk = own_valid && nb > 0 && !fallback;

      // ---- pass 2b: the selected block's products of the own row
      {
        // Warp-cooperative reload: lane group rg fetches target lane t's block
        // segment (one 128-byte row segment per group per instruction, the
        // coalesced pattern of pass 1) into t's row of a shared tile, instead
        // of every lane gathering its own 32 values from 32 different lines
        // per instruction (~31 L1 tag requests each, the largest tag-request
        // source at small K).  The tile is the remnant tile (rows of walking
        // lanes only; a fallback lane's remnant row is left intact) or, with
        // no remnant, S (free once every lane has read its bounds).
        T* tile = rem > 0 ? RT : S;
        __syncwarp();
        const uint32_t wmask = __ballot_sync(FULL, walk);
        const int bbi = (int)bb;
#pragma unroll
        for (int i = 0; i < 32 / R; ++i) {
          const int t = i * R + rg;
          const int32_t wt = __shfl_sync(FULL, own_word, t);
          const int32_t dt = __shfl_sync(FULL, own_doc, t);
          const int bt = __shfl_sync(FULL, bbi, t);
          if ((wmask >> t) & 1u) {
            Seg<T, E, (VEC != 0)> x, th;
            x.load(p.phi + (int64_t)wt * p.ld_phi + bt + s * E);
            th.load(p.theta + (int64_t)dt * p.ld_theta + bt + s * E);
            T a[E];
#pragma unroll
            for (int e = 0; e < E; ++e) a[e] = mul_rn(th.v[e], x.v[e]);
            store_seg(tile + t * TS + s * E, a);
          }
        }
        __syncwarp();
        if (walk) {
#pragma unroll
          for (int g = 0; g < W / E; ++g) {
            T a[E];
            load_seg_smem(a, tile + lane * TS + g * E);
#pragma unroll
            for (int e = 0; e < E; ++e) cur[g * E + e] = a[e];
          }
        }
      }

      if (own_valid) {
        int result = 0;
        if (walk) {
          T low = prev;
          int lo = 0;
          Walk<T, W / 2>::run(cur, low, high, stop, r, lo);
          result = (int)bb + lo;
        }
        if (fallback) {
          // linear remnant fallback (kernels.py:354-361), products from the tile(s)
          T a2 = T(0);
          for (int t = 0; t < rem; ++t) {
            const T a = (MODE == MODE_LDA && async_rem) ? mul_rn(__ldg(town + t), RT[own * TS + t]) : RT[own * TS + t];
            a2 = add_rn(a2, a);
            if (stop < a2) { result = t; break; }
          }
        }
        p.z[zidx] = result;
        if (MODE == MODE_LDA) {
          if (p.word_topic) atomicAdd(p.word_topic + (int64_t)own_word * K + result, 1);
          if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)own_doc * K + result, 1);
        }
      }
    }
    __syncwarp();
  }
}

// ================================================ rows, one block
// Standalone rows with K = NB * W (no remnant; dispatched for NB = 1): every block of a
// chunk's 32 rows is staged in shared memory as it is loaded, so pass 2
// reads the selected block from there instead of re-gathering it from
// global memory (at K = 32 / 64 that per-lane re-gather -- 32 lines per
// instruction -- made the per-row kernel L1-bound at ~2.7 / 4.8 TB/s).
// Same loads, tree, running sums, bisection and walk as bfly_kernel.
template <typename T, int W, int NB>
__global__ void __launch_bounds__(128, 6) rows_stash_kernel(DrawParams<T> p) {
  using GW = Geo<W>;
  constexpr int E = GW::E, L = GW::L, R = GW::R;
  constexpr int TS = W + 4;  // 16-byte aligned rows, conflict-free 128-bit accesses
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* tile = reinterpret_cast<T*>(smem_raw) + (size_t)wib * NB * 32 * TS;  // [NB][32 rows][TS]
  const int s = lane % L;
  const int rg = lane / L;
  const int own = s * R + rg;  // interleaved rows (bfly_kernel, MODE_ROWS)
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t wpb = blockDim.x >> 5;
  const uint64_t pol = make_l2_policy(p.l2_policy_x);
  for (int64_t c = (int64_t)blockIdx.x * wpb + wib; c < n_chunks; c += (int64_t)gridDim.x * wpb) {
    const int64_t tok0 = c << 5;
    RowSet<T, L> prow;
    RowSet<T, (L < 2 ? 2 : L)> trow;
    prow.base = reinterpret_cast<const char*>(p.phi + s * E);
    prow.ldb = (uint32_t)(p.ld_phi * sizeof(T));
    trow.base = nullptr;
    trow.ldb = 0;
#pragma unroll
    for (int i = 0; i < (L < 2 ? 2 : L); ++i) trow.idx[i] = 0;
    bool rvalid[L];
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const int k = kk * R + rg;
      rvalid[kk] = tok0 + k < n;
      prow.idx[kk] = (uint32_t)(rvalid[kk] ? tok0 + k : tok0);
    }
    T S[NB];
    T acc = T(0);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      BlockRegs<T, W, true, MODE_ROWS, 1> cur;
      cur.load(prow, trow, (int64_t)b * W, pol, pol);
#pragma unroll
      for (int kk = 0; kk < L; ++kk) store_seg(tile + ((size_t)b * 32 + kk * R + rg) * TS + s * E, cur.x[kk].v);
      const T t = cur.reduce(rvalid, s, 0u);
      acc = add_rn(acc, t);  // sequential running sums (kernels.py:221-223)
      S[b] = acc;
    }
    __syncwarp();
    const int64_t own_tok = tok0 + own;
    if (own_tok < n) {
      uint64_t ka, kb;
      unsigned long long ekey;
      int r;
      int64_t zidx;
      token_keys<T, MODE_ROWS>(p, own_tok, 0, W, ka, kb, ekey, r, zidx);
      const T total = acc;
      const T stop = make_stop<T>(p, zidx, total, ka, kb, true);
      if (!(total > T(0))) atomicMin(p.err, ekey);
      // bisection over the NB running sums: the first block whose sum exceeds stop
      int j = NB - 1;
#pragma unroll
      for (int b = NB - 2; b >= 0; --b)
        if (stop < S[b]) j = b;
      const T prev = j > 0 ? S[j - 1] : T(0);
      T high = S[j];
      T cur[W];
      const T* row = tile + ((size_t)j * 32 + own) * TS;
#pragma unroll
      for (int g = 0; g < W / E; ++g) {
        T a[E];
        load_seg_smem(a, row + g * E);
#pragma unroll
        for (int e = 0; e < E; ++e) cur[g * E + e] = a[e];
      }
      T low = prev;
      int lo = 0;
      Walk<T, W / 2>::run(cur, low, high, stop, r, lo);
      p.z[zidx] = j * W + lo;
    }
    __syncwarp();
  }
}

// rows_stash_kernel with the chunk loads double-buffered by cp.async
// (fp32, 16-byte segments): chunk c + stride is in flight while chunk c is
// searched, so each warp always has one chunk of loads outstanding (the
// single-buffer kernel exposed a DRAM round trip per chunk: K = 32 at 49% of
// DRAM bandwidth with 22 warps per SM).  The loads are coalesced (a warp
// instruction copies R whole row segments); each lane then reads ITS OWN row
// from the tile and forms the block totals as the pairwise tree in registers
// -- the same additions the shuffle transpose-reduce performs, so the same
// bits, without its shuffles and second pass over the tile (ncu: the
// transposed variant was short-scoreboard / shared-memory bound).
template <typename T, int W, int NB>
__global__ void __launch_bounds__(128, (NB == 1 ? 6 : 3)) rows_stash2_kernel(DrawParams<T> p) {
  using GW = Geo<W>;
  constexpr int E = GW::E, L = GW::L, R = GW::R;
  static_assert(E * sizeof(T) == 16, "16-byte segments");
  constexpr int TS = W + 4;
  constexpr int STAGE = NB * 32 * TS;  // elements per stage
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* tiles = reinterpret_cast<T*>(smem_raw) + (size_t)wib * 2 * STAGE;  // [2][NB][32 rows][TS]
  const int s = lane % L;
  const int rg = lane / L;
  const int own = lane;  // own row: consecutive lanes read rows TS apart (conflict-free)
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
  auto issue = [&](int64_t c, T* tile) {
    const int64_t tok0 = c << 5;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const int k = kk * R + rg;
      const int64_t row = tok0 + k < n ? tok0 + k : tok0;  // tail rows read a valid row
      const T* src = p.phi + row * p.ld_phi + s * E;
#pragma unroll
      for (int b = 0; b < NB; ++b) cp_async16(tile + ((size_t)b * 32 + k) * TS + s * E, src + b * W);
    }
    cp_async_commit();
  };
  int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (c < n_chunks) issue(c, tiles);
  for (int st = 0; c < n_chunks; c += stride, st ^= 1) {
    if (c + stride < n_chunks) issue(c + stride, tiles + (st ^ 1) * STAGE);
    else cp_async_commit();  // empty group: the wait below still means "chunk c landed"
    cp_async_wait_n<1>();
    __syncwarp();
    T* tile = tiles + st * STAGE;
    const int64_t tok0 = c << 5;
    {
      // the lane reads its own row from the tile and forms each block total
      // as the same pairwise tree the transpose-reduce computes (no
      // shuffles); pass 2 re-reads the selected block from the tile
      const int64_t own_tok = tok0 + own;
      if (own_tok < n) {
        const T* row = tile + (size_t)own * TS;
        T cur[W];
        auto load_own = [&](int b) {
#pragma unroll
          for (int g = 0; g < W / E; ++g) {
            T a[E];
            load_seg_smem(a, row + (size_t)b * 32 * TS + g * E);
#pragma unroll
            for (int e = 0; e < E; ++e) cur[g * E + e] = a[e];
          }
        };
        T S[NB];
        T acc = T(0);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          load_own(b);
          acc = add_rn(acc, Tree<T, W>::sum(cur));  // sequential running sums (kernels.py:221-223)
          S[b] = acc;
        }
        const T total = acc;
        uint64_t ka, kb;
        unsigned long long ekey;
        int r;
        int64_t zidx;
        token_keys<T, MODE_ROWS>(p, own_tok, 0, W, ka, kb, ekey, r, zidx);
        const T stop = make_stop<T>(p, zidx, total, ka, kb, true);
        if (!(total > T(0))) atomicMin(p.err, ekey);
        int j = NB - 1;
#pragma unroll
        for (int b = NB - 2; b >= 0; --b)
          if (stop < S[b]) j = b;
        if (NB > 1 && j != NB - 1) load_own(j);
        T low = j > 0 ? S[j - 1] : T(0);
        T high = S[j];
        int lo = 0;
        Walk<T, W / 2>::run(cur, low, high, stop, r, lo);
        p.z[zidx] = j * W + lo;
      }
    }
    __syncwarp();  // every lane is done with this stage before it is refilled
  }
  cp_async_wait_n<0>();
}

// ========================================================= prefix table
// The paper's comparison baseline: a full per-token prefix-sum table
// (kernels.py:129-167 compute_partial_sums_transposed + kernels.py:248-260
// _prefix_binary_search; arithmetic identical to draw_z_basic,
// kernels.py:380-401).  Loads are the same coalesced vector loads as the
// butterfly kernel; the products are transposed back to their row through a
// padded shared-memory tile (the "pay the piper" gather),
// summed sequentially, and EVERY running sum is stored to a per-lane table in
// global scratch (the paper's local-memory table, interleaved by lane so the
// stores coalesce).  The bisection then reads that table.
template <typename T, bool VEC, int MODE>
__global__ void __launch_bounds__(128) prefix_kernel(DrawParams<T> p, T* __restrict__ table,
                                                     int64_t stride) {
  constexpr int W = 32;
  using G = Geo<W>;
  constexpr int E = G::E, L = G::L, R = G::R;
  constexpr int TP = W + 1;  // padded tile row
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* tile = reinterpret_cast<T*>(smem_raw) + (size_t)wib * 32 * TP;
  const int K = p.K;
  const int nb = K / W, rem = K % W;
  const int s = lane % L;
  const int rg = lane / L;
  const int64_t gl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // table column
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t wpb = blockDim.x >> 5;
  const int WR = p.lanes;
  for (int64_t c = (int64_t)blockIdx.x * wpb + wib; c < n_chunks; c += (int64_t)gridDim.x * wpb) {
    const int64_t tok0 = c << 5;
    bool my_valid = tok0 + lane < n;
    int32_t my_doc = 0, my_word = 0;
    if (MODE == MODE_LDA && my_valid) {
      my_doc = p.token_doc[tok0 + lane];
      my_word = p.words[tok0 + lane];
      if (p.token_pos != nullptr) my_valid = p.token_pos[tok0 + lane] >= 0;  // padding slot
    }
    const T* pown = p.phi + (MODE == MODE_LDA ? (int64_t)my_word : tok0 + lane) * p.ld_phi;
    const T* town = MODE == MODE_LDA ? p.theta + (int64_t)my_doc * p.ld_theta : nullptr;
    T acc = T(0);
    if (my_valid) {
      for (int t = 0; t < rem; ++t) {
        T a = MODE == MODE_LDA ? mul_rn(__ldg(town + t), __ldg(pown + t)) : __ldg(pown + t);
        acc = add_rn(acc, a);
        table[(int64_t)t * stride + gl] = acc;
      }
    }
    for (int b = 0; b < nb; ++b) {
      const int64_t off = (int64_t)rem + (int64_t)b * W;
#pragma unroll
      for (int kk = 0; kk < L; ++kk) {
        const int k = kk * R + rg;
        const int32_t wk = __shfl_sync(FULL, my_word, k);
        const int32_t dk = __shfl_sync(FULL, my_doc, k);
        Seg<T, E, (VEC != 0)> x;
        const bool v = tok0 + k < n;
        if (v) x.load(p.phi + (MODE == MODE_LDA ? (int64_t)wk : tok0 + k) * p.ld_phi + off + s * E);
        else x.zero();
        if (MODE == MODE_LDA) {
          Seg<T, E, (VEC != 0)> th;
          if (v) th.load(p.theta + (int64_t)dk * p.ld_theta + off + s * E); else th.zero();
#pragma unroll
          for (int e = 0; e < E; ++e) x.v[e] = mul_rn(th.v[e], x.v[e]);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) tile[k * TP + s * E + e] = x.v[e];
      }
      __syncwarp();
#pragma unroll 8
      for (int t = 0; t < W; ++t) {
        acc = add_rn(acc, tile[lane * TP + t]);
        table[(off + t) * stride + gl] = acc;
      }
      __syncwarp();
    }
    const T total = acc;
    if (my_valid) {
      uint64_t ka, kb;
      unsigned long long ekey;
      int r;
      int64_t zidx;
      token_keys<T, MODE>(p, tok0 + lane, my_doc, WR, ka, kb, ekey, r, zidx);
      const T stop = make_stop<T>(p, zidx, total, ka, kb, MODE == MODE_ROWS);
      if (!(total > T(0))) atomicMin(p.err, ekey);
      int j = 0, k = K - 1;  // samp.py:65-77 bisection over the table
      while (j < k) {
        const int mid = (j + k) >> 1;
        if (stop < table[(int64_t)mid * stride + gl]) k = mid; else j = mid + 1;
      }
      p.z[zidx] = j;
      if (MODE == MODE_LDA) {
        if (p.word_topic) atomicAdd(p.word_topic + (int64_t)my_word * K + j, 1);
        if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)my_doc * K + j, 1);
      }
    }
    __syncwarp();
  }
}

}  // namespace wd
