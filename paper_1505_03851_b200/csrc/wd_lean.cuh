// wd_lean.cuh -- the register-lean LDA draw for large K (fp32, W = 32,
// 256-bit lane segments, K a multiple of 32).
//
// Same arithmetic as bfly_kernel<float, 32, 2, MODE_LDA, 1, KV_*> (and so the
// reference's draw_z_butterfly, kernels.py:487-539): per W-topic block the
// own row's pairwise tree (Tree<8> in-lane + the shuffle transpose-reduce),
// sequential running sums over blocks, stop = fl(total * fl(u)), the block
// bisection and the add-or-subtract walk selected by the bits of doc mod W.
// What differs is the register budget.  The gathers of this path are served
// by L2 and their rate is set by the bytes in flight per SM (microbenchmark
// tools/stage_probe.cu at K = 4096: 14.4 / 16.4 / 18.3 TB/s with 5 / 6 / 8
// resident CTAs of the same loop; per-lane bulk-async copies into a shared
// ring topped out at 6 TB/s, the copy engine serialising the 128-512-byte
// row segments).  The general kernel needs 80-96 registers (5-6 CTAs/SM)
// because every theta path (one, two or per-row documents), the remnant
// tile and the coarse-group recompute share one allocation.  This kernel
// keeps only what a vocabulary tile padded to the lane-group height needs:
//
//   * each lane's 4 chunk rows belong to one document (run padding 4), so a
//     block is 4 phi segments + 1 theta segment in flight (40 registers); a
//     chunk that breaks this (a tile built without padding, a chunk tail)
//     takes the per-row theta loop in halves, which holds the same 32
//     registers of loads;
//   * no remnant (K % 32 == 0): the first block starts at topic 0 and the
//     remnant fallback of kernels.py:354-361 cannot trigger (stop >= S_{j-1});
//   * at most NBC running sums per lane in shared memory (every G-th block,
//     G = ceil(nb / NBC)); after the bisection the selected group's block
//     totals are recomputed from the own row one 8-topic segment at a time
//     (16 registers of loads), then the selected block is loaded for the walk.
//
// __launch_bounds__(128, 8): 64 registers, 32 warps per SM.
#pragma once

#include "wd_draw.cuh"

namespace wd {

#ifndef WD_LEAN_MIN_BLOCKS
#define WD_LEAN_MIN_BLOCKS 8
#endif
#ifndef WD_LEAN_PIPE2
#define WD_LEAN_PIPE2 0
#endif
#ifndef WD_LEAN_NBC
#define WD_LEAN_NBC 32  // running sums kept per lane (4 KB of S per warp)
#endif
constexpr int kLeanNbc = WD_LEAN_NBC;
// product tile of the cooperative pass 2: 32 rows, stride 36 floats (16-byte
// aligned 128-bit accesses), aliasing S
constexpr int kLeanTile = 36;
constexpr int kLeanWarpFloats = kLeanNbc * 32 > 32 * kLeanTile ? kLeanNbc * 32 : 32 * kLeanTile;

// Block totals of the 4 rows a lane loads, each at ITS row's block (the
// owner's bj, shuffled), in pass 1's geometry: segment s of rows rg*4 + kk,
// two rows in flight at a time; the transpose-reduce hands lane (s, rg) the
// total of its own row rg*4 + s.  Same tree as BlockRegs::reduce.
__device__ __forceinline__ float lean_coop_block_total(const RowSet<float, 4>& prow, const RowSet<float, 4>& trow,
                                                       int bj, int s, int rg, uint64_t px, uint64_t pt) {
  float q[4];
#pragma unroll
  for (int h = 0; h < 4; h += 2) {
    Seg<float, 8, true> x[2], t[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int jb = __shfl_sync(FULL, bj, rg * 4 + h + u);
      x[u].load(prow.ptr(h + u, (int64_t)jb * 32), px);
      t[u].load(trow.ptr(h + u, (int64_t)jb * 32), pt);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float a[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = mul_rn(t[u].v[e], x[u].v[e]);
      q[h + u] = Tree<float, 8>::sum(a);
    }
  }
  return xreduce<float, 4>(q, s);
}

// block total of the own row's block at topic `base` (pairwise Tree<32> as
// ((T8 + T8) + (T8 + T8)), the sums BlockRegs::reduce forms), one segment
// of phi and theta in flight at a time
__device__ __forceinline__ float lean_own_block_total(const float* __restrict__ pown,
                                                      const float* __restrict__ town, int64_t base) {
  float q[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    Seg<float, 8, true> x, t;
    x.load(pown + base + g * 8);
    t.load(town + base + g * 8);
    float a[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = mul_rn(t.v[e], x.v[e]);
    q[g] = Tree<float, 8>::sum(a);
  }
  return add_rn(add_rn(q[0], q[1]), add_rn(q[2], q[3]));
}

template <int MINB, bool COOP2>
__global__ void __launch_bounds__(128, MINB) lda_lean_kernel(DrawParams<float> p) {
  constexpr int W = 32, E = 8, L = 4, R = 8;
  using Regs = BlockRegs<float, W, 2, MODE_LDA, 1>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int K = p.K;
  const int nb = K / W;
  const int G = nb > kLeanNbc ? (nb + kLeanNbc - 1) / kLeanNbc : 1;
  const int nbc = (nb + G - 1) / G;
  float* S = reinterpret_cast<float*>(smem_raw) + (size_t)wib * kLeanWarpFloats;
  const int s = lane % L;
  const int rg = lane / L;
  const int own = rg * L + s;  // lane-contiguous rows: lane (s, rg) loads rows rg*L + kk
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t wpb = blockDim.x >> 5;
  const uint64_t pol_x = make_l2_policy(p.l2_policy_x);
  const uint64_t pol_t = make_l2_policy(p.l2_policy_t);
  for (int64_t c = (int64_t)blockIdx.x * wpb + wib; c < n_chunks; c += (int64_t)gridDim.x * wpb) {
    const int64_t tok0 = c << 5;
    bool my_valid = tok0 + lane < n;
    int32_t my_doc = 0, my_word = 0;
    if (my_valid) {
      my_doc = p.token_doc[tok0 + lane];
      my_word = p.words[tok0 + lane];
      if (p.token_pos != nullptr) my_valid = p.token_pos[tok0 + lane] >= 0;  // run padding slot
    }
    const uint32_t vmask = __ballot_sync(FULL, my_valid);
    RowSet<float, L> prow;
    RowSet<float, L> trow;
    prow.base = reinterpret_cast<const char*>(p.phi + s * E);
    prow.ldb = (uint32_t)(p.ld_phi * sizeof(float));
    trow.base = reinterpret_cast<const char*>(p.theta + s * E);
    trow.ldb = (uint32_t)(p.ld_theta * sizeof(float));
    bool rvalid[L];
    int32_t d1 = -1;  // the document of the lane's valid rows (-1: none yet)
    bool single = true;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const int k = rg * L + kk;
      rvalid[kk] = (vmask >> k) & 1u;
      // an invalid row reads the phi row of a valid row of the same load
      // instruction (rows k ^ j*L): merged by the coalescer, sums discarded
      int src = k;
      if (!rvalid[kk]) {
#pragma unroll
        for (int j = R - 1; j >= 1; --j)
          if ((vmask >> (k ^ (j * L))) & 1u) src = k ^ (j * L);
      }
      prow.idx[kk] = (uint32_t)__shfl_sync(FULL, my_word, src);
      const int32_t dk = __shfl_sync(FULL, my_doc, k);
      trow.idx[kk] = (uint32_t)dk;
      if (rvalid[kk]) {
        if (d1 < 0) d1 = dk;
        else if (dk != d1) single = false;
      }
    }
    const int32_t own_doc = __shfl_sync(FULL, my_doc, own);
    const int32_t own_word = __shfl_sync(FULL, my_word, own);
    const bool own_valid = (vmask >> own) & 1u;

    // ---- pass 1: running block sums of the own row (every G-th kept)
    float acc = 0.f;
    if (__all_sync(FULL, single)) {
      RowSet<float, L> th1 = trow;
      th1.idx[0] = (uint32_t)(d1 < 0 ? (int32_t)trow.idx[0] : d1);
      const int pf = p.theta_prefetch;
      const char* tpf = th1.base + (uint64_t)th1.idx[0] * th1.ldb;  // the lane's theta row (segment s)
#if WD_LEAN_PIPE2
      // two blocks in flight per warp: block b+1's loads issued before block
      // b's arithmetic (needs ~100 registers: 5 CTAs per SM)
      Regs cur;
      if (nb > 0) cur.load(prow, th1, 0, pol_x, pol_t);
      for (int b = 0; b < nb; ++b) {
        Regs nxt;
        if (b + 1 < nb) nxt.load(prow, th1, (int64_t)(b + 1) * W, pol_x, pol_t);
        const float t = cur.reduce(rvalid, s, 0u);
        acc = add_rn(acc, t);
        store_s(S, b, nb, G, lane, acc);
        cur = nxt;
      }
      if (false)
#endif
#pragma unroll 2
      for (int b = 0; b < nb; ++b) {
        Regs cur;
        cur.load(prow, th1, (int64_t)b * W, pol_x, pol_t);
        // theta streams from HBM once per tile pass: fetch block b + pf's
        // segment into L2 now, so the block's loads wait on L2, not DRAM
        if (pf > 0 && b + pf < nb)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(tpf + (size_t)(b + pf) * W * sizeof(float)));
        const float t = cur.reduce(rvalid, s, 0u);
        acc = add_rn(acc, t);
        store_s(S, b, nb, G, lane, acc);
      }
    } else {  // rows from several documents: per-row theta, half a block at a time
      for (int b = 0; b < nb; ++b) {
        const float t = block_total_nd0<float, W, 2>(prow, trow, (int64_t)b * W, rvalid, s, pol_x, pol_t);
        acc = add_rn(acc, t);
        store_s(S, b, nb, G, lane, acc);
      }
    }
    __syncwarp();
    const float total = acc;

    // ---- pass 2 (own row): stop, bisection, group recompute, walk
    if constexpr (!COOP2) {
      if (own_valid) {
        uint64_t ka, kb;
        unsigned long long ekey;
        int r;
        int64_t zidx;
        token_keys<float, MODE_LDA>(p, tok0 + own, own_doc, W, ka, kb, ekey, r, zidx);
        const float stop = make_stop<float>(p, zidx, total, ka, kb, false);
        if (!(total > 0.f)) atomicMin(p.err, ekey);
        const float* pown = p.phi + (int64_t)own_word * p.ld_phi;
        const float* town = p.theta + (int64_t)own_doc * p.ld_theta;
        // the first kept running sum that exceeds stop (S is nondecreasing)
        int lo2 = 0, hi2 = nbc - 1;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (stop < S[mid * 32 + lane]) hi2 = mid; else lo2 = mid + 1;
        }
        int j;
        float prev, high;
        if (G == 1) {
          j = lo2;
          prev = j > 0 ? S[(j - 1) * 32 + lane] : 0.f;
          high = S[j * 32 + lane];
        } else {
          float run = lo2 > 0 ? S[(lo2 - 1) * 32 + lane] : 0.f;
          const int b0 = lo2 * G, b1 = min(b0 + G, nb);
          j = b1 - 1;
          prev = run;
          high = run;
          for (int bj = b0; bj < b1; ++bj) {
            const float sb = add_rn(run, lean_own_block_total(pown, town, (int64_t)bj * W));
            if (stop < sb || bj == b1 - 1) {
              j = bj;
              prev = run;
              high = sb;
              break;
            }
            run = sb;
          }
        }
        // the selected block's products, then the walk (kernels.py:268-314)
        float cur[W];
        const int64_t bb = (int64_t)j * W;
#pragma unroll
        for (int g = 0; g < W / E; ++g) {
          Seg<float, 8, true> x, t;
          x.load(pown + bb + g * E);
          t.load(town + bb + g * E);
#pragma unroll
          for (int e = 0; e < E; ++e) cur[g * E + e] = mul_rn(t.v[e], x.v[e]);
        }
        float low = j > 0 ? prev : 0.f;
        int lo = 0;
        Walk<float, W / 2>::run(cur, low, high, stop, r, lo);
        const int result = (int)bb + lo;
        p.z[zidx] = result;
        if (p.word_topic) atomicAdd(p.word_topic + (int64_t)own_word * K + result, 1);
        if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)own_doc * K + result, 1);
      }
    } else {
      // Warp-cooperative pass 2: every block this pass reads (the selected
      // group's blocks when G > 1, then the selected block) is loaded in
      // pass 1's geometry -- lane (s, rg) fetches segment s of its 4 rows,
      // each at that row's own block -- so a warp instruction covers 8 rows'
      // 128-byte lines instead of 32 lanes' lines (per-lane gathers were
      // ~20% of the L1 wavefronts at K = 1024).  Block totals come out of the
      // same tree + transpose-reduce as pass 1; the selected block's products
      // go through a shared tile [32 rows][36] (aliasing S) to their owner.
      uint64_t ka = 0, kb = 0;
      unsigned long long ekey = 0;
      int r = 0;
      int64_t zidx = 0;
      float stop = 0.f;
      if (own_valid) {
        token_keys<float, MODE_LDA>(p, tok0 + own, own_doc, W, ka, kb, ekey, r, zidx);
        stop = make_stop<float>(p, zidx, total, ka, kb, false);
        if (!(total > 0.f)) atomicMin(p.err, ekey);
      }
      int lo2 = 0, hi2 = nbc - 1;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2) >> 1;
        if (stop < S[mid * 32 + lane]) hi2 = mid; else lo2 = mid + 1;
      }
      int j;
      float prev, high;
      if (G == 1) {
        j = lo2;
        prev = j > 0 ? S[(j - 1) * 32 + lane] : 0.f;
        high = S[j * 32 + lane];
      } else {
        float run = lo2 > 0 ? S[(lo2 - 1) * 32 + lane] : 0.f;
        const int b0 = lo2 * G, b1 = min(b0 + G, nb);
        j = b1 - 1;
        prev = run;
        high = run;
        bool found = false;
        for (int gi = 0; gi < G; ++gi) {  // warp-uniform trip count
          const int bj = min(b0 + gi, b1 - 1);
          const float t = lean_coop_block_total(prow, trow, bj, s, rg, pol_x, pol_t);
          if (!found && b0 + gi < b1) {
            const float sb = add_rn(run, t);
            if (stop < sb || b0 + gi == b1 - 1) {
              found = true;
              j = b0 + gi;
              prev = run;
              high = sb;
            }
            run = sb;
          }
        }
      }
      __syncwarp();  // every lane is done with S: it becomes the product tile
      float* tile = S;
#pragma unroll
      for (int h = 0; h < L; h += 2) {
        Seg<float, 8, true> x[2], t[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int jb = __shfl_sync(FULL, j, rg * L + h + q);
          x[q].load(prow.ptr(h + q, (int64_t)jb * W), pol_x);
          t[q].load(trow.ptr(h + q, (int64_t)jb * W), pol_t);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float a[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) a[e] = mul_rn(t[q].v[e], x[q].v[e]);
          store_seg(tile + (rg * L + h + q) * kLeanTile + s * E, a);
        }
      }
      __syncwarp();
      if (own_valid) {
        float cur[W];
#pragma unroll
        for (int g = 0; g < W / E; ++g) {
          float a[8];
          load_seg_smem(a, tile + own * kLeanTile + g * E);
#pragma unroll
          for (int e = 0; e < E; ++e) cur[g * E + e] = a[e];
        }
        float low = j > 0 ? prev : 0.f;
        int lo = 0;
        Walk<float, W / 2>::run(cur, low, high, stop, r, lo);
        const int result = j * W + lo;
        p.z[zidx] = result;
        if (p.word_topic) atomicAdd(p.word_topic + (int64_t)own_word * K + result, 1);
        if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)own_doc * K + result, 1);
      }
    }
    __syncwarp();
  }
}

}  // namespace wd
