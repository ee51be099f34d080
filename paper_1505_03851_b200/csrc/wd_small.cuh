// wd_small.cuh -- the LDA draw at small K (configs[2]: K = 200): fp32, W = 32,
// 256-bit lane segments, K = 8 * RM + 32 * NB with NB <= 8, RM <= 3.
//
// Same arithmetic as bfly_kernel<float, 32, 2, MODE_LDA, 1, KV_SMALL> and the
// reference's draw_z_butterfly (kernels.py:487-539): remnant running sums
// first (kernels.py:199-205), the pairwise tree per W-topic block
// (kernels.py:206-224), sequential running block sums, stop =
// fl(total * fl(u)), block bisection, the add-or-subtract walk
// (kernels.py:268-314) and the remnant fallback (kernels.py:354-361).
//
// At K = 200 a token's row is only 800 bytes: ncu on the general kernel
// (profiles/ncu_r02_kernels.md) shows the pass-1 loop at ~1/3 of the stall
// samples and shared-memory wavefronts at 42% of the L1 traffic -- the
// remnant tile, the running-sum array S and the cooperative pass-2 reload
// tile.  Here:
//
//   * the NB running sums live in registers (NB is a template parameter);
//   * the walk's first two levels read the selected block's 8-topic segment
//     totals T8 (the tree nodes Tree<16> and Tree<8> are sums of them), which
//     pass 1 stashes in shared memory with one 128-bit store per lane per
//     block (each lane already holds the T8 of its segment for its 4 rows);
//     levels 4, 2, 1 need only the live segment's 8 products: one 256-bit
//     phi and one theta load of the own row instead of the whole block;
//   * the remnant (RM segments) is the own row's products, gathered per lane
//     with 256-bit loads and summed in registers -- no remnant tile;
//   * chunks whose lanes' rows are not single-document (tiles without run
//     padding, chunk tails) take per-row theta loads in halves.
// Shared memory: the T8 stash, [block][segment][row] with a 40-float segment
// stride (the 128-bit stores of a quarter warp hit 8 distinct bank groups),
// NB * 4 * 40 floats per warp.
#pragma once

#include "wd_draw.cuh"

namespace wd {

#ifndef WD_SMALL_GROUP  // blocks whose loads may be in flight together (the opaque dependency every GROUP blocks)
#define WD_SMALL_GROUP 1
#endif
#ifndef WD_SMALL_EARLY
#define WD_SMALL_EARLY 0  // measured at K = 200: 14.8 vs 13.6 ms (register pressure)
#endif
#ifndef WD_SMALL_LDA_MIN_BLOCKS  // measured at K = 200: 5 / 6 / 7 / 8 CTAs per SM -> 13.85 / 13.58 / 13.82 / 15.07 ms
#define WD_SMALL_LDA_MIN_BLOCKS 6
#endif

template <int NB, int RM>
__global__ void __launch_bounds__(128, WD_SMALL_LDA_MIN_BLOCKS) lda_small_kernel(DrawParams<float> p) {
  constexpr int W = 32, E = 8, L = 4, R = 8;
  constexpr int REM = 8 * RM;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  constexpr int TS = 40;  // floats per (block, segment) row of the stash
  float* T8 = reinterpret_cast<float*>(smem_raw) + (size_t)wib * NB * 4 * TS;  // [b][seg][row]
  const int K = p.K;
  const int s = lane % L;
  const int rg = lane / L;
  const int own = rg * L + s;
  const int64_t n = p.n_tokens;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t wpb = blockDim.x >> 5;
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
    prow.base = reinterpret_cast<const char*>(p.phi + REM + s * E);
    prow.ldb = (uint32_t)(p.ld_phi * sizeof(float));
    int32_t d1 = -1;
    bool single = true;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
      const int k = rg * L + kk;
      const bool rv = (vmask >> k) & 1u;
      int src = k;  // invalid rows read a valid row of the same load instruction
      if (!rv) {
#pragma unroll
        for (int j = R - 1; j >= 1; --j)
          if ((vmask >> (k ^ (j * L))) & 1u) src = k ^ (j * L);
      }
      prow.idx[kk] = (uint32_t)__shfl_sync(FULL, my_word, src);
      const int32_t dk = __shfl_sync(FULL, my_doc, k);
      if (rv) {
        if (d1 < 0) d1 = dk;
        else if (dk != d1) single = false;
      }
    }
    const int32_t own_doc = __shfl_sync(FULL, my_doc, own);
    const int32_t own_word = __shfl_sync(FULL, my_word, own);
    const bool own_valid = (vmask >> own) & 1u;

    // remnant of the own row: its products, summed sequentially (re-read
    // for the rare fallback scan instead of being kept live)
    float acc = 0.f;
#pragma unroll
    for (int g = 0; g < RM; ++g) {
      Seg<float, 8, true> x, t;
      x.load(p.phi + (int64_t)own_word * p.ld_phi + g * 8);
      t.load(p.theta + (int64_t)own_doc * p.ld_theta + g * 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = add_rn(acc, mul_rn(t.v[e], x.v[e]));
    }
    const float prem = acc;

    // the own token's keys and u (or explicit stop) before pass 1: the hash
    // chain and the key loads overlap the block loads (WD_SMALL_EARLY)
    uint64_t ka = 0, kb = 0;
    unsigned long long ekey = 0;
    int r = 0;
    int64_t zidx = 0;
    float pre = 0.f;
    if (WD_SMALL_EARLY && own_valid) {
      token_keys<float, MODE_LDA>(p, tok0 + own, own_doc, W, ka, kb, ekey, r, zidx);
      pre = stop_pre<float>(p, zidx, ka, kb, false);
    }

    // ---- pass 1: block totals of the own row, T8 stash, running sums in registers
    float S[NB];
    const bool fast = __all_sync(FULL, single);
    // the lane's document (any valid one when its rows are all padding)
    const float* tseg = p.theta + REM + s * E + (int64_t)(d1 < 0 ? my_doc : d1) * p.ld_theta;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      // block b's loads depend on block b-1's sum through an opaque runtime
      // zero: one block in flight per warp, so the unrolled loop keeps the
      // register budget of one block
      const int64_t col = (int64_t)b * W + ((b % WD_SMALL_GROUP) == 0 ? (int64_t)(__float_as_uint(acc) & p.opaque_zero) : 0);
      float q[L];
      if (fast) {
        // all five loads of the block in flight together: every consumer
        // depends on every load through the opaque zero (BlockRegs::join),
        // so ptxas cannot interleave them with the arithmetic
        BlockRegs<float, W, 2, MODE_LDA, 1> blk;
#pragma unroll
        for (int kk = 0; kk < L; ++kk) blk.x[kk].load(prow.ptr(kk, col));
        blk.th[0].load(tseg + col);
        blk.join(p.opaque_zero);
#pragma unroll
        for (int kk = 0; kk < L; ++kk) {
          float a[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) a[e] = mul_rn(blk.th[0].v[e], blk.x[kk].v[e]);
          q[kk] = Tree<float, 8>::sum(a);
        }
      } else {
#pragma unroll
        for (int h = 0; h < L; h += 2) {
          Seg<float, 8, true> x[2], th[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {  // per-row theta (rows of several documents)
            const int32_t du = __shfl_sync(FULL, my_doc, rg * L + h + u);
            x[u].load(prow.ptr(h + u, col));
            th[u].load(p.theta + REM + s * E + (int64_t)du * p.ld_theta + col);
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float a[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) a[e] = mul_rn(th[u].v[e], x[u].v[e]);
            q[h + u] = Tree<float, 8>::sum(a);
          }
        }
      }
      // segment totals of this lane's 4 rows (rows rg*4 .. rg*4+3, segment s)
      *reinterpret_cast<float4*>(T8 + (b * 4 + s) * TS + rg * L) = make_float4(q[0], q[1], q[2], q[3]);
      acc = add_rn(acc, xreduce<float, L>(q, s));
      S[b] = acc;
    }
    const float total = acc;
    __syncwarp();

    // ---- pass 2 (own row)
    if (own_valid) {
      if (!WD_SMALL_EARLY) {
        token_keys<float, MODE_LDA>(p, tok0 + own, own_doc, W, ka, kb, ekey, r, zidx);
        pre = stop_pre<float>(p, zidx, ka, kb, false);
      }
      const float stop = stop_finish<float>(p, pre, total);
      const bool live = total > 0.f;
      if (!live) atomicMin(p.err, ekey);
      int j = 0;  // first block whose running sum exceeds stop (nb - 1 if none)
#pragma unroll
      for (int b = 0; b + 1 < NB; ++b) j += (S[b] <= stop) ? 1 : 0;
      float prev = prem, high = 0.f;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (b == j) high = S[b];
        if (b + 1 == j) prev = S[b];
      }
      const float* pown = p.phi + (int64_t)own_word * p.ld_phi;
      const float* town = p.theta + (int64_t)own_doc * p.ld_theta;
      const int bb = REM + j * W;
      if (bb == 0) prev = 0.f;
      const bool fallback = bb > 0 && stop < prev && live;
      int result = 0;
      if (!fallback) {
        // levels 16 and 8 from the stashed segment totals (Tree<16> of a
        // half = the sum of its two T8; Tree<8> of a quarter = its T8)
        float t8[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) t8[g] = T8[(j * 4 + g) * TS + own];
        float low = prev;
        int seg;
        {
          const float cmp = (r & 16) ? sub_rn(high, add_rn(t8[2], t8[3])) : add_rn(low, add_rn(t8[0], t8[1]));
          const bool less = stop < cmp;
          if (less) high = cmp; else low = cmp;
          seg = less ? 0 : 2;
        }
        {
          const float lo8 = seg == 0 ? t8[0] : t8[2];
          const float hi8 = seg == 0 ? t8[1] : t8[3];
          const float cmp = (r & 8) ? sub_rn(high, hi8) : add_rn(low, lo8);
          const bool less = stop < cmp;
          if (less) high = cmp; else low = cmp;
          seg += less ? 0 : 1;
        }
        // levels 4, 2, 1 on the live segment's 8 products (own row)
        float cur[8];
        {
          Seg<float, 8, true> x, t;
          x.load(pown + bb + seg * 8);
          t.load(town + bb + seg * 8);
#pragma unroll
          for (int e = 0; e < 8; ++e) cur[e] = mul_rn(t.v[e], x.v[e]);
        }
        int lo = 0;
        Walk<float, 4>::run(cur, low, high, stop, r, lo);
        result = bb + seg * 8 + lo;
      } else {
        // linear remnant fallback: first t with stop < P[t] (same additions)
        float a2 = 0.f;
        int t = 0;
#pragma unroll
        for (int g = 0; g < RM; ++g) {
          Seg<float, 8, true> x, th;
          x.load(pown + g * 8);
          th.load(town + g * 8);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            a2 = add_rn(a2, mul_rn(th.v[e], x.v[e]));
            t += (a2 <= stop) ? 1 : 0;
          }
        }
        if (t < REM) result = t;
      }
      p.z[zidx] = result;
      if (p.word_topic) atomicAdd(p.word_topic + (int64_t)own_word * K + result, 1);
      if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)own_doc * K + result, 1);
    }
    __syncwarp();
  }
}

}  // namespace wd
