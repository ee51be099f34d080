// wd_shared.cuh -- one shared weight vector, many draws: build the butterfly
// table ONCE, then every draw is a search (the reference's sample_butterfly,
// bench.py:129-147: build_block_tables on lanes identical rows, then one
// butterfly_search per draw).
//
// With identical rows every lane's running block sums are the same, and the
// node the reference's cross-lane fetch returns at walk level `bit` is the
// pairwise-tree node of the block over the span the lane's r bit selects
// (kernels.py:268-314).  So the table is: the remnant prefix P[rem], the block
// running sums S[nb] and every block's pairwise-tree nodes, levels 0 (the
// weights) to log2(W)-1, formed with the same IEEE additions as Tree<T, W>.
// A draw then costs log2(nb) + log2(W) table reads instead of K weight reads.
#pragma once

#include "wd_draw.cuh"

namespace wd {

template <int W> struct SharedGeo {
  static constexpr int NODES = 2 * W - 2;  // levels 0 .. log2(W)-1
  // offset of level l (span 2^l): W + W/2 + ... over the lower levels
  static __host__ __device__ constexpr int off(int span) { return 2 * W - 2 * W / span; }
};

inline size_t shared_table_elems(int W, int K) {
  const int nb = K / W, rem = K % W;
  return (size_t)rem + (size_t)nb + (size_t)nb * (size_t)(2 * W - 2);
}

// layout: P[rem] | S[nb] | nodes[nb][2W-2]; one CTA
template <typename T, int W>
__global__ void __launch_bounds__(256) shared_build_kernel(const T* __restrict__ w, int K, T* __restrict__ tab) {
  using SG = SharedGeo<W>;
  const int nb = K / W, rem = K % W;
  T* P = tab;
  T* S = tab + rem;
  T* N = S + nb;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const T* x = w + rem + (size_t)b * W;
    T* nd = N + (size_t)b * SG::NODES;
    for (int t = 0; t < W; ++t) nd[t] = x[t];
    int prev = 0;
    for (int span = 2; span < W; span *= 2) {
      const int o = SG::off(span);
      for (int i = 0; i < W / span; ++i) nd[o + i] = add_rn(nd[prev + 2 * i], nd[prev + 2 * i + 1]);
      prev = o;
    }
    S[b] = add_rn(nd[prev], nd[prev + 1]);  // block total, Tree<T, W>::sum
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // sequential remnant prefix, then block running sums
    T s = T(0);
    for (int t = 0; t < rem; ++t) {
      s = add_rn(s, w[t]);
      P[t] = s;
    }
    for (int b = 0; b < nb; ++b) {
      s = add_rn(s, S[b]);
      S[b] = s;
    }
  }
}

template <typename T, int W>
__global__ void __launch_bounds__(256) shared_draw_kernel(DrawParams<T> p, const T* __restrict__ tab) {
  using SG = SharedGeo<W>;
  const int K = p.K, nb = K / W, rem = K % W;
  const T* P = tab;
  const T* S = tab + rem;
  const T* N = S + nb;
  const T prem = rem > 0 ? P[rem - 1] : T(0);
  const T total = nb > 0 ? S[nb - 1] : prem;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n_tokens;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t ka, kb;
    unsigned long long ekey;
    int r;
    int64_t zidx;
    token_keys<T, MODE_ROWS>(p, i, 0, W, ka, kb, ekey, r, zidx);
    const T stop = make_stop<T>(p, zidx, total, ka, kb, true);
    if (!(total > T(0))) atomicMin(p.err, ekey);
    // block bisection (kernels.py:337-346)
    int lo2 = 0, hi2 = nb > 0 ? nb - 1 : 0;
    while (lo2 < hi2) {
      const int mid = (lo2 + hi2) >> 1;
      if (stop < __ldg(S + mid)) hi2 = mid;
      else lo2 = mid + 1;
    }
    const int j = lo2;
    const int64_t bb = (int64_t)rem + (int64_t)j * W;
    T prev = bb == 0 ? T(0) : (j > 0 ? __ldg(S + j - 1) : prem);
    T high = nb > 0 ? __ldg(S + j) : T(0);
    const bool fallback = bb > 0 && stop < prev && total > T(0);
    int result = 0;
    if (nb > 0 && !fallback) {  // the walk (kernels.py:268-314) on the stored nodes
      const T* nd = N + (size_t)j * SG::NODES;
      T low = prev;
      int lo = 0;
#pragma unroll
      for (int bit = W / 2; bit >= 1; bit >>= 1) {
        const int o = SG::off(bit);
        const T cmp = (r & bit) ? sub_rn(high, __ldg(nd + o + (lo + bit) / bit)) : add_rn(low, __ldg(nd + o + lo / bit));
        if (stop < cmp) {
          high = cmp;
        } else {
          low = cmp;
          lo += bit;
        }
      }
      result = (int)bb + lo;
    }
    if (fallback) {  // linear remnant fallback (kernels.py:354-361)
      for (int t = 0; t < rem; ++t)
        if (stop < __ldg(P + t)) {
          result = t;
          break;
        }
    }
    p.z[zidx] = result;
  }
}

}  // namespace wd
