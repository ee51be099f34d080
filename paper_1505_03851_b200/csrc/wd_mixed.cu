// wd_mixed.cu -- the LDA draw with float32 theta and float64 phi.
//
// The reference forms every product as theta_local[..] * phi[..] in numpy and
// stores it into a float32 table (kernels.py:209 into a RegisterArray of
// theta's dtype; kernels.py:391 `(row * phi[w]).astype(dtype)`), so with a
// float64 phi each product is fl32(fl64(theta * phi)) -- rounded twice.  The
// float32 kernels would need phi cast to float32 first, which rounds the
// other way for ~25% of products.  This path computes the product exactly as
// the reference does (the float32 theta value is exact in float64) and runs
// the rest of the draw in float32, one thread per token:
//
//   WD_BUTTERFLY  remnant running sums (kernels.py:199-205), one pairwise
//                 Tree<W> per W-topic block, running block sums; stop; the
//                 first block whose running sum exceeds it (== the
//                 reference's bisection, the sums are nondecreasing) found by
//                 re-forming the same sums; the add-or-subtract walk on that
//                 block (Walk<float, W/2>); the remnant fallback.
//   WD_PREFIX     the sequential prefix (np.cumsum) and the first index
//                 whose prefix exceeds stop (== binary_search /
//                 _prefix_binary_search on a nondecreasing table).
//
// Where the reference rounds differs by kernel: draw_z_basic rounds every
// product to float32 and sums in float32 (kernels.py:391-392); the warp
// kernels (transposed, butterfly) store the block products into float32
// registers but add each REMNANT product (the K mod W leading topics)
// unrounded to the float32 sum in float64 and round the sum
// (kernels.py:162-165, 199-203).
//
// Rare-path code (the reference's own run_gibbs never mixes dtypes): simple
// and exact rather than fast -- two passes over the products per token.
#include <cuda_runtime.h>

#include <cstdint>

#include "warpdraw_b200.h"
#include "wd_draw.cuh"

namespace wd {

int device_sm_count();
void set_last_cuda_error(cudaError_t e);

__device__ __forceinline__ float prod_mixed(const float* th, const double* ph, int64_t k) {
  return __double2float_rn(__dmul_rn((double)th[k], ph[k]));
}
// a remnant step of the warp kernels: `sums = (sums + prod).astype(dtype)`
// with prod the float64 product itself (kernels.py:162-165, 199-203): one
// rounding of the float64 sum, not of the product
__device__ __forceinline__ float add_rem_mixed(float acc, const float* th, const double* ph, int64_t k) {
  return __double2float_rn(__dadd_rn((double)acc, __dmul_rn((double)th[k], ph[k])));
}

template <int W, bool BFLY>
__global__ void __launch_bounds__(128) lda_mixed_kernel(DrawParams<float> p) {
  const double* phi64 = reinterpret_cast<const double*>(p.phi);
  const int K = p.K;
  const int rem = K % W, nb = K / W;
  for (int64_t tok = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; tok < p.n_tokens;
       tok += (int64_t)gridDim.x * blockDim.x) {
    if (p.token_pos != nullptr && p.token_pos[tok] < 0) continue;  // run padding slot
    const int32_t doc = p.token_doc[tok];
    const int32_t word = p.words[tok];
    const float* th = p.theta + (int64_t)doc * p.ld_theta;
    const double* ph = phi64 + (int64_t)word * p.ld_phi;
    uint64_t ka, kb;
    unsigned long long ekey;
    int r;
    int64_t zidx;
    token_keys<float, MODE_LDA>(p, tok, doc, W, ka, kb, ekey, r, zidx);
    // warp kernels (butterfly, transposed = master keys) vs draw_z_basic
    const bool warp_rem = BFLY || p.key_rule == WD_KEYS_MASTER;
    auto step = [&](float a, int64_t t) {
      return (warp_rem && t < rem) ? add_rem_mixed(a, th, ph, t) : add_rn(a, prod_mixed(th, ph, t));
    };
    // pass A: the total, in the reference's order
    float acc = 0.f;
    for (int t = 0; t < (BFLY ? rem : K); ++t) acc = step(acc, t);
    const float prem = acc;
    if (BFLY) {
      for (int b = 0; b < nb; ++b) {
        float c[W];
#pragma unroll
        for (int e = 0; e < W; ++e) c[e] = prod_mixed(th, ph, rem + (int64_t)b * W + e);
        acc = add_rn(acc, Tree<float, W>::sum(c));
      }
    }
    const float total = acc;
    const float stop = make_stop<float>(p, zidx, total, ka, kb, false);
    const bool live = total > 0.f;
    if (!live) atomicMin(p.err, ekey);
    int result = 0;
    if (!BFLY) {
      // first index whose running sum exceeds stop (K - 1 if none)
      float run = 0.f;
      result = K - 1;
      for (int t = 0; t < K; ++t) {
        run = step(run, t);
        if (stop < run) { result = t; break; }
      }
    } else {
      // pass B: the first block whose running sum exceeds stop (nb - 1 if none)
      float run = prem, prev = prem, high = 0.f;
      int j = nb - 1;
      for (int b = 0; b < nb; ++b) {
        float c[W];
#pragma unroll
        for (int e = 0; e < W; ++e) c[e] = prod_mixed(th, ph, rem + (int64_t)b * W + e);
        const float sb = add_rn(run, Tree<float, W>::sum(c));
        if (stop < sb || b == nb - 1) {
          j = b;
          prev = run;
          high = sb;
          break;
        }
        run = sb;
      }
      const int bb = rem + j * W;
      if (bb == 0) prev = 0.f;
      const bool fallback = bb > 0 && stop < prev && live;
      if (nb > 0 && !fallback) {
        float c[W];
#pragma unroll
        for (int e = 0; e < W; ++e) c[e] = prod_mixed(th, ph, bb + e);
        float low = prev;
        int lo = 0;
        Walk<float, W / 2>::run(c, low, high, stop, r, lo);
        result = bb + lo;
      }
      if (fallback || (nb == 0 && live)) {
        float a2 = 0.f;
        for (int t = 0; t < rem; ++t) {
          a2 = step(a2, t);
          if (stop < a2) { result = t; break; }
        }
      }
    }
    p.z[zidx] = result;
    if (p.word_topic) atomicAdd(p.word_topic + (int64_t)word * K + result, 1);
    if (p.doc_topic) atomicAdd(p.doc_topic + (int64_t)doc * K + result, 1);
  }
}

template <int W, bool BFLY>
static int launch_mixed_w(const DrawParams<float>& p, cudaStream_t st) {
  int64_t grid = (p.n_tokens + 127) / 128;
  const int64_t cap = (int64_t)device_sm_count() * 16;
  if (grid > cap) grid = cap;
  if (grid <= 0) return WD_OK;
  lda_mixed_kernel<W, BFLY><<<(int)grid, 128, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

template <bool BFLY>
static int launch_mixed_b(int W, const DrawParams<float>& p, cudaStream_t st) {
  switch (W) {
    case 2: return launch_mixed_w<2, BFLY>(p, st);
    case 4: return launch_mixed_w<4, BFLY>(p, st);
    case 8: return launch_mixed_w<8, BFLY>(p, st);
    case 16: return launch_mixed_w<16, BFLY>(p, st);
    case 32: return launch_mixed_w<32, BFLY>(p, st);
    case 64: return launch_mixed_w<64, BFLY>(p, st);
    default: return WD_ERR_UNSUPPORTED;
  }
}

// variant WD_BUTTERFLY or WD_PREFIX (the basic / transposed prefix table);
// p.phi points at float64 rows (ld_phi in doubles)
int launch_draw_mixed(int variant, int W, const DrawParams<float>& p, cudaStream_t st) {
  return variant == WD_BUTTERFLY ? launch_mixed_b<true>(W, p, st) : launch_mixed_b<false>(W, p, st);
}

}  // namespace wd
