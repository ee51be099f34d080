// wd_device.cuh -- device building blocks shared by the sm_100a kernels.
//
// All floating-point arithmetic goes through the *_rn intrinsics below so that
// no FMA contraction can change a bit (the file is also compiled with
// -fmad=false); nothing here flushes subnormals (never --use_fast_math).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "warpdraw_b200.h"

namespace wd {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// nextafter(x, 0) for finite x > 0 (kernels.py:99: np.nextafter(sums, 0))
__device__ __forceinline__ float next_below(float x) { return __int_as_float(__float_as_int(x) - 1); }
__device__ __forceinline__ double next_below(double x) {
  return __longlong_as_double(__double_as_longlong(x) - 1);
}

// ------------------------------------------------------------------ u stream
// rng.py:16-40 (SplitMix64 key folding) and rng.py:101-122 (first output of
// xoshiro256** seeded by SplitMix64; only state[1] feeds that output).
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) { return fin64(x + GAMMA); }
__host__ __device__ __forceinline__ uint64_t unit_bits(uint64_t h) {
  uint64_t x = fin64(h + 2ull * GAMMA) * 5ull;
  x = (x << 7) | (x >> 57);
  return (x * 9ull) >> 11;  // 53 significant bits
}
// units_for(seed, a, b) as the 53-bit integer; u = bits * 2^-53
__device__ __forceinline__ uint64_t unit_bits2(uint64_t seed, uint64_t a, uint64_t b) {
  return unit_bits(mix64(mix64(seed ^ a) ^ b));
}
__device__ __forceinline__ uint64_t unit_bits1(uint64_t seed, uint64_t a) {
  return unit_bits(mix64(seed ^ a));
}
// fl_T(u): u is exact in binary64; the float conversion of bits*2^-53 equals
// RN(bits)*2^-53 because the scale is a power of two and the result is normal.
template <typename T> __device__ __forceinline__ T unit_to(uint64_t bits);
template <> __device__ __forceinline__ float unit_to<float>(uint64_t bits) {
  return __fmul_rn(__ull2float_rn(bits), 0x1p-53f);
}
template <> __device__ __forceinline__ double unit_to<double>(uint64_t bits) {
  return __dmul_rn(__ull2double_rn(bits), 0x1p-53);
}
template <typename T> __device__ __forceinline__ T from_double(double u);
template <> __device__ __forceinline__ float from_double<float>(double u) { return __double2float_rn(u); }
template <> __device__ __forceinline__ double from_double<double>(double u) { return u; }

// Philox4x32-10 (Salmon et al., SC'11; Random123's constants): one 128-bit
// block for a 128-bit counter under a 64-bit key.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                               uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Opt-in Philox4x32-10 stops (WD_STOPS_PHILOX): counter (doc, key), key = seed.
// Not reference-parity; 53-bit unit from 2 words.
__device__ __forceinline__ uint64_t philox_bits(uint64_t seed, uint64_t a, uint64_t b) {
  const uint4 r = philox4x32_10((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32), (uint32_t)seed,
                                (uint32_t)(seed >> 32));
  return ((uint64_t)r.x << 21) | (uint64_t)(r.y >> 11);
}

// ------------------------------------------------------------- L2 policies
// 0 = evict_normal, 1 = evict_last (phi: keep the gathered rows resident),
// 2 = evict_first (theta / weights: streamed once).
__device__ __forceinline__ uint64_t make_l2_policy(int kind) {
  uint64_t pol;
  if (kind == 1) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else if (kind == 2) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// ------------------------------------------------------------- segment loads
// E consecutive elements starting at p.  VEC: p is aligned to min(16, E*sizeof(T)).
template <typename T, int E, bool VEC> struct Seg {
  T v[E];
  __device__ __forceinline__ void load(const T* __restrict__ p) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = __ldg(p + e);
  }
  __device__ __forceinline__ void load(const T* __restrict__ p, uint64_t) { load(p); }
  __device__ __forceinline__ void load_na(const T* __restrict__ p, uint64_t pol) { load(p, pol); }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = T(0);
  }
};
template <> struct Seg<float, 4, true> {
  float v[4];
  __device__ __forceinline__ void load(const float* __restrict__ p) {
    float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  // 128-bit read-only load carrying an L2 eviction-priority policy
  __device__ __forceinline__ void load(const float* __restrict__ p, uint64_t pol) {
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p), "l"(pol));
  }
  // ... that does not allocate in L1 (rows streamed once per chunk)
  __device__ __forceinline__ void load_na(const float* __restrict__ p, uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
        : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void zero() { v[0] = v[1] = v[2] = v[3] = 0.f; }
};
// 256-bit segment (sm_100 LDG.E.256): 8 fp32 topics per lane, 32-byte aligned
template <> struct Seg<float, 8, true> {
  float v[8];
  __device__ __forceinline__ void load(const float* __restrict__ p) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
  }
  __device__ __forceinline__ void load(const float* __restrict__ p, uint64_t pol) {
    asm("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void load_na(const float* __restrict__ p, uint64_t pol) { load(p, pol); }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = 0.f;
  }
};
template <> struct Seg<float, 2, true> {
  float v[2];
  __device__ __forceinline__ void load(const float* __restrict__ p) {
    float2 t = __ldg(reinterpret_cast<const float2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
  __device__ __forceinline__ void load(const float* __restrict__ p, uint64_t) { load(p); }
  __device__ __forceinline__ void load_na(const float* __restrict__ p, uint64_t pol) { load(p, pol); }
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.f; }
};
// 4 fp64 = one 256-bit load (the fp64 vector path requires 32-byte alignment)
template <> struct Seg<double, 4, true> {
  double v[4];
  __device__ __forceinline__ void load(const double* __restrict__ p) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  }
  __device__ __forceinline__ void load(const double* __restrict__ p, uint64_t pol) {
    asm("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "l"(p), "l"(pol));
  }
  __device__ __forceinline__ void load_na(const double* __restrict__ p, uint64_t pol) { load(p, pol); }
  __device__ __forceinline__ void zero() { v[0] = v[1] = v[2] = v[3] = 0.0; }
};
template <> struct Seg<double, 2, true> {
  double v[2];
  __device__ __forceinline__ void load(const double* __restrict__ p) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = a.x; v[1] = a.y;
  }
  __device__ __forceinline__ void load(const double* __restrict__ p, uint64_t) { load(p); }
  __device__ __forceinline__ void load_na(const double* __restrict__ p, uint64_t pol) { load(p, pol); }
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.0; }
};

// Balanced aligned pairwise tree over N consecutive values (N power of two):
// exactly the sums the reference's log2(W) shuffle_xor sets produce
// (kernels.py:206-224; butterfly.py:58-75 closed form).
template <typename T, int N> struct Tree {
  static __device__ __forceinline__ T sum(const T* x) {
    return add_rn(Tree<T, N / 2>::sum(x), Tree<T, N / 2>::sum(x + N / 2));
  }
};
template <typename T> struct Tree<T, 1> {
  static __device__ __forceinline__ T sum(const T* x) { return x[0]; }
};

// Geometry of the vector-widened butterfly for a W-topic block:
//   E lanes' worth of consecutive topics per lane (one 16-byte vector for fp32),
//   L = W/E lanes cover one document row of the block,
//   R = 32/L document rows per warp-wide load instruction.
template <int W> struct Geo {
  static constexpr int E = W >= 4 ? 4 : W;
  static constexpr int L = W / E;
  static constexpr int R = 32 / L;
  static_assert(L >= 1 && L <= 32 && (L & (L - 1)) == 0, "W must be a power of two in [2, 128]");
};
// ... by vector level: V = 2 widens the lane segment to 8 fp32 topics (one
// 256-bit load), so L halves: half the loads, shuffles and selects per block.
template <int W, int V> struct GeoV {
  static constexpr int E = (V == 2 && W >= 8) ? 8 : Geo<W>::E;
  static constexpr int L = W / E;
  static constexpr int R = 32 / L;
};

}  // namespace wd
