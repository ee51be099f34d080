// theta_probe.cu -- microbenchmark for the K = 4096 LDA draw's pass 1 with
// theta streamed from HBM (configs[4]): does reading each chunk's theta
// rows from DRAM (a document's row is read by one chunk per vocabulary tile)
// cost the L2-bound phi gather its rate, and does an L2 prefetch win it back?
//
// Pattern (tools/stage_probe.cu's V0, the lean kernel's geometry): a 40 MB
// L2-resident phi slice of K = 4096 fp32 rows; a warp takes chunks of 32
// random rows and streams every row block by block (W = 32 topics = 128 B,
// lane (s, rg) loads segment s of rows rg*4 + kk with one 256-bit load),
// multiplying by the theta segment of the chunk's document (lane groups 0-3
// document 2c, 4-7 document 2c + 1: ~2 documents per chunk as at configs[4]).
//
//   resident   theta rows from a 16 MB table (L2 hits; the old probe)
//   stream     theta rows 2c, 2c + 1 of a 4 GB table (each read once: DRAM)
//   +ef        theta loads with an L2 evict_first policy
//   +pfN       prefetch.global.L2 of the theta segment N blocks ahead
//   +bulk      cp.async.bulk.prefetch.L2 of the next chunk's two theta rows
//              (32 KB) at chunk start
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o theta_probe theta_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int K = 4096;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ void ld_v8(float (&a)[8], const float* p) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7])
               : "l"(p));
}
__device__ __forceinline__ void ld_v8_pol(float (&a)[8], const float* p, uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7])
               : "l"(p), "l"(pol));
}

// MODE 0 resident, 1 stream; EF evict_first on theta; PF prefetch distance
// in blocks (0 off); BULK next-chunk bulk prefetch
template <int MODE, bool EF, int PF, bool BULK>
__global__ void __launch_bounds__(128, 8) probe(const float* __restrict__ phi, const float* __restrict__ theta,
                                                const int* __restrict__ rows, int n_chunks, int n_theta,
                                                float* out) {
  const int lane = threadIdx.x & 31, s = lane & 3, rg = lane >> 2;
  const int wpb = blockDim.x >> 5;
  uint64_t pol = 0;
  if (EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  float acc = 0.f;
  const int cs = gridDim.x * wpb;
  for (int c = blockIdx.x * wpb + (threadIdx.x >> 5); c < n_chunks; c += cs) {
    const int my = rows[c * 32 + lane];
    uint32_t r[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) r[kk] = __shfl_sync(FULL, my, rg * 4 + kk);
    int doc;
    if (MODE == 0) doc = (2 * c + (rg >> 2)) & 1023;
    else if (MODE == 1) doc = (2 * c + (rg >> 2)) % n_theta;
    else if (MODE == 2) {  // stream, the 8 CTAs an SM holds (blockIdx j + 148 i) on adjacent rows
      const int k = c / cs, per = gridDim.x / 8;
      const int blk = (blockIdx.x % per) * 8 + blockIdx.x / per;
      doc = (2 * ((k * gridDim.x + blk) * wpb + (threadIdx.x >> 5)) + (rg >> 2)) % n_theta;
    } else if (MODE == 3) doc = (2 * c + (rg >> 2)) % 4096;  // 64 MB table: mostly L2 hits, 32 pages
    else if (MODE == 4) doc = ((2 * c + (rg >> 2)) & 1023) * 16;  // 16 MB of rows over 256 MB (128 pages)
    else if (MODE == 5) doc = ((2 * c + (rg >> 2)) & 1023) * 4;   // 16 MB of rows over 64 MB (32 pages)
    else if (MODE == 6) doc = (2 * c + (rg >> 2)) & 2047;         // 32 MB table
    else if (MODE == 7) doc = c % n_theta;                        // stream, one document per chunk
    else doc = (2 * (c >> 1) + (rg >> 2)) % n_theta;              // stream, a row pair shared by 2 chunks

    const float* th = theta + (size_t)doc * K + s * 8;
    if (BULK && lane < 2) {
      const int nc = c + cs;
      if (nc < n_chunks) {
        const float* nrow = theta + (size_t)((2 * nc + lane) % n_theta) * K;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nrow), "r"(K * 4) : "memory");
      }
    }
    float run = 0.f;
#pragma unroll 2
    for (int b = 0; b < K / 32; ++b) {
      float x[4][8], t[8];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ld_v8(x[kk], phi + (size_t)r[kk] * K + b * 32 + s * 8);
      if (EF) ld_v8_pol(t, th + b * 32, pol);
      else ld_v8(t, th + b * 32);
      if (PF > 0 && b + PF < K / 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(th + (b + PF) * 32));
      // PF < 0: every -PF blocks, one bulk L2 prefetch per document of the
      // theta span -PF blocks ahead (-PF x 128 contiguous bytes)
      if (PF < 0 && (b % -PF) == 0 && (lane & 15) == 0 && b + -PF < K / 32)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(th + (b + -PF) * 32), "r"(-PF * 128)
                     : "memory");
      if (PF < 0 && b == 0 && (lane & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(th), "r"(-PF * 128) : "memory");
      float q[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a += x[kk][e] * t[e];
        q[kk] = a;
      }
      float v = (s & 1) ? q[1] + __shfl_xor_sync(FULL, q[0], 1) : q[0] + __shfl_xor_sync(FULL, q[1], 1);
      float w = (s & 1) ? q[3] + __shfl_xor_sync(FULL, q[2], 1) : q[2] + __shfl_xor_sync(FULL, q[3], 1);
      float z = (s & 2) ? w + __shfl_xor_sync(FULL, v, 2) : v + __shfl_xor_sync(FULL, w, 2);
      run += z;
    }
    acc += run;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// theta through a per-lane cp.async ring: lane copies its own 32-byte
// theta segment of block b + D into slot (b + D) % (D + 1) (no registers
// held while the copy is in flight) and reads block b's from shared memory
template <int MODE, int D>
__global__ void __launch_bounds__(128, 8) probe_ring(const float* __restrict__ phi, const float* __restrict__ theta,
                                                     const int* __restrict__ rows, int n_chunks, int n_theta,
                                                     float* out) {
  __shared__ __align__(16) float ring[4][D + 1][32][8];
  const int lane = threadIdx.x & 31, s = lane & 3, rg = lane >> 2, wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  float acc = 0.f;
  const int cs = gridDim.x * wpb;
  auto copy = [&](const float* src, int slot) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&ring[wib][slot][lane][0]);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(src + 4) : "memory");
  };
  for (int c = blockIdx.x * wpb + wib; c < n_chunks; c += cs) {
    const int my = rows[c * 32 + lane];
    uint32_t r[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) r[kk] = __shfl_sync(FULL, my, rg * 4 + kk);
    const int doc = MODE == 0 ? ((2 * c + (rg >> 2)) & 1023) : ((2 * c + (rg >> 2)) % n_theta);
    const float* th = theta + (size_t)doc * K + s * 8;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      copy(th + d * 32, d);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float run = 0.f;
#pragma unroll 2
    for (int b = 0; b < K / 32; ++b) {
      float x[4][8], t[8];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ld_v8(x[kk], phi + (size_t)r[kk] * K + b * 32 + s * 8);
      if (b + D < K / 32) copy(th + (b + D) * 32, (b + D) % (D + 1));
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");
      const float4 t0 = *reinterpret_cast<const float4*>(&ring[wib][b % (D + 1)][lane][0]);
      const float4 t1 = *reinterpret_cast<const float4*>(&ring[wib][b % (D + 1)][lane][4]);
      t[0] = t0.x; t[1] = t0.y; t[2] = t0.z; t[3] = t0.w; t[4] = t1.x; t[5] = t1.y; t[6] = t1.z; t[7] = t1.w;
      float q[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a += x[kk][e] * t[e];
        q[kk] = a;
      }
      float v = (s & 1) ? q[1] + __shfl_xor_sync(FULL, q[0], 1) : q[0] + __shfl_xor_sync(FULL, q[1], 1);
      float w = (s & 1) ? q[3] + __shfl_xor_sync(FULL, q[2], 1) : q[2] + __shfl_xor_sync(FULL, q[3], 1);
      float z = (s & 2) ? w + __shfl_xor_sync(FULL, v, 2) : v + __shfl_xor_sync(FULL, w, 2);
      run += z;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    acc += run;
  }
  if (acc == 1234.5f) out[0] = acc;
}

// theta from shared memory (TS = 1: two LDS.128 per block from a per-warp
// tile holding 16 blocks of the chunk's two documents' rows, the lane group's
// document selecting the half; TS = 2: no theta load at all, a register
// constant) -- what the L1 data pipe charges for the theta operand
template <int TS>
__global__ void __launch_bounds__(128, 8) probe_smem(const float* __restrict__ phi, const int* __restrict__ rows,
                                                     int n_chunks, float* out, const float* __restrict__ theta_g) {
  __shared__ __align__(16) float tile[4][2][16][32];  // [warp][doc][block mod 16][topic]
  const int lane = threadIdx.x & 31, s = lane & 3, rg = lane >> 2, wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  for (int i = threadIdx.x; i < 4 * 2 * 16 * 32; i += blockDim.x) (&tile[0][0][0][0])[i] = 1.f + (i & 7);
  __syncthreads();
  float acc = 0.f;
  const int cs = gridDim.x * wpb;
  const float* tw = &tile[wib][rg >> 2][0][s * 8];
  for (int c = blockIdx.x * wpb + wib; c < n_chunks; c += cs) {
    const int my = rows[c * 32 + lane];
    uint32_t r[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) r[kk] = __shfl_sync(FULL, my, rg * 4 + kk);
    float run = 0.f;
#pragma unroll 2
    for (int b = 0; b < K / 32; ++b) {
      float x[4][8], t[8];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ld_v8(x[kk], phi + (size_t)r[kk] * K + b * 32 + s * 8);
      if (TS == 3) {  // theta LDG by the two leader lane groups only (8 lanes), others a constant
        if ((rg & 3) == 0) ld_v8(t, theta_g + (size_t)((2 * c + (rg >> 2)) & 1023) * K + b * 32 + s * 8);
        else {
#pragma unroll
          for (int e = 0; e < 8; ++e) t[e] = 1.f + e;
        }
      } else if (TS == 4) {  // leader lanes load, store to smem, all lanes read back (broadcast)
        float* slot = &tile[wib][rg >> 2][b & 15][s * 8];
        if ((rg & 3) == 0) {
          float u8[8];
          ld_v8(u8, theta_g + (size_t)((2 * c + (rg >> 2)) & 1023) * K + b * 32 + s * 8);
          *reinterpret_cast<float4*>(slot) = make_float4(u8[0], u8[1], u8[2], u8[3]);
          *reinterpret_cast<float4*>(slot + 4) = make_float4(u8[4], u8[5], u8[6], u8[7]);
        }
        __syncwarp();
        const float4 t0 = *reinterpret_cast<const float4*>(slot);
        const float4 t1 = *reinterpret_cast<const float4*>(slot + 4);
        t[0] = t0.x; t[1] = t0.y; t[2] = t0.z; t[3] = t0.w; t[4] = t1.x; t[5] = t1.y; t[6] = t1.z; t[7] = t1.w;
      } else if (TS == 1) {
        const float4 t0 = *reinterpret_cast<const float4*>(tw + (b & 15) * 32);
        const float4 t1 = *reinterpret_cast<const float4*>(tw + (b & 15) * 32 + 4);
        t[0] = t0.x; t[1] = t0.y; t[2] = t0.z; t[3] = t0.w; t[4] = t1.x; t[5] = t1.y; t[6] = t1.z; t[7] = t1.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) t[e] = 1.f + e + (float)(b & 1);
      }
      float q[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a += x[kk][e] * t[e];
        q[kk] = a;
      }
      float v = (s & 1) ? q[1] + __shfl_xor_sync(FULL, q[0], 1) : q[0] + __shfl_xor_sync(FULL, q[1], 1);
      float w = (s & 1) ? q[3] + __shfl_xor_sync(FULL, q[2], 1) : q[2] + __shfl_xor_sync(FULL, q[3], 1);
      float z = (s & 2) ? w + __shfl_xor_sync(FULL, v, 2) : v + __shfl_xor_sync(FULL, w, 2);
      run += z;
    }
    acc += run;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int n_chunks = argc > 1 ? atoi(argv[1]) : 131072;
  const int vrows = argc > 2 ? atoi(argv[2]) * 64 : 2560;  // phi slice, MB (default 40)
  const int n_theta = 262144;  // 4 GB of theta rows: 2 per chunk, each read once
  float *phi, *theta, *out;
  int* rows;
  CK(cudaMalloc(&phi, (size_t)vrows * K * 4));
  CK(cudaMalloc(&theta, (size_t)n_theta * K * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&rows, (size_t)n_chunks * 32 * 4));
  std::vector<int> h((size_t)n_chunks * 32);
  srand(1);
  for (auto& x : h) x = rand() % vrows;
  CK(cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(phi, 0, (size_t)vrows * K * 4));
  CK(cudaMemset(theta, 0, (size_t)n_theta * K * 4));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double bytes = (double)n_chunks * 32 * K * 4;  // phi bytes (the algorithmic gather)
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int i = 0; i < 3; ++i) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %8.1f GB/s of phi\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  const int grid = sms * 8;
#define RUN(NAME, ...) timeit(NAME, [&] { probe<__VA_ARGS__><<<grid, 128>>>(phi, theta, rows, n_chunks, n_theta, out); })
  if (argc > 3 && argv[3][0] == 's') {  // theta operand source
    RUN("resident (theta LDG, L2)", 0, false, 0, false);
    timeit("theta from smem (2x LDS.128)", [&] { probe_smem<1><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("no theta load", [&] { probe_smem<2><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("theta LDG by leader lanes", [&] { probe_smem<3><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("leader LDG + smem bcast", [&] { probe_smem<4><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    RUN("resident (theta LDG, L2)", 0, false, 0, false);
    timeit("theta from smem (2x LDS.128)", [&] { probe_smem<1><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("no theta load", [&] { probe_smem<2><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("theta LDG by leader lanes", [&] { probe_smem<3><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
    timeit("leader LDG + smem bcast", [&] { probe_smem<4><<<grid, 128>>>(phi, rows, n_chunks, out, theta); });
  } else if (argc > 3) {  // short list
    RUN("resident", 0, false, 0, false);
    RUN("stream", 1, false, 0, false);
    RUN("stream+ef", 1, true, 0, false);
    RUN("32 MB table", 6, false, 0, false);
#define RUNR(NAME, ...) timeit(NAME, [&] { probe_ring<__VA_ARGS__><<<grid, 128>>>(phi, theta, rows, n_chunks, n_theta, out); })
    RUNR("resident ring D2", 0, 2);
    RUNR("stream ring D2", 1, 2);
    RUNR("stream ring D4", 1, 4);
    RUNR("stream ring D6", 1, 6);
    RUN("stream+bulk span 4", 1, false, -4, false);
    RUN("stream+bulk span 8", 1, false, -8, false);
    RUN("stream+bulk span 16", 1, false, -16, false);
    RUN("stream+bulk span 32", 1, false, -32, false);
    RUN("stream+ef+bulk span 8", 1, true, -8, false);
    RUN("stream, 1 doc per chunk", 7, false, 0, false);
    RUN("stream, rows shared by 2 chunks", 8, false, 0, false);
  } else {
    RUN("resident", 0, false, 0, false);
    RUN("stream", 1, false, 0, false);
    RUN("stream+ef", 1, true, 0, false);
    RUN("stream+pf2", 1, false, 2, false);
    RUN("stream+pf4", 1, false, 4, false);
    RUN("stream+pf8", 1, false, 8, false);
    RUN("stream+ef+pf4", 1, true, 4, false);
    RUN("stream+bulk", 1, false, 0, true);
    RUN("stream+ef+bulk", 1, true, 0, true);
    RUN("stream, SM-local rows", 2, false, 0, false);
    RUN("64 MB table", 3, false, 0, false);
    RUN("64 MB table+ef", 3, true, 0, false);
    RUN("16 MB rows over 256 MB", 4, false, 0, false);
    RUN("16 MB rows over 64 MB", 5, false, 0, false);
    RUN("32 MB table", 6, false, 0, false);
    RUN("resident", 0, false, 0, false);
    RUN("stream", 1, false, 0, false);
  }
  CK(cudaGetLastError());
  return 0;
}
