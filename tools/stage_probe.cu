// stage_probe.cu -- microbenchmark for the LDA phi gather at large K:
// is bulk-async (TMA engine) staging into a per-warp shared-memory ring
// faster than register loads?  Pattern: a 40 MB L2-resident phi slice of
// K = 4096 fp32 rows; each warp takes chunks of 32 random rows and streams
// every row block by block (W = 32 topics = 128 B), multiplying by a theta
// segment and reducing -- the bytes and order of the draw's pass 1.
//
//   V0  register LDG.256 (the current kernel's geometry, L = 4 loads/lane/block)
//   V1  per-lane cp.async.bulk of SPAN bytes of its row into a ring of NS
//       stages per warp (mbarrier complete_tx), consumer LDS.128
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stage_probe stage_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int K = 4096;
constexpr int FULL = 0xffffffff;

__device__ __forceinline__ void ld_v8(float (&a)[8], const float* p) {
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3]), "=f"(a[4]), "=f"(a[5]), "=f"(a[6]), "=f"(a[7]) : "l"(p));
}

// V0: registers.  lane (s = lane % 4, rg = lane / 4): rows rg*4 + kk, topics s*8..s*8+7 of the block
template <int MINB, int NT = 1>
__global__ void __launch_bounds__(128, MINB) v0(const float* __restrict__ phi, const float* __restrict__ theta,
                                                const int* __restrict__ rows, int n_chunks, float* out) {
  extern __shared__ float smv0[];
  const int lane = threadIdx.x & 31, s = lane & 3, rg = lane >> 2;
  const int wpb = blockDim.x >> 5;
  float acc = 0.f;
  for (int c = blockIdx.x * wpb + (threadIdx.x >> 5); c < n_chunks; c += gridDim.x * wpb) {
    const int my = rows[c * 32 + lane];
    uint32_t r[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) r[kk] = __shfl_sync(FULL, my, rg * 4 + kk);
    const float* th = theta + (c & 1023) * K + s * 8;
    float run = 0.f;
#pragma unroll 2
    for (int b = 0; b < K / 32; ++b) {
      float x[4][8], t[NT][8];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) ld_v8(x[kk], phi + (size_t)r[kk] * K + b * 32 + s * 8);
#pragma unroll
      for (int i = 0; i < NT; ++i) ld_v8(t[i], th + i * 7 * K + b * 32);
      float q[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a += x[kk][e] * t[(NT > 1 && (kk & 1)) ? NT - 1 : 0][e];
        q[kk] = a;
      }
      // transpose-reduce over 4 lanes (2 levels)
      float v = (s & 1) ? q[1] + __shfl_xor_sync(FULL, q[0], 1) : q[0] + __shfl_xor_sync(FULL, q[1], 1);
      float w = (s & 1) ? q[3] + __shfl_xor_sync(FULL, q[2], 1) : q[2] + __shfl_xor_sync(FULL, q[3], 1);
      float z = (s & 2) ? w + __shfl_xor_sync(FULL, v, 2) : v + __shfl_xor_sync(FULL, w, 2);
      run += z;
    }
    acc += run;
    if (threadIdx.x == 0 && acc == 1.5f) smv0[c & 7] = acc;
  }
  if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}

// V1: ring of NS stages per warp, stage = 32 rows x SPAN floats (+ theta SPAN floats)
template <int SPAN, int NS, int WPB>
__global__ void __launch_bounds__(WPB * 32) v1(const float* __restrict__ phi, const float* __restrict__ theta,
                                               const int* __restrict__ rows, int n_chunks, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  constexpr int STAGE = (32 + 1) * SPAN * 4;  // 32 phi rows + 1 theta row
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int s = lane & 7, rg = lane >> 3;  // LDS.128: 8 lanes per row, 4 rows per instruction
  float* ring = reinterpret_cast<float*>(sm + (size_t)wib * NS * STAGE);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)WPB * NS * STAGE) + wib * NS;
  if (lane == 0)
    for (int i = 0; i < NS; ++i) mbar_init(bar + i, 1);
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  constexpr int NSEG = K / SPAN;  // stages per chunk
  float acc = 0.f;
  const int c0 = blockIdx.x * WPB + wib, cs = gridDim.x * WPB;
  const int my_chunks = c0 < n_chunks ? (n_chunks - c0 + cs - 1) / cs : 0;
  const int total = my_chunks * NSEG;  // stage sequence of this warp
  int my_row = 0;
  auto issue = [&](int g) {  // stage sequence number g -> chunk, segment
    const int ci = g / NSEG, seg = g % NSEG;
    const int c = c0 + ci * cs;
    float* st = ring + (size_t)(g % NS) * (STAGE / 4);
    const int r = rows[c * 32 + lane];
    if (lane == 0) mbar_expect_tx(bar + g % NS, STAGE);
    __syncwarp();
    bulk_g2s(st + lane * SPAN, phi + (size_t)r * K + seg * SPAN, SPAN * 4, bar + g % NS);
    if (lane == 0) bulk_g2s(st + 32 * SPAN, theta + (size_t)(c & 1023) * K + seg * SPAN, SPAN * 4, bar + g % NS);
  };
  for (int g = 0; g < NS - 1 && g < total; ++g) issue(g);
  float run = 0.f;
  for (int g = 0; g < total; ++g) {
    if (g + NS - 1 < total) issue(g + NS - 1);
    mbar_wait(bar + g % NS, (g / NS) & 1);
    const float* st = ring + (size_t)(g % NS) * (STAGE / 4);
#pragma unroll
    for (int b = 0; b < SPAN / 32; ++b) {
      const float4 t = *reinterpret_cast<const float4*>(st + 32 * SPAN + b * 32 + s * 4);
      float q[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const float4 x = *reinterpret_cast<const float4*>(st + (rg * 8 + kk) * SPAN + b * 32 + s * 4);
        q[kk] = x.x * t.x + x.y * t.y + x.z * t.z + x.w * t.w;
      }
      // transpose-reduce over 8 lanes (3 levels)
#pragma unroll
      for (int bit = 1, n = 8; bit < 8; bit <<= 1, n >>= 1)
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
          const bool hi = (s & bit) != 0;
          const float send = hi ? q[2 * i] : q[2 * i + 1], keep = hi ? q[2 * i + 1] : q[2 * i];
          q[i] = keep + __shfl_xor_sync(FULL, send, bit);
        }
      run += q[0];
    }
    __syncwarp();  // every lane has read the stage before it is refilled
    if ((g + 1) % NSEG == 0) { acc += run; run = 0.f; }
  }
  if (acc == 1234.5f) out[0] = acc;
  (void)my_row;
}

int main(int argc, char** argv) {
  const int vrows = 2560;  // 40 MB slice
  const int n_chunks = argc > 1 ? atoi(argv[1]) : 200000;
  float *phi, *theta, *out;
  int* rows;
  CK(cudaMalloc(&phi, (size_t)vrows * K * 4));
  CK(cudaMalloc(&theta, (size_t)1024 * K * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&rows, (size_t)n_chunks * 32 * 4));
  std::vector<int> h((size_t)n_chunks * 32);
  srand(1);
  for (auto& x : h) x = rand() % vrows;
  CK(cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(phi, 0, (size_t)vrows * K * 4));
  CK(cudaMemset(theta, 0, (size_t)1024 * K * 4));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double bytes = (double)n_chunks * 32 * K * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.3f ms  %8.1f GB/s\n", name, ms / 3, bytes / (ms / 3 * 1e-3) / 1e9);
  };
  timeit("v0 regs minb5", [&] { v0<5><<<sms * 5, 128>>>(phi, theta, rows, n_chunks, out); });
  timeit("v0 regs minb6", [&] { v0<6><<<sms * 6, 128>>>(phi, theta, rows, n_chunks, out); });
  timeit("v0 regs minb8", [&] { v0<8><<<sms * 8, 128>>>(phi, theta, rows, n_chunks, out); });
  timeit("v0 regs minb8 nt2", [&] { v0<8, 2><<<sms * 8, 128>>>(phi, theta, rows, n_chunks, out); });
  timeit("v0 regs minb6 nt2", [&] { v0<6, 2><<<sms * 6, 128>>>(phi, theta, rows, n_chunks, out); });
  for (int kb : {4, 8, 12, 16, 20, 24}) {
    CK(cudaFuncSetAttribute(v0<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
    char nm[64];
    snprintf(nm, sizeof nm, "v0 regs minb8 smem %dK/CTA", kb);
    timeit(nm, [&] { v0<8><<<sms * 8, 128, kb * 1024>>>(phi, theta, rows, n_chunks, out); });
  }
  for (int kb : {8, 16, 24, 32}) {
    CK(cudaFuncSetAttribute(v0<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
    char nm[64];
    snprintf(nm, sizeof nm, "v0 regs minb6 smem %dK/CTA", kb);
    timeit(nm, [&] { v0<6><<<sms * 6, 128, kb * 1024>>>(phi, theta, rows, n_chunks, out); });
  }
#define RUN_V1(SPAN, NS, WPB, CTAS)                                                                          \
  {                                                                                                          \
    const int smem = WPB * NS * (33 * SPAN * 4) + WPB * NS * 8;                                              \
    CK(cudaFuncSetAttribute(v1<SPAN, NS, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));          \
    char nm[96];                                                                                             \
    snprintf(nm, sizeof nm, "v1 span%d ns%d wpb%d ctas/sm%d smem%dK", SPAN, NS, WPB, CTAS, smem / 1024);     \
    timeit(nm, [&] { v1<SPAN, NS, WPB><<<sms * CTAS, WPB * 32, smem>>>(phi, theta, rows, n_chunks, out); }); \
  }
  RUN_V1(32, 4, 4, 4);
  RUN_V1(128, 3, 2, 4);
  CK(cudaGetLastError());
  return 0;
}
