// l2_width_probe.cu -- L2 -> SM read rate by load width: grid-stride sweeps of
// an L2-resident buffer with U independent loads per thread of 64, 128 or 256
// bits (ld.global.cg / .nc), best over grid sizes.  Is the in-run ceiling
// (wd_l2_read_probe, 256-bit) a property of L2 or of the load width?
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2w tools/l2_width_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int BITS, int U, bool NC>
__global__ void __launch_bounds__(512) sweep(const float* __restrict__ p, int64_t n, int reps, float* sink) {
  constexpr int E = BITS / 32;  // floats per load
  const int64_t ne = n / E;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    // each rep starts 3/7 of the buffer further on: a thread never re-reads
    // the lines it read in the previous rep (no L1 hits for .nc loads)
    const int64_t rot = (int64_t)(r % 7) * (ne / 7) * 3;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += U * stride) {
      float v[U][E];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = i + u * stride;
#pragma unroll
        for (int e = 0; e < E; ++e) v[u][e] = 0.f;
        if (j < ne) {
          int64_t jr = j + rot;
          if (jr >= ne) jr -= ne;
          const float* q = p + E * jr;
          if constexpr (BITS == 256) {
            if (NC)
              asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                           : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]),
                             "=f"(v[u][5]), "=f"(v[u][6]), "=f"(v[u][7]) : "l"(q));
            else
              asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                           : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]),
                             "=f"(v[u][5]), "=f"(v[u][6]), "=f"(v[u][7]) : "l"(q));
          } else if constexpr (BITS == 128) {
            if (NC)
              asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]) : "l"(q));
            else
              asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]) : "l"(q));
          } else {
            if (NC)
              asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v[u][0]), "=f"(v[u][1]) : "l"(q));
            else
              asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(v[u][0]), "=f"(v[u][1]) : "l"(q));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < E; ++e) acc += v[u][e];
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t bytes = 32ll << 20;
  float *p, *sink;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(p, 0, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern) {
    double best = 0;
    int best_g = 0;
    for (int g : {sms * 2, sms * 4, sms * 8}) {
      kern<<<g, 512>>>(p, bytes / 4, 2, sink);
      cudaEventRecord(a);
      kern<<<g, 512>>>(p, bytes / 4, 100, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gbs = (double)bytes * 100 / (ms * 1e-3) / 1e9;
      if (gbs > best) best = gbs, best_g = g;
    }
    printf("%-22s %9.1f GB/s (grid %d)\n", name, best, best_g);
  };
  for (int pass = 0; pass < 2; ++pass) {
    run("256-bit cg U8", sweep<256, 8, false>);
    run("256-bit nc U8", sweep<256, 8, true>);
    run("256-bit nc U4", sweep<256, 4, true>);
    run("128-bit cg U8", sweep<128, 8, false>);
    run("128-bit nc U8", sweep<128, 8, true>);
    run("128-bit nc U16", sweep<128, 16, true>);
    run("64-bit nc U16", sweep<64, 16, true>);
    run("256-bit cg U4", sweep<256, 4, false>);
  }
  CK(cudaGetLastError());
  return 0;
}
