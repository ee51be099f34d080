// wd_probe.cu -- the L2 read-bandwidth probe behind bench.py's roofline.
//
// The vocabulary-tiled LDA draw is served by L2 (each tile's phi slice stays
// resident while theta streams), so its roofline is the L2 -> SM read rate,
// not HBM.  This kernel measures that ceiling in the same process as the
// draw: a grid-stride sweep of U independent 256-bit loads per thread
// (ld.global.cg, L1 bypassed) over an L2-resident buffer, repeated `reps`
// times.  Bytes read per rep = the whole buffer (wd_l2_probe_bytes).
#include <cuda_runtime.h>

#include <cstdint>

#include "warpdraw_b200.h"

namespace wd {
void set_last_cuda_error(cudaError_t e);

constexpr int kProbeU = 8;
constexpr int kProbeThreads = 512;

__global__ void __launch_bounds__(kProbeThreads) l2_read_probe(const float* __restrict__ p, int64_t n8, int reps,
                                                               float* __restrict__ sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += kProbeU * stride) {
      // U independent loads in flight per thread; the tail of the last sweep
      // is predicated off, so every 32-byte element is read once per rep
      float v[kProbeU][8];
#pragma unroll
      for (int u = 0; u < kProbeU; ++u) {
        const int64_t j = i + u * stride;
#pragma unroll
        for (int e = 0; e < 8; ++e) v[u][e] = 0.f;
        if (j < n8)
          asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                         "=f"(v[u][6]), "=f"(v[u][7])
                       : "l"(p + 8 * j));
      }
#pragma unroll
      for (int u = 0; u < kProbeU; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += v[u][e];
    }
  if (acc == 1234.5f) sink[0] = acc;  // keeps the loads live
}

}  // namespace wd

extern "C" {

int64_t wd_l2_probe_bytes(int64_t buffer_bytes, int blocks) {
  (void)blocks;  // every 32-byte element of the buffer is read once per rep, for any grid
  return (buffer_bytes / 32) * 32;
}

int wd_l2_read_probe(const void* buffer, int64_t buffer_bytes, int reps, int blocks, float* sink, void* stream) {
  if (!buffer || !sink || buffer_bytes < 32 || reps < 1 || blocks < 1 || ((uintptr_t)buffer & 31))
    return WD_ERR_INVALID_ARGUMENT;
  wd::l2_read_probe<<<blocks, wd::kProbeThreads, 0, (cudaStream_t)stream>>>((const float*)buffer, buffer_bytes / 32,
                                                                            reps, sink);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    wd::set_last_cuda_error(e);
    return WD_ERR_CUDA;
  }
  return WD_OK;
}

}  // extern "C"
