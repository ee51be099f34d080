"""Measure the L2 -> SM read bandwidth of this GPU (the roofline the vocabulary-
tiled LDA draw runs against once its phi slice is L2-resident).

A grid-stride kernel of 128-bit loads re-reads an L2-resident buffer (default
32 MB) many times; bytes delivered / CUDA-event time.  Also reports the HBM
read bandwidth on a 4 GB buffer with the same kernel, for comparison with the
copy-based MEASURED_PEAKS.json figure.

    python tools/l2_peak.py [--mb 32] [--out profiles/l2_peak.json]
"""

from __future__ import annotations

import argparse
import json

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <cuda_runtime.h>
#include <torch/extension.h>
// U independent 256-bit loads (LDG.E.256) in flight per thread and iteration
template <int U>
__global__ void rd(const float* __restrict__ p, long n8, int reps, float* out) {
  float acc = 0.f;
  const long stride = (long)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i + (U - 1) * stride < n8; i += U * stride) {
      float v[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                       "=f"(v[u][6]), "=f"(v[u][7])
                     : "l"(p + 8 * (i + u * stride)));
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += v[u][e];
    }
  if (acc == 1234.5f) out[0] = acc;
}
void run(torch::Tensor x, int reps, torch::Tensor out, int blocks) {
  long n8 = x.numel() / 8;
  rd<8><<<blocks, 512, 0, at::cuda::getCurrentCUDAStream()>>>(x.data_ptr<float>(), n8, reps,
                                                             out.data_ptr<float>());
}
"""
CPP = "void run(torch::Tensor x, int reps, torch::Tensor out, int blocks);"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=32)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    mod = load_inline("l2peak", CPP, cuda_sources=SRC.replace("#include <torch/extension.h>",
                                                              "#include <torch/extension.h>\n#include <ATen/cuda/CUDAContext.h>"),
                      functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      verbose=False)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(1, device="cuda")
    res = {}
    for name, mbs, reps in (("l2", [16, 24, 32, 40, 48], 200), ("hbm", [4096], 3)):
      best, best_mb = 0.0, None
      for mb in mbs:
        x = torch.rand(mb * (1 << 20) // 4, device="cuda")
        for blocks in (sms * 2, sms * 4, sms * 8, sms * 16):
            mod.run(x, 1, out, blocks)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            mod.run(x, reps, out, blocks)
            e.record()
            torch.cuda.synchronize()
            # bytes actually read: whole U * stride sweeps only (32 B per element)
            stride = blocks * 512
            n8 = x.numel() // 8
            n_read = (n8 // (8 * stride)) * 8 * stride if n8 >= 8 * stride else 0
            gbs = n_read * 32 * reps / (s.elapsed_time(e) / 1e3) / 1e9
            if gbs > best:
                best, best_mb = gbs, mb
        del x
      res[f"{name}_read_gbs"] = best
      res[f"{name}_buffer_mb"] = best_mb
    res["device"] = torch.cuda.get_device_name()
    print(json.dumps(res))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
