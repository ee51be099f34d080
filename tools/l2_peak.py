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
__global__ void rd(const float4* __restrict__ p, long n, int reps, float* out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) out[0] = acc;
}
void run(torch::Tensor x, int reps, torch::Tensor out, int blocks) {
  long n = x.numel() / 4;
  rd<<<blocks, 512, 0, at::cuda::getCurrentCUDAStream()>>>((const float4*)x.data_ptr<float>(), n, reps,
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
    for name, mb, reps in (("l2", a.mb, 200), ("hbm", 4096, 3)):
        x = torch.rand(mb * (1 << 20) // 4, device="cuda")
        best = 0.0
        for blocks in (sms * 2, sms * 4, sms * 8):
            mod.run(x, 1, out, blocks)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            mod.run(x, reps, out, blocks)
            e.record()
            torch.cuda.synchronize()
            gbs = x.numel() * 4 * reps / (s.elapsed_time(e) / 1e3) / 1e9
            best = max(best, gbs)
        res[f"{name}_read_gbs"] = best
        res[f"{name}_buffer_mb"] = mb
        del x
    res["device"] = torch.cuda.get_device_name()
    print(json.dumps(res))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
