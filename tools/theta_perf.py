"""Time the device theta resample (wd_resample_theta) on the bench corpus
shape: 1M documents, Poisson(200) lengths, z from DeviceLDA's own draw, at
K = 200 / 1024 / 2048 / 4096 (CUDA events, mean of 10 after warm-up).

    python tools/theta_perf.py [--docs 1000000] [--ks 200,1024,2048,4096]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import _lib  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--ks", default="200,1024,2048,4096")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    M, V = a.docs, 40_000
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lengths, 0)
    words = torch.randint(0, V, (int(off[-1]),), generator=g, device="cuda", dtype=torch.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    L = _lib.load()
    for K in [int(k) for k in a.ks.split(",")]:
        lda = DeviceLDA(dc, K, V, seed=1)
        lda.init_uniform()
        lda.iterate(0)
        torch.cuda.synchronize()

        def step(t):
            _lib.check(L.wd_resample_theta(lda._dt, lda.z.data_ptr(), dc.offsets.data_ptr(), dc.n_docs, K, lda.alpha,
                                           1000 + t, 0, lda.theta.data_ptr(), lda.theta.stride(0),
                                           _lib.stream_handle()), "theta")
        for t in range(3):
            step(t)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for t in range(10):
            step(t)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(json.dumps({"K": K, "docs": M, "theta_ms": ms, "G_gammas_per_s": M * K / ms / 1e6}), flush=True)
        del lda
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
