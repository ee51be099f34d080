"""Draw time with and without the fused word-topic counts, uniform vs Zipf words (K=200, 1M docs)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_1505_03851_b200 as wd  # noqa: E402
from configs import make_corpus, timed  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
dev = torch.device("cuda", 0)
for kind in ("uniform", "zipf"):
    g = torch.Generator(device=dev).manual_seed(2026)
    off, words = make_corpus(1_000_000, 40_000, 200.0, kind, g, dev)
    dc = wd.DeviceCorpus.from_csr(off, words, vocab_size=40_000)
    theta = wd.kernels.to_block_aligned(torch.rand((dc.n_docs, K), generator=g, device=dev) * 0.9 + 0.1)
    phi = wd.kernels.to_block_aligned(torch.rand((40_000, K), generator=g, device=dev) * 0.9 + 0.1)
    z = torch.empty(dc.n_tokens, dtype=torch.int32, device=dev)
    wt = torch.zeros((40_000, K), dtype=torch.int32, device=dev)
    err = torch.empty(2, dtype=torch.int64, device=dev)
    for counts in (False, True):
        dt = timed(lambda: wd.draw_z_device("butterfly", dc, theta, phi, wd.SeededStops(3), 32, z=z, err=err,
                                            word_topic=wt if counts else None, check=False), 5)
        print(f"{kind:8s} counts={counts!s:5s} draw {dt * 1e3:7.2f} ms  {dc.n_tokens / dt / 1e9:6.2f} G tok/s", flush=True)
    del dc, theta, phi, z, wt
