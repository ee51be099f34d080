"""Draw time vs vocabulary-tile size: python tools/exp_tiles.py [docs] [K] [MB list]."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402
from configs import make_corpus, timed  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
MBS = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "10,16,20,27,32,41").split(",")]
V = 40000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
off, words = make_corpus(M, V, 200.0, "uniform", g, dev)
dc = wd.DeviceCorpus.from_csr(off, words)
T = dc.n_tokens
for mb in MBS:
    lda = DeviceLDA(dc, K, V, vocab_tile_bytes=mb << 20)
    lda.init_uniform()
    ms = timed(lambda: lda.draw(0), 3) * 1e3
    print(f"tile {mb}MB tiles={lda.tiles.n_tiles} pad={lda.tiles.run_pad} draw {ms:.2f} ms  "
          f"{T / ms / 1e6:.3f} Gtok/s", flush=True)
    del lda
lda = DeviceLDA(dc, K, V)
lda.init_uniform()
lda.draw(0)
print(f"resample {timed(lambda: lda.resample(0), 3) * 1e3:.2f} ms (theta {M}x{K}, phi {V}x{K})")
