"""Draw time vs vocabulary-tile size (K=1024, V=40k, 200k docs) + resample timing."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
M, V = int(sys.argv[1]) if len(sys.argv) > 1 else 200000, 40000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
MBS = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "10,16,20,27,32,41").split(",")]
lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
off[1:] = torch.cumsum(lengths, 0)
T = int(off[-1])
words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
dc = wd.DeviceCorpus.from_csr(off, words)


def timeit(f, n=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    c.record()
    torch.cuda.synchronize()
    return a.elapsed_time(c) / n


for mb in MBS:
    lda = DeviceLDA(dc, K, V, vocab_tile_bytes=mb << 20)
    lda.init_uniform()
    ms = timeit(lambda: lda.draw(0))
    print(f"tile {mb}MB tiles={lda.tiles.n_tiles} draw {ms:.2f} ms  {T/ms/1e6:.3f} Gtok/s", flush=True)
    del lda
lda = DeviceLDA(dc, K, V)
lda.init_uniform()
lda.draw(0)
print(f"resample {timeit(lambda: lda.resample(0)):.2f} ms (theta {M}x{K}, phi {V}x{K})")
