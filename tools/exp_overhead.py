"""Host overhead per DeviceLDA.iterate on a tiny corpus (BASELINE configs[0] shape)."""
import sys
import time

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402
from configs import make_corpus  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
off, words = make_corpus(1024, 5000, 100.0, "uniform", g, dev)
dc = wd.DeviceCorpus.from_csr(off, words)
lda = DeviceLDA(dc, 64, 5000, seed=1)
lda.init_uniform()
for t in range(20):
    lda.iterate(t)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for t in range(n):
    lda.iterate(t)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / n:.3f} ms/iter, wall {1e3 * (t2 - t0) / n:.3f} ms/iter")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for t in range(50):
    lda.iterate(t)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
