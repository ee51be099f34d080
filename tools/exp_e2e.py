"""e2e variants on the bench shape: z D2H int32 / int16 / none."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
M, V, K = 1_000_000, 40_000, 1024
lengths = torch.poisson(torch.full((M,), 200.0, device=dev), generator=g).clamp_(min=1).long()
off = torch.zeros(M + 1, dtype=torch.int64, device=dev)
off[1:] = torch.cumsum(lengths, 0)
T = int(off[-1])
words = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int32)
lda = DeviceLDA(wd.DeviceCorpus.from_csr(off, words), K, V, seed=3)
lda.init_uniform()
h_theta = lda.theta.cpu().pin_memory()
h_phi = lda.phi.cpu().pin_memory()
for name, zh in (("none", None), ("int32", torch.empty(T, dtype=torch.int32).pin_memory()),
                 ("int16", torch.empty(T, dtype=torch.int16).pin_memory())):
    lda.iterate_from_host(0, 2, h_theta, h_phi, zh)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lda.iterate_from_host(10, 6, h_theta, h_phi, zh)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 6
    print(f"z={name}: {ms:.1f} ms/step  {T / ms / 1e6:.3f} G tokens/s", flush=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for t in range(6):
    lda.iterate(t)
b.record()
torch.cuda.synchronize()
print(f"resident: {a.elapsed_time(b) / 6:.1f} ms/step")
