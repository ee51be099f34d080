"""LDA draw time vs vocabulary size at fixed tokens (K=1024): L2/TLB sensitivity."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda").manual_seed(0)
M = 200_000
lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
off[1:] = torch.cumsum(lengths, 0)
T = int(off[-1])
theta = torch.rand((M, K), generator=g, device="cuda") * 0.9 + 0.1
z = torch.empty(T, dtype=torch.int32, device="cuda")
err = torch.empty(2, dtype=torch.int64, device="cuda")
for V in (1000, 5000, 10000, 20000, 40000, 80000):
    words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    phi = torch.rand((V, K), generator=g, device="cuda") * 0.9 + 0.1
    f = lambda: wd.draw_z_device("butterfly", dc, theta, phi, wd.SeededStops(3), 32, z=z, err=err, check=False)
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"V={V} phi={V*K*4/1e6:.0f}MB ms={ms:.2f} Gtok/s={T/ms/1e6:.3f} algGB/s={T*(4*K+8)/ms/1e6:.0f}", flush=True)
    del phi, words, dc
