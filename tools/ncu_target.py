"""Minimal launches for ncu captures: `python tools/ncu_target.py rows|lda|prefix K [n]`."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402

what = sys.argv[1]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n = int(sys.argv[3]) if len(sys.argv) > 3 else (1 << 20)
g = torch.Generator(device="cuda").manual_seed(0)
if what in ("rows", "prefix"):
    w = torch.rand((n, K), generator=g, device="cuda") * 0.9 + 0.1
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    err = torch.empty(2, dtype=torch.int64, device="cuda")
    for _ in range(4):
        wd.sample_rows(w, 5, variant="butterfly" if what == "rows" else "prefix", out=out, err=err, check=False)
elif what == "resample":
    from paper_1505_03851_b200.device_lda import DeviceLDA

    M, V = n, 40000
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    lda = DeviceLDA(wd.DeviceCorpus.from_csr(off, words), K, V)
    lda.init_uniform()
    for t in range(3):
        lda.iterate(t)
else:
    M, V = n, 40000
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    theta = torch.rand((M, K), generator=g, device="cuda") * 0.9 + 0.1
    phi = torch.rand((V, K), generator=g, device="cuda") * 0.9 + 0.1
    z = torch.empty(T, dtype=torch.int32, device="cuda")
    err = torch.empty(2, dtype=torch.int64, device="cuda")
    wt = torch.zeros((V, K), dtype=torch.int32, device="cuda")
    kern = "butterfly" if what in ("lda", "ldatiled") else "transposed"
    run_pad = 8 if len(sys.argv) <= 4 else int(sys.argv[4])  # DeviceLDA's rule at K=1024
    tiles = dc.vocab_tiles((40 << 20) // (4 * K), run_pad) if what == "ldatiled" else None
    err = torch.empty((tiles.n_tiles if tiles else 1, 2), dtype=torch.int64, device="cuda")
    for _ in range(4):
        wd.draw_z_device(kern, dc, theta, phi, wd.SeededStops(3), 32, z=z, err=err, word_topic=wt, check=False,
                         tiles=tiles)
torch.cuda.synchronize()
print("done", what, K, n)
