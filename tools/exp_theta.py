"""Theta resample on the bench shape: time it and save a checksum slice (A/B across library builds)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import _lib  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else None
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
M = 1_000_000
lengths = torch.poisson(torch.full((M,), 200.0, device=dev), generator=g).clamp_(min=1).long()
off = torch.zeros(M + 1, dtype=torch.int64, device=dev)
off[1:] = torch.cumsum(lengths, 0)
T = int(off[-1])
z = torch.randint(0, K, (T,), generator=g, device=dev, dtype=torch.int32)
theta = torch.empty((M, K), dtype=torch.float32, device=dev)
L = _lib.load()
st = _lib.stream_handle()


def run():
    _lib.check(L.wd_resample_theta(0, z.data_ptr(), off.data_ptr(), M, K, 0.1, 777, 0, theta.data_ptr(), K, st), "t")


for _ in range(2):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    run()
b.record()
torch.cuda.synchronize()
print(f"theta resample K={K}: {a.elapsed_time(b) / 5:.3f} ms", flush=True)
if out:
    np.save(out, theta[::997].cpu().numpy())
