import sys, json, torch
sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd
from paper_1505_03851_b200 import _lib
L = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
for K in (200, 1024, 2048):
    M = 1_000_000
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda"); off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    z = torch.randint(0, K, (T,), generator=g, device="cuda", dtype=torch.int32)
    theta = torch.empty((M, K), dtype=torch.float32, device="cuda")
    f = lambda: _lib.check(L.wd_resample_theta(0, z.data_ptr(), off.data_ptr(), M, K, 0.1, 5, 0, theta.data_ptr(), K, _lib.stream_handle()), "t")
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    print(json.dumps({"K": K, "theta_ms": s.elapsed_time(e) / 10}), flush=True)
    del z, theta
