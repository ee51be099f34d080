"""Device throughput of the sequential-stream samplers (SAMPLERS binary /
alias) and of the shared-vector butterfly sampler, n = 2^24 draws."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1505_03851_b200 import _lib, samplers  # noqa: E402
from paper_1505_03851_b200.rng import derive_seed  # noqa: E402


def timed(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


n = 1 << 24
L = _lib.load()
out = torch.empty(n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(L.wd_stream_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
for K in (19, 256, 1024, 65536):
    w = np.random.default_rng(K).uniform(0.1, 1.0, size=K)
    wt = torch.from_numpy(w).cuda()
    table = torch.empty_like(wt)
    L.wd_prefix_f64(wt.data_ptr(), K, table.data_ptr(), _lib.stream_handle())
    th, al = samplers.alias_table(w)
    th = torch.from_numpy(th.view(np.int64)).cuda()
    al = torch.from_numpy(al).cuda()
    row = {"K": K}
    for name, m in (("binary", _lib.WD_STREAM_BINARY), ("alias", _lib.WD_STREAM_ALIAS)):
        def f():
            L.wd_stream_draws(m, table.data_ptr(), th.data_ptr(), al.data_ptr(), K, derive_seed(1, 4), n,
                              out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
        row[name + "_Gdraws"] = n / timed(f) / 1e9
    w32 = torch.from_numpy(w.astype(np.float32)).cuda()
    row["butterfly_f32_Gdraws"] = n / timed(lambda: samplers.sample_rows(w32, 3, n=n, out=out, check=False)) / 1e9
    w64 = torch.from_numpy(w).cuda()
    row["butterfly_f64_lanes8_Gdraws"] = n / timed(lambda: samplers.sample_rows(w64, 3, lanes=8, n=n, out=out, check=False)) / 1e9
    print(json.dumps(row), flush=True)
