"""Quick kernel timing (CUDA events) for development; not the bench contract."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402


def t_events(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    res = {}
    what = sys.argv[2] if len(sys.argv) > 2 else "both"
    n = 1 << 20 if what != "lda" else 0
    g = torch.Generator(device="cuda").manual_seed(0)
    for K in [int(k) for k in (sys.argv[1] if len(sys.argv) > 1 else "32,64,128,256,512,1024,2048").split(",")] if n else []:
        w = torch.rand((n, K), generator=g, device="cuda") * 0.9 + 0.1
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        err = torch.empty(2, dtype=torch.int64, device="cuda")
        row = {}
        for var in ("butterfly", "prefix"):
            dt = t_events(lambda: wd.sample_rows(w, 5, variant=var, out=out, err=err, check=False))
            row[var] = {"ms": dt * 1e3, "Gdraws": n / dt / 1e9, "GBps": n * (4 * K + 4) / dt / 1e9}
        row["speedup"] = row["prefix"]["ms"] / row["butterfly"]["ms"]
        res[f"rows_K{K}"] = row
        print(K, json.dumps(row), flush=True)
        del w
    if what == "rows":
        return
    # LDA draw, cfg4-like but 200k docs
    M, V, K = 200_000, 40_000, 1024
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
    for kern in ("butterfly",):
        dt = t_events(lambda: wd.draw_z_device(kern, dc, theta, phi, wd.SeededStops(3), 32, z=z, err=err,
                                               check=False), iters=5, warm=2)
        nb = T * (4 * K + 4 * K * M / T + 8)
        res[f"lda_{kern}"] = {"ms": dt * 1e3, "Gtok": T / dt / 1e9, "GBps": nb / dt / 1e9}
        print(kern, res[f"lda_{kern}"], flush=True)
    dt = t_events(lambda: wd.draw_z_device("butterfly", dc, theta, phi, wd.SeededStops(3), 32, z=z, err=err,
                                           word_topic=wt, check=False), iters=5, warm=2)
    res["lda_butterfly_counts"] = {"ms": dt * 1e3, "Gtok": T / dt / 1e9}
    print(res["lda_butterfly_counts"])
    json.dump(res, open("gpurun_out/quick_perf.json", "w"), indent=1)


if __name__ == "__main__":
    main()
