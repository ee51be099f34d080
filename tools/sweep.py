"""The paper's comparison on the B200: butterfly vs full prefix-sum table, swept over K.

    python tools/sweep.py [--out profiles/sweep_r01] [--rows 1048576] [--docs 200000]

Two sweeps, CUDA-event timed over a CUDA graph of 10 launches (3 warm-up
launches first; inputs larger than L2, or L2 flushed by a 256 MB write before
each launch with the flush time subtracted):
  * standalone independent rows (BASELINE configs[1]): n rows of K fp32
    weights, algorithmic bytes 4K + 4 per draw;
  * LDA z draw (configs[2] shape, scaled to --docs documents): butterfly vs
    the paper's transposed prefix-table kernel, 4K + 4K/Nbar + 8 B/token.
K covers the paper's eight points (16..240) and powers of two to 2048/4096.
Writes <out>.json and <out>.md.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import RUN_PAD_MIN_MEAN_RUN, lean_draw  # noqa: E402


def _graph(body, iters):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            body()
    return g


def _replay_ms(g):
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def timed(fn, flush, iters=10, warm=3):
    """Device time per call: `iters` calls captured in one CUDA graph (no host
    launch overhead in the measurement); with `flush`, a 256 MB write before
    every call evicts L2 and its own time is subtracted."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if flush is None:
        return _replay_ms(_graph(fn, iters)) / iters / 1e3

    def body():
        flush.zero_()
        fn()

    t_all = _replay_ms(_graph(body, iters))
    t_flush = _replay_ms(_graph(flush.zero_, iters))
    return (t_all - t_flush) / iters / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/sweep")
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--docs", type=int, default=200_000)
    ap.add_argument("--vocab", type=int, default=40_000)
    ap.add_argument("--ks", default="16,32,48,64,80,112,128,144,176,200,208,240,256,512,1024,2048,4096")
    ap.add_argument("--lda-ks", default="16,48,80,112,144,176,208,240,256,512,1024,2048")
    a = ap.parse_args()
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    n = a.rows
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    err = torch.empty(2, dtype=torch.int64, device="cuda")
    for K in [int(x) for x in a.ks.split(",")]:
        w = torch.rand((n, K), generator=g, device="cuda") * 0.9 + 0.1
        fl = flush if n * K * 4 < (512 << 20) else None
        r = {"K": K}
        for var in ("butterfly", "prefix"):
            # errors accumulate over the timed calls (one reset, checked after):
            # the per-call reset is a separate stream operation as long as a
            # small-K draw (WD_ERR_ACCUMULATE)
            err.fill_(-1)
            dt = timed(lambda: wd.sample_rows(w, 5, variant=var, out=out, err=err, check=False,
                                              accumulate_err=True), fl)
            if err.cpu().numpy().view(np.uint64)[0] != np.uint64(2**64 - 1):
                raise RuntimeError("a sweep row summed to zero")
            r[var] = {"ms": dt * 1e3, "draws_per_s": n / dt, "frac": n * (4 * K + 4) / dt / 1e9 / peak}
        r["speedup"] = r["prefix"]["ms"] / r["butterfly"]["ms"]
        rows.append(r)
        print("rows", json.dumps(r), flush=True)
        del w
    torch.cuda.empty_cache()
    # LDA draw sweep
    M, V = a.docs, a.vocab
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    z = torch.empty(T, dtype=torch.int32, device="cuda")
    lda = []
    for K in [int(x) for x in a.lda_ks.split(",")]:
        # the product's layout (DeviceLDA): line-aligned theta/phi blocks,
        # vocabulary tiles when phi exceeds ~40 MB, and for the butterfly
        # kernel the token list (document, word)-ordered in every tile with
        # (tile, document) runs padded to the 4-row lane groups by
        # DeviceLDA's rule (device_lda.py); the prefix-table baseline keeps
        # CSR order unless phi needs tiling
        theta = wd.kernels.to_block_aligned(torch.rand((M, K), generator=g, device="cuda") * 0.9 + 0.1)
        phi = wd.kernels.to_block_aligned(torch.rand((V, K), generator=g, device="cuda") * 0.9 + 0.1)
        r = {"K": K}
        tiled = V * K * 4 > (40 << 20)
        rows_t = (40 << 20) // (4 * K) if tiled else V
        n_tiles = -(-V // rows_t)
        pad = 4 if (K // 32 <= 32 and T / M / n_tiles >= RUN_PAD_MIN_MEAN_RUN) else 0
        if lean_draw(K, 32, 4):
            pad = 4
        r["vocab_tiles"] = n_tiles
        r["run_pad"] = pad
        terr = torch.empty((n_tiles, 2), dtype=torch.int64, device="cuda")
        bfly_tiles = dc.vocab_tiles(rows_t, pad)
        for kern in ("butterfly", "transposed"):
            tiles = bfly_tiles if kern == "butterfly" else (dc.vocab_tiles(rows_t, 0) if tiled else None)
            dt = timed(lambda: wd.draw_z_device(kern, dc, theta, phi, wd.SeededStops(3), 32, z=z, err=terr,
                                                check=False, tiles=tiles), flush, iters=5, warm=2)
            r[kern] = {"ms": dt * 1e3, "tokens_per_s": T / dt,
                       "alg_GBps": T * (4 * K + 4 * K * M / T + 8) / dt / 1e9}
        r["speedup"] = r["transposed"]["ms"] / r["butterfly"]["ms"]
        lda.append(r)
        print("lda", json.dumps(r), flush=True)
        del theta, phi
    res = {"peak_hbm_gbs": peak, "rows_n": n, "lda_docs": M, "lda_tokens": T, "rows": rows, "lda": lda,
           "device": torch.cuda.get_device_name()}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as fh:
        fh.write(f"# Butterfly vs full prefix-sum table on {res['device']}\n\n")
        fh.write(f"Standalone rows: n = {n} independent fp32 rows, W = 32, HBM peak {peak} GB/s (measured).\n\n")
        fh.write("| K | butterfly draws/s | frac of HBM | prefix-table draws/s | frac | speedup |\n|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write(f"| {r['K']} | {r['butterfly']['draws_per_s']:.3e} | {r['butterfly']['frac']:.2f} | "
                     f"{r['prefix']['draws_per_s']:.3e} | {r['prefix']['frac']:.2f} | {r['speedup']:.2f}x |\n")
        fh.write(f"\nLDA z draw: {M} docs, {T} tokens (Poisson(200)), V = {V}, fp32, W = 32.\n\n")
        fh.write("| K | vocab tiles | butterfly tokens/s | alg. GB/s | prefix-table (transposed) tokens/s | speedup |\n"
                 "|---|---|---|---|---|---|\n")
        for r in lda:
            fh.write(f"| {r['K']} | {r['vocab_tiles']} | {r['butterfly']['tokens_per_s']:.3e} | "
                     f"{r['butterfly']['alg_GBps']:.0f} | {r['transposed']['tokens_per_s']:.3e} | {r['speedup']:.2f}x |\n")
    print("wrote", a.out + ".md")


if __name__ == "__main__":
    main()
