"""Every BASELINE.json config on one B200 through the product path (DeviceLDA /
sample_rows), uniform and Zipf ("Wikipedia-shaped") word frequencies.

    python tools/configs.py [--only cfg3,cfg5] [--out gpurun_out/configs.json]

One "iteration" is DeviceLDA.iterate (butterfly draw with fused word-topic
counts + phi/theta device resample), timed with CUDA events after warm-up;
the draw alone is timed too, and its algorithmic bytes per token
4K + 4K/Nbar + 8 give the draw's GB/s.  configs[4] (10M docs
over 8 GPUs) runs ONE rank's shard (1.25M documents) on the single GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402

CONFIGS = {
    # name: (docs, vocab, topics, mean length, words, iterations timed)
    "cfg1": (1024, 5000, 64, 100.0, "uniform", 10),
    "cfg3": (1_000_000, 40_000, 200, 200.0, "uniform", 5),
    "cfg3_zipf": (1_000_000, 40_000, 200, 200.0, "zipf", 5),
    "cfg4": (1_000_000, 40_000, 1024, 200.0, "uniform", 5),
    "cfg4_zipf": (1_000_000, 40_000, 1024, 200.0, "zipf", 5),
    "k2048": (1_000_000, 40_000, 2048, 200.0, "uniform", 3),
    "cfg5_shard": (1_250_000, 40_000, 4096, 200.0, "uniform", 3),
}


def make_corpus(M, V, mean, words_kind, g, dev):
    lengths = torch.poisson(torch.full((M,), mean, device=dev), generator=g).clamp_(min=1).long()
    if M % 32:  # Corpus.padded (lda.py:56-63): empty documents up to a multiple of W
        lengths = torch.cat([lengths, torch.zeros(32 - M % 32, dtype=torch.long, device=dev)])
        M = lengths.numel()
    off = torch.zeros(M + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    if words_kind == "uniform":
        words = torch.randint(0, V, (T,), generator=g, device=dev, dtype=torch.int32)
    else:
        # Zipf(s=1) over ranks 1..V; word id = rank - 1 (frequency-sorted
        # vocabulary, as dictionary-built corpora are)
        p = 1.0 / torch.arange(1, V + 1, device=dev, dtype=torch.float64)
        cdf = torch.cumsum(p / p.sum(), 0)
        u = torch.rand(T, generator=g, device=dev, dtype=torch.float64)
        words = torch.searchsorted(cdf, u).clamp_(max=V - 1).to(torch.int32)
        del u
    return off, words


def timed(fn, n, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / n


def run(name, peak, run_pad=None, dtype="float32", lanes=32, tile_mb=None):
    M, V, K, mean, kind, iters = CONFIGS[name]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(2026)
    off, words = make_corpus(M, V, mean, kind, g, dev)
    dc = wd.DeviceCorpus.from_csr(off, words, vocab_size=V)
    T = dc.n_tokens
    kw = {} if tile_mb is None else {"vocab_tile_bytes": int(tile_mb * (1 << 20))}
    lda = DeviceLDA(dc, K, V, seed=2026, run_pad=run_pad, dtype=getattr(torch, dtype), lanes=lanes, **kw)
    lda.init_uniform()
    it = [0]

    def step():
        lda.iterate(it[0])
        it[0] += 1

    def draw():
        lda.draw(it[0])
        it[0] += 1

    t_iter = timed(step, iters)
    t_draw = timed(draw, iters)
    lda.check_errors()
    esz = 8 if dtype == "float64" else 4
    bpt = esz * K + esz * K * dc.n_docs / T + 8
    top_share = None
    if kind == "zipf":
        top_share = float((words == 0).sum().item()) / T
    res = {
        "config": name, "dtype": dtype, "lanes": lanes, "docs": dc.n_docs, "vocab": V, "topics": K, "tokens": T, "words": kind,
        "vocab_tiles": lda.tiles.n_tiles if lda.tiles is not None else 1,
        "run_pad": lda.tiles.run_pad if lda.tiles is not None else 0,
        "padded_slots": (lda.tiles.bounds[-1] - T) if lda.tiles is not None else 0,
        "iter_ms": t_iter * 1e3, "tokens_per_s_iter": T / t_iter,
        "draw_ms": t_draw * 1e3, "draw_tokens_per_s": T / t_draw,
        "draw_alg_gbs": T * bpt / t_draw / 1e9, "draw_alg_frac_hbm": T * bpt / t_draw / 1e9 / peak,
        "bytes_per_token": bpt, "top_word_share": top_share,
    }
    del lda, dc, off, words
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(CONFIGS))
    ap.add_argument("--out", default="gpurun_out/configs.json")
    ap.add_argument("--run-pad", type=int, default=None, help="force VocabTiles.run_pad (default: DeviceLDA's rule)")
    ap.add_argument("--tile-mb", type=float, default=None, help="vocabulary tile size (default: DeviceLDA's 40 MB)")
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--lanes", type=int, default=32)
    args = ap.parse_args()
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    out = []
    for name in args.only.split(","):
        t0 = time.time()
        r = run(name, peak, args.run_pad, args.dtype, args.lanes, args.tile_mb)
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)
        out.append(r)
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        json.dump({"hbm_peak_gbs": peak, "gpu": torch.cuda.get_device_name(0), "results": out},
                  open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
