"""Reproduce the paper's own experiment on the B200:
whole-application LDA time, butterfly-table draw vs full prefix-sum-table
draw, K in {16, 48, ..., 240}, 100 Gibbs iterations, on a synthetic corpus
with the paper's Wikipedia shape (M = 43,556 documents, V = 37,286 words,
3,072,662 tokens: mean length 70.5, max ~307).

The paper (Titan Black) reports the butterfly version faster for K >= 80
and more than 2x faster for K >= 200, over the whole application.

    python tools/paper_repro.py [--iters 100] [--out profiles/paper_repro_r01]
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
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402


def corpus(seed=1505):
    gen = np.random.default_rng(seed)
    M, V, T = 43_556, 37_286, 3_072_662
    lengths = np.minimum(np.maximum(gen.poisson(70.5, size=M), 1), 307)
    lengths = np.floor(lengths * (T / lengths.sum())).astype(np.int64)  # total ~= the paper's token count
    lengths = np.maximum(lengths, 1)
    pad = (-M) % 32
    lengths = np.concatenate([lengths, np.zeros(pad, dtype=np.int64)])
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
    return off, words, V


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--out", default="profiles/paper_repro")
    a = ap.parse_args()
    off, words, V = corpus()
    dc = wd.DeviceCorpus.from_csr(off, words)
    rows = []
    for K in (16, 48, 80, 112, 144, 176, 208, 240):
        r = {"K": K}
        for kern in ("butterfly", "transposed"):
            lda = DeviceLDA(dc, K, V, seed=7, kernel=kern)
            lda.init_from_assignments()
            lda.iterate(0)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for t in range(a.iters):
                lda.iterate(1 + t)
            e.record()
            torch.cuda.synchronize()
            lda.check_errors()
            r[kern] = {"app_s": s.elapsed_time(e) / 1e3, "log_likelihood": lda.log_likelihood()}
            del lda
        r["speedup"] = r["transposed"]["app_s"] / r["butterfly"]["app_s"]
        rows.append(r)
        print(json.dumps(r), flush=True)
    res = {"corpus": {"docs": int(off.size - 1), "vocab": V, "tokens": int(off[-1])}, "iters": a.iters, "rows": rows,
           "device": torch.cuda.get_device_name()}
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    with open(a.out + ".md", "w") as fh:
        fh.write(f"# Paper experiment on {res['device']}: whole LDA application, {a.iters} iterations\n\n")
        fh.write(f"Synthetic Wikipedia-shaped corpus: {res['corpus']['docs']} docs (32-padded), V = {V}, "
                 f"{res['corpus']['tokens']} tokens; fp32, W = 32; device resample included.\n\n")
        fh.write("| K | butterfly app time (s) | prefix-table app time (s) | speedup |\n|---|---|---|---|\n")
        for r in rows:
            fh.write(f"| {r['K']} | {r['butterfly']['app_s']:.3f} | {r['transposed']['app_s']:.3f} | "
                     f"{r['speedup']:.2f}x |\n")
    print("wrote", a.out + ".md")


if __name__ == "__main__":
    main()
