"""Corpus I/O at configs[4] scale: a 10M-document
synthetic corpus (Poisson(200) lengths, V = 40,000) written once as .wdc
(uint16 ids, ~4 GB), then timed into HBM by corpus_io.load_device_corpus
(whole corpus on one GPU, and one rank's shard of 8), plus the native text
parser on a 1M-document text corpus.  Prints one JSON line."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1505_03851_b200 import corpus_io as C  # noqa: E402
from paper_1505_03851_b200 import lda  # noqa: E402


def main():
    import torch

    out = {}
    d = os.environ.get("IO_BENCH_DIR", "/tmp/wd_io_bench")
    os.makedirs(d, exist_ok=True)
    M = int(os.environ.get("IO_BENCH_DOCS", 10_000_000))
    rng = np.random.default_rng(2026)
    N = np.maximum(rng.poisson(200, M), 1).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(N)])
    T = int(off[-1])
    path = os.path.join(d, "cfg5.wdc")
    t0 = time.perf_counter()
    with open(path, "wb") as fh:
        fh.write(C.HEADER.pack(C.MAGIC, 1, 2, M, T, 40000, 0, bytes(16)))
        fh.write(off.astype("<i8").tobytes())
        step = 1 << 28
        for a in range(0, T, step):
            rng.integers(0, 40000, min(step, T - a), dtype=np.uint16).tofile(fh)
    out["write_s"] = time.perf_counter() - t0
    out["file_bytes"] = os.path.getsize(path)
    torch.cuda.init()
    torch.empty(1, device="cuda")
    for label, kw in (("whole_first_call", {}), ("whole", {}), ("rank0_of_8", {"rank": 0, "world": 8})):
        tim = {}
        dc = C.load_device_corpus(path, timing=tim, **kw)
        out[label] = {"docs": dc.n_docs, "tokens": dc.n_tokens, **{k: round(v, 3) for k, v in tim.items()}}
        out[label]["gb_per_s"] = tim["bytes"] / tim["total_s"] / 1e9
        del dc
        torch.cuda.empty_cache()
    # native text parser on 1M documents
    Mt = 1_000_000
    corp = lda.Corpus(40000, N[:Mt], C.RaggedWords(off[: Mt + 1], np.zeros(int(off[Mt]), np.int32)))
    corp.words.flat[:] = rng.integers(0, 40000, corp.words.flat.size)
    tp = os.path.join(d, "cfg3.txt")
    t0 = time.perf_counter()
    lda.save_corpus(corp, tp)
    out["text_1M_write_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    back = lda.load_corpus(tp)
    out["text_1M_parse_s"] = time.perf_counter() - t0
    assert np.array_equal(back.csr()[1], corp.words.flat)
    out["cores"] = len(os.sched_getaffinity(0))
    os.remove(path)
    os.remove(tp)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
