"""Fused word-topic counts in the draw vs a separate counts pass (bench shape)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import _lib  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402
from configs import make_corpus, timed  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kind = sys.argv[2] if len(sys.argv) > 2 else "uniform"
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(2026)
off, words = make_corpus(1_000_000, 40_000, 200.0, kind, g, dev)
dc = wd.DeviceCorpus.from_csr(off, words, vocab_size=40_000)
lda = DeviceLDA(dc, K, 40_000, seed=1)
lda.init_uniform()
L = _lib.load()


def fused():
    lda.draw(0)


def nofuse():
    lda.draw(0, fused_counts=False)


def separate():
    lda.draw(0, fused_counts=False)
    lda.word_topic.zero_()
    _lib.check(L.wd_topic_counts(dc.words.data_ptr(), None, lda.z.data_ptr(), dc.n_tokens, K, None,
                                 lda.word_topic.data_ptr(), _lib.stream_handle()), "counts")


for name, f in (("fused", fused), ("no counts", nofuse), ("separate pass", separate)):
    print(f"K={K} {kind:8s} {name:14s} {timed(f, 5) * 1e3:8.2f} ms", flush=True)
