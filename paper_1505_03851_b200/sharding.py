"""Document sharding for multi-GPU runs.

Shards are contiguous ranges of documents cut on `align`-document boundaries
(align = W, so a master-index group of W documents -- kernels.py:520-536 --
never straddles two GPUs and `doc mod W` is the same on every layout), and
balanced by TOKEN count (the draw cost is per token), not by document count.
Every rank keeps the global id of its first document (doc_base); the u hash
and the theta Gamma stream are keyed by global ids, so z and the counts are
identical for any number of ranks.
"""

from __future__ import annotations

import numpy as np


def shard_ranges(lengths, world: int, align: int = 32):
    """[(doc_lo, doc_hi)] for `world` ranks: aligned cuts near equal token counts."""
    lengths = np.asarray(lengths, dtype=np.int64)
    M = lengths.size
    if world < 1:
        raise ValueError("world must be >= 1")
    if M % align:
        raise ValueError("document count must be a multiple of the alignment (pad upstream)")
    groups = M // align
    gtok = lengths.reshape(groups, align).sum(axis=1) if groups else np.zeros(0, np.int64)
    cum = np.concatenate([[0], np.cumsum(gtok)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        g = int(np.searchsorted(cum, target))
        if g > 0 and abs(cum[g - 1] - target) <= abs(cum[min(g, groups)] - target):
            g -= 1
        g = min(max(g, cuts[-1]), groups)
        cuts.append(g)
    cuts.append(groups)
    return [(cuts[r] * align, cuts[r + 1] * align) for r in range(world)]


def shard_csr(offsets, words, lo: int, hi: int):
    """Local CSR (offsets rebased to 0, words slice) of documents [lo, hi)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    a, b = int(offsets[lo]), int(offsets[hi])
    return offsets[lo : hi + 1] - a, np.asarray(words)[a:b]


def count_chunks(vocab_size: int, rows_per_tile: int | None):
    """word_topic row ranges reduced one by one: the vocabulary tiles, derived
    from V and the tile height only, so every rank has the same list."""
    if not rows_per_tile:
        return [(0, int(vocab_size))]
    return [(lo, min(int(vocab_size), lo + int(rows_per_tile))) for lo in range(0, int(vocab_size), int(rows_per_tile))]


class TileAllReduce:
    """Issues the word-topic count all-reduce tile by tile behind the draw.

    A vocabulary tile's draw touches only the count rows of its own words,
    so once its launch is enqueued those rows are final on the stream and
    their all-reduce can run (NCCL stream) while the next tile draws.  Ranks
    skip launches for tiles their shard has no tokens in, so issuing is
    driven by the row range reached, not by launch count: every rank issues
    the same chunk sequence in the same order (a collective requirement).

    all_reduce(view) -> work (with .wait()) is the collective, e.g.
    lambda v: dist.all_reduce(v, group=pg, async_op=True).
    """

    def __init__(self, counts, chunks, all_reduce):
        self.counts = counts
        self.chunks = list(chunks)
        self.all_reduce = all_reduce
        self.next = 0
        self.works = []

    def after_tile(self, t, lo, hi):
        while self.next < len(self.chunks) and self.chunks[self.next][1] <= hi:
            a, b = self.chunks[self.next]
            self.works.append(self.all_reduce(self.counts[a:b]))
            self.next += 1

    def finish(self):
        """Issue the chunks no launch reached (tiles empty on this rank)."""
        if self.chunks:
            self.after_tile(-1, self.chunks[-1][1], self.chunks[-1][1])
        return self.works

    def wait(self):
        for w in self.works:
            w.wait()
        self.works = []
