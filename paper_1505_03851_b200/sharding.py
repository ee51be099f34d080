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
