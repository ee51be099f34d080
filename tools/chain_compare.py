"""Throughput-mode chain (DeviceLDA: device Gammas) vs parity-mode chain
(reference-exact: numpy Gammas, lda.py:185-208) from the same start state on
a cfg3-shaped corpus; prints LL trajectories and per-topic total statistics.

    python tools/chain_compare.py [--docs 200000] [--topics 200] [--iters 10] [--zipf]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import lda as L  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402


def corpus(M, V, mean, zipf, seed):
    g = np.random.default_rng(seed)
    N = np.maximum(g.poisson(mean, size=M), 1).astype(np.int64)
    T = int(N.sum())
    if zipf:
        p = 1.0 / np.arange(1, V + 1)
        words = g.choice(V, size=T, p=p / p.sum())
    else:
        words = g.integers(0, V, size=T)
    off = np.concatenate([[0], np.cumsum(N)])
    return L.Corpus(vocab_size=V, lengths=N, words=[words[off[m]:off[m + 1]] for m in range(M)])


def run(M, V, K, iters, zipf, seed=11):
    c = corpus(M, V, 200.0, zipf, seed).padded(32)
    cfg = wd.WarpConfig(32, 4)
    z = L.init_assignments(c, K, seed)
    params = L.resample_params(c, z, K, 0.1, 0.01, seed, -1, dtype=np.float32)
    dc = c.to_device()
    lda = DeviceLDA(dc, K, V, seed=seed)
    lda.theta.copy_(torch.from_numpy(params.theta))
    lda.phi.copy_(torch.from_numpy(params.phi))
    ref_lda = DeviceLDA(dc, K, V, seed=seed)  # only its LL evaluator is used
    ll_ref, ll_dev, first_equal = [], [], None
    t0 = time.time()
    for t in range(iters):
        params, z = L.gibbs_iterate(c, params, z, "butterfly", cfg, seed, t, dtype=np.float32, _dcorpus=dc)
        lda.iterate(t)
        if t == 0:  # same start, same draw stream: iteration 0's z must be identical
            first_equal = bool(np.array_equal(np.concatenate(z).astype(np.int32), lda.z.cpu().numpy()))
        ref_lda.theta.copy_(torch.from_numpy(params.theta))
        ref_lda.phi.copy_(torch.from_numpy(params.phi))
        ll_ref.append(ref_lda.log_likelihood())
        ll_dev.append(lda.log_likelihood())
    lda.check_errors()
    tot_ref = np.bincount(np.concatenate(z), minlength=K).astype(np.float64)
    tot_dev = np.bincount(lda.z.cpu().numpy(), minlength=K).astype(np.float64)
    stat = float(np.sum((tot_ref - tot_dev) ** 2 / np.maximum(tot_ref + tot_dev, 1)))
    return {"docs": M, "topics": K, "iters": iters, "zipf": zipf, "tokens": int(dc.n_tokens),
            "first_iteration_z_equal": first_equal, "ll_ref": ll_ref, "ll_dev": ll_dev,
            "ll_rel": [abs(a - b) / abs(a) for a, b in zip(ll_ref, ll_dev)],
            "topic_total_chi2": stat, "dof": K - 1, "wall_s": time.time() - t0,
            "tot_rel_sd": float(np.std((tot_dev - tot_ref) / tot_ref))}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=200_000)
    ap.add_argument("--topics", type=int, default=200)
    ap.add_argument("--vocab", type=int, default=40_000)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--zipf", action="store_true")
    a = ap.parse_args()
    print(json.dumps(run(a.docs, a.vocab, a.topics, a.iters, a.zipf)))
