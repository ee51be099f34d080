"""Strong-scaling model of configs[3] (the bench corpus, K = 1024) on 2/4/8 GPUs,
measured one shard at a time on ONE GPU (the only hardware this round has).

For N in 1, 2, 4, 8 the 1M-document corpus is cut exactly as `bench.py
--gpus N` cuts it (sharding.shard_ranges: 32-aligned, token-balanced) and
the first and last rank's shards are run alone through DeviceLDA (no process
group): draw, theta resample and phi resample timed separately with CUDA
events.  A rank's iteration at N GPUs is then

    T_N = draw_N + theta_N + phi + allreduce_tail_N

with phi resampled whole on every rank ("replicated_phi"), or sharded
("sharded_phi", DeviceLDA's default for N > 1):

    T_N = draw_N + allreduce_tail_N + phi_share_N + 2 partial all-gathers
          + max(theta_N, phi rows all-gather)

(the rows' all-gather runs on the NCCL stream while theta resamples).  The
count all-reduce is hidden behind the next vocabulary tile's draw
except the LAST tile's rows (DeviceLDA draw(overlap_allreduce=True)), whose
all-reduce is exposed: bytes = (V / tiles) x K x 4, time = 2 (N-1)/N x bytes
/ busbw (ring all-reduce), busbw an assumption given on the command line
(default 700 GB/s: NCCL all-reduce bus bandwidth on 8 x B200 NVLink 5; NVLS
in-switch reduction would only lower it).  Predicted strong-scaling
efficiency = T_1 / (N * max(T_N over ranks)).  Prints one JSON object.

    python tools/scaling_model.py [--busbw-gbs 700] [--steps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import _lib  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402
from paper_1505_03851_b200.rng import derive_seed  # noqa: E402


def time_shard(args, rank, world, dev):
    a = argparse.Namespace(**vars(args))
    a.scaling = "strong"
    off, words, doc_base = bench.make_shard(torch, rank, world, a, dev)
    dc = wd.DeviceCorpus.from_csr(off, words, doc_base=doc_base, vocab_size=a.vocab)
    del words
    lda = DeviceLDA(dc, a.topics, a.vocab, lanes=32, seed=a.seed)
    lda.init_uniform()
    for t in range(2):
        lda.iterate(t)
    torch.cuda.synchronize()
    L = _lib.load()
    st = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for s in range(args.steps):
        t = 10 + s
        e = ev[s]
        e[0].record(st)
        lda.draw(t)
        e[1].record(st)
        _lib.check(L.wd_resample_theta(lda._dt, lda.z.data_ptr(), dc.offsets.data_ptr(), dc.n_docs, lda.K, lda.alpha,
                                       derive_seed(lda.seed, 2, t, 0), dc.doc_base, lda.theta.data_ptr(),
                                       lda.theta.stride(0), _lib.stream_handle()), "theta")
        e[2].record(st)
        _lib.check(L.wd_resample_phi(lda._dt, lda.word_topic.data_ptr(), lda.V, lda.K, lda.beta,
                                     derive_seed(lda.seed, 2, t, 1), lda.phi.data_ptr(), lda.phi.stride(0),
                                     lda._phi_ws.data_ptr(), lda._phi_ws.numel(), _lib.stream_handle()), "phi")
        e[3].record(st)
    torch.cuda.synchronize()
    mean = lambda i, j: sum(x[i].elapsed_time(x[j]) for x in ev) / len(ev)  # noqa: E731
    # the sharded phi resample's compute on this rank: its 1/world share of
    # the fixed row chunks, three passes (+ the two column-partial folds)
    G = int(L.wd_resample_phi_chunks())
    c0, c1 = rank * G // world, (rank + 1) * G // world
    part = torch.empty((G, lda.K), dtype=torch.float32, device=dev)
    colstat = torch.zeros(2 * lda.K, dtype=torch.float32, device=dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for s in range(args.steps):
        for pss in (0, 1, 2):
            _lib.check(L.wd_resample_phi_pass(lda._dt, pss, lda.word_topic.data_ptr(), lda.V, lda.K, lda.beta, 99 + s,
                                              lda.phi.data_ptr(), lda.phi.stride(0), c0, c1, G, part.data_ptr(),
                                              colstat.data_ptr(), _lib.stream_handle()), "phi pass")
            if pss < 2:
                _lib.check(L.wd_resample_phi_reduce(pss, part.data_ptr(), G, lda.K, colstat.data_ptr(),
                                                    _lib.stream_handle()), "phi reduce")
    b.record(st)
    torch.cuda.synchronize()
    out = {"rank": rank, "docs": dc.n_docs, "tokens": dc.n_tokens, "draw_ms": mean(0, 1), "theta_ms": mean(1, 2),
           "phi_ms": mean(2, 3), "iter_ms": mean(0, 3), "vocab_tiles": lda.tiles.n_tiles,
           "rows_per_tile": lda.tiles.rows_per_tile, "phi_shard_ms": a.elapsed_time(b) / args.steps,
           "phi_bytes": (-(-lda.V // G) * G) * lda.phi.stride(0) * lda.phi.element_size()}
    del lda, dc
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--busbw-gbs", type=float, default=700.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--collective-latency-us", type=float, default=25.0,
                    help="latency of one small (2.4 MB) all-gather of column partials")
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--topics", type=int, default=1024)
    ap.add_argument("--vocab", type=int, default=40_000)
    ap.add_argument("--mean-len", type=float, default=200.0)
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--only-n", type=int, default=None,
                    help="model this world size only (e.g. configs[4]: --docs 10000000 --topics 4096 --only-n 8)")
    ap.add_argument("--all-ranks", action="store_true", help="time every rank's shard (default: first and last)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = {"assumption": f"ring all-reduce busbw {args.busbw_gbs} GB/s (NVLink 5); only the last vocabulary tile's "
                         "count all-reduce is exposed", "per_n": {}}
    t1 = None
    total_tokens = None
    for N in ((args.only_n,) if args.only_n else (1, 2, 4, 8)):
        ranks = list(range(N)) if args.all_ranks else sorted({0, N - 1})
        shards = [time_shard(args, r, N, dev) for r in ranks]
        if args.all_ranks:
            total_tokens = sum(x["tokens"] for x in shards)
        worst = max(shards, key=lambda s: s["iter_ms"])
        tile_bytes = worst["rows_per_tile"] * args.topics * 4
        ar_ms = 0.0 if N == 1 else 2 * (N - 1) / N * tile_bytes / (args.busbw_gbs * 1e9) * 1e3
        t_n = worst["iter_ms"] + ar_ms
        if N == 1:
            t1 = t_n
            total_tokens = shards[0]["tokens"]
        eff = (lambda t: t1 / (N * t)) if t1 else (lambda t: None)
        # sharded phi (DeviceLDA default for N > 1): the rank's phi share, two
        # column-partial all-gathers (~latency), then the rows' all-gather
        # overlapping the theta resample
        ag_ms = 0.0 if N == 1 else (N - 1) / N * worst["phi_bytes"] / (args.busbw_gbs * 1e9) * 1e3
        part_ms = 0.0 if N == 1 else 2 * args.collective_latency_us / 1e3
        t_sh = (worst["draw_ms"] + ar_ms + worst["phi_shard_ms"] + part_ms + max(worst["theta_ms"], ag_ms)
                if N > 1 else t_n)
        res["per_n"][N] = {"shards": shards, "exposed_allreduce_ms": ar_ms,
                           "replicated_phi": {"predicted_iter_ms": t_n, "predicted_tokens_per_s": total_tokens / (t_n / 1e3),
                                              "predicted_efficiency": eff(t_n)},
                           "sharded_phi": {"phi_allgather_ms": ag_ms, "partials_allgather_ms": part_ms,
                                           "predicted_iter_ms": t_sh,
                                           "predicted_tokens_per_s": total_tokens / (t_sh / 1e3),
                                           "predicted_efficiency": eff(t_sh)}}
        if args.all_ranks:
            res["per_n"][N]["sum_of_shard_iterations_ms"] = sum(x["iter_ms"] for x in shards)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
