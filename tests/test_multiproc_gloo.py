"""World-size-2 (gloo, CPU) coverage of the N>1 path: 32-aligned token-balanced
document shards, global doc ids, per-rank draws and the word-topic all-reduce
must reproduce the single-process result exactly.  The per-rank draw here is
the CPU oracle (the device kernel is checked against the same oracle and the
same doc_base semantics in tests/test_gpu_parity.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_03851_b200.sharding import shard_csr, shard_ranges


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=3):
    gen = np.random.default_rng(seed)
    M, V, K = 256, 120, 48
    N = np.maximum(gen.poisson(15, size=M), 0)
    N[::17] = 0
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int64)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    return M, V, K, N, off, words, theta, phi


def _worker(rank, world, port, out_dir):
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M, V, K, N, off, words, theta, phi = _problem()
    lo, hi = shard_ranges(N, world)[rank]
    soff, swords = shard_csr(off, words, lo, hi)
    seed = O.derive_seed(7, 1, 0)
    z, err = O.draw_z_csr(theta[lo:hi], phi, soff, swords, W=32, seed=seed, doc_base=lo)
    assert err is None
    _, wt = O.topic_counts(soff, swords, z, K, V)
    wt_t = torch.from_numpy(wt.astype(np.int32))
    dist.all_reduce(wt_t)
    np.save(os.path.join(out_dir, f"z{rank}.npy"), z)
    np.save(os.path.join(out_dir, f"wt{rank}.npy"), wt_t.numpy())
    dist.destroy_process_group()


def test_shard_ranges_aligned_and_balanced():
    gen = np.random.default_rng(0)
    N = gen.poisson(200, size=32 * 1000)
    for world in (1, 2, 3, 4, 8):
        r = shard_ranges(N, world)
        assert r[0][0] == 0 and r[-1][1] == N.size
        assert all(a % 32 == 0 and b % 32 == 0 and a <= b for a, b in r)
        assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        tok = [int(N[a:b].sum()) for a, b in r]
        assert max(tok) - min(tok) <= 2 * int(N.reshape(-1, 32).sum(1).max())
    with pytest.raises(ValueError):
        shard_ranges(np.ones(33), 2)


def test_two_rank_gloo_matches_single_process(tmp_path):
    from oracle import oracle as O

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    M, V, K, N, off, words, theta, phi = _problem()
    z_full, err = O.draw_z_csr(theta, phi, off, words, W=32, seed=O.derive_seed(7, 1, 0))
    _, wt_full = O.topic_counts(off, words, z_full, K, V)
    z_parts = np.concatenate([np.load(tmp_path / f"z{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(z_parts, z_full)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"wt{r}.npy"), wt_full)


def _tile_worker(rank, world, port, out_dir):
    """Per-tile overlapped all-reduce (sharding.TileAllReduce as DeviceLDA
    drives it): counts are produced tile by tile, each rank skips the tiles
    its shard has no tokens in, and the collective sequence must still line
    up across ranks and give the full counts."""
    from oracle import oracle as O
    from paper_1505_03851_b200.sharding import TileAllReduce, count_chunks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M, V, K, N, off, words, theta, phi = _problem()
    # rank 1 has no tokens in words [40, 80): drop them from its shard
    lo, hi = shard_ranges(N, world)[rank]
    soff, swords = shard_csr(off, words, lo, hi)
    z, err = O.draw_z_csr(theta[lo:hi], phi, soff, swords, W=32, seed=O.derive_seed(7, 1, 0), doc_base=lo)
    keep = np.ones(swords.size, bool) if rank == 0 else ~((swords >= 40) & (swords < 80))
    rows = 20
    wt = torch.zeros((V, K), dtype=torch.int32)
    red = TileAllReduce(wt, count_chunks(V, rows), lambda v: dist.all_reduce(v, async_op=True))
    tile = swords // rows
    for t in range(int(tile.max()) + 1):
        sel = keep & (tile == t)
        if not sel.any():
            continue  # no launch for an empty tile
        np.add.at(wt.numpy(), (swords[sel], z[sel]), 1)
        red.after_tile(t, t * rows, min(V, (t + 1) * rows))
    red.finish()
    red.wait()
    local = np.zeros((V, K), np.int64)
    np.add.at(local, (swords[keep], z[keep]), 1)
    np.save(os.path.join(out_dir, f"tiles_wt{rank}.npy"), wt.numpy())
    np.save(os.path.join(out_dir, f"tiles_local{rank}.npy"), local)
    dist.destroy_process_group()


def test_count_chunks_cover_vocab():
    from paper_1505_03851_b200.sharding import count_chunks

    assert count_chunks(100, None) == [(0, 100)]
    c = count_chunks(101, 20)
    assert c[0] == (0, 20) and c[-1] == (100, 101) and all(c[i][1] == c[i + 1][0] for i in range(len(c) - 1))


def test_two_rank_gloo_tile_allreduce(tmp_path):
    world = 2
    mp.start_processes(_tile_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    total = sum(np.load(tmp_path / f"tiles_local{r}.npy") for r in range(world))
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"tiles_wt{r}.npy"), total)


def _bench_args(scaling):
    import argparse

    return argparse.Namespace(seed=5, docs=1000, mean_len=20.0, vocab=300, scaling=scaling)


def _strong_shard_worker(rank, world, port, out_dir):
    """bench.make_shard under --scaling strong: every rank generates the same
    corpus and keeps its shard_ranges slice; the gathered shards must tile
    the corpus exactly (documents, offsets, words, global doc ids)."""
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, words, doc_base = bench.make_shard(torch, rank, world, _bench_args("strong"), torch.device("cpu"))
    meta = torch.tensor([doc_base, off.numel() - 1, words.numel()], dtype=torch.int64)
    metas = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(metas, meta)
    np.save(os.path.join(out_dir, f"off{rank}.npy"), off.numpy())
    np.save(os.path.join(out_dir, f"words{rank}.npy"), words.numpy())
    np.save(os.path.join(out_dir, f"meta{rank}.npy"), torch.stack(metas).numpy())
    dist.destroy_process_group()


def test_two_rank_gloo_strong_shards_tile_the_corpus(tmp_path):
    import bench

    world = 2
    mp.start_processes(_strong_shard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    off1, words1, base1 = bench.make_shard(torch, 0, 1, _bench_args("strong"), torch.device("cpu"))
    assert base1 == 0
    metas = np.load(tmp_path / "meta0.npy")
    np.testing.assert_array_equal(metas, np.load(tmp_path / "meta1.npy"))
    assert metas[0, 0] == 0 and metas[1, 0] == metas[0, 1]  # contiguous, 32-aligned cuts
    assert metas[1, 0] % 32 == 0 and metas[:, 1].sum() == off1.numel() - 1
    words = np.concatenate([np.load(tmp_path / f"words{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(words, words1.numpy())
    lens = np.concatenate([np.diff(np.load(tmp_path / f"off{r}.npy")) for r in range(world)])
    np.testing.assert_array_equal(lens, np.diff(off1.numpy()))
    tok = metas[:, 2]
    assert abs(int(tok[0]) - int(tok[1])) < 0.05 * tok.sum()  # token-balanced
    # weak scaling: rank r's corpus is its own (seed + r), doc_base = r x M
    offw, _, basew = bench.make_shard(torch, 1, 2, _bench_args("weak"), torch.device("cpu"))
    assert basew == offw.numel() - 1
