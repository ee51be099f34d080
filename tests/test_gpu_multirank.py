"""Multi-rank DeviceLDA on ONE GPU (gloo backend, both ranks on cuda:0): a
2-shard run must reproduce the single-process run exactly -- z, the
all-reduced word-topic counts, phi and theta -- because shards are
32-aligned, keys use global document ids and every Gamma stream is keyed by
(seed, global row, topic).  This exercises the same code path bench.py runs
over NCCL on N GPUs (only the all-reduce transport differs)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    gen = np.random.default_rng(12)
    M, V, K = 512, 700, 96
    N = np.maximum(gen.poisson(40, size=M), 0)
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
    return M, V, K, N, off, words


def _run(rank, world, port, out_dir, iters, host=False):
    import paper_1505_03851_b200 as wd
    from paper_1505_03851_b200.device_lda import DeviceLDA
    from paper_1505_03851_b200.sharding import shard_csr, shard_ranges

    torch.cuda.set_device(0)
    M, V, K, N, off, words = _problem()
    pg = None
    lo, hi = 0, M
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist.group.WORLD
        lo, hi = shard_ranges(N, world)[rank]
    soff, swords = shard_csr(off, words, lo, hi)
    dc = wd.DeviceCorpus.from_csr(soff, swords, doc_base=lo)
    lda = DeviceLDA(dc, K, V, seed=5, process_group=pg, vocab_tile_bytes=64 * K * 4)
    lda.init_from_assignments()
    if host:  # parameters entering from pinned host memory each iteration
        th_h = lda.theta.cpu().pin_memory()
        ph_h = lda.phi.cpu().pin_memory()
        lda.iterate_from_host(0, iters, th_h, ph_h)
        torch.cuda.synchronize()
    else:
        for t in range(iters):
            lda.iterate(t)
    lda.check_errors()
    ll = lda.log_likelihood()
    np.savez(os.path.join(out_dir, f"{'h' if host else 'r'}{world}_{rank}.npz"), z=lda.z.cpu().numpy(), theta=lda.theta.cpu().numpy(),
             phi=lda.phi.cpu().numpy(), wt=lda.word_topic.cpu().numpy(), ll=np.array(ll),
             sharded=np.array(lda.shard_phi))
    if world > 1:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ranks_reproduce_one(tmp_path, world):
    """N > 1 runs the sharded phi resample (each rank its share of the row
    chunks, column partials and rows all-gathered): phi must still be the
    1-rank phi bit for bit, and with it the whole chain."""
    iters = 3
    _run(0, 1, 0, str(tmp_path), iters)
    mp.start_processes(_run, args=(world, _free_port(), str(tmp_path), iters), nprocs=world, join=True,
                       start_method="spawn")
    one = np.load(tmp_path / "r1_0.npz")
    parts = [np.load(tmp_path / f"r{world}_{r}.npz") for r in range(world)]
    assert all(bool(p["sharded"]) for p in parts)
    np.testing.assert_array_equal(np.concatenate([p["z"] for p in parts]), one["z"])
    np.testing.assert_array_equal(np.concatenate([p["theta"] for p in parts]), one["theta"])
    for p in parts:
        np.testing.assert_array_equal(p["wt"], one["wt"])
        np.testing.assert_array_equal(p["phi"], one["phi"])
        assert abs(float(p["ll"]) - float(one["ll"])) <= 1e-9 * abs(float(one["ll"]))


def test_two_ranks_reproduce_one_from_host(tmp_path):
    """iterate_from_host (double-buffered theta / phi uploads) with the
    sharded phi resample: 2 ranks equal 1 rank."""
    iters = 2
    _run(0, 1, 0, str(tmp_path), iters, True)
    mp.start_processes(_run, args=(2, _free_port(), str(tmp_path), iters, True), nprocs=2, join=True,
                       start_method="spawn")
    one = np.load(tmp_path / "h1_0.npz")
    parts = [np.load(tmp_path / f"h2_{r}.npz") for r in range(2)]
    np.testing.assert_array_equal(np.concatenate([p["z"] for p in parts]), one["z"])
    for p in parts:
        np.testing.assert_array_equal(p["phi"], one["phi"])


def test_bench_nccl_path_world1():
    """bench.py's N > 1 code path (NCCL process group, per-tile async count
    all-reduces, max-over-ranks timing) exercised at world size 1 under
    torchrun: one valid JSON line."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1", "--force-dist", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--no-sampler", "--no-dropin", "--docs", "64000", "--vocab", "40000"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["roofline"]["launches_per_draw"] == 4
    assert line["roofline"]["bound"] == "l2" and 0 < line["roofline"]["frac"] <= 1.2
    assert line["scaling"] == "strong" and line["tokens_per_step"] == line["tokens_rank0"]
    assert "nranks 1" in r.stderr or "nRanks 1" in r.stderr  # NCCL communicator line (NCCL_DEBUG=INFO)


@pytest.mark.parametrize("world", [2, 4])
def test_bench_multirank_flow_gloo(world):
    """bench.py --gpus N as the driver launches it (torchrun, N ranks), with
    the gloo backend so every rank can share the one GPU: the sharded
    corpus, per-tile count all-reduces, sharded phi resample, max-over-ranks
    timing and the single JSON line from rank 0 (numbers meaningless: the
    ranks share a GPU)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(world),
           "--dist-backend", "gloo", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-sampler", "--no-dropin",
           "--docs", "64000", "--vocab", "40000"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"].startswith(f"dp{world}")
    assert line["tokens_per_step"] > line["tokens_rank0"] > 0
    assert line["roofline"]["draw_ms_max_over_ranks"] >= line["roofline"]["draw_ms"] * 0.999
