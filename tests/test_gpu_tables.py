"""GPU: the split table / search API (build_block_tables kernels.py:580-600,
butterfly_search kernels.py:317-362) against golden vectors the reference
produced (tests/golden/make_golden_tables.py): every table entry and every
index bit-exact, W = 2..64, fp32 / fp64, K below / at / above W with
remnants, batched and unbatched, all-zero lanes."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402


def _cases(golden):
    g = golden("tables")
    for ci, (W, K, nbatch, esz) in enumerate(g["meta"]):
        yield ci, int(W), int(K), int(nbatch), g


def test_tables_and_search_match_reference_golden(golden):
    n = 0
    for ci, W, K, nbatch, g in _cases(golden):
        prods = g[f"prods_{ci}"]
        warp, p, sums = wd.build_block_tables(prods, wd.WarpConfig(lanes=W, elem_size=prods.dtype.itemsize))
        assert p.data.shape == g[f"p_{ci}"].shape and p.length == K
        np.testing.assert_array_equal(p.numpy(), g[f"p_{ci}"], err_msg=f"case {ci} W={W} K={K}")
        np.testing.assert_array_equal(sums, g[f"sums_{ci}"], err_msg=f"case {ci}")
        idx = wd.butterfly_search(warp, p, sums, g[f"stops_{ci}"])
        np.testing.assert_array_equal(idx, g[f"idx_{ci}"], err_msg=f"case {ci} W={W} K={K}")
        snap = wd.table_snapshot(p, sums)
        assert snap.lanes == W and np.array_equal(snap.p, g[f"p_{ci}"])
        n += 1
    assert n == 144


def test_search_errors_and_broadcast_stops():
    W, K = 8, 21
    prods = np.random.default_rng(1).uniform(0.1, 1, size=(4, W, K)).astype(np.float32)
    warp, p, sums = wd.build_block_tables(prods, wd.WarpConfig(lanes=W))
    bad = sums.copy()  # stop == sum is out of range
    with pytest.raises(wd.StopOutOfRangeError, match=r"stop values must lie in \[0, sum\)"):
        wd.butterfly_search(warp, p, sums, bad)
    with pytest.raises(wd.StopOutOfRangeError):
        wd.butterfly_search(warp, p, sums, -np.ones_like(sums))
    with pytest.raises(NotImplementedError):
        wd.butterfly_search(warp, p, sums, sums * 0, observer=lambda s: None)
    # one shared row of stops broadcast over the batch (bench.py:146 style)
    stops = (sums[0] * 0.5).astype(np.float32)
    got = wd.butterfly_search(warp, p, np.broadcast_to(sums, sums.shape), np.broadcast_to(stops, sums.shape))
    assert got.shape == (4, W) and got.dtype == np.int64
    with pytest.raises(ValueError, match="one row per lane"):
        wd.build_block_tables(prods[:, :4], wd.WarpConfig(lanes=W))
    with pytest.raises(ValueError, match="batched builds cannot be traced"):
        wd.build_block_tables(prods, wd.WarpConfig(lanes=W), trace=wd.Trace())


def test_large_batch_matches_fused_row_sampler():
    """2^16 warp groups through build + search equal the fused standalone
    sampler (wd_sample_rows) drawing the same rows with the same stops."""
    W, K, G = 32, 200, 1 << 12
    rng = np.random.default_rng(3)
    prods = rng.uniform(0.0, 1.0, size=(G, W, K)).astype(np.float32)
    warp, p, sums = wd.build_block_tables(prods, wd.WarpConfig(lanes=W))
    u = rng.random(sums.shape)
    stops = np.minimum((sums * u.astype(np.float32)).astype(np.float32),
                       np.nextafter(sums, 0).astype(np.float32))
    idx = wd.butterfly_search(warp, p, sums, stops)
    # the same rows as independent standalone rows (row id = g * W + lane: r = lane)
    rows = torch.from_numpy(prods.reshape(G * W, K)).cuda()
    fused = wd.sample_rows(rows, 0, lanes=W, stops=torch.from_numpy(stops.reshape(-1)).cuda()).cpu().numpy()
    np.testing.assert_array_equal(idx.reshape(-1), fused)
