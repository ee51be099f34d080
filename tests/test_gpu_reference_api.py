"""GPU: the drop-in through the reference's OWN public API, and the boundary's
robustness cases.

The reference package `warpdraw` is imported unmodified from baseline/_ref
(pip-installed there, git-ignored, travels to the GPU box) or from
/root/reference in the build container.  integrate.install() patches its
registries; the reference's own run_gibbs (lda.py:245-286) must then
reproduce the golden output the unpatched reference produced (cfg1.npz:
z, theta/phi SHA-256, log-likelihood trajectory, BASELINE configs[0])."""

import hashlib
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import _lib  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402
from oracle import oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_path():
    for cand in (os.environ.get("WARPDRAW_REF"), os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if cand and os.path.isdir(os.path.join(cand, "warpdraw")):
            return cand
    return None


@pytest.fixture
def warpdraw():
    ref = _reference_path()
    if ref is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    sys.path.insert(0, ref)
    import warpdraw as w
    import warpdraw.bench  # noqa: F401
    import warpdraw.kernels  # noqa: F401
    import warpdraw.lda  # noqa: F401
    from paper_1505_03851_b200 import integrate

    integrate.install()
    try:
        yield w
    finally:
        integrate.uninstall()
        sys.path.remove(ref)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_reference_run_gibbs_through_install_equals_golden(warpdraw, golden):
    """warpdraw.lda.run_gibbs(cfg1) with draw_z patched onto the GPU: z, the
    numpy-resampled theta/phi (SHA-256) and the log-likelihood trajectory are
    the unpatched reference's, bit for bit."""
    g = golden("cfg1")
    N = g["N"]
    off = np.concatenate([[0], np.cumsum(N)])
    words = g["words"].astype(np.int64)
    corpus = warpdraw.lda.Corpus(vocab_size=5000, lengths=N,
                                 words=[words[off[m]:off[m + 1]] for m in range(N.size)])
    params, z, ll = warpdraw.lda.run_gibbs(corpus, 64, 10, "butterfly", warpdraw.warp.WarpConfig(32, 4), 7,
                                           dtype=np.float32)
    np.testing.assert_array_equal(np.concatenate(z), g["z"].astype(np.int64))
    assert _sha(params.theta) == str(g["theta_sha"])
    assert _sha(params.phi) == str(g["phi_sha"])
    np.testing.assert_array_equal(ll, g["ll"])


def test_reference_draw_z_registry_equals_golden(warpdraw, golden):
    """warpdraw.kernels.draw_z / KERNELS[...] (patched) on the golden ragged
    LDA cases: every kernel, seeded and injected stops."""
    g = golden("lda")
    n = 0
    for i in range(int(g["n_cases"])):
        W, K, M, V, seed, dt_code, injected = (int(x) for x in g[f"c{i}_meta"])
        N = g[f"c{i}_N"]
        off = np.concatenate([[0], np.cumsum(N)])
        flat = g[f"c{i}_words"].astype(np.int64)
        w = [flat[off[m]:off[m + 1]] for m in range(N.size)]
        theta, phi = g[f"c{i}_theta"], g[f"c{i}_phi"]
        if injected:
            u = g[f"c{i}_units"]
            stops = warpdraw.kernels.InjectedStops([u[off[m]:off[m + 1]] for m in range(N.size)])
        else:
            stops = warpdraw.kernels.SeededStops(seed)
        for kname in ("butterfly", "transposed", "basic"):
            z = warpdraw.kernels.draw_z(kname, N, theta, phi, w, warpdraw.warp.WarpConfig(W, theta.itemsize), stops)
            got = np.concatenate([np.asarray(x) for x in z])
            np.testing.assert_array_equal(got, g[f"c{i}_z_{kname}"].astype(np.int64), err_msg=f"case {i} {kname}")
            assert all(x.dtype == np.int64 for x in z)
            n += 1
    assert n > 0


def test_reference_errors_through_install(warpdraw):
    """AllZeroError / OutOfBoundsError come out as the reference's classes."""
    N = np.array([3] + [0] * 31)
    w = [np.array([0, 1, 2])] + [np.zeros(0, np.int64)] * 31
    phi = np.ones((4, 8), np.float32)
    theta = np.zeros((32, 8), np.float32)
    cfg = warpdraw.warp.WarpConfig(32, 4)
    with pytest.raises(warpdraw.sampling.AllZeroError, match="document 0: all products are zero"):
        warpdraw.kernels.draw_z("butterfly", N, theta, phi, w, cfg, warpdraw.kernels.SeededStops(1))
    theta[:] = 1
    w[0] = np.array([0, 9, 2])  # word 9 >= V = 4
    with pytest.raises(warpdraw.warp.OutOfBoundsError):
        warpdraw.kernels.draw_z("butterfly", N, theta, phi, w, cfg, warpdraw.kernels.SeededStops(1))


# ------------------------------------------------------ boundary robustness
def test_word_id_out_of_range_raises_before_launch():
    off = np.array([0, 2, 4], dtype=np.int64)
    dc = wd.DeviceCorpus.from_csr(off, np.array([0, 5, 1, 2], np.int32))
    theta = torch.ones((2, 32), device="cuda")
    phi = torch.ones((5, 32), device="cuda")
    with pytest.raises(wd.OutOfBoundsError):
        wd.draw_z_device("basic", dc, theta, phi, wd.SeededStops(1))
    dc2 = wd.DeviceCorpus.from_csr(off, np.array([0, -1, 1, 2], np.int32))
    with pytest.raises(IndexError):
        wd.draw_z_device("basic", dc2, theta, phi, wd.SeededStops(1))
    with pytest.raises(wd.OutOfBoundsError):
        wd.DeviceCorpus.from_csr(off, np.array([0, 1 << 40, 1, 2], np.int64))


def test_empty_vocabulary_tiles_and_empty_shard_do_not_raise():
    """A shard with no tokens in some vocabulary tiles (the err rows of the
    tiles it skips must read ERR_NONE), and a shard with no tokens at all."""
    gen = np.random.default_rng(5)
    M, V, K = 64, 4000, 64
    N = np.maximum(gen.poisson(20, size=M), 1)
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    # words in the first and last eighth of V only: the middle tiles are empty
    words = gen.integers(0, V // 4, size=int(off[-1]))
    words = np.where(words < V // 8, words, words + 3 * V // 4).astype(np.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    lda = DeviceLDA(dc, K, V, seed=3, vocab_tile_bytes=K * 4 * 500)  # 8 tiles, 6 of them empty
    assert lda.tiles.n_tiles == 8
    assert sum(b > a for a, b in zip(lda.tiles.bounds[:-1], lda.tiles.bounds[1:])) == 2
    lda.err.fill_(0)  # stale garbage in every row
    lda.init_uniform()
    lda.iterate(0)
    torch.cuda.synchronize()
    lda.check_errors()
    # empty shard (32 empty documents)
    dc0 = wd.DeviceCorpus.from_csr(np.zeros(33, np.int64), np.zeros(0, np.int32))
    lda0 = DeviceLDA(dc0, K, V, seed=3, vocab_tile_bytes=K * 4 * 500)
    lda0.err.fill_(0)
    lda0.init_uniform()
    lda0.iterate(0)
    torch.cuda.synchronize()
    lda0.check_errors()
    z = wd.draw_z_device("butterfly", dc0, lda0.theta, lda0.phi, wd.SeededStops(1), tiles=dc0.vocab_tiles(500))
    assert z.numel() == 0


def test_host_corpus_cache_hits_and_invalidates():
    """The reference-signature path caches the CSR upload per word-list
    object: the second call reuses it; a changed list or changed lengths
    rebuild it (same z as a fresh call either way)."""
    from paper_1505_03851_b200 import kernels as K

    gen = np.random.default_rng(9)
    M, V, Kt = 64, 300, 40
    N = np.maximum(gen.poisson(10, size=M), 1)
    w = [gen.integers(0, V, size=int(n)) for n in N]
    theta = gen.uniform(0.1, 1, size=(M, Kt)).astype(np.float32)
    phi = gen.uniform(0.1, 1, size=(V, Kt)).astype(np.float32)
    K._host_corpora.clear()
    cfg = wd.WarpConfig(32, 4)
    z1 = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(4))
    c1 = K._host_corpora.entries[0][3]
    z2 = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(4))
    assert K._host_corpora.entries[0][3] is c1
    for a, b in zip(z1, z2):
        np.testing.assert_array_equal(a, b)
    w[3] = (w[3] + 1) % V  # a new array object in the same list
    z3 = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(4))
    assert K._host_corpora.entries[0][3] is not c1
    K._host_corpora.clear()
    z4 = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(4))
    for a, b in zip(z3, z4):
        np.testing.assert_array_equal(a, b)


def test_large_call_pinned_result_buffers():
    """Above _ASYNC_OUT_MIN tokens the reference-signature call returns z as
    views of a pooled pinned buffer: results kept by the caller are never
    overwritten by later calls (the pool hands out only buffers with no live
    views, and falls back to fresh memory when all are held), equal the
    oracle, and an AllZero document still raises after the asynchronous
    download."""
    from paper_1505_03851_b200 import kernels as K

    gen = np.random.default_rng(21)
    M, V, Kt = 2048, 500, 72
    N = np.maximum(gen.poisson(60, size=M), 1)
    assert N.sum() >= K._ASYNC_OUT_MIN
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    flat = gen.integers(0, V, size=int(off[-1]))
    w = [flat[a:b] for a, b in zip(off[:-1], off[1:])]
    theta = gen.uniform(0.1, 1, size=(M, Kt)).astype(np.float32)
    phi = gen.uniform(0.1, 1, size=(V, Kt)).astype(np.float32)
    cfg = wd.WarpConfig(32, 4)
    K._z_out_pool.clear()
    kept = []
    for seed in range(K._Z_OUT_POOL_MAX + 2):  # more results held than pool buffers
        z = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(seed))
        kept.append((seed, z))
    assert len(K._z_out_pool) == K._Z_OUT_POOL_MAX
    for seed, z in kept:
        exp, err = O.draw_z_csr(theta, phi, off, flat, W=32, seed=seed, threads=8)
        assert err is None
        np.testing.assert_array_equal(np.concatenate(z), exp)
        assert z[0].dtype == np.int64 and len(z) == M
    # dropping a result frees its buffer for the next call (no new buffer)
    bufs = [e[0].data_ptr() for e in K._z_out_pool]
    del kept[1:3]
    z = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(99))
    assert [e[0].data_ptr() for e in K._z_out_pool] == bufs
    exp, _ = O.draw_z_csr(theta, phi, off, flat, W=32, seed=99, threads=8)
    np.testing.assert_array_equal(np.concatenate(z), exp)
    np.testing.assert_array_equal(np.concatenate(kept[0][1]),
                                  O.draw_z_csr(theta, phi, off, flat, W=32, seed=0, threads=8)[0])
    # the other two kernels and injected stops on the same path
    u = gen.random(int(off[-1]))
    ragged_u = [u[a:b] for a, b in zip(off[:-1], off[1:])]
    for kern, variant, rule in (("transposed", O.PREFIX, O.KEY_MASTER), ("basic", O.PREFIX, O.KEY_POSITION)):
        z = wd.draw_z(kern, N, theta, phi, w, cfg, wd.SeededStops(5))
        exp, _ = O.draw_z_csr(theta, phi, off, flat, W=32, seed=5, variant=variant, key_rule=rule, threads=8)
        np.testing.assert_array_equal(np.concatenate(z), exp)
    z = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.InjectedStops(ragged_u))
    np.testing.assert_array_equal(np.concatenate(z), O.draw_z_csr(theta, phi, off, flat, W=32, units_=u, threads=8)[0])
    # the error check still runs on the asynchronous path
    theta[777] = 0
    with pytest.raises(wd.AllZeroError, match=r"^document 777: all products are zero$"):
        wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(1))
    with pytest.raises(wd.AllZeroError, match=r"^document 777, word 0: all products are zero$"):
        wd.draw_z("basic", N, theta, phi, w, cfg, wd.SeededStops(1))


def test_topic_counts_through_install_equal_numpy(warpdraw):
    """warpdraw.lda.topic_counts after install(): the GPU counts equal the
    reference's own np.add.at counts, including its index rules (negative z
    wraps, z >= K and word ids >= V raise IndexError)."""
    from paper_1505_03851_b200 import integrate

    ref = integrate._saved["lda"][2]  # the reference's own topic_counts
    gpu = warpdraw.lda.topic_counts
    assert gpu is not ref
    gen = np.random.default_rng(31)
    M, V, Kt = 96, 150, 24
    N = gen.poisson(12, size=M)
    N[5] = 0
    w = [gen.integers(0, V, size=int(n)) for n in N]
    corpus = warpdraw.lda.Corpus(lengths=N.astype(np.int64), words=w, vocab_size=V)
    z = [gen.integers(0, Kt, size=int(n)) for n in N]
    z[7] = z[7] - Kt  # negative topics wrap in np.add.at
    exp_dt, exp_wt = ref(corpus, z, Kt)
    got_dt, got_wt = gpu(corpus, z, Kt)
    assert got_dt.dtype == np.int64 and got_wt.dtype == np.int64
    np.testing.assert_array_equal(got_dt, exp_dt)
    np.testing.assert_array_equal(got_wt, exp_wt)
    bad = list(z)
    bad[3] = bad[3].copy()
    bad[3][0] = Kt
    with pytest.raises(IndexError):
        gpu(corpus, bad, Kt)
    w_bad = list(w)
    w_bad[2] = w_bad[2].copy()
    w_bad[2][0] = V
    with pytest.raises(IndexError):
        gpu(warpdraw.lda.Corpus(lengths=corpus.lengths, words=w_bad, vocab_size=V), z, Kt)
