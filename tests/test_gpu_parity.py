"""GPU parity: the sm_100a kernels against the reference's golden vectors and
the pinned CPU oracle, bit-exact (integer z / index outputs)."""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------ u stream
def test_device_units_match_reference_kat(golden):
    g = golden("units")
    got = wd.units_for(int(g["big_seed"]), g["bm"], g["bk"])
    np.testing.assert_array_equal(got, g["ubig"])
    seeds, k0, k1, sidx = g["seeds"], g["k0"], g["k1"], g["sidx"]
    for s_i in np.unique(sidx)[:16]:
        sel = sidx == s_i
        np.testing.assert_array_equal(wd.units_for(int(seeds[s_i]), k0[sel], k1[sel]), g["u2"][sel])
        np.testing.assert_array_equal(wd.units_for(int(seeds[s_i]), k0[sel]), g["u1"][sel])
    assert wd.units_for(0) == 0.6012629994179048


def test_device_units_million_keys_vs_oracle():
    gen = np.random.default_rng(1)
    m = gen.integers(0, 10**7, size=1 << 20)
    i = gen.integers(0, 4096, size=1 << 20)
    seed = wd.derive_seed(2026, 1, 3)
    np.testing.assert_array_equal(wd.units_for(seed, m, i), O.units(seed, m, i))


# ----------------------------------------------------------- standalone rows
def _row_cases(g):
    for i in range(int(g["n_cases"])):
        yield i, g[f"c{i}_meta"], g[f"c{i}_w"], g[f"c{i}_stops"], g[f"c{i}_idx"]


def test_rows_vs_reference_golden(golden):
    g = golden("rows")
    for i, meta, w, stops, idx in _row_cases(g):
        W, K, rows, seed, dt_code, kind = (int(x) for x in meta)
        wt = _cuda(w)
        if kind == 0:
            got = wd.sample_rows(wt, seed, lanes=W, check=False)
        else:
            got = wd.sample_rows(wt, lanes=W, stops=_cuda(stops), check=False)
        np.testing.assert_array_equal(got.cpu().numpy(), idx, err_msg=f"case {i} W={W} K={K} dt={dt_code}")


def test_shared_vector_samplers_vs_reference_golden(golden):
    g = golden("rows")
    np.testing.assert_array_equal(wd.sample_butterfly(g["sampler_w"], 20000, seed=61), g["sampler_draws"])
    np.testing.assert_array_equal(wd.sample_butterfly(g["sampler_w32"], 5000, seed=5, lanes=32),
                                  g["sampler_draws32"])
    assert set(wd.SAMPLERS) >= {"butterfly", "prefix"}


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("K", [1, 5, 19, 32, 64, 100, 200, 256, 1000, 1024, 2048, 4096])
def test_rows_vs_oracle(dtype, K):
    gen = np.random.default_rng(K)
    n = 2048 if K <= 1024 else 512
    w = gen.uniform(0.1, 1.0, size=(n, K)).astype(dtype)
    if K > 8:
        w[:, 3::7] = 0
    seed = 1234 + K
    for W in (32, 8) if dtype == np.float32 else (32,):
        got = wd.sample_rows(_cuda(w), seed, lanes=W).cpu().numpy()
        exp = O.sample_rows(w, W, wd.derive_seed(seed, 6), threads=8)
        np.testing.assert_array_equal(got, exp, err_msg=f"W={W}")
    got = wd.sample_rows(_cuda(w), seed, lanes=32, variant="prefix").cpu().numpy()
    exp = O.sample_rows(w, 32, wd.derive_seed(seed, 6), variant=O.PREFIX, threads=8)
    np.testing.assert_array_equal(got, exp)


def test_rows_kernel_smem_revisit():
    """One kernel instantiation launched with a large, then a smaller, then the
    large dynamic shared-memory size again (the opt-in limit is per function and
    must never be lowered under a cached launch configuration)."""
    gen = np.random.default_rng(5)
    for K in (1024, 512, 1024, 2048, 512, 2048):
        w = gen.uniform(0.1, 1.0, size=(1024, K)).astype(np.float32)
        got = wd.sample_rows(_cuda(w), K, lanes=32).cpu().numpy()
        np.testing.assert_array_equal(got, O.sample_rows(w, 32, wd.derive_seed(K, 6), threads=8), err_msg=f"K={K}")


@pytest.mark.parametrize("W", [2, 4, 16, 64])
def test_rows_other_lane_counts_vs_oracle(W):
    gen = np.random.default_rng(W)
    for K in (W - 1, W, 3 * W + 1, 7 * W):
        if K < 1:
            continue
        w = gen.uniform(0, 1, size=(640, K))
        got = wd.sample_rows(_cuda(w), 9, lanes=W).cpu().numpy()
        np.testing.assert_array_equal(got, O.sample_rows(w, W, wd.derive_seed(9, 6)))


def test_rows_strided_and_row_base():
    gen = np.random.default_rng(3)
    big = gen.uniform(0.1, 1, size=(1000, 260)).astype(np.float32)
    view = _cuda(big)[:, :200]  # ld = 260, vector path
    got = wd.sample_rows(view, 5, lanes=32, row_base=777).cpu().numpy()
    exp = O.sample_rows(np.ascontiguousarray(big[:, :200]), 32, wd.derive_seed(5, 6), row0=777)
    np.testing.assert_array_equal(got, exp)
    view = _cuda(big)[:, 1:200]  # misaligned rows -> scalar path
    got = wd.sample_rows(view, 5, lanes=32).cpu().numpy()
    exp = O.sample_rows(np.ascontiguousarray(big[:, 1:200]), 32, wd.derive_seed(5, 6))
    np.testing.assert_array_equal(got, exp)


def test_rows_integer_regime_midpoints_exact():
    gen = np.random.default_rng(14)
    for W, K in ((8, 19), (32, 240), (32, 1024)):
        w = gen.integers(1, 2**20, size=(256, K)).astype(np.float64)
        prefix = np.cumsum(w, axis=-1)
        target = gen.integers(0, K, size=256)
        stops = prefix[np.arange(256), target] - 0.5
        got = wd.sample_rows(_cuda(w), lanes=W, stops=_cuda(stops)).cpu().numpy()
        np.testing.assert_array_equal(got, target)


def test_stop_out_of_range_and_allzero_rows():
    w = torch.ones((8, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(wd.StopOutOfRangeError):
        wd.sample_rows(w, lanes=8, stops=torch.full((8,), -0.1, dtype=torch.float64))
    with pytest.raises(wd.StopOutOfRangeError):
        wd.sample_rows(w, lanes=8, stops=torch.full((8,), 8.0, dtype=torch.float64))
    z = torch.zeros((4, 40), dtype=torch.float32, device="cuda")
    with pytest.raises(wd.AllZeroError):
        wd.sample_rows(z, 1)
    # the reference's search returns K-1 for an all-zero row (discarded lanes)
    assert (wd.sample_rows(z, 1, check=False).cpu().numpy() == 39).all()


def test_rows_empty():
    w = torch.ones((0, 16), dtype=torch.float32, device="cuda")
    assert wd.sample_rows(w, 1).numel() == 0


# ---------------------------------------------------------------- LDA draw
def _lda_cases(g):
    for i in range(int(g["n_cases"])):
        W, K, M, V, seed, dt_code, injected = (int(x) for x in g[f"c{i}_meta"])
        N = g[f"c{i}_N"]
        off = np.concatenate([[0], np.cumsum(N)])
        words = g[f"c{i}_words"]
        w = [words[off[m]:off[m + 1]].astype(np.int64) for m in range(M)]
        units = g[f"c{i}_units"] if injected else None
        yield i, W, K, seed, N, w, g[f"c{i}_theta"], g[f"c{i}_phi"], units


@pytest.mark.parametrize("kernel", ["basic", "transposed", "butterfly"])
def test_draw_z_vs_reference_golden(golden, kernel):
    g = golden("lda")
    for i, W, K, seed, N, w, theta, phi, units in _lda_cases(g):
        if units is None:
            stops = wd.SeededStops(seed)
        else:
            off = np.concatenate([[0], np.cumsum(N)])
            stops = wd.InjectedStops([units[off[m]:off[m + 1]] for m in range(len(N))])
        z = wd.draw_z(kernel, N, theta, phi, w, wd.WarpConfig(lanes=W, elem_size=theta.itemsize), stops)
        got = np.concatenate(z) if len(z) else np.zeros(0)
        np.testing.assert_array_equal(got, g[f"c{i}_z_{kernel}"], err_msg=f"case {i} W={W} K={K}")


def test_allzero_messages_match_reference(golden):
    g = golden("lda")
    theta = np.ones((8, 5), dtype=np.float32)
    theta[3] = 0
    theta[6] = 0
    phi = np.ones((4, 5), dtype=np.float32)
    N = np.array([1, 2, 0, 3, 1, 1, 2, 1])
    w = [np.zeros(int(n), dtype=np.int64) for n in N]
    for kern, msg in zip(("basic", "transposed", "butterfly"), g["allzero_msgs"]):
        with pytest.raises(wd.AllZeroError) as exc:
            wd.draw_z(kern, N, theta, phi, w, wd.WarpConfig(lanes=8, elem_size=4), wd.SeededStops(3))
        assert str(exc.value) == str(msg)


def test_draw_z_errors_and_hooks():
    N = np.array([1] * 6)
    theta = np.ones((6, 4))
    phi = np.ones((2, 4))
    w = [np.zeros(1, dtype=np.int64)] * 6
    with pytest.raises(ValueError, match="multiple"):
        wd.draw_z_butterfly(N, theta, phi, w, wd.WarpConfig(lanes=8), wd.SeededStops(1))
    with pytest.raises(ValueError, match="unknown kernel"):
        wd.draw_z("fancy", N, theta, phi, w, wd.WarpConfig(lanes=8), wd.SeededStops(1))
    with pytest.raises(NotImplementedError):
        wd.draw_z_butterfly(np.array([1] * 8), np.ones((8, 4)), phi, [np.zeros(1, dtype=np.int64)] * 8,
                            wd.WarpConfig(lanes=8), wd.SeededStops(1), step_hook=lambda *a: None)


def _random_corpus(gen, M, V, mean, zero_frac=0.05):
    N = gen.poisson(mean, size=M).astype(np.int64)
    N[gen.random(M) < zero_frac] = 0
    off = np.concatenate([[0], np.cumsum(N)])
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int64)
    return N, off, words


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("K", [1, 17, 64, 100, 200, 1024, 8192])
def test_lda_draw_vs_oracle(dtype, K):
    """Every kernel variant (all-remnant K < W, small, fine, coarse up to
    K = 8192; 256-bit segments when 32-byte aligned, 128-bit at K = 100
    whose remnant of 4 breaks that alignment) against the oracle, fp32 and
    fp64."""
    gen = np.random.default_rng(K)
    M, V = (1024, 700) if K <= 1024 else (128, 50)
    N, off, words = _random_corpus(gen, M, V, 30 if K < 1024 else 8)
    theta = gen.dirichlet(np.full(K, 0.1), size=M).astype(dtype)
    phi = gen.uniform(0.01, 1, size=(V, K)).astype(dtype)
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
    th, ph = _cuda(theta), _cuda(phi)
    seed = wd.derive_seed(7, 1, 0)
    for kernel, variant, rule in (("butterfly", O.BUTTERFLY, O.KEY_MASTER), ("transposed", O.PREFIX, O.KEY_MASTER),
                                  ("basic", O.PREFIX, O.KEY_POSITION)):
        z = wd.draw_z_device(kernel, dc, th, ph, wd.SeededStops(seed), 32).cpu().numpy()
        exp, err = O.draw_z_csr(theta, phi, off, words, W=32, seed=seed, variant=variant, key_rule=rule, threads=8)
        assert err is None
        np.testing.assert_array_equal(z, exp, err_msg=kernel)


def test_lda_injected_and_fused_counts_vs_oracle():
    gen = np.random.default_rng(5)
    M, V, K = 512, 300, 200
    N, off, words = _random_corpus(gen, M, V, 50)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    u = gen.random(int(off[-1]))
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
    wt = torch.zeros((V, K), dtype=torch.int32, device="cuda")
    dtc = torch.zeros((M, K), dtype=torch.int32, device="cuda")
    z = wd.draw_z_device("butterfly", dc, _cuda(theta), _cuda(phi), _cuda(u), 32, word_topic=wt, doc_topic=dtc)
    exp, _ = O.draw_z_csr(theta, phi, off, words, W=32, units_=u)
    np.testing.assert_array_equal(z.cpu().numpy(), exp)
    dt_e, wt_e = O.topic_counts(off, words, exp, K, V)
    np.testing.assert_array_equal(wt.cpu().numpy(), wt_e)
    np.testing.assert_array_equal(dtc.cpu().numpy(), dt_e)


def test_lda_shard_doc_base_matches_whole_corpus():
    """A 32-aligned document shard drawn with its global doc_base reproduces
    the whole-corpus draw for its tokens (multi-GPU parity)."""
    gen = np.random.default_rng(8)
    M, V, K = 256, 100, 64
    N, off, words = _random_corpus(gen, M, V, 20)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    seed = 99
    full = wd.draw_z_device("butterfly", wd.DeviceCorpus.from_csr(off, words.astype(np.int32)), _cuda(theta),
                            _cuda(phi), wd.SeededStops(seed), 32).cpu().numpy()
    lo, hi = 96, 224
    soff = off[lo:hi + 1] - off[lo]
    swords = words[off[lo]:off[hi]]
    dc = wd.DeviceCorpus.from_csr(soff, swords.astype(np.int32), doc_base=lo)
    part = wd.draw_z_device("butterfly", dc, _cuda(theta[lo:hi]), _cuda(phi), wd.SeededStops(seed), 32).cpu().numpy()
    np.testing.assert_array_equal(part, full[off[lo]:off[hi]])


def test_lda_empty_and_degenerate():
    dc = wd.DeviceCorpus.from_csr(np.zeros(33, dtype=np.int64), np.zeros(0, dtype=np.int32))
    z = wd.draw_z_device("butterfly", dc, torch.ones((32, 4), device="cuda"), torch.ones((3, 4), device="cuda"),
                         wd.SeededStops(1), 32)
    assert z.numel() == 0
    # K = 1: every draw is topic 0
    N = np.array([3] * 32)
    z = wd.draw_z_butterfly(N, np.ones((32, 1), np.float32), np.ones((5, 1), np.float32),
                            [np.array([0, 1, 2])] * 32, wd.WarpConfig(32, 4), wd.SeededStops(2))
    assert all((x == 0).all() for x in z)


# -------------------------------------------------------------- whole runs
def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_run_gibbs_whole_run_parity(golden, tag):
    g = golden("gibbs")
    M, V, K, iters, W, dt_code, seed = (int(x) for x in g[f"{tag}_meta"])
    kernel = str(g[f"{tag}_kernel"])
    N = g[f"{tag}_N"]
    off = np.concatenate([[0], np.cumsum(N)])
    words = g[f"{tag}_words"]
    corpus = wd.Corpus(vocab_size=V, lengths=N, words=[words[off[m]:off[m + 1]].astype(np.int64) for m in range(M)])
    dtype = np.float32 if dt_code == 0 else np.float64
    params, z, ll = wd.run_gibbs(corpus, K, iters, kernel, wd.WarpConfig(lanes=W, elem_size=np.dtype(dtype).itemsize),
                                 seed, dtype=dtype)
    np.testing.assert_array_equal(np.concatenate(z), g[f"{tag}_z"])
    assert _sha(params.theta) == str(g[f"{tag}_theta_sha"])
    assert _sha(params.phi) == str(g[f"{tag}_phi_sha"])
    np.testing.assert_array_equal(ll, g[f"{tag}_ll"])


def test_config1_whole_run_parity(golden):
    """BASELINE configs[0]: D=1000, V=5000, K=64, 10 iterations, fp32 butterfly."""
    import os

    from conftest import GOLDEN

    if not os.path.exists(os.path.join(GOLDEN, "cfg1.npz")):
        pytest.skip("cfg1 golden not generated")
    g = golden("cfg1")
    N = g["N"]
    off = np.concatenate([[0], np.cumsum(N)])
    words = g["words"].astype(np.int64)
    corpus = wd.Corpus(vocab_size=5000, lengths=N, words=[words[off[m]:off[m + 1]] for m in range(N.size)])
    params, z, ll = wd.run_gibbs(corpus, 64, 10, "butterfly", wd.WarpConfig(32, 4), 7, dtype=np.float32)
    np.testing.assert_array_equal(np.concatenate(z), g["z"].astype(np.int64))
    assert _sha(params.theta) == str(g["theta_sha"])
    assert _sha(params.phi) == str(g["phi_sha"])
    np.testing.assert_array_equal(ll, g["ll"])


# -------------------------------------------- full-size properties (bench shape)
def test_full_size_rows_k1024_properties():
    """n = 2^20 rows, K = 1024 (the bench shape): in-range, zero weights never
    drawn, a 4096-row random subset bit-exact vs the oracle, and the
    butterfly/prefix disagreement rate bounded (1.2e-4)."""
    n, K = 1 << 20, 1024
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.rand((n, K), generator=g, device="cuda", dtype=torch.float32) * 0.9 + 0.1
    w[:, 5::97] = 0
    zb = wd.sample_rows(w, 2026, lanes=32)
    zp = wd.sample_rows(w, 2026, lanes=32, variant="prefix")
    zbn = zb.cpu().numpy()
    assert zbn.min() >= 0 and zbn.max() < K
    picked = w.gather(1, zb.long()[:, None])
    assert bool((picked > 0).all())
    mism = float((zb != zp).float().mean())
    assert mism < 1e-3
    rows = np.sort(np.random.default_rng(1).choice(n, 4096, replace=False))
    sub = w[torch.from_numpy(rows).cuda()].cpu().numpy()
    seed6 = wd.derive_seed(2026, 6)
    exp = np.array([O.sample_rows(sub[j:j + 1], 32, seed6, row0=int(r))[0] for j, r in enumerate(rows)])
    np.testing.assert_array_equal(zbn[rows], exp)


@pytest.mark.parametrize("run_pad", [0, 8])
@pytest.mark.parametrize("kernel", ["butterfly", "transposed", "basic"])
def test_vocab_tiled_draw_identical(kernel, run_pad):
    """Drawing tile by tile over the vocabulary (phi slices L2-resident) gives
    the same z and counts as the untiled draw, for every kernel and stop mode,
    with and without (tile, document) runs padded to the lane-group height."""
    gen = np.random.default_rng(11)
    M, V, K = 640, 1000, 128
    N, off, words = _random_corpus(gen, M, V, 40)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
    th, ph = _cuda(theta), _cuda(phi)
    tiles = dc.vocab_tiles(137, run_pad)
    assert tiles.n_tiles == -(-V // 137)
    if run_pad:
        pos = tiles.token_pos.cpu().numpy()
        assert (pos >= 0).sum() == dc.n_tokens and tiles.bounds[-1] == pos.size > dc.n_tokens
        assert all(b % run_pad == 0 for b in tiles.bounds)
    else:
        assert tiles.bounds[-1] == dc.n_tokens
    u = _cuda(gen.random(int(off[-1])))
    for stops in (wd.SeededStops(5), u):
        wt0 = torch.zeros((V, K), dtype=torch.int32, device="cuda")
        wt1 = torch.zeros((V, K), dtype=torch.int32, device="cuda")
        z0 = wd.draw_z_device(kernel, dc, th, ph, stops, 32, word_topic=wt0)
        z1 = wd.draw_z_device(kernel, dc, th, ph, stops, 32, word_topic=wt1, tiles=tiles)
        np.testing.assert_array_equal(z0.cpu().numpy(), z1.cpu().numpy())
        np.testing.assert_array_equal(wt0.cpu().numpy(), wt1.cpu().numpy())
    exp, _ = O.draw_z_csr(theta, phi, off, words, W=32, seed=5,
                          variant=O.BUTTERFLY if kernel == "butterfly" else O.PREFIX,
                          key_rule=O.KEY_POSITION if kernel == "basic" else O.KEY_MASTER)
    z = wd.draw_z_device(kernel, dc, th, ph, wd.SeededStops(5), 32, tiles=tiles).cpu().numpy()
    np.testing.assert_array_equal(z, exp)


@pytest.mark.parametrize("K,M,words_kind,tiles", [(1024, 1_000_000, "uniform", 4), (1024, 1_000_000, "zipf", 4),
                                                   (200, 1_000_000, "zipf", 1), (2048, 1_000_000, "uniform", 8),
                                                   (4096, 1_250_016, "uniform", 16)])
def test_full_size_lda_sampled_tokens(K, M, words_kind, tiles):
    """The BASELINE shapes at full size through DeviceLDA (vocabulary-tiled,
    (document, word)-ordered, run-padded): configs[3] per GPU (1M documents,
    Poisson(200) lengths, V=40k, K=1024) uniform and Zipf; configs[2]
    Wikipedia-shaped (K=200, Zipf words: the small-K kernel); K=2048 and one
    rank's shard of configs[4] (1.25M documents, K=4096: the register-lean
    kernel).  4096 randomly chosen tokens are re-drawn one by one by the
    oracle from the same theta/phi rows, u and master-index key, and must
    match bit-for-bit; the fused word-topic counts must sum to the token
    count."""
    from paper_1505_03851_b200.device_lda import DeviceLDA

    g = torch.Generator(device="cuda").manual_seed(3 + K)
    V = 40_000
    lengths = torch.poisson(torch.full((M,), 200.0, device="cuda"), generator=g).clamp_(min=1).long()
    off = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1])
    if words_kind == "uniform":
        words = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    else:
        p = 1.0 / torch.arange(1, V + 1, device="cuda", dtype=torch.float64)
        cdf = torch.cumsum(p / p.sum(), 0)
        words = torch.searchsorted(cdf, torch.rand(T, generator=g, device="cuda", dtype=torch.float64))
        words = words.clamp_(max=V - 1).to(torch.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    lda = DeviceLDA(dc, K, V, seed=11)
    lda.init_uniform()
    assert lda.tiles is not None and lda.tiles.n_tiles == tiles and lda.tiles.run_pad == 4
    lda.draw(0)
    lda.check_errors()
    assert int(lda.word_topic.sum()) == T
    z = lda.z
    offh = off.cpu().numpy()
    Nh = np.diff(offh)
    rng = np.random.default_rng(0)
    toks = np.sort(rng.choice(T, 4096, replace=False))
    docs = np.searchsorted(offh, toks, side="right") - 1
    seed = wd.derive_seed(11, 1, 0)
    th = lda.theta[torch.from_numpy(docs).cuda()].cpu().numpy()
    wt = words[torch.from_numpy(toks).cuda()].long()
    ph = lda.phi[wt].cpu().numpy()
    zs = z[torch.from_numpy(toks).cuda()].cpu().numpy()
    gmax = Nh.reshape(-1, 32).max(axis=1)
    for j, (t, m) in enumerate(zip(toks, docs)):
        i = t - offh[m]
        key = gmax[m // 32] - 1 if i == Nh[m] - 1 else i
        u = O.units(seed, [m], [key])[0]
        a = (th[j] * ph[j]).astype(np.float32)
        idx, _, _ = O.draw_one(a, 32, int(m % 32), u=u)
        assert idx == zs[j], (t, m, i)


@pytest.mark.parametrize("run_pad", [0, 1])
@pytest.mark.parametrize("K,W,dtype", [(4096, 32, np.float32), (200, 32, np.float32), (640, 8, np.float32),
                                       (320, 64, np.float32), (1024, 32, np.float64)])
def test_lda_large_k_and_lanes_tiled_vs_oracle(K, W, dtype, run_pad):
    """K up to 4096 (BASELINE configs[4] row length), other lane counts and
    float64, drawn through vocabulary tiles, against the oracle."""
    gen = np.random.default_rng(K + W)
    M, V = 256, 300
    N, off, words = _random_corpus(gen, M, V, 20)
    theta = gen.dirichlet(np.full(K, 0.1), size=M).astype(dtype)
    phi = gen.uniform(0.01, 1, size=(V, K)).astype(dtype)
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
    tiles = dc.vocab_tiles(64, run_pad * W // 4)  # run_pad: the lane-group height W/4
    seed = 77
    z = wd.draw_z_device("butterfly", dc, _cuda(theta), _cuda(phi), wd.SeededStops(seed), W, tiles=tiles).cpu().numpy()
    exp, err = O.draw_z_csr(theta, phi, off, words, W=W, seed=seed, threads=8)
    assert err is None
    np.testing.assert_array_equal(z, exp)


@pytest.mark.parametrize("kernel", ["butterfly", "basic"])
def test_philox_stops_match_host_twin(kernel):
    """The opt-in Philox4x32-10 stream on the device (PhiloxStops) gives the
    same z as the host twin's u injected per token (rng.philox_units, pinned
    to the Random123 known answers)."""
    gen = np.random.default_rng(31)
    M, V, K = 96, 200, 200
    N, off, words = _random_corpus(gen, M, V, 20)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32), doc_base=64)
    seed = 0x1234_5678_9ABC
    z_p = wd.draw_z_device(kernel, dc, _cuda(theta), _cuda(phi), wd.kernels.PhiloxStops(seed), 32).cpu().numpy()
    doc = np.repeat(np.arange(M), N) + 64
    pos = np.arange(int(off[-1])) - np.repeat(off[:-1], N)
    u = wd.rng.philox_units(seed, doc, pos)
    z_u = wd.draw_z_device(kernel, dc, _cuda(theta), _cuda(phi), _cuda(u), 32).cpu().numpy()
    np.testing.assert_array_equal(z_p, z_u)
