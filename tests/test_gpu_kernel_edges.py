"""GPU: the round-2 kernels (small-K LDA, register-lean large-K LDA) on the
edge cases the reference tests for the draw: an all-zero
document (AllZeroError with the reference's message, kernels.py:421-425),
injected and Philox stops, shards with a non-zero doc_base, padded and
unpadded vocabulary tiles and the untiled CSR-order draw (which takes the
small-K kernel up to K = 256), against the oracle / the host twin."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.kernels import to_block_aligned  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _corpus(gen, M, V, mean):
    N = gen.poisson(mean, size=M).astype(np.int64)
    N[gen.random(M) < 0.05] = 0
    off = np.concatenate([[0], np.cumsum(N)])
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int64)
    return N, off, words


def _dev(a):
    return to_block_aligned(torch.from_numpy(np.ascontiguousarray(a)).cuda())


@pytest.mark.parametrize("K", [200, 232, 2048, 4096])
@pytest.mark.parametrize("pad", [0, 4, None])  # None: the untiled CSR-order draw
def test_allzero_document(K, pad):
    gen = np.random.default_rng(K + (pad if pad is not None else 7))
    M, V = 256, 300
    N, off, words = _corpus(gen, M, V, 12)
    dead = int(np.flatnonzero(N > 0)[7])
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    theta[dead] = 0
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
    tiles = None if pad is None else dc.vocab_tiles(64, pad)
    with pytest.raises(wd.AllZeroError, match=rf"^document {dead}: all products are zero$"):
        wd.draw_z_device("butterfly", dc, _dev(theta), _dev(phi), wd.SeededStops(3), 32, tiles=tiles)
    _, err = O.draw_z_csr(theta, phi, off, words, W=32, seed=3)
    assert err is not None and (err >> 40) * 32 + (err & 0xFF) == dead  # the oracle's first dead document


@pytest.mark.parametrize("K", [72, 200, 256, 2048])
@pytest.mark.parametrize("tiled", [True, False])
def test_injected_philox_and_doc_base(K, tiled):
    """A shard starting at global document 96: seeded keys use global ids;
    injected u per token; Philox stops equal their host twin's u."""
    gen = np.random.default_rng(K)
    M, V = 160, 250
    N, off, words = _corpus(gen, M, V, 15)
    theta = gen.uniform(0.05, 1, size=(M, K)).astype(np.float32)
    phi = gen.uniform(0.05, 1, size=(V, K)).astype(np.float32)
    base = 96
    dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32), doc_base=base)
    tiles = dc.vocab_tiles(80, 4) if tiled else None
    th, ph = _dev(theta), _dev(phi)
    # seeded (global document ids in the keys and in doc mod W)
    z = wd.draw_z_device("butterfly", dc, th, ph, wd.SeededStops(9), 32, tiles=tiles).cpu().numpy()
    exp, err = O.draw_z_csr(theta, phi, off, words, W=32, seed=9, doc_base=base)
    assert err is None
    np.testing.assert_array_equal(z, exp)
    # injected u per token (CSR order)
    u = gen.random(int(off[-1]))
    z = wd.draw_z_device("butterfly", dc, th, ph, torch.from_numpy(u).cuda(), 32, tiles=tiles).cpu().numpy()
    exp, _ = O.draw_z_csr(theta, phi, off, words, W=32, units_=u, doc_base=base)
    np.testing.assert_array_equal(z, exp)
    # Philox stops == the host twin's u injected
    seed = 0xFEED_5EED
    z_p = wd.draw_z_device("butterfly", dc, th, ph, wd.kernels.PhiloxStops(seed), 32, tiles=tiles).cpu().numpy()
    doc = np.repeat(np.arange(M), N) + base
    pos = np.arange(int(off[-1])) - np.repeat(off[:-1], N)
    z_u = wd.draw_z_device("butterfly", dc, th, ph, torch.from_numpy(wd.rng.philox_units(seed, doc, pos)).cuda(), 32,
                           tiles=tiles).cpu().numpy()
    np.testing.assert_array_equal(z_p, z_u)


def test_sampler_error_accumulation():
    """WD_ERR_ACCUMULATE: one caller-owned err over a batch of draws keeps the
    first batch's AllZero row; a normal call resets it."""
    gen = np.random.default_rng(5)
    for K in (16, 1024):
        w = torch.from_numpy(gen.uniform(0.1, 1, size=(300, K)).astype(np.float32)).cuda()
        wz = w.clone()
        wz[123] = 0
        err = torch.empty(2, dtype=torch.int64, device="cuda")
        err.fill_(-1)
        wd.sample_rows(wz, 1, err=err, check=False, accumulate_err=True)
        wd.sample_rows(w, 2, err=err, check=False, accumulate_err=True)
        e = err.cpu().numpy().view(np.uint64)
        assert int(e[0]) == 123 and int(e[1]) == (1 << 64) - 1
        wd.sample_rows(w, 3, err=err, check=False)  # resets first
        assert int(err.cpu().numpy().view(np.uint64)[0]) == (1 << 64) - 1
        with pytest.raises(ValueError, match="caller-owned err"):
            wd.sample_rows(w, 3, accumulate_err=True)
