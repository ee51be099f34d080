"""GPU: binary CSR corpus straight into HBM (corpus_io.load_device_corpus),
sharded like the multi-GPU run, and the draw over it.

A shard read from the .wdc file must be exactly the in-memory shard
(sharding.shard_ranges cuts, doc_base = first global document), and z drawn
shard by shard must equal z drawn over the whole corpus (global document ids
in the hash keys), so the file path feeds the same bits as the bench."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200 import corpus_io as C  # noqa: E402
from paper_1505_03851_b200 import lda  # noqa: E402
from paper_1505_03851_b200.sharding import shard_ranges  # noqa: E402


def _corpus(M, V, seed=11):
    rng = np.random.default_rng(seed)
    N = rng.poisson(40, M)
    N[rng.integers(0, M, M // 50)] = 0  # empty documents
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    words = rng.integers(0, V, int(off[-1])).astype(np.int32)
    return lda.Corpus(V, N.astype(np.int64), C.RaggedWords(off, words)), off, words


@pytest.mark.parametrize("V", [5000, 70000])
def test_device_corpus_from_file_and_shards(tmp_path, V):
    corp, off, words = _corpus(20_000, V)
    p = str(tmp_path / "c.wdc")
    C.save_corpus_bin(corp, p)
    t = {}
    dc = C.load_device_corpus(p, timing=t)
    assert dc.n_docs == 20_000 and dc.doc_base == 0 and t["total_s"] > 0
    assert np.array_equal(dc.offsets.cpu().numpy(), off)
    assert np.array_equal(dc.words.cpu().numpy(), words)
    assert dc.word_max == int(words.max())
    cuts = shard_ranges(np.diff(off), 3)
    for r in range(3):
        s = C.load_device_corpus(p, rank=r, world=3)
        lo, hi = cuts[r]
        assert s.doc_base == lo and s.n_docs == hi - lo
        assert np.array_equal(s.offsets.cpu().numpy(), off[lo:hi + 1] - off[lo])
        assert np.array_equal(s.words.cpu().numpy(), words[off[lo]:off[hi]])


def test_sharded_draw_from_file_equals_whole_corpus(tmp_path):
    M, V, K = 8192, 3000, 96
    corp, off, words = _corpus(M, V, seed=12)
    p = str(tmp_path / "c.wdc")
    C.save_corpus_bin(corp, p)
    g = torch.Generator(device="cuda").manual_seed(3)
    theta = torch.rand((M, K), generator=g, device="cuda") + 0.05
    phi = torch.rand((V, K), generator=g, device="cuda") + 0.05
    stops = wd.SeededStops(wd.derive_seed(9, 1, 0))
    whole = C.load_device_corpus(p)
    z_all = wd.draw_z_device("butterfly", whole, theta, phi, stops, 32).cpu().numpy()
    parts = []
    for r in range(2):
        s = C.load_device_corpus(p, rank=r, world=2)
        th = theta[s.doc_base:s.doc_base + s.n_docs]
        parts.append(wd.draw_z_device("butterfly", s, th, phi, stops, 32).cpu().numpy())
    assert np.array_equal(np.concatenate(parts), z_all)


def test_injected_stop_file_drives_the_device_draw(tmp_path):
    """The stop-inject file (cli.py:213-230) -> row t of load_injected_units
    -> WD_STOPS_UNITS: the same z as InjectedStops over the ragged values."""
    M, V, K = 256, 500, 40
    corp, off, words = _corpus(M, V, seed=13)
    rng = np.random.default_rng(1)
    u = rng.random(int(off[-1]) * 2)
    f = tmp_path / "u.txt"
    f.write_text("\n".join(repr(float(x)) for x in u) + "\n")
    units = C.load_injected_units(str(f), corp.lengths, 2)
    theta = rng.uniform(0.1, 1, (M, K)).astype(np.float32)
    phi = rng.uniform(0.1, 1, (V, K)).astype(np.float32)
    dc = corp.to_device()
    th, ph = torch.from_numpy(theta).cuda(), torch.from_numpy(phi).cuda()
    for t in range(2):
        z_dev = wd.draw_z_device("butterfly", dc, th, ph, torch.from_numpy(units[t]).cuda(), 32).cpu().numpy()
        ragged = [units[t][a:b] for a, b in zip(off[:-1], off[1:])]
        z_ref = wd.draw_z_device("butterfly", dc, th, ph, wd.InjectedStops(ragged), 32).cpu().numpy()
        assert np.array_equal(z_dev, z_ref)
