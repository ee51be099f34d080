"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, the host logic of the API mirror matches the reference semantics,
and the product path refuses to run without CUDA (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1505_03851_b200 as wd
from paper_1505_03851_b200 import _lib
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "warpdraw_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|int64_t|size_t)\s+(wd_\w+)\(", text, re.M)))


def test_header_declares_the_bound_exports():
    assert _declared_symbols() == sorted(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    from paper_1505_03851_b200 import build

    path = build.build()
    L = ctypes.CDLL(path)
    for name in _declared_symbols():
        assert hasattr(L, name), name
    h = _lib.load(path)
    assert h.wd_abi_version() == 1
    assert h.wd_status_string(0) == b"ok"


def test_invalid_arguments_rejected_without_gpu():
    L = _lib.load()
    # validation happens before any device work
    assert L.wd_draw_z(0, 0, 3, None, 0, None, 0, 8, None, None, None, None, None, 0, 0, 0, 0, 0, 0, None, None,
                       None, None, None, None, None, 0, None) == 1  # lanes=3
    assert L.wd_units(0, 3, None, None, 1, None, None) == 1
    assert L.wd_sample_rows(0, 2, 32, None, 0, 1, 8, 0, 0, 0, None, None, None, None, None, 0, None) == 1


def test_product_path_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeLibraryError):
        wd.sample_rows(torch.ones((4, 4)), 1)
    with pytest.raises(_lib.NativeLibraryError):
        wd.draw_z("butterfly", [1] * 8, np.ones((8, 4)), np.ones((2, 4)), [np.zeros(1, np.int64)] * 8,
                  wd.WarpConfig(lanes=8), wd.SeededStops(1))
    with pytest.raises(_lib.NativeLibraryError):
        wd.units_for(1, np.arange(3))


def test_host_seed_plumbing_matches_oracle():
    gen = np.random.default_rng(0)
    for _ in range(200):
        s = int(gen.integers(0, 2**63))
        ks = [int(k) for k in gen.integers(-(2**40), 2**40, size=int(gen.integers(0, 4)))]
        assert wd.derive_seed(s, *ks) == O.derive_seed(s, *ks)
        assert wd.unit_for(s, *ks) == O.units(s, *[[k] for k in ks])[0] if len(ks) <= 3 else True
    assert wd.derive_seed(7, 1, 0) == 0xB5D8C8503FA207B1


def test_warp_config_validation():
    with pytest.raises(ValueError):
        wd.WarpConfig(lanes=3)
    with pytest.raises(ValueError):
        wd.WarpConfig(lanes=128)
    with pytest.raises(ValueError):
        wd.WarpConfig(elem_size=2)
    assert wd.WarpConfig(lanes=64).log2_lanes == 6


def test_corpus_padding_and_csr():
    c = wd.Corpus(vocab_size=5, lengths=np.array([2, 0, 3]), words=[np.array([1, 2]), np.zeros(0), np.array([4, 0, 1])])
    p = c.padded(8)
    assert p.n_docs == 8 and p.padding == 5 and p.n_real_docs == 3
    off, words = p.csr()
    np.testing.assert_array_equal(off, [0, 2, 2, 5, 5, 5, 5, 5, 5])
    np.testing.assert_array_equal(words, [1, 2, 4, 0, 1])
    assert c.padded(3) is c


def test_injected_stops_from_file(tmp_path):
    lengths = [2, 0, 1]
    path = tmp_path / "stops.txt"
    path.write_text("0.1\n0.2\n0.3\n")
    stops = wd.InjectedStops.from_file(path, lengths)
    np.testing.assert_array_equal(stops.units(np.array([0, 0, 2]), np.array([0, 1, 0]), None), [0.1, 0.2, 0.3])
    np.testing.assert_array_equal(stops.flat(lengths), [0.1, 0.2, 0.3])
    path.write_text("0.1\n")
    with pytest.raises(ValueError, match="holds 1"):
        wd.InjectedStops.from_file(path, lengths)
    path.write_text("0.1\n0.2\n1.0\n")
    with pytest.raises(ValueError, match=r"\[0, 1\)"):
        wd.InjectedStops.from_file(path, lengths)


def test_corpus_file_roundtrip(tmp_path):
    c = wd.Corpus(vocab_size=9, lengths=np.array([3, 1]), words=[np.array([1, 8, 2]), np.array([0])])
    p = tmp_path / "c.txt"
    wd.save_corpus(c, p)
    d = wd.load_corpus(p)
    assert d.vocab_size == 9
    np.testing.assert_array_equal(d.lengths, [3, 1])
    p.write_text("#2 5\n1 2\n7\n")
    with pytest.raises(wd.WordIdOutOfRangeError):
        wd.load_corpus(p)
    p.write_text("1 x\n")
    with pytest.raises(wd.CorpusParseError):
        wd.load_corpus(p)


def test_corpus_npz_roundtrip(tmp_path):
    c = wd.Corpus(vocab_size=9, lengths=np.array([3, 0, 1]), words=[np.array([1, 8, 2]), np.zeros(0), np.array([0])])
    p = tmp_path / "c.npz"
    wd.save_corpus_npz(c.padded(4), p)
    d = wd.load_corpus_npz(p)
    assert d.vocab_size == 9 and d.padding == 1 and d.n_docs == 4
    np.testing.assert_array_equal(d.lengths, [3, 0, 1, 0])
    np.testing.assert_array_equal(d.words[0], [1, 8, 2])


def test_init_assignments_matches_reference_stream():
    c = wd.Corpus(vocab_size=5, lengths=np.array([4, 0, 2]), words=[np.zeros(4), np.zeros(0), np.zeros(2)])
    z = wd.init_assignments(c, 7, 11)
    gen = np.random.default_rng(O.derive_seed(11, 0))
    exp = [gen.integers(0, 7, size=n) for n in (4, 0, 2)]
    for a, b in zip(z, exp):
        np.testing.assert_array_equal(a, b)


def test_chi_square():
    stat, dof = wd.chi_square([10, 10], [0.5, 0.5])
    assert stat == 0.0 and dof == 1
    assert abs(wd.chi_square_critical(18) - 42.3124) < 1e-3


@pytest.mark.parametrize("run_pad", [0, 8])
def test_vocab_tile_builder_cpu(run_pad):
    """The vocabulary-tile regrouping (plain torch ops, runs on CPU tensors):
    every token appears exactly once with its (document, position); tiles
    hold their word range ordered by (document, word, position); with
    run_pad every (tile, document)
    run starts and ends on a multiple of run_pad, padding slots carry
    token_pos = -1 and their run's document."""
    import torch

    from paper_1505_03851_b200.kernels import DeviceCorpus, _build_vocab_tiles

    gen = np.random.default_rng(5)
    M, V, rows = 96, 70, 16
    N = gen.poisson(9, size=M)
    N[::7] = 0
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
    td = np.repeat(np.arange(M), N).astype(np.int32)
    c = DeviceCorpus(torch.from_numpy(off), torch.from_numpy(words), torch.from_numpy(td), M, int(off[-1]))
    t = _build_vocab_tiles(c, rows, run_pad)
    w, d, p = t.words.numpy(), t.token_doc.numpy(), t.token_pos.numpy()
    assert t.n_tiles == -(-int(words.max() + 1) // rows) and t.bounds[-1] == w.size
    real = p >= 0
    assert real.sum() == words.size
    # each real slot is a distinct original token, with its word
    orig = off[d[real]] + p[real]
    assert np.array_equal(np.sort(orig), np.arange(words.size))
    assert np.array_equal(w[real], words[orig])
    for ti in range(t.n_tiles):
        a, b = t.bounds[ti], t.bounds[ti + 1]
        assert np.all(w[a:b] // rows == ti)
        rr = real[a:b]
        o = orig[np.cumsum(real)[a:b][rr] - 1]  # original token index of the tile's real slots
        dd, ww = d[a:b][rr].astype(np.int64), w[a:b][rr].astype(np.int64)
        key = (dd * V + ww) * words.size + o
        assert np.all(np.diff(key) > 0)  # (document, word, position) order
        if run_pad:
            assert (b - a) % run_pad == 0
            dd = d[a:b]
            starts = np.flatnonzero(np.r_[True, dd[1:] != dd[:-1]])
            assert np.all(starts % run_pad == 0)
    if not run_pad:
        assert real.all()


def test_philox_known_answers():
    """Philox4x32-10 against the Random123 known-answer vectors (the opt-in
    PhiloxStops stream; the device kernel is checked against this twin in
    tests/test_gpu_parity.py)."""
    from paper_1505_03851_b200.rng import philox4x32_10

    kat = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF, 0xFFFFFFFF], [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, out in kat:
        assert [int(x) for x in philox4x32_10(ctr, key)] == out


def test_host_helper_ragged_loops_match_numpy():
    """csrc/wd_host.c (the boundary's ragged <-> CSR loops) against numpy."""
    from paper_1505_03851_b200 import kernels as K

    assert K._wdhost is not None, "host helper not built"
    gen = np.random.default_rng(4)
    N = gen.integers(0, 9, size=500)
    for dt in (np.int64, np.int32, np.int16, np.uint16, np.uint8):
        w = [gen.integers(0, 200, size=int(n) + int(gen.integers(0, 3))).astype(dt) for n in N]
        off, flat = K.ragged_to_csr(N, w)
        ref = np.concatenate([x[:n] for x, n in zip(w, N)]).astype(np.int32)
        np.testing.assert_array_equal(flat, ref)
        assert flat.dtype == np.int32 and off[-1] == N.sum()
    with pytest.raises(ValueError, match="shorter"):
        K.ragged_to_csr([3], [np.arange(2)])
    with pytest.raises(wd.OutOfBoundsError):
        K.ragged_to_csr([2], [np.array([1, 1 << 40])])
    # non-ndarray elements take the numpy path
    off, flat = K.ragged_to_csr([2, 1], [[1, 2], (7,)])
    np.testing.assert_array_equal(flat, [1, 2, 7])
    z = np.arange(int(N.sum()), dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(N)])
    views = K.csr_to_ragged(z, off)
    assert len(views) == N.size and all(v.dtype == np.int64 for v in views)
    for m in range(N.size):
        np.testing.assert_array_equal(views[m], z[off[m]:off[m + 1]])
    ids = K._wdhost.list_ids(views)
    assert K._wdhost.ids_equal(views, ids)
    views2 = list(views)
    views2[7] = views2[7].copy()
    assert not K._wdhost.ids_equal(views2, ids)
    assert not K._wdhost.ids_equal(views[:-1], ids)


def test_flat_topics_follows_np_add_at_index_rules():
    """The GPU topic_counts' host-side flattening of a ragged z: CSR order,
    each document's first `length` entries, negative topics wrapped as
    np.add.at wraps them, out-of-range topics rejected with IndexError --
    with the native helper and through the numpy path alike."""
    from paper_1505_03851_b200 import kernels as Kmod
    from paper_1505_03851_b200.lda import _flat_topics

    K = 7
    z = [np.array([0, 6, -1]), np.array([], dtype=np.int64), np.array([-7, 3], dtype=np.int32)]
    lengths = np.array([3, 0, 2], dtype=np.int64)
    exp = np.array([0, 6, 6, 0, 3], dtype=np.int32)
    np.testing.assert_array_equal(_flat_topics(z, lengths, K), exp)
    saved = Kmod._wdhost
    try:
        Kmod._wdhost = None  # the numpy path
        np.testing.assert_array_equal(_flat_topics(z, lengths, K), exp)
        with pytest.raises(IndexError, match="out of bounds"):
            _flat_topics([np.array([7])], np.array([1]), K)
    finally:
        Kmod._wdhost = saved
    for bad in (7, -8, 1 << 40):
        with pytest.raises(IndexError, match="out of bounds"):
            _flat_topics([np.array([1, bad])], np.array([2]), K)
