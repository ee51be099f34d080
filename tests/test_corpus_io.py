"""CPU: the native corpus / stop-file / CSV formats (corpus_io, libwdio.so)
against the reference's Python semantics (lda.py:66-118, cli.py:213-273).

The reference's parsers and writers are plain Python over the standard
library; each expectation below is that same Python code path (the
reference's line parser kept as lda._load_corpus_python, csv.writer with
repr(float(x)), np.loadtxt), run on the same file."""

import csv
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1505_03851_b200 import corpus_io as C
from paper_1505_03851_b200 import lda

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_wdio_header_declares_the_exports():
    text = open(os.path.join(ROOT, "include", "wdio.h")).read()
    names = set(re.findall(r"^\s*(?:int|void)\s+(wdio_\w+)\(", text, re.M))
    L = C._io()
    assert names and all(hasattr(L, n) for n in names)


def test_repr_matches_python():
    rng = np.random.default_rng(0)
    vals = [float(x) for x in rng.standard_normal(20000) * 10.0 ** rng.integers(-300, 300, 20000)]
    vals += [float(np.float32(x)) for x in rng.random(5000)]
    vals += [0.0, -0.0, 1.0, 0.1, 1e-5, 1e-4, 9.999e-5, 123.0, 1e15, 1e16, 1.5e16, 1e22, 5e-324,
             1.7976931348623157e308, float("nan"), float("inf"), -float("inf"), 2.0 ** 60, 0.30000000000000004]
    for v in vals:
        assert C.repr_float(v) == repr(v), v


CORPORA = [
    "#3 10\n1 2 3\n\n 4  5\t9 \n",
    "1 2 3\r\n0\r\n7",
    "1 2 3\n\n\n",
    "",
    "\n",
    "   \n5",
    "#2 6\n+5 007\n-0 1\n",
    "1 2 3\r4 5\n",           # lone CR: a line break in text mode
    "1\x0b2\x0c3\n",          # vertical tab / form feed are whitespace for str.split
    "1_0 2\n",                # underscore: int() accepts it (Python path)
    "12345678901234567890123 1\n",  # beyond int64: Python path
]


@pytest.mark.parametrize("text", CORPORA)
def test_load_corpus_matches_reference_parser(tmp_path, text):
    p = tmp_path / "c.txt"
    p.write_bytes(text.encode())
    try:
        exp = lda._load_corpus_python(str(p))
    except Exception as e:  # noqa: BLE001
        with pytest.raises(type(e)) as got:
            lda.load_corpus(str(p))
        assert str(got.value) == str(e)
        return
    got = lda.load_corpus(str(p))
    assert got.vocab_size == exp.vocab_size and got.n_docs == exp.n_docs
    assert np.array_equal(got.lengths, exp.lengths)
    for a, b in zip(got.words, exp.words):
        assert a.dtype == np.int64 and np.array_equal(a, b)


BAD = [
    "#3\n1 2\n",             # header must be '#M V'
    "#x 4\n1\n",             # bad header
    "#2 10\n1 2\n",          # header count mismatch
    "1 2\n3 x\n",            # bad token, line 2
    "1 2\n3 -4\n",           # negative id
    "1 2\n3 4.5\n",          # bad token
    "1 2\n3 9\n",            # id >= V (vocab_size=5)
    "1 \xe9\n",              # non-ASCII token
]


@pytest.mark.parametrize("text", BAD)
def test_load_corpus_errors_are_the_reference_errors(tmp_path, text):
    p = tmp_path / "c.txt"
    p.write_bytes(text.encode())
    with pytest.raises(Exception) as exp:
        lda._load_corpus_python(str(p), vocab_size=5)
    with pytest.raises(type(exp.value)) as got:
        lda.load_corpus(str(p), vocab_size=5)
    assert str(got.value) == str(exp.value)


def test_large_corpus_parses_in_parallel_and_round_trips(tmp_path):
    rng = np.random.default_rng(3)
    M = 60000
    N = rng.poisson(30, M)
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    words = rng.integers(0, 5000, int(off[-1])).astype(np.int32)
    corp = lda.Corpus(5000, N.astype(np.int64), C.RaggedWords(off, words))
    p = tmp_path / "big.txt"
    lda.save_corpus(corp, str(p))
    # the reference's writer (lda.py:113-118) byte for byte
    ref = f"#{M} 5000\n" + "".join(" ".join(str(int(x)) for x in words[a:b]) + "\n"
                                   for a, b in zip(off[:-1], off[1:]))
    assert p.read_bytes() == ref.encode()
    back = lda.load_corpus(str(p))
    assert isinstance(back.words, C.RaggedWords)
    o2, w2 = back.csr()
    assert np.array_equal(o2, off) and np.array_equal(w2, words)


def test_padded_csr_corpus_keeps_csr():
    off = np.array([0, 2, 2, 5], dtype=np.int64)
    corp = lda.Corpus(9, np.diff(off), C.RaggedWords(off, np.array([1, 2, 3, 4, 5], np.int32)))
    p = corp.padded(4)
    assert p.n_docs == 4 and p.padding == 1 and isinstance(p.words, C.RaggedWords)
    assert len(p.words[3]) == 0 and np.array_equal(p.csr()[0], [0, 2, 2, 5, 5])


def test_binary_corpus_round_trip_and_validation(tmp_path):
    rng = np.random.default_rng(4)
    N = rng.poisson(20, 1000)
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    for V, wb in ((40000, 2), (70000, 4)):
        words = rng.integers(0, V, int(off[-1])).astype(np.int32)
        corp = lda.Corpus(V, N.astype(np.int64), C.RaggedWords(off, words), padding=0)
        p = tmp_path / f"c{V}.wdc"
        C.save_corpus_bin(corp, str(p))
        h = C.read_bin_header(str(p))
        assert h["word_bytes"] == wb and h["n_docs"] == 1000 and h["n_tokens"] == off[-1]
        back = C.load_corpus_bin(str(p))
        assert back.vocab_size == V and np.array_equal(back.csr()[1], words)
    raw = bytearray((tmp_path / "c40000.wdc").read_bytes())
    (tmp_path / "trunc.wdc").write_bytes(bytes(raw[:-2]))
    with pytest.raises(ValueError, match="does not match the header"):
        C.load_corpus_bin(str(tmp_path / "trunc.wdc"))
    raw[:8] = b"NOTACORP"
    (tmp_path / "bad.wdc").write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="not a version-1"):
        C.load_corpus_bin(str(tmp_path / "bad.wdc"))


def _ref_injected(path, lengths, iterations):
    """cli._load_injected_iterations (cli.py:213-230) restated."""
    flat = np.loadtxt(path, dtype=np.float64, ndmin=1)
    per_iter = int(np.sum(lengths))
    if flat.size != per_iter * iterations:
        raise ValueError(f"stop file holds {flat.size} values; need {per_iter} x {iterations} iterations")
    if np.any(flat < 0) or np.any(flat >= 1):
        raise ValueError("injected values must lie in [0, 1)")
    return flat


@pytest.mark.parametrize("fmt", ["repr", "%.6e", "%.3f", "mixed"])
def test_injected_units_file(tmp_path, fmt):
    rng = np.random.default_rng(5)
    lengths = np.array([3, 0, 5, 2])
    iters = 3
    u = rng.random(int(lengths.sum()) * iters)
    p = tmp_path / "u.txt"
    if fmt == "repr":
        text = "\n".join(repr(float(x)) for x in u) + "\n"
    elif fmt == "mixed":
        text = "\n".join((f"  {x:.17g}\t" if i % 2 else f"{x:.5E}") for i, x in enumerate(u)) + "\n\n"
    else:
        text = "\n".join(fmt % x for x in u)
    p.write_text(text)
    got = C.load_injected_units(str(p), lengths, iters)
    exp = _ref_injected(str(p), lengths, iters)
    assert got.shape == (iters, lengths.sum()) and np.array_equal(got.ravel(), exp)
    # InjectedStops.from_file (kernels.py:74-83) over one iteration's worth
    p1 = tmp_path / "u1.txt"
    p1.write_text("\n".join(repr(float(x)) for x in u[: lengths.sum()]) + "\n")
    st = lda.InjectedStops.from_file(str(p1), lengths)
    assert np.array_equal(st.flat(lengths), u[: lengths.sum()])


def test_injected_units_errors(tmp_path):
    p = tmp_path / "u.txt"
    p.write_text("0.5\n0.25\n")
    with pytest.raises(C.StopFileError, match=r"stop file holds 2 values; need 3 x 1 iterations"):
        C.load_injected_units(str(p), [3], 1)
    p.write_text("0.5\n1.0\n")
    with pytest.raises(C.StopFileError, match=r"injected values must lie in \[0, 1\)"):
        C.load_injected_units(str(p), [2], 1)
    p.write_text("# comment\n0.5\n0.25\n")  # np.loadtxt semantics (Python path)
    assert np.array_equal(C.load_injected_units(str(p), [2], 1).ravel(), [0.5, 0.25])


def _csv_bytes(rows):
    import io

    buf = io.StringIO(newline="")
    w = csv.writer(buf)
    for r in rows:
        w.writerow(r)
    return buf.getvalue().encode()


def test_output_writers_match_cmd_lda(tmp_path):
    """z.csv, likelihood.csv, theta.csv, phi.csv exactly as cmd_lda writes
    them (cli.py:232-273: csv.writer, repr(float(x)))."""
    rng = np.random.default_rng(6)
    lengths = np.array([4, 0, 3, 6, 1, 0])
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    z = rng.integers(0, 17, int(off[-1])).astype(np.int32)
    theta = rng.dirichlet(np.full(17, 0.1), size=8).astype(np.float32)
    theta[0, 3] = 0.0
    phi = rng.dirichlet(np.full(30, 0.01), size=17).T.copy()
    traj = [-12345.678, -1e-7, float(np.float32(-3.25))]
    n_docs = 5  # cmd_lda writes the loaded (unpadded) corpus only
    C.write_outputs(str(tmp_path), n_docs, z, off, theta, phi, traj)
    zr = [["doc", "pos", "topic"]] + [[m, i, int(z[off[m] + i])] for m in range(n_docs) for i in range(lengths[m])]
    assert (tmp_path / "z.csv").read_bytes() == _csv_bytes(zr)
    lr = [["iteration", "log_likelihood"]] + [[t, repr(float(v))] for t, v in enumerate(traj)]
    assert (tmp_path / "likelihood.csv").read_bytes() == _csv_bytes(lr)
    assert (tmp_path / "theta.csv").read_bytes() == _csv_bytes([[repr(float(x)) for x in r] for r in theta[:n_docs]])
    assert (tmp_path / "phi.csv").read_bytes() == _csv_bytes([[repr(float(x)) for x in r] for r in phi])
    # ragged z (the reference's run_gibbs output) and strided matrices
    C.write_z_csv(str(tmp_path / "z2.csv"), [z[a:b].astype(np.int64) for a, b in zip(off[:-1], off[1:])][:n_docs],
                  off[: n_docs + 1])
    assert (tmp_path / "z2.csv").read_bytes() == _csv_bytes(zr)
    C.write_matrix_csv(str(tmp_path / "s.csv"), phi[:, ::2])
    assert (tmp_path / "s.csv").read_bytes() == _csv_bytes([[repr(float(x)) for x in r] for r in phi[:, ::2]])


def test_native_loader_has_no_cpu_compute_dependency():
    """libwdio is host I/O only: it never links the CUDA library."""
    path = os.path.join(ROOT, "paper_1505_03851_b200", "_lib", "libwdio.so")
    ctypes.CDLL(path)
    with open(path, "rb") as fh:
        assert b"libcudart" not in fh.read()
