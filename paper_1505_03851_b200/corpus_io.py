"""Corpus and output formats at configs[2]-[4] scale.

The reference keeps a corpus as a Python list of per-document arrays
(`Corpus.words`, lda.py:30-63), parses its text format line by line
(`load_corpus`, lda.py:66-110), reads injected stop values with np.loadtxt
(`_load_injected_iterations`, cli.py:213-230; `InjectedStops.from_file`,
kernels.py:74-83) and writes `z.csv` / `theta.csv` / `phi.csv` /
`likelihood.csv` through the csv module (cli.py:232-273).  Here the same
formats go through native code (csrc/wd_io.c, libwdio.so) straight to and
from flat CSR buffers -- offsets int64 [M+1], words int32 [sum N] -- that
`DeviceCorpus` consumes, with no per-document Python object:

  load_corpus(path)          the reference's text format -> Corpus whose
                             `words` is a RaggedWords view of the CSR
  save_corpus(corpus, path)  the reference's text format
  save_corpus_bin / load_corpus_bin
                             binary CSR file (.wdc, below)
  load_device_corpus(path, rank=, world=)
                             .wdc -> DeviceCorpus: this rank's 32-aligned,
                             token-balanced document shard only, read by
                             parallel preads into pinned memory and copied to
                             HBM chunk by chunk behind the reads
  load_injected_units(path, lengths, iterations)
                             the stop-inject file -> float64 [iterations, sum N]
                             (row t is iteration t's u per token, CSR order: the
                             device draw's WD_STOPS_UNITS input)
  write_outputs(outdir, ...) cmd_lda's four CSV files, byte-identical
  write_z_csv / write_matrix_csv / write_likelihood_csv

Parsing semantics are the reference's: inputs the C parser does not accept
verbatim (non-ASCII, underscores, negative ids, malformed tokens, '#'
comments in stop files, several values per line) are re-read by the
reference's own Python logic, so errors carry the reference's messages.

.wdc layout (little endian): 64-byte header
    magic b"WDCORPUS", u32 version = 1, u32 word_bytes (2 or 4),
    u64 n_docs, u64 n_tokens, u64 vocab_size, u64 padding, 16 reserved bytes
then offsets int64 [n_docs + 1], then words as uint16 (word_bytes 2, used
when vocab_size <= 65536: half the bytes to read) or int32.
"""

from __future__ import annotations

import ctypes
import os
import struct
from collections.abc import Sequence

import numpy as np

from . import _lib

MAGIC = b"WDCORPUS"
HEADER = struct.Struct("<8sIIQQQQ16s")
assert HEADER.size == 64

_WDIO = None


def _io():
    """libwdio.so (built by paper_1505_03851_b200.build); host-side only, no GPU needed."""
    global _WDIO
    if _WDIO is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libwdio.so")
        if not os.path.exists(path):
            raise _lib.NativeLibraryError(f"{path} is missing: run python -m paper_1505_03851_b200.build")
        L = ctypes.CDLL(path)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        pi64, pi32, pvp = ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(vp)
        L.wdio_scan_corpus.argtypes = [ctypes.c_char_p, i64, ctypes.c_int, pvp, pi64, pi64, pi32]
        L.wdio_fill_corpus.argtypes = [vp, vp, vp]
        L.wdio_release.argtypes = [vp]
        L.wdio_release.restype = None
        L.wdio_scan_floats.argtypes = [ctypes.c_char_p, ctypes.c_int, pvp, pi64]
        L.wdio_fill_floats.argtypes = [vp, vp]
        L.wdio_release_floats.argtypes = [vp]
        L.wdio_release_floats.restype = None
        L.wdio_pread.argtypes = [ctypes.c_char_p, i64, i64, vp, ctypes.c_int]
        L.wdio_write_z_csv.argtypes = [ctypes.c_char_p, vp, ctypes.c_int, vp, i64, ctypes.c_int]
        L.wdio_write_matrix_csv.argtypes = [ctypes.c_char_p, vp, ctypes.c_int, i64, i64, i64, ctypes.c_int]
        L.wdio_write_corpus_text.argtypes = [ctypes.c_char_p, vp, vp, i64, i64, i64, ctypes.c_int]
        L.wdio_repr.argtypes = [ctypes.c_double, ctypes.c_char_p]
        for f in ("wdio_scan_corpus", "wdio_fill_corpus", "wdio_scan_floats", "wdio_fill_floats", "wdio_pread",
                  "wdio_write_z_csv", "wdio_write_matrix_csv", "wdio_write_corpus_text", "wdio_repr"):
            getattr(L, f).restype = ctypes.c_int
        _WDIO = L
    return _WDIO


def _threads() -> int:
    try:
        return max(1, min(64, len(os.sched_getaffinity(0))))
    except AttributeError:  # pragma: no cover
        return max(1, min(64, os.cpu_count() or 1))


def _check_rc(rc: int, what: str, path=None):
    if rc < 0:
        raise OSError(-rc, f"{what}: {os.strerror(-rc)}", None if path is None else str(path))
    if rc == 12:  # pragma: no cover
        raise MemoryError(what)


def _cpath(path) -> bytes:
    return os.fsencode(os.fspath(path))


# ------------------------------------------------------------------ ragged view
class RaggedWords(Sequence):
    """`Corpus.words` backed by one CSR buffer: element m is document m's
    word ids as a fresh int64 array (the reference's element type,
    lda.py:101), made on access.  `csr()` hands the flat buffers to the
    device path without any per-document work."""

    def __init__(self, offsets, flat):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.flat = np.ascontiguousarray(flat, dtype=np.int32)
        if self.offsets.ndim != 1 or self.offsets.size < 1 or self.offsets[0] != 0 or \
                int(self.offsets[-1]) != self.flat.size:
            raise ValueError("RaggedWords: offsets must start at 0 and end at len(flat)")

    def __len__(self):
        return self.offsets.size - 1

    def __getitem__(self, m):
        if isinstance(m, slice):
            return [self[i] for i in range(*m.indices(len(self)))]
        n = len(self)
        m = int(m)
        if m < 0:
            m += n
        if not 0 <= m < n:
            raise IndexError("document index out of range")
        return self.flat[self.offsets[m]:self.offsets[m + 1]].astype(np.int64)

    def __iter__(self):
        for m in range(len(self)):
            yield self[m]

    def __add__(self, other):  # list(words) + [...] in Corpus.padded-style code
        return list(self) + list(other)

    def csr(self):
        return self.offsets, self.flat

    def padded(self, extra: int) -> "RaggedWords":
        """`extra` empty documents appended (Corpus.padded, lda.py:56-63)."""
        if extra <= 0:
            return self
        off = np.concatenate([self.offsets, np.full(extra, self.offsets[-1], dtype=np.int64)])
        return RaggedWords(off, self.flat)


# ------------------------------------------------------------------ text corpus
def _corpus_cls():
    from .lda import Corpus, CorpusParseError, WordIdOutOfRangeError

    return Corpus, CorpusParseError, WordIdOutOfRangeError


def _read_header(path):
    """(declared_m, declared_v, byte offset of the first document line) of
    the optional "#M V" first line (lda.py:79-87); errors as the reference."""
    _, CorpusParseError, _ = _corpus_cls()
    with open(path, "rb") as fh:
        first = fh.readline()
    try:
        text = first.decode("utf-8")
    except UnicodeDecodeError:
        return None  # the Python parser raises the reference's decode error
    if text.endswith("\r\n"):
        text = text[:-2]
    elif text.endswith("\n") or text.endswith("\r"):
        text = text[:-1]
    if "\r" in text:
        return None  # a lone CR is a line break in text mode: Python path
    if not text.startswith("#"):
        return None, None, 0
    fields = text[1:].split()
    if len(fields) != 2:
        raise CorpusParseError(f"{path}:1: header must be '#M V'")
    try:
        m, v = int(fields[0]), int(fields[1])
    except ValueError as exc:
        raise CorpusParseError(f"{path}:1: bad header {text!r}") from exc
    return m, v, len(first)


def parse_corpus_csr(path):
    """(offsets int64 [M+1], words int32 [sum N], declared_m, declared_v,
    max_word) of a text corpus by the native parser, or None when the file
    needs the reference's Python parser (exotic-but-valid syntax or an
    error, which that parser then reports)."""
    hdr = _read_header(path)
    if hdr is None:
        return None
    dm, dv, start = hdr
    L = _io()
    h = ctypes.c_void_p()
    nd, nt, mx = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    rc = L.wdio_scan_corpus(_cpath(path), start, _threads(), ctypes.byref(h), ctypes.byref(nd), ctypes.byref(nt),
                            ctypes.byref(mx))
    if rc == 1:
        return None
    _check_rc(rc, "load_corpus", path)
    try:
        off = np.empty(nd.value + 1, dtype=np.int64)
        words = np.empty(nt.value, dtype=np.int32)
        L.wdio_fill_corpus(h, off.ctypes.data, words.ctypes.data)
    finally:
        L.wdio_release(h)
    return off, words, dm, dv, int(mx.value)


def load_corpus(path, vocab_size: int | None = None):
    """lda.load_corpus (lda.py:66-110) into a CSR-backed Corpus: the same
    documents, vocabulary rule and errors (CorpusParseError with the line
    number, WordIdOutOfRangeError naming the first offending document)."""
    Corpus, CorpusParseError, WordIdOutOfRangeError = _corpus_cls()
    res = parse_corpus_csr(path)
    if res is None:
        from .lda import _load_corpus_python

        return _load_corpus_python(path, vocab_size)
    off, words, dm, dv, mx = res
    M = off.size - 1
    if dm is not None and M != dm:
        raise CorpusParseError(f"{path}: header declares {dm} documents, found {M}")
    if dv is not None:
        vocab_size = dv
    if vocab_size is None:
        vocab_size = mx + 1
    if mx >= vocab_size:
        bad = int(np.argmax(words >= vocab_size))
        m = int(np.searchsorted(off, bad, side="right") - 1)
        doc_max = int(words[off[m]:off[m + 1]].max())
        raise WordIdOutOfRangeError(f"{path}: document {m} holds word id {doc_max} >= V={vocab_size}")
    return Corpus(vocab_size=vocab_size, lengths=np.diff(off), words=RaggedWords(off, words))


def corpus_csr(corpus):
    """(offsets, words int32) of any Corpus (RaggedWords: no copy)."""
    if isinstance(corpus.words, RaggedWords):
        off, flat = corpus.words.csr()
        if off.size - 1 == corpus.n_docs and np.array_equal(np.diff(off), corpus.lengths):
            return off, flat
    from .kernels import ragged_to_csr

    return ragged_to_csr(corpus.lengths, corpus.words)


def save_corpus(corpus, path):
    """lda.save_corpus (lda.py:113-118): "#M V" header (real documents only),
    one line of space-separated ids per document."""
    off, words = corpus_csr(corpus)
    M = corpus.n_real_docs
    _check_rc(_io().wdio_write_corpus_text(_cpath(path), words.ctypes.data, off.ctypes.data, M, M,
                                            int(corpus.vocab_size), _threads()), "save_corpus", path)


# ---------------------------------------------------------------- binary CSR
def save_corpus_bin(corpus, path, word_bytes: int | None = None):
    """Binary CSR (.wdc).  word_bytes defaults to 2 when every id fits uint16."""
    off, words = corpus_csr(corpus)
    V = int(corpus.vocab_size)
    if word_bytes is None:
        word_bytes = 2 if V <= 65536 else 4
    if word_bytes == 2 and words.size and (int(words.min()) < 0 or int(words.max()) > 65535):
        raise ValueError("word ids do not fit uint16")
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, 1, word_bytes, off.size - 1, words.size, V, int(corpus.padding), bytes(16)))
        fh.write(np.ascontiguousarray(off, dtype="<i8").tobytes())
        w = words.astype("<u2" if word_bytes == 2 else "<i4", copy=False)
        w.tofile(fh)


def read_bin_header(path) -> dict:
    with open(path, "rb") as fh:
        raw = fh.read(HEADER.size)
    if len(raw) != HEADER.size:
        raise ValueError(f"{path}: not a .wdc corpus (short header)")
    magic, ver, wb, M, T, V, pad, _ = HEADER.unpack(raw)
    if magic != MAGIC or ver != 1 or wb not in (2, 4):
        raise ValueError(f"{path}: not a version-1 .wdc corpus")
    size = os.path.getsize(path)
    words_at = HEADER.size + 8 * (M + 1)
    if size != words_at + wb * T:
        raise ValueError(f"{path}: file size {size} does not match the header (expected {words_at + wb * T})")
    return {"word_bytes": wb, "n_docs": M, "n_tokens": T, "vocab_size": V, "padding": pad, "words_at": words_at}


def _pread(path, off, nbytes, dst_ptr):
    if nbytes:
        _check_rc(_io().wdio_pread(_cpath(path), int(off), int(nbytes), dst_ptr, _threads()), "pread", path)


def _read_offsets(path, h, lo=0, hi=None):
    hi = h["n_docs"] if hi is None else hi
    off = np.empty(hi - lo + 1, dtype=np.int64)
    _pread(path, HEADER.size + 8 * lo, 8 * off.size, off.ctypes.data)
    if off.size and (off[0] < 0 or np.any(np.diff(off) < 0) or off[-1] > h["n_tokens"]):
        raise ValueError(f"{path}: corrupt offsets")
    return off


def load_corpus_bin(path):
    """.wdc -> Corpus (CSR-backed, no per-document objects)."""
    Corpus, _, WordIdOutOfRangeError = _corpus_cls()
    h = read_bin_header(path)
    off = _read_offsets(path, h)
    if off[0] != 0 or off[-1] != h["n_tokens"]:
        raise ValueError(f"{path}: corrupt offsets")
    raw = np.empty(h["n_tokens"], dtype=np.uint16 if h["word_bytes"] == 2 else np.int32)
    _pread(path, h["words_at"], raw.nbytes, raw.ctypes.data)
    words = raw.astype(np.int32) if raw.dtype != np.int32 else raw
    if words.size and (int(words.min()) < 0 or int(words.max()) >= h["vocab_size"]):
        raise WordIdOutOfRangeError(f"{path}: word id out of range for V={h['vocab_size']}")
    return Corpus(vocab_size=h["vocab_size"], lengths=np.diff(off), words=RaggedWords(off, words),
                  padding=h["padding"])


_CHUNK = 256 << 20
_PINNED: dict = {}


def _pinned_stage(i: int, nbytes: int):
    import torch

    buf = _PINNED.get(i)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        _PINNED[i] = buf
    return buf[:nbytes]


def load_device_corpus(path, *, rank: int = 0, world: int = 1, device=None, doc_range=None, timing=None):
    """.wdc -> DeviceCorpus of this rank's shard (sharding.shard_ranges:
    32-document-aligned cuts balanced by tokens, doc_base = the shard's first
    global document), or of doc_range=(lo, hi).  Words are read in 256 MB
    pieces by parallel preads into two pinned buffers; each piece's H2D copy
    (side stream) overlaps the read of the next; uint16 ids are widened to
    int32 on the device."""
    import time

    import torch

    from .kernels import DeviceCorpus
    from .sharding import shard_ranges

    _lib.require_cuda()
    t0 = time.perf_counter()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    h = read_bin_header(path)
    if doc_range is None:
        if world > 1:
            full = _read_offsets(path, h)
            lo, hi = shard_ranges(np.diff(full), world)[rank]
        else:
            lo, hi = 0, h["n_docs"]
    else:
        lo, hi = int(doc_range[0]), int(doc_range[1])
        if lo % 32 or not 0 <= lo <= hi <= h["n_docs"]:
            raise ValueError("doc_range must start on a 32-document boundary inside the corpus")
    off = _read_offsets(path, h, lo, hi)
    a, b = int(off[0]), int(off[-1])
    n = b - a
    wb = h["word_bytes"]
    src_dt = torch.int16 if wb == 2 else torch.int32
    words_raw = torch.empty(n, dtype=src_dt, device=dev)
    per = max(1, _CHUNK // wb)
    # two pinned staging buffers, cached across calls (pinning 512 MB costs
    # ~0.8 s, more than reading a 1.25M-document shard)
    pins = [_pinned_stage(i, per * wb).view(src_dt)[:min(per, max(n, 1))] for i in range(2 if n > per else 1)]
    side = torch.cuda.Stream(device=dev)
    done = [None] * len(pins)
    t1 = time.perf_counter()
    for k, s in enumerate(range(0, n, per)):
        e = min(n, s + per)
        slot = k % len(pins)
        if done[slot] is not None:
            done[slot].synchronize()  # the H2D that last used this pinned buffer has finished
        buf = pins[slot]
        _pread(path, h["words_at"] + wb * (a + s), wb * (e - s), buf.data_ptr())
        with torch.cuda.stream(side):
            words_raw[s:e].copy_(buf[:e - s], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        done[slot] = ev
    torch.cuda.current_stream(dev).wait_stream(side)
    t2 = time.perf_counter()
    words = (words_raw.to(torch.int32) & 0xFFFF) if wb == 2 else words_raw
    del words_raw
    dc = DeviceCorpus.from_csr(torch.from_numpy(off - a), words, doc_base=lo, vocab_size=h["vocab_size"],
                               device=dev)
    if dc.n_tokens and dc.word_max >= h["vocab_size"]:
        from .lda import WordIdOutOfRangeError

        raise WordIdOutOfRangeError(f"{path}: word id {dc.word_max} >= V={h['vocab_size']}")
    torch.cuda.synchronize(dev)
    if timing is not None:
        timing.update(header_and_offsets_s=t1 - t0, words_read_and_h2d_s=t2 - t1,
                      prepare_s=time.perf_counter() - t2, total_s=time.perf_counter() - t0, bytes=wb * n + 8 * off.size)
    return dc


# ---------------------------------------------------------------- stop files
class StopFileError(ValueError):
    """The stop-inject file does not fit the corpus (cli.py ConfigError messages)."""


def read_floats(path) -> np.ndarray:
    """np.loadtxt(path, dtype=float64, ndmin=1) for one value per line, by the
    native parser; other layouts go through np.loadtxt itself (flattened)."""
    L = _io()
    h = ctypes.c_void_p()
    n = ctypes.c_int64()
    rc = L.wdio_scan_floats(_cpath(path), _threads(), ctypes.byref(h), ctypes.byref(n))
    if rc == 1:
        return np.loadtxt(path, dtype=np.float64, ndmin=1).ravel()
    _check_rc(rc, "read_floats", path)
    try:
        out = np.empty(n.value, dtype=np.float64)
        L.wdio_fill_floats(h, out.ctypes.data)
    finally:
        L.wdio_release_floats(h)
    return out


def load_injected_units(path, lengths, iterations: int) -> np.ndarray:
    """cli._load_injected_iterations (cli.py:213-230) as one float64 array
    [iterations, sum N]: row t holds iteration t's u per token in (document,
    word) order -- exactly the flat CSR-order units the device draw takes
    (pass row t as the `stops` tensor).  Same size / range checks and
    messages as the reference."""
    flat = read_floats(path)
    per_iter = int(np.sum(np.asarray(lengths, dtype=np.int64)))
    if flat.size != per_iter * iterations:
        raise StopFileError(f"stop file holds {flat.size} values; need {per_iter} x {iterations} iterations")
    if np.any(flat < 0) or np.any(flat >= 1):
        raise StopFileError("injected values must lie in [0, 1)")
    return flat.reshape(iterations, per_iter)


# ------------------------------------------------------------------- writers
def write_z_csv(path, z, offsets):
    """z.csv of cmd_lda (cli.py:259-264) from flat CSR-order z (any signed
    integer dtype; numpy or a torch tensor) and its offsets."""
    if isinstance(z, (list, tuple)):  # the reference's ragged z (run_gibbs output)
        z = np.concatenate([np.asarray(a, dtype=np.int64) for a in z]) if len(z) else np.zeros(0, np.int64)
    z = _host_array(z)
    if z.dtype not in (np.int16, np.int32, np.int64):
        z = z.astype(np.int64)
    z = np.ascontiguousarray(z)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    if off.size < 1 or int(off[-1]) > z.size:
        raise ValueError("offsets do not fit z")
    _check_rc(_io().wdio_write_z_csv(_cpath(path), z.ctypes.data, z.itemsize, off.ctypes.data, off.size - 1,
                                      _threads()), "write_z_csv", path)


def write_matrix_csv(path, matrix):
    """_write_matrix_csv (cli.py:232-236): repr(float(x)) per field."""
    m = _host_array(matrix)
    if m.ndim != 2:
        m = np.atleast_2d(m)
    if m.dtype not in (np.float32, np.float64):
        m = m.astype(np.float64)
    if m.shape[1] == 0 or m.strides[1] != m.itemsize or m.strides[0] % m.itemsize:
        m = np.ascontiguousarray(m)
    if m.shape[1] == 0:  # csv.writer writes an empty row as a bare line end
        with open(path, "wb") as fh:
            fh.write(b"\r\n" * m.shape[0])
        return
    _check_rc(_io().wdio_write_matrix_csv(_cpath(path), m.ctypes.data, m.itemsize, m.shape[0], m.shape[1],
                                           m.strides[0] // m.itemsize, _threads()), "write_matrix_csv", path)


def write_likelihood_csv(path, trajectory):
    """likelihood.csv (cli.py:265-269)."""
    L = _io()
    buf = ctypes.create_string_buffer(40)
    rows = ["iteration,log_likelihood"]
    for t, ll in enumerate(trajectory):
        L.wdio_repr(float(ll), buf)
        rows.append(f"{t},{buf.value.decode()}")
    with open(path, "wb") as fh:
        fh.write(("\r\n".join(rows) + "\r\n").encode())


def write_outputs(outdir, n_docs: int, z, offsets, theta, phi, trajectory):
    """The four files cmd_lda writes (cli.py:256-273): z.csv over the first
    n_docs documents (the corpus cmd_lda loaded), likelihood.csv,
    theta.csv (first n_docs rows), phi.csv."""
    os.makedirs(outdir, exist_ok=True)
    off = np.ascontiguousarray(offsets, dtype=np.int64)[: n_docs + 1]
    write_z_csv(os.path.join(outdir, "z.csv"), z, off)
    write_likelihood_csv(os.path.join(outdir, "likelihood.csv"), trajectory)
    write_matrix_csv(os.path.join(outdir, "theta.csv"), _host_array(theta)[:n_docs])
    write_matrix_csv(os.path.join(outdir, "phi.csv"), phi)


def repr_float(x: float) -> str:
    """Python repr(float(x)) computed by the native writer (tests pin it)."""
    buf = ctypes.create_string_buffer(40)
    _io().wdio_repr(float(x), buf)
    return buf.value.decode()


def _host_array(x):
    try:
        import torch

        if torch.is_tensor(x):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)
