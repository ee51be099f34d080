"""Drop-in replacement for the reference's kernel registry (kernels.py:542-555).

Same names, signatures, error types and messages as
/root/reference/pkg/src/warpdraw/kernels.py; the work runs in the sm_100a
kernels of libwarpdraw_b200.so:

    draw_z_butterfly   -> wd_draw_z(WD_BUTTERFLY, keys = master index)
    draw_z_transposed  -> wd_draw_z(WD_PREFIX,    keys = master index)
    draw_z_basic       -> wd_draw_z(WD_PREFIX,    keys = word position)

z is bit-identical to the reference for float32 and float64 inputs (see
tests/test_gpu_parity.py).  Two entry levels:

  * the reference signature (host numpy in, ragged int64 lists out);
  * draw_z_device: device-resident corpus/parameters (DeviceCorpus + torch
    CUDA tensors), z as an int32 CUDA tensor, optional fused topic counts --
    the fast path the LDA driver and bench.py use.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .sampling import AllZeroError

try:  # host helper of the boundary (csrc/wd_host.c; built by build.py)
    from . import _wdhost
except ImportError:  # pragma: no cover - numpy fallback for the host-side loops only
    _wdhost = None
from .warp import OutOfBoundsError, Trace, WarpConfig

__all__ = [
    "VocabTiles",
    "block_aligned_rows",
    "combine_err",
    "StopOutOfRangeError",
    "SeededStops",
    "InjectedStops",
    "PhiloxStops",
    "DeviceCorpus",
    "draw_z_device",
    "draw_z_basic",
    "draw_z_transposed",
    "draw_z_butterfly",
    "KERNELS",
    "draw_z",
]


class StopOutOfRangeError(ValueError):
    """A search was handed a stop value outside [0, sum)."""


# --- stop randomness providers (kernels.py:42-92) ---


class SeededStops:
    """Fresh hashed stream per (document, master iteration) (kernels.py:42-53).

    On the device the hash is evaluated inline at each stored token's final
    key, so no redundant redraws are executed.
    """

    def __init__(self, seed: int):
        self.seed = int(seed)

    def units(self, m, i, i_master):
        from .rng import units_for

        return units_for(self.seed, m, i_master)


class InjectedStops:
    """Pre-drawn unit values looked up by (document, word index) (kernels.py:56-92)."""

    def __init__(self, units):
        self._units = [np.asarray(u, dtype=np.float64) for u in units]
        self._csr = None  # (lengths, flat) when built from one flat CSR-order array

    @classmethod
    def from_flat(cls, flat, lengths) -> "InjectedStops":
        """u per token in CSR (document, word) order, e.g. one row of
        corpus_io.load_injected_units; the flat array is kept as the device
        layout (no per-document concatenation in flat())."""
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        lengths = np.asarray(lengths, dtype=np.int64)
        off = np.concatenate([[0], np.cumsum(lengths)])
        if flat.size != int(off[-1]):
            raise ValueError(f"{flat.size} values for {int(off[-1])} tokens")
        st = cls(csr_to_ragged(flat, off))
        st._csr = (lengths, flat)
        return st

    @classmethod
    def from_seed(cls, seed: int, lengths) -> "InjectedStops":
        from .rng import units_for

        return cls([units_for(seed, np.full(int(n), m), np.arange(int(n))) for m, n in enumerate(lengths)])

    @classmethod
    def from_file(cls, path, lengths) -> "InjectedStops":
        from .corpus_io import read_floats  # np.loadtxt semantics, native parser

        flat = read_floats(path)
        if flat.size != int(np.sum(lengths)):
            raise ValueError(
                f"stop file {path} holds {flat.size} values, corpus needs {int(np.sum(lengths))}"
            )
        if np.any(flat < 0) or np.any(flat >= 1):
            raise ValueError("injected values must lie in [0, 1)")
        return cls.from_flat(flat, lengths)

    def units(self, m, i, i_master):
        mm = np.atleast_1d(np.asarray(m))
        ii = np.atleast_1d(np.asarray(i))
        out = np.zeros(mm.shape, dtype=np.float64)
        for t in range(mm.size):
            row = self._units[int(mm.flat[t])]
            out.flat[t] = row[int(ii.flat[t])] if row.size else 0.0
        return out

    def flat(self, lengths) -> np.ndarray:
        """u in CSR token order (doc-major), the device layout."""
        lengths = np.asarray(lengths, dtype=np.int64)
        if self._csr is not None and np.array_equal(self._csr[0], lengths):
            return self._csr[1]
        if len(self._units) == lengths.size:
            lens = np.fromiter(map(len, self._units), dtype=np.int64, count=lengths.size)
            if np.array_equal(lens, lengths):
                return np.concatenate(self._units) if lengths.size else np.zeros(0)
        parts = []
        for m, n in enumerate(lengths):
            n = int(n)
            if n == 0:
                continue
            row = self._units[m]
            parts.append(row[:n] if row.size else np.zeros(n))
        return np.concatenate(parts) if parts else np.zeros(0)


class PhiloxStops:
    """Opt-in counter-based Philox4x32-10 stream keyed by (seed, doc, word).

    NOT reference-parity (the reference's stream is the SplitMix64/xoshiro
    hash); provided for users who want a standard counter RNG.
    """

    def __init__(self, seed: int):
        self.seed = int(seed)


# --- device corpus ---


def _torch():
    import torch

    return torch


@dataclass
class DeviceCorpus:
    """A CSR corpus shard resident in HBM.

    offsets [n_docs+1] int64, words [n_tokens] int32, token_doc [n_tokens]
    int32, last_key [n_docs] int32 (master-index key of each doc's last
    word for `lanes`-doc groups).  doc_base is the global id of local doc 0.
    """

    offsets: object
    words: object
    token_doc: object
    n_docs: int
    n_tokens: int
    doc_base: int = 0
    vocab_size: int | None = None
    _last_key: dict = field(default_factory=dict)
    word_min: int = 0
    word_max: int = -1

    def check_words(self, n_rows: int):
        """Word ids must index phi's rows: the reference raises OutOfBoundsError
        from GlobalArray2D._check (warp.py:234-240; IndexError in basic's numpy
        indexing).  Checked once per call from the range cached at build time,
        before any launch (a bad id would read and, with fused counts, write
        outside phi / word_topic)."""
        if self.n_tokens and (self.word_min < 0 or self.word_max >= n_rows):
            bad = self.word_min if self.word_min < 0 else self.word_max
            raise OutOfBoundsError(f"phi[{bad}, :]: word id out of bounds for {n_rows} rows")

    @classmethod
    def from_csr(cls, offsets, words, doc_base: int = 0, vocab_size: int | None = None, device=None):
        torch = _torch()
        _lib.require_cuda()
        dev = device or torch.device("cuda")
        off = torch.as_tensor(np.asarray(offsets, dtype=np.int64) if not torch.is_tensor(offsets) else offsets,
                              dtype=torch.int64).to(dev).contiguous()
        if torch.is_tensor(words):
            if words.dtype != torch.int32:
                lo, hi = torch.aminmax(words) if words.numel() else (0, -1)
                _check_int32(int(lo), int(hi))
            wd = words.to(device=dev, dtype=torch.int32).contiguous()
        else:
            words = np.asarray(words)
            if words.dtype != np.int32:
                if words.size:
                    _check_int32(int(words.min()), int(words.max()))
                words = words.astype(np.int32)
            wd = torch.from_numpy(np.ascontiguousarray(words)).to(dev)
        n_docs = off.numel() - 1
        n_tokens = wd.numel()
        wmin, wmax = (0, -1)
        if n_tokens:
            lo, hi = torch.aminmax(wd)
            wmin, wmax = int(lo), int(hi)
        td = torch.empty(n_tokens, dtype=torch.int32, device=dev)
        L = _lib.load()
        _lib.check(L.wd_corpus_prepare(off.data_ptr(), n_docs, n_tokens, int(doc_base), 32, td.data_ptr(), None,
                                       _lib.stream_handle()), "wd_corpus_prepare")
        return cls(off, wd, td, n_docs, n_tokens, int(doc_base), vocab_size, word_min=wmin, word_max=wmax)

    @classmethod
    def from_ragged(cls, lengths, words, doc_base: int = 0, vocab_size: int | None = None):
        offsets, flat = ragged_to_csr(lengths, words)
        return cls.from_csr(offsets, flat, doc_base, vocab_size)

    def vocab_tiles(self, rows_per_tile: int, run_pad: int = 0) -> VocabTiles:
        """Token list regrouped by vocabulary tile (cached per tile size)."""
        key = ("tiles", int(rows_per_tile), int(run_pad))
        if key not in self._last_key:
            self._last_key[key] = _build_vocab_tiles(self, int(rows_per_tile), int(run_pad))
        return self._last_key[key]

    def last_key(self, lanes: int):
        if lanes not in self._last_key:
            torch = _torch()
            lk = torch.empty(max(self.n_docs, 1), dtype=torch.int32, device=self.offsets.device)
            L = _lib.load()
            _lib.check(L.wd_corpus_prepare(self.offsets.data_ptr(), self.n_docs, self.n_tokens, self.doc_base,
                                           int(lanes), None, lk.data_ptr(), _lib.stream_handle()),
                       "wd_corpus_prepare")
            self._last_key[lanes] = lk
        return self._last_key[lanes]


def _check_int32(lo: int, hi: int):
    if lo < -(1 << 31) or hi >= (1 << 31):
        raise OutOfBoundsError(f"word id {hi if hi >= (1 << 31) else lo} does not fit the int32 device layout")


def ragged_to_csr(lengths, words):
    """(offsets[M+1] int64, words[sum N] int32) of a ragged corpus: document m
    contributes words[m][:lengths[m]] (the reference reads w[m][i] for i < N[m],
    kernels.py:364-377).  One np.concatenate, no per-document Python work
    when every list is exactly N[m] long (the Corpus invariant, lda.py:42-53)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    M = lengths.size
    offsets = np.zeros(M + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    if M == 0 or offsets[-1] == 0:
        return offsets, np.zeros(0, np.int32)
    if isinstance(words, np.ndarray) and words.ndim == 2:  # dense [M, >= max N]
        if words.shape[1] < lengths.max():
            raise ValueError("word lists shorter than the document lengths")
        mask = np.arange(words.shape[1])[None, :] < lengths[:, None]
        flat = words[:M][mask]
    else:
        if _wdhost is not None and isinstance(words, list) and len(words) == M:
            try:
                flat, _, _ = _wdhost.concat_ragged(words, lengths)
                return offsets, flat
            except TypeError:
                pass  # not plain integer ndarrays: numpy below
            except OverflowError as exc:
                raise OutOfBoundsError(str(exc)) from None
        arrs = [np.asarray(words[m]) for m in range(M)] if not isinstance(words, list) else words
        lens = np.fromiter(map(len, arrs), dtype=np.int64, count=M)
        if np.any(lens < lengths):
            raise ValueError("word lists shorter than the document lengths")
        if np.array_equal(lens, lengths):
            flat = np.concatenate(arrs)
        else:
            flat = np.concatenate([np.asarray(a)[:n] for a, n in zip(arrs, lengths.tolist())])
    if flat.dtype != np.int32:
        if flat.size and (int(flat.min()) < -(1 << 31) or int(flat.max()) >= (1 << 31)):
            _check_int32(int(flat.min()), int(flat.max()))
        flat = flat.astype(np.int32)
    return offsets, flat


def csr_to_ragged(z, offsets) -> list:
    """Ragged list of int64 arrays (views into one fresh int64 buffer) from a
    flat z and its CSR offsets: the reference's output shape
    (`_ragged_zeros`, kernels.py:364-369), without a per-document copy."""
    if _wdhost is not None and isinstance(z, np.ndarray) and z.ndim == 1 and z.flags.c_contiguous:
        return _wdhost.ragged_views(z, np.ascontiguousarray(offsets, dtype=np.int64))
    ol = offsets.tolist() if isinstance(offsets, np.ndarray) else list(offsets)
    return [z[a:b] for a, b in zip(ol[:-1], ol[1:])]


@dataclass
class VocabTiles:
    """The corpus' tokens regrouped by vocabulary tile.

    Tile t holds the tokens whose word lies in [t*rows, (t+1)*rows), ordered
    by (document, word, position): documents stay contiguous and a
    document's repeated words sit on adjacent rows (their phi loads hit L1).  Drawing tile by tile
    keeps the active slice of phi (rows x K) resident in the 126 MB L2 while
    theta rows stream; z, units and the hash keys still use each token's
    original (document, position), so results are bit-identical to the
    untiled draw.

    run_pad > 0: every (tile, document) run of tokens is padded to a multiple
    of run_pad slots (8 = the L consecutive chunk rows a lane group of the
    butterfly kernel loads), so no lane group straddles two documents and
    each lane needs ONE theta segment per block (no per-row selection).
    Padding slots carry token_pos = -1, their run's document and its last
    word: valid loads, nothing drawn.
    """

    words: object
    token_doc: object
    token_pos: object
    bounds: list
    rows_per_tile: int
    run_pad: int = 0
    n_tokens: int = 0

    @property
    def n_tiles(self) -> int:
        return len(self.bounds) - 1


def _build_vocab_tiles(corpus: "DeviceCorpus", rows_per_tile: int, run_pad: int = 0) -> VocabTiles:
    torch = _torch()
    tile = torch.div(corpus.words, rows_per_tile, rounding_mode="floor").to(torch.int32)
    # order: (tile, document, word).  Documents stay contiguous inside a tile
    # (the draw's theta-segment sharing), and a document's repeated words
    # become adjacent rows, whose phi loads then hit L1 instead of L2.
    V = int(corpus.words.max().item()) + 1 if corpus.n_tokens else 1
    M = max(1, corpus.n_docs)
    key = (tile.to(torch.int64) * M + corpus.token_doc.to(torch.int64)) * V + corpus.words.to(torch.int64)
    _, order = torch.sort(key, stable=True)
    del key
    words = corpus.words[order].contiguous()
    doc = corpus.token_doc[order].contiguous()
    pos = (order - corpus.offsets[doc.long()]).to(torch.int32).contiguous()
    tile = tile[order]
    del order
    n_tiles = int(tile.max().item()) + 1 if corpus.n_tokens else 1
    T = corpus.n_tokens
    if run_pad > 1 and T:
        dev = words.device
        brk = torch.ones(T, dtype=torch.bool, device=dev)
        brk[1:] = (doc[1:] != doc[:-1]) | (tile[1:] != tile[:-1])
        run_start = brk.nonzero().squeeze(1)
        run_len = torch.diff(run_start, append=torch.tensor([T], device=dev))
        plen = (run_len + run_pad - 1) // run_pad * run_pad
        new_start = torch.cumsum(plen, 0) - plen
        run_id = torch.cumsum(brk.to(torch.int64), 0) - 1
        del brk
        dest = new_start[run_id] + (torch.arange(T, device=dev) - run_start[run_id])
        slot_run = torch.repeat_interleave(torch.arange(run_start.numel(), device=dev), plen)
        pw = words[run_start + run_len - 1][slot_run]
        pd = doc[run_start][slot_run]
        pp = torch.full((slot_run.numel(),), -1, dtype=torch.int32, device=dev)
        pw[dest] = words
        pp[dest] = pos
        counts = torch.zeros(n_tiles, dtype=torch.int64, device=dev).index_add_(0, tile[run_start].long(), plen)
        counts = counts.cpu().numpy()
        del dest, slot_run, run_id, new_start, run_start, run_len, plen
        words, doc, pos = pw.contiguous(), pd.contiguous(), pp.contiguous()
    else:
        counts = torch.bincount(tile.long(), minlength=n_tiles).cpu().numpy()
    bounds = [0] + np.cumsum(counts).tolist()
    del tile
    return VocabTiles(words, doc, pos, [int(b) for b in bounds], int(rows_per_tile), int(run_pad), int(T))


def block_aligned_rows(n_rows: int, K: int, dtype=None, device=None, lanes: int = 32):
    """An [n_rows, K] theta/phi buffer whose W-topic blocks start on 128-byte
    lines: a view into a row-padded allocation, offset so that column
    K mod W (the first block; the remnant comes first, kernels.py:199-205)
    is line-aligned, with a leading dimension of whole lines.  With K = 200 a
    dense row is 800 B and every 128-byte block segment straddles two L1/L2
    lines (two wavefronts per row per load); aligned, it touches one.  Same
    values, same results, ~12% more memory at K = 200, none when K % 32 == 0."""
    torch = _torch()
    dtype = dtype or torch.float32
    esz = torch.empty(0, dtype=dtype).element_size()
    line = 128 // esz
    lead = (-(K % lanes)) % line
    ld = -(-(lead + K) // line) * line
    if lead == 0 and ld == K:
        return torch.empty((n_rows, K), dtype=dtype, device=device)
    return torch.empty((n_rows, ld), dtype=dtype, device=device)[:, lead : lead + K]


def to_block_aligned(t, lanes: int = 32):
    """Copy of a 2-D CUDA tensor in the block_aligned_rows layout."""
    out = block_aligned_rows(t.shape[0], t.shape[1], t.dtype, t.device, lanes)
    out.copy_(t)
    return out


_DTYPES = {"float32": _lib.WD_FLOAT32, "float64": _lib.WD_FLOAT64}


def _dtype_code(t) -> int:
    name = str(t.dtype).replace("torch.", "")
    if name not in _DTYPES:
        raise TypeError(f"theta/phi must be float32 or float64, got {t.dtype}")
    return _DTYPES[name]


_workspace_cache: dict = {}


def _workspace(variant, dtype_code, lanes, K, device):
    L = _lib.load()
    nbytes = int(L.wd_workspace_bytes(variant, dtype_code, lanes, int(K)))
    if nbytes == 0:
        return None, 0
    torch = _torch()
    key = (str(device), variant)
    buf = _workspace_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        _workspace_cache[key] = buf
    return buf, nbytes


_KERNEL_SPEC = {
    # name: (variant, key rule, requires M % W == 0)
    "basic": (_lib.WD_PREFIX, _lib.WD_KEYS_POSITION, False),
    "transposed": (_lib.WD_PREFIX, _lib.WD_KEYS_MASTER, True),
    "butterfly": (_lib.WD_BUTTERFLY, _lib.WD_KEYS_MASTER, True),
}


def _token_positions(corpus: DeviceCorpus):
    """Host (m, i) of every token in CSR order (only for generic stop providers)."""
    off = corpus.offsets.cpu().numpy()
    lengths = np.diff(off)
    m = np.repeat(np.arange(corpus.n_docs), lengths)
    i = np.arange(corpus.n_tokens) - np.repeat(off[:-1], lengths)
    return m, i, lengths


def _stop_args(stops, corpus: DeviceCorpus, key_rule: int, lanes: int, device):
    """Map a stops provider to (mode, seed, units tensor)."""
    torch = _torch()
    if isinstance(stops, SeededStops):
        return _lib.WD_STOPS_SEEDED, stops.seed, None
    if isinstance(stops, PhiloxStops):
        return _lib.WD_STOPS_PHILOX, stops.seed, None
    if isinstance(stops, InjectedStops):
        lengths = np.diff(corpus.offsets.cpu().numpy())
        flat = stops.flat(lengths)
        return _lib.WD_STOPS_UNITS, 0, torch.from_numpy(np.ascontiguousarray(flat)).to(device)
    if torch.is_tensor(stops):  # u per token, float64, CSR order
        return _lib.WD_STOPS_UNITS, 0, stops.to(device=device, dtype=torch.float64).contiguous()
    if hasattr(stops, "units"):
        # duck-typed provider: evaluate .units at each stored token's final
        # key (kernels.py:520-536 master-index rule) on the host
        m, i, lengths = _token_positions(corpus)
        i_master = i.copy()
        if key_rule == _lib.WD_KEYS_MASTER and corpus.n_docs:
            gm = corpus.doc_base + np.arange(corpus.n_docs)
            q = gm // lanes
            gmax = np.zeros(q.max() + 1, dtype=np.int64)
            np.maximum.at(gmax, q, lengths)
            last = i == lengths[m] - 1
            i_master[last] = gmax[q[m[last]]] - 1
        u = np.asarray(stops.units(corpus.doc_base + m, i, i_master), dtype=np.float64)
        return _lib.WD_STOPS_UNITS, 0, torch.from_numpy(np.ascontiguousarray(u)).to(device)
    raise TypeError(f"unsupported stops provider {type(stops).__name__}")


def raise_for_err(err_host, key_rule: int, lanes: int):
    allzero, stop_bad = int(err_host[0]), int(err_host[1]) != _lib.ERR_NONE
    if stop_bad:
        raise StopOutOfRangeError("stop values must lie in [0, sum)")
    if allzero != _lib.ERR_NONE:
        if key_rule == _lib.WD_KEYS_POSITION:
            m, i = allzero >> 32, allzero & 0xFFFFFFFF
            raise AllZeroError(f"document {m}, word {i}: all products are zero")
        q, r = allzero >> 40, allzero & 0xFF
        raise AllZeroError(f"document {q * lanes + r}: all products are zero")


def draw_z_device(kernel: str, corpus: DeviceCorpus, theta, phi, stops, lanes: int = 32, *, z=None,
                  word_topic=None, doc_topic=None, err=None, check: bool = True, stream=None,
                  tiles: VocabTiles | None = None, after_tile=None):
    """Device-resident draw.  theta [n_docs, K], phi [V, K] CUDA tensors
    (float32 or float64, same dtype, row stride = leading dim).  Returns z
    (int32 CUDA tensor, CSR token order).  word_topic / doc_topic (int32) are
    incremented in the same kernel when given.  tiles (corpus.vocab_tiles)
    draws tile by tile so each phi slice stays L2-resident; z is identical.
    check=False skips the host synchronisation on the error word (err, shape
    [n_launches, 2], must then be supplied and inspected by the caller with
    raise_for_err(combine_err(err))).  after_tile(t, word_lo, word_hi) is
    called right after tile t's launch is enqueued: the word_topic rows
    [word_lo, word_hi) are final on the stream from that point (a tile's
    tokens are exactly the words of its range), which lets a caller start
    their all-reduce while the next tile draws."""
    torch = _torch()
    if kernel not in _KERNEL_SPEC:
        raise ValueError(f"unknown kernel {kernel!r}; pick one of {sorted(_KERNEL_SPEC)}")
    variant, key_rule, needs_pad = _KERNEL_SPEC[kernel]
    if needs_pad and (corpus.n_docs % lanes or corpus.doc_base % lanes):
        raise ValueError("document count must be a multiple of the lane count (pad upstream)")
    _lib.require_cuda()
    # float32 theta with float64 phi: the reference forms fl32(fl64(theta *
    # phi)) (numpy promotion, kernels.py:209, 391) -- a dedicated path keeps
    # phi in float64 (csrc/wd_mixed.cu); float64 theta with float32 phi is
    # exact after widening phi
    mixed = theta.dtype == torch.float32 and phi.dtype == torch.float64
    if theta.dtype != phi.dtype and not mixed:
        phi = phi.to(theta.dtype)
    if theta.stride(-1) != 1 or phi.stride(-1) != 1:
        raise ValueError("theta/phi rows must be contiguous")
    K = int(theta.shape[1])
    if int(phi.shape[1]) != K:
        raise ValueError("theta and phi disagree on the topic count")
    if theta.shape[0] < corpus.n_docs:
        raise ValueError("theta has fewer rows than the corpus has documents")
    dev = theta.device
    dt = _lib.WD_FLOAT32_PHI64 if mixed else _dtype_code(theta)
    mode, seed, units = _stop_args(stops, corpus, key_rule, lanes, dev)
    if mode == _lib.WD_STOPS_UNITS and units.numel() < corpus.n_tokens:
        raise ValueError("units do not cover every token")
    if z is None:
        z = torch.empty(corpus.n_tokens, dtype=torch.int32, device=dev)
    if tiles is None:
        launches = [(corpus.words, corpus.token_doc, None, 0, corpus.n_tokens, 0)]
    else:
        launches = [(tiles.words, tiles.token_doc, tiles.token_pos, a, b - a, t)
                    for t, (a, b) in enumerate(zip(tiles.bounds[:-1], tiles.bounds[1:])) if b > a]
    if err is None or err.numel() < 2 * max(1, len(launches)):
        err = torch.empty((max(1, len(launches)), 2), dtype=torch.int64, device=dev)
    err2 = err.view(-1, 2)
    # ERR_NONE in every row: rows beyond this call's launches (e.g. vocabulary
    # tiles this shard has no tokens in) must not hold stale words
    err2.fill_(-1)
    corpus.check_words(int(phi.shape[0]))
    last_key = corpus.last_key(lanes) if (mode == _lib.WD_STOPS_SEEDED and key_rule == _lib.WD_KEYS_MASTER) else None
    ws, ws_bytes = (None, 0) if mixed else _workspace(variant, dt, lanes, K, dev)
    L = _lib.load()
    st = _lib.stream_handle(stream)
    for li, (wds, tdoc, tpos, a, n, t) in enumerate(launches):
        _lib.check(
            L.wd_draw_z(variant, dt, int(lanes), theta.data_ptr(), theta.stride(0), phi.data_ptr(), phi.stride(0), K,
                        corpus.offsets.data_ptr(), wds.data_ptr() + 4 * a, tdoc.data_ptr() + 4 * a,
                        None if tpos is None else tpos.data_ptr() + 4 * a, _lib.ptr(last_key), corpus.n_docs, n,
                        corpus.doc_base, mode, key_rule, int(seed) & ((1 << 64) - 1), _lib.ptr(units), None,
                        z.data_ptr(), _lib.ptr(word_topic), _lib.ptr(doc_topic), err2[li].data_ptr(), _lib.ptr(ws),
                        ws_bytes, st),
            "wd_draw_z")
        if after_tile is not None:
            V = int(phi.shape[0])
            lo, hi = (0, V) if tiles is None else (t * tiles.rows_per_tile, min(V, (t + 1) * tiles.rows_per_tile))
            after_tile(t, lo, hi)
    if check:
        raise_for_err(combine_err(err2[: max(1, len(launches))]), key_rule, lanes)
    return z


def combine_err(err) -> np.ndarray:
    """Fold per-launch error words [n, 2] into one (min AllZero key, any range flag)."""
    e = err.reshape(-1, 2).cpu().numpy().view(np.uint64)
    return np.array([e[:, 0].min(), e[:, 1].min()], dtype=np.uint64)


class _HostCorpusCache:
    """DeviceCorpus of the ragged word lists a reference-signature call was
    last made with.  gibbs_iterate passes the same `corpus.words` list every
    iteration (lda.py:229-238), so the host->CSR conversion and the corpus
    upload happen once per corpus, not once per call.  A hit needs the same
    list object holding the same array objects (ids compared: ~50 ms for 1M
    documents) and the same lengths; the arrays themselves are treated as
    immutable, as the reference's Corpus treats them."""

    def __init__(self, size: int = 2):
        self.size = size
        self.entries = []  # (w, ids, N, corpus)

    @staticmethod
    def _ids(w):
        if not isinstance(w, list):
            return None
        if _wdhost is not None:
            return _wdhost.list_ids(w)
        return np.fromiter(map(id, w), dtype=np.int64, count=len(w))

    @staticmethod
    def _same(w, ids):
        if _wdhost is not None:
            return _wdhost.ids_equal(w, ids)
        return ids.size == len(w) and np.array_equal(ids, np.fromiter(map(id, w), dtype=np.int64, count=len(w)))

    def get(self, N, w):
        for ent in self.entries:
            ew, eids, eN, corpus = ent
            if ew is w and np.array_equal(eN, N) and self._same(w, eids):
                return corpus
        ids = self._ids(w)
        corpus = DeviceCorpus.from_ragged(N, w)
        if ids is not None:
            self.entries.insert(0, (w, ids, N.copy(), corpus))
            del self.entries[self.size:]
        return corpus

    def clear(self):
        self.entries = []


_host_corpora = _HostCorpusCache()
_host_bufs: dict = {}


def _pinned(slot, nbytes):
    torch = _torch()
    buf = _host_bufs.get(slot)
    if buf is None or buf.numel() < nbytes:
        _host_bufs.pop(slot, None)
        buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8).pin_memory()
        _host_bufs[slot] = buf
    return buf


_H2D_CHUNKS = 4


def _upload_params(x, lanes, slot):
    """Host theta/phi -> a cached device buffer in the block_aligned_rows
    layout: row chunks are copied into a cached pinned buffer by torch's
    multi-threaded copy, each chunk's H2D enqueued behind it (the copy of
    chunk i+1 overlaps the transfer of chunk i).  No allocation after the
    first call; the next call reuses the pinned buffer only after this call's
    draw has synchronised."""
    torch = _torch()
    x = np.ascontiguousarray(x)
    key = (slot, x.shape, x.dtype.str)
    buf = _host_bufs.get(key)
    if buf is None:
        _host_bufs.pop(next((k for k in _host_bufs if isinstance(k, tuple) and k[0] == slot), None), None)
        buf = block_aligned_rows(x.shape[0], x.shape[1], getattr(torch, x.dtype.name), torch.device("cuda"), lanes)
        _host_bufs[key] = buf
    src = torch.from_numpy(x)
    pin = _pinned("pin_" + slot, x.nbytes).view(src.dtype)[: x.size].view(x.shape)
    rows = x.shape[0]
    step = max(1, -(-rows // _H2D_CHUNKS))
    for a in range(0, rows, step):
        pin[a:a + step].copy_(src[a:a + step])
        buf[a:a + step].copy_(pin[a:a + step], non_blocking=True)
    return buf


_ASYNC_OUT_MIN = 1 << 16  # tokens: below this the synchronous path is as fast


def _to_host_ragged(z_dev, offsets_host):
    """z (int32, device) -> list of int64 arrays: D2H into a cached pinned
    buffer, widened by torch's multi-threaded copy into one fresh int64
    buffer, then one view per document (csr_to_ragged)."""
    torch = _torch()
    n = z_dev.numel()
    pin = _pinned("z", 4 * n).view(torch.int32)[:n]
    pin.copy_(z_dev)  # synchronous D2H
    if _wdhost is not None and hasattr(_wdhost, "widen_i32"):
        # a fresh huge-page mapping filled by several threads (the page
        # faults of a fresh 4K-page buffer cost more than the copy)
        z64 = _wdhost.widen_i32(pin.data_ptr(), n, max(1, min(16, len(os.sched_getaffinity(0)))))
    else:
        z64 = torch.empty(n, dtype=torch.int64)
        z64.copy_(pin)
        z64 = z64.numpy()
    return csr_to_ragged(z64, offsets_host)


# Pinned int64 host buffers the reference-signature call returns z in (its
# per-document arrays are views of one).  An entry is [tensor, weakref to the
# ndarray handed out]: it is reused once every view of that ndarray is gone
# (the weakref is dead), so a caller that keeps the previous call's z while
# making the next call (run_gibbs) alternates between two buffers.  At most
# _Z_OUT_POOL_MAX buffers; a caller holding more results gets the pageable
# path (_to_host_ragged).
_Z_OUT_POOL_MAX = 3
_z_out_pool: list = []


def _z_out_buffer(n):
    """(pinned int64 tensor, its ndarray) with room for n values and no live
    views, or None when the pool is full of buffers still referenced."""
    import weakref

    torch = _torch()
    free = [e for e in _z_out_pool if e[1] is None or e[1]() is None]
    ent = next((e for e in free if e[0].numel() >= n), None)
    if ent is None:
        if free:  # a free buffer that is too small: replace it
            _z_out_pool.remove(free[0])
        elif len(_z_out_pool) >= _Z_OUT_POOL_MAX:
            return None
        # page-locked memory is taken from the host: keep the pool under a
        # quarter of physical memory
        held = sum(e[0].numel() * 8 for e in _z_out_pool)
        try:
            phys = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        except (ValueError, OSError, AttributeError):
            phys = 0
        if phys and held + 8 * int(n) > phys // 4:
            return None
        ent = [torch.empty(max(int(n), 1), dtype=torch.int64).pin_memory(), None]
        _z_out_pool.append(ent)
    full = ent[0].numpy()
    ent[1] = weakref.ref(full)
    return ent[0], full


# wall-clock phases of the last reference-signature call (seconds): corpus
# lookup/upload, theta+phi upload enqueue, then on the synchronous path the
# draw (incl. its error check) and the z download; on the pinned-buffer path
# (large corpora) upload_and_draw is the enqueue of everything plus the
# host-side views, download the remaining wait for the stream
last_host_timing: dict = {}


def _host_call(kernel, N, theta, phi, w, lanes, stops, trace, threads, step_hook):
    if step_hook is not None:
        raise NotImplementedError("step_hook is an emulator instrumentation hook; not available on the device path")
    theta = np.asarray(theta)
    phi = np.asarray(phi)
    if theta.dtype not in (np.float32, np.float64):
        theta = theta.astype(np.float64)
    N = np.asarray(N, dtype=np.int64)
    M = theta.shape[0] if kernel != "basic" else len(N)
    if kernel != "basic" and M % lanes:
        raise ValueError("document count must be a multiple of the lane count (pad upstream)")
    _lib.require_cuda()
    import time

    t0 = time.perf_counter()
    corpus = _host_corpora.get(N, w)
    t1 = time.perf_counter()
    th = _upload_params(theta, lanes, "theta")
    # float32 theta keeps a float64 phi as is (the reference's promotion);
    # otherwise phi takes theta's dtype (float64 theta: exact widening)
    keep64 = theta.dtype == np.float32 and phi.dtype == np.float64
    ph = _upload_params(phi if keep64 else phi.astype(theta.dtype, copy=False), lanes, "phi")
    t2 = time.perf_counter()
    off = np.zeros(N.size + 1, dtype=np.int64)
    np.cumsum(N, out=off[1:])
    n = corpus.n_tokens
    slot = _z_out_buffer(n) if (n >= _ASYNC_OUT_MIN and _wdhost is not None) else None
    if slot is None:
        z = draw_z_device(kernel, corpus, th, ph, stops, lanes)  # synchronises (error check)
        t3 = time.perf_counter()
        out = _to_host_ragged(z, off)
    else:
        # everything on the stream at once -- uploads, draw, int64 widening,
        # D2H into the pinned result buffer -- while the host builds the
        # per-document views of that buffer (they need its address, not its
        # contents); then one synchronisation and the error check
        torch = _torch()
        key_rule = _KERNEL_SPEC[kernel][1]
        err = torch.empty((1, 2), dtype=torch.int64, device=th.device)
        z = draw_z_device(kernel, corpus, th, ph, stops, lanes, err=err, check=False)
        host_t, full = slot
        host_t[:n].copy_(z.to(torch.int64), non_blocking=True)
        out = csr_to_ragged(full[:n], off)
        t3 = time.perf_counter()
        e = combine_err(err)  # synchronises
        raise_for_err(e, key_rule, lanes)
    t4 = time.perf_counter()
    last_host_timing.update(corpus=t1 - t0, upload_enqueue=t2 - t1, upload_and_draw=t3 - t1, download=t4 - t3,
                            total=t4 - t0)
    return out


def draw_z_basic(N, theta, phi, w, stops) -> list:
    """Sequential-order prefix table per word (kernels.py:380-401), on the GPU."""
    return _host_call("basic", N, theta, phi, w, 32, stops, None, 1, None)


def draw_z_transposed(N, theta, phi, w, config: WarpConfig, stops, trace: Trace | None = None, threads: int = 1,
                      step_hook=None) -> list:
    """The paper's full prefix-sum-table kernel (kernels.py:428-484), on the GPU."""
    return _host_call("transposed", N, theta, phi, w, config.lanes, stops, trace, threads, step_hook)


def draw_z_butterfly(N, theta, phi, w, config: WarpConfig, stops, trace: Trace | None = None, threads: int = 1,
                     step_hook=None) -> list:
    """Butterfly-patterned partial sums (kernels.py:487-539), on the GPU."""
    return _host_call("butterfly", N, theta, phi, w, config.lanes, stops, trace, threads, step_hook)


KERNELS = {
    "basic": draw_z_basic,
    "transposed": draw_z_transposed,
    "butterfly": draw_z_butterfly,
}


def draw_z(kernel: str, N, theta, phi, w, config: WarpConfig, stops, **kwargs):
    """Dispatch a kernel by name with a uniform signature (kernels.py:549-555)."""
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}; pick one of {sorted(KERNELS)}")
    if kernel == "basic":
        return draw_z_basic(N, theta, phi, w, stops)
    return KERNELS[kernel](N, theta, phi, w, config, stops, **kwargs)
