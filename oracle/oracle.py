"""ctypes front-end to the CPU oracle (oracle/wd_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs as the parity checker.  The product package
(paper_1505_03851_b200) never imports this module.

Parity: pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libwd_oracle.so")
_lib = None

KEY_MASTER = 0
KEY_POSITION = 1
BUTTERFLY = 0
PREFIX = 1


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "wd_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "-B", "libwd_oracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, i32, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.wdo_derive_seed.restype = u64
        L.wdo_derive_seed.argtypes = [u64, vp, i32]
        L.wdo_unit.restype = dbl
        L.wdo_unit.argtypes = [u64, vp, i32]
        L.wdo_units.restype = None
        L.wdo_units.argtypes = [u64, i32, vp, vp, vp, i64, vp]
        for sfx in ("f32", "f64"):
            f = getattr(L, f"wdo_draw_one_{sfx}")
            f.restype = i64
            f.argtypes = [i32, vp, i64, i32, i32, i32, dbl, vp, vp]
            f = getattr(L, f"wdo_sample_rows_{sfx}")
            f.restype = None
            f.argtypes = [i32, i32, vp, i64, i64, i64, i64, u64, vp, vp, vp, i32]
            f = getattr(L, f"wdo_draw_z_{sfx}")
            f.restype = i32
            f.argtypes = [i32, i32, i32, vp, i64, vp, i64, vp, vp, i64, i64, i64, u64, vp, vp, vp, i32]
        L.wdo_topic_counts.restype = None
        L.wdo_topic_counts.argtypes = [vp, vp, vp, i64, i64, vp, vp]
        L.wdo_max_threads.restype = i32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _sfx(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"unsupported dtype {dt}")


def max_threads() -> int:
    return int(lib().wdo_max_threads())


def derive_seed(seed: int, *keys: int) -> int:
    k = np.asarray([int(x) & ((1 << 64) - 1) for x in keys], dtype=np.uint64).view(np.int64)
    return int(lib().wdo_derive_seed(int(seed) & ((1 << 64) - 1), _p(k) if k.size else None, len(keys)))


def units(seed: int, *key_arrays) -> np.ndarray:
    keys = [np.ascontiguousarray(np.asarray(k, dtype=np.int64).ravel()) for k in key_arrays]
    n = keys[0].size if keys else 1
    out = np.empty(n, dtype=np.float64)
    ps = [_p(k) for k in keys] + [None] * (3 - len(keys))
    lib().wdo_units(int(seed) & ((1 << 64) - 1), len(keys), ps[0], ps[1], ps[2], n, _p(out))
    return out


def draw_one(a, W: int, r: int, *, u=None, stop=None, variant=BUTTERFLY):
    """One token: returns (index, total, stop) in a.dtype."""
    a = np.ascontiguousarray(a)
    total = np.zeros(1, a.dtype)
    st = np.zeros(1, a.dtype)
    have = stop is not None
    v = float(stop if have else u)
    idx = getattr(lib(), f"wdo_draw_one_{_sfx(a.dtype)}")(variant, _p(a), a.size, W, r, int(have), v, _p(total), _p(st))
    return int(idx), total[0], st[0]


def sample_rows(weights, W: int, seed: int = 0, *, row0: int = 0, units_=None, stops=None,
                variant=BUTTERFLY, n=None, threads: int = 1) -> np.ndarray:
    """weights [n, K] (or [K] shared with n given); returns int64 indices."""
    w = np.ascontiguousarray(weights)
    if w.ndim == 1:
        K, ld = w.size, 0
        assert n is not None
    else:
        n, K = w.shape
        ld = K
    out = np.empty(n, dtype=np.int64)
    u = None if units_ is None else np.ascontiguousarray(units_, dtype=np.float64)
    s = None if stops is None else np.ascontiguousarray(stops, dtype=w.dtype)
    getattr(lib(), f"wdo_sample_rows_{_sfx(w.dtype)}")(
        variant, W, _p(w), n, K, ld, row0, int(seed) & ((1 << 64) - 1), _p(u), _p(s), _p(out), threads)
    return out


def draw_z_csr(theta, phi, offsets, words, *, W: int, seed: int = 0, units_=None,
               variant=BUTTERFLY, key_rule=KEY_MASTER, doc_base: int = 0, threads: int = 1):
    """LDA draw over CSR; returns (z int64[sum N], err_key or None)."""
    theta = np.ascontiguousarray(theta)
    phi = np.ascontiguousarray(phi, dtype=theta.dtype)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    words = np.ascontiguousarray(words, dtype=np.int64)
    M = offsets.size - 1
    K = theta.shape[1]
    z = np.zeros(words.size, dtype=np.int64)
    err = np.zeros(1, dtype=np.uint64)
    u = None if units_ is None else np.ascontiguousarray(units_, dtype=np.float64)
    rc = getattr(lib(), f"wdo_draw_z_{_sfx(theta.dtype)}")(
        variant, key_rule, W, _p(theta), theta.shape[1], _p(phi), phi.shape[1], _p(offsets), _p(words),
        M, K, doc_base, int(seed) & ((1 << 64) - 1), _p(u), _p(z), _p(err), threads)
    return z, (int(err[0]) if rc else None)


def topic_counts(offsets, words, z, K: int, V: int):
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    words = np.ascontiguousarray(words, dtype=np.int64)
    z = np.ascontiguousarray(z, dtype=np.int64)
    M = offsets.size - 1
    dt = np.zeros((M, K), dtype=np.int64)
    wt = np.zeros((V, K), dtype=np.int64)
    lib().wdo_topic_counts(_p(offsets), _p(words), _p(z), M, K, _p(dt), _p(wt))
    return dt, wt


def ragged_to_csr(lengths, words):
    lengths = np.asarray(lengths, dtype=np.int64)
    offsets = np.zeros(lengths.size + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    flat = np.concatenate([np.asarray(w, dtype=np.int64).ravel() for w in words]) if len(words) else np.zeros(0, np.int64)
    return offsets, flat
