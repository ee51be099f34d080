"""ctypes binding of the C ABI in include/warpdraw_b200.h.

This is the whole host->device boundary: the Python API mirrors the
reference package and calls these entry points with device pointers taken
from torch tensors and the current torch CUDA stream.  There is no CPU
fallback: without the built library or a CUDA device every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "_lib", "libwarpdraw_b200.so")

WD_OK = 0
WD_FLOAT32, WD_FLOAT64, WD_FLOAT32_PHI64 = 0, 1, 2
WD_BUTTERFLY, WD_PREFIX = 0, 1
WD_STOPS_SEEDED, WD_STOPS_UNITS, WD_STOPS_EXPLICIT, WD_STOPS_PHILOX = 0, 1, 2, 3
WD_KEYS_MASTER, WD_KEYS_POSITION = 0, 1
WD_STREAM_BINARY, WD_STREAM_ALIAS = 0, 1
ERR_NONE = (1 << 64) - 1
WD_ERR_ACCUMULATE = 1

EXPORTS = (
    "wd_abi_version",
    "wd_status_string",
    "wd_last_cuda_error",
    "wd_corpus_prepare",
    "wd_workspace_bytes",
    "wd_draw_z",
    "wd_sample_rows",
    "wd_units",
    "wd_topic_counts",
    "wd_log_gamma_draws",
    "wd_resample_theta",
    "wd_resample_phi_workspace_bytes",
    "wd_resample_phi",
    "wd_log_likelihood",
    "wd_prefix_f64",
    "wd_stream_workspace_bytes",
    "wd_stream_draws",
    "wd_l2_probe_bytes",
    "wd_l2_read_probe",
    "wd_build_block_tables",
    "wd_butterfly_search",
    "wd_sample_rows_ex",
    "wd_resample_phi_chunks",
    "wd_resample_phi_pass",
    "wd_resample_phi_reduce",
)


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or returned an error."""


_lock = threading.Lock()
_lib = None


def _declare(L):
    i32, i64, u64, vp, sz = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
    L.wd_abi_version.restype = i32
    L.wd_abi_version.argtypes = []
    L.wd_status_string.restype = ctypes.c_char_p
    L.wd_status_string.argtypes = [i32]
    L.wd_last_cuda_error.restype = ctypes.c_char_p
    L.wd_last_cuda_error.argtypes = []
    L.wd_corpus_prepare.restype = i32
    L.wd_corpus_prepare.argtypes = [vp, i64, i64, i64, i32, vp, vp, vp]
    L.wd_workspace_bytes.restype = sz
    L.wd_workspace_bytes.argtypes = [i32, i32, i32, ctypes.c_int32]
    L.wd_draw_z.restype = i32
    L.wd_draw_z.argtypes = [i32, i32, i32, vp, i64, vp, i64, ctypes.c_int32, vp, vp, vp, vp, vp, i64, i64, i64,
                            i32, i32, u64, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    L.wd_sample_rows.restype = i32
    L.wd_sample_rows.argtypes = [i32, i32, i32, vp, i64, i64, ctypes.c_int32, i64, i32, u64, vp, vp, vp, vp, vp,
                                 sz, vp]
    L.wd_sample_rows_ex.restype = i32
    L.wd_sample_rows_ex.argtypes = [i32, i32, i32, vp, i64, i64, ctypes.c_int32, i64, i32, u64, vp, vp, vp, vp, vp,
                                    sz, i32, vp]
    L.wd_units.restype = i32
    L.wd_units.argtypes = [u64, i32, vp, vp, i64, vp, vp]
    L.wd_topic_counts.restype = i32
    L.wd_topic_counts.argtypes = [vp, vp, vp, i64, ctypes.c_int32, vp, vp, vp]
    dbl = ctypes.c_double
    L.wd_log_gamma_draws.restype = i32
    L.wd_log_gamma_draws.argtypes = [u64, vp, vp, vp, i64, vp, vp]
    L.wd_resample_theta.restype = i32
    L.wd_resample_theta.argtypes = [i32, vp, vp, i64, ctypes.c_int32, dbl, u64, i64, vp, i64, vp]
    L.wd_resample_phi_workspace_bytes.restype = sz
    L.wd_resample_phi_workspace_bytes.argtypes = [ctypes.c_int32]
    L.wd_resample_phi.restype = i32
    L.wd_resample_phi.argtypes = [i32, vp, i64, ctypes.c_int32, dbl, u64, vp, i64, vp, sz, vp]
    L.wd_log_likelihood.restype = i32
    L.wd_log_likelihood.argtypes = [i32, vp, i64, vp, i64, vp, vp, i64, i64, i64, ctypes.c_int32, vp, vp, sz, vp]
    L.wd_prefix_f64.restype = i32
    L.wd_prefix_f64.argtypes = [vp, i64, vp, vp]
    L.wd_stream_workspace_bytes.restype = sz
    L.wd_stream_workspace_bytes.argtypes = [i64]
    L.wd_stream_draws.restype = i32
    L.wd_stream_draws.argtypes = [i32, vp, vp, vp, i64, u64, i64, vp, vp, sz, vp]
    L.wd_l2_probe_bytes.restype = i64
    L.wd_l2_probe_bytes.argtypes = [i64, i32]
    L.wd_l2_read_probe.restype = i32
    L.wd_l2_read_probe.argtypes = [vp, i64, i32, i32, vp, vp]
    L.wd_build_block_tables.restype = i32
    L.wd_build_block_tables.argtypes = [i32, i32, vp, ctypes.c_int32, i64, vp, vp, vp]
    L.wd_resample_phi_chunks.restype = i32
    L.wd_resample_phi_chunks.argtypes = []
    L.wd_resample_phi_pass.restype = i32
    L.wd_resample_phi_pass.argtypes = [i32, i32, vp, i64, ctypes.c_int32, ctypes.c_double, u64, vp, i64, i32, i32, i32,
                                       vp, vp, vp]
    L.wd_resample_phi_reduce.restype = i32
    L.wd_resample_phi_reduce.argtypes = [i32, vp, i32, ctypes.c_int32, vp, vp]
    L.wd_butterfly_search.restype = i32
    L.wd_butterfly_search.argtypes = [i32, i32, vp, vp, vp, ctypes.c_int32, i64, vp, vp, vp]


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            p = path or os.environ.get("WARPDRAW_B200_LIB", LIB_PATH)
            if not os.path.exists(p):
                raise NativeLibraryError(
                    f"{p} not built; run `python -m paper_1505_03851_b200.build` (no CPU fallback exists)")
            L = ctypes.CDLL(p)
            _declare(L)
            _lib = L
    return _lib


def check(status: int, what: str):
    if status != WD_OK:
        L = load()
        msg = L.wd_status_string(status).decode()
        cuda = L.wd_last_cuda_error().decode()
        raise NativeLibraryError(f"{what}: {msg}" + (f" ({cuda})" if cuda else ""))


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the warpdraw B200 path has no CPU fallback")
    load()


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
