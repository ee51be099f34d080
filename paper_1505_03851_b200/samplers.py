"""Standalone samplers: the reference's SAMPLERS registry (bench.py:118-154)
plus the batched independent-row API used by the K sweep (BASELINE configs[1]).

    sample_butterfly(weights, n, seed, lanes=8)   bench.py:129-147, on the GPU
    sample_prefix(weights, n, seed, lanes=8)      same u stream, prefix table
    sample_binary(weights, n, seed)               bench.py:118-121, sequential xoshiro stream
    sample_alias(weights, n, seed)                bench.py:123-126, exact Vose table
    sample_rows(weights[n, K], seed, ...)         one independent row per draw

The u stream is units_for(derive_seed(seed, 6), draw_id) exactly as in
bench.py:141-143; results are bit-identical to the reference.  The binary
and alias samplers consume ONE sequential xoshiro256** stream in the
reference; on the device every thread jumps to its own stream position
(wd_stream_draws), so they are bit-identical too.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import _lib
from .kernels import StopOutOfRangeError, _workspace
from .rng import derive_seed
from .sampling import AllZeroError, EmptyWeightsError

_VARIANTS = {"butterfly": _lib.WD_BUTTERFLY, "prefix": _lib.WD_PREFIX}


def _dtype_code(t):
    import torch

    if t.dtype == torch.float32:
        return _lib.WD_FLOAT32
    if t.dtype == torch.float64:
        return _lib.WD_FLOAT64
    raise TypeError(f"weights must be float32 or float64, got {t.dtype}")


def sample_rows(weights, seed: int | None = None, *, lanes: int = 32, variant: str = "butterfly", row_base: int = 0,
                units=None, stops=None, out=None, n: int | None = None, err=None, check: bool = True, stream=None,
                raw_seed: int | None = None, accumulate_err: bool = False):
    """Draw one index per row of `weights` ([n, K] CUDA tensor, float32/64).

    A 1-D weights tensor is one shared vector; pass n for the number of draws.
    Row id = row_base + i; u = units_for(derive_seed(seed, 6), id) unless
    `units` (float64 per row) or `stops` (explicit, weights dtype) are given.
    Returns an int32 CUDA tensor.  Rows summing to zero raise AllZeroError
    when check=True (the reference's search returns index K-1 for them).
    accumulate_err=True (with a caller-owned err and check=False): err is not
    reset first, so a batch of calls shares one reset and one check
    (WD_ERR_ACCUMULATE) instead of a reset per call.
    """
    import torch

    _lib.require_cuda()
    if variant not in _VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if weights.dim() == 1:
        if n is None:
            raise ValueError("a shared weight vector needs n")
        ld = 0
        K = int(weights.shape[0])
    else:
        n, K = int(weights.shape[0]), int(weights.shape[1])
        if weights.stride(-1) != 1:
            raise ValueError("weight rows must be contiguous")
        ld = weights.stride(0)
    dt = _dtype_code(weights)
    dev = weights.device
    mode, sd, u_t, s_t = _lib.WD_STOPS_SEEDED, 0, None, None
    if stops is not None:
        mode = _lib.WD_STOPS_EXPLICIT
        s_t = torch.as_tensor(stops, dtype=weights.dtype).to(dev).contiguous()
    elif units is not None:
        mode = _lib.WD_STOPS_UNITS
        u_t = torch.as_tensor(units, dtype=torch.float64).to(dev).contiguous()
    else:
        sd = raw_seed if raw_seed is not None else derive_seed(int(seed), 6)
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=dev)
    own_err = err is None
    if own_err:
        err = torch.empty(2, dtype=torch.int64, device=dev)
    L = _lib.load()
    v = _VARIANTS[variant]
    ws, nbytes = _workspace(v, dt, int(lanes), K, dev)
    if accumulate_err and (own_err or check):
        raise ValueError("accumulate_err needs a caller-owned err and check=False")
    _lib.check(L.wd_sample_rows_ex(v, dt, int(lanes), weights.data_ptr(), ld, n, K, int(row_base), mode,
                                   int(sd) & ((1 << 64) - 1), _lib.ptr(u_t), _lib.ptr(s_t), out.data_ptr(),
                                   err.data_ptr(), _lib.ptr(ws), nbytes,
                                   _lib.WD_ERR_ACCUMULATE if accumulate_err else 0, _lib.stream_handle(stream)),
               "wd_sample_rows")
    if check:
        e = err.cpu().numpy().view(np.uint64)
        if int(e[1]) != _lib.ERR_NONE:
            raise StopOutOfRangeError("stop values must lie in [0, sum)")
        if int(e[0]) != _lib.ERR_NONE and stops is None:
            raise AllZeroError(f"row {int(e[0])}: all weights are zero")
    return out


def _shared(weights, n, seed, lanes, variant):
    import torch

    w = np.asarray(weights, dtype=np.float64)
    if n <= 0:
        return np.zeros(0, dtype=np.int64)
    wt = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    # bench.py:129-147 builds no AllZero check; the search returns K-1 there
    idx = sample_rows(wt, seed, lanes=lanes, variant=variant, n=int(n), check=False)
    return idx.cpu().numpy().astype(np.int64)


def sample_butterfly(weights, n: int, seed: int, lanes: int = 8) -> np.ndarray:
    """Draw through the butterfly table and search (bench.py:129-147)."""
    return _shared(weights, n, seed, lanes, "butterfly")


def sample_prefix(weights, n: int, seed: int, lanes: int = 8) -> np.ndarray:
    """Same u stream through the full prefix-sum table (the paper's baseline)."""
    return _shared(weights, n, seed, lanes, "prefix")


def _as_weights(weights) -> np.ndarray:
    """sampling.py:27-33: non-empty 1-D float64, no negative entries."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.size == 0:
        raise EmptyWeightsError("need a non-empty 1-D weight vector")
    if np.any(w < 0):
        raise ValueError("weights must be non-negative")
    return w


def alias_table(weights):
    """Exact Vose alias table (sampling.py:101-131) as device-ready arrays.

    Returns (thresh uint64[K], alias int32[K]) with thresh[k] =
    ceil(F[k] * 2^53): for a 53-bit unit u = b * 2^-53 the reference's exact
    test u < F[k] is b < thresh[k].  The worklists are stacks (pop from the
    end) and a scaled weight of exactly 1 counts as large, so the pairing --
    and hence every alias -- is the reference's.
    """
    w = _as_weights(weights)
    exact = [Fraction(x) for x in w.tolist()]
    total = sum(exact, Fraction(0))
    if total <= 0:
        raise AllZeroError("weights sum to zero")
    K = len(exact)
    scaled = [x * K / total for x in exact]
    accept: list = [Fraction(1)] * K
    alias = np.arange(K, dtype=np.int32)
    small = [k for k, x in enumerate(scaled) if x < 1]
    large = [k for k, x in enumerate(scaled) if x >= 1]
    while small and large:
        lo, hi = small.pop(), large.pop()
        accept[lo], alias[lo] = scaled[lo], hi
        scaled[hi] -= 1 - scaled[lo]
        (small if scaled[hi] < 1 else large).append(hi)
    # leftovers (either list) keep acceptance 1
    thresh = np.array([-((-f.numerator << 53) // f.denominator) for f in accept], dtype=np.uint64)
    return thresh, alias


def _stream_draws(method, n, seed, table=None, thresh=None, alias=None, K=0):
    import torch

    _lib.require_cuda()
    n = int(n)
    if n < 0:
        raise ValueError("n must be non-negative")
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    L = _lib.load()
    ws = torch.empty(int(L.wd_stream_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    _lib.check(L.wd_stream_draws(method, _lib.ptr(table), _lib.ptr(thresh), _lib.ptr(alias), int(K),
                                 int(seed) & ((1 << 64) - 1), n, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                 _lib.stream_handle()), "wd_stream_draws")
    return out[:n].cpu().numpy().astype(np.int64)


def sample_binary(weights, n: int, seed: int) -> np.ndarray:
    """Prefix table + bisection, u from one xoshiro256** stream seeded
    derive_seed(seed, 4) (bench.py:118-121, sampling.py:46-92)."""
    import torch

    w = _as_weights(weights)
    if np.isnan(w).any() or not (w > 0).any():  # float64 running total not > 0
        raise AllZeroError("weights sum to zero")
    _lib.require_cuda()
    wt = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    table = torch.empty_like(wt)
    L = _lib.load()
    _lib.check(L.wd_prefix_f64(wt.data_ptr(), wt.numel(), table.data_ptr(), _lib.stream_handle()), "wd_prefix_f64")
    return _stream_draws(_lib.WD_STREAM_BINARY, n, derive_seed(int(seed), 4), table=table, K=w.size)


def sample_alias(weights, n: int, seed: int) -> np.ndarray:
    """Vose alias table, two units per draw from one xoshiro256** stream
    seeded derive_seed(seed, 5) (bench.py:123-126, sampling.py:134-138)."""
    import torch

    thresh, alias = alias_table(weights)
    _lib.require_cuda()
    th = torch.from_numpy(thresh.view(np.int64)).cuda()
    al = torch.from_numpy(alias).cuda()
    return _stream_draws(_lib.WD_STREAM_ALIAS, n, derive_seed(int(seed), 5), thresh=th, alias=al, K=alias.size)


SAMPLERS = {
    "binary": sample_binary,
    "alias": sample_alias,
    "butterfly": sample_butterfly,
    "prefix": sample_prefix,
}


def chi_square(observed, expected) -> tuple[float, int]:
    """Pearson statistic and degrees of freedom (bench.py:30-50)."""
    obs = np.asarray(observed, dtype=np.float64)
    exp = np.asarray(expected, dtype=np.float64)
    if obs.shape != exp.shape or obs.ndim != 1 or obs.size < 2:
        raise ValueError("need matching 1-D bins, at least two")
    if np.any(exp <= 0):
        raise ValueError("expected probabilities must be positive")
    n = obs.sum()
    stat = float(np.sum((obs - exp * n) ** 2 / (exp * n)))
    return stat, obs.size - 1


def chi_square_critical(dof: int, significance: float = 0.001) -> float:
    from scipy import stats

    return float(stats.chi2.ppf(1.0 - significance, dof))
