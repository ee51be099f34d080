"""The reference's counter-style unit stream (rng.py:15-122).

derive_seed / mix64 / unit_for are scalar host utilities (seed plumbing).
units_for, the vectorised stream the kernels consume, is evaluated on the
device (wd_units); the draw kernels hash the same function inline.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_UNIT_SCALE = 2.0**-53


def _fin(z: int) -> int:
    z = ((z ^ (z >> 30)) * _MIX1) & _MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & _MASK64
    return z ^ (z >> 31)


def mix64(x: int) -> int:
    """One SplitMix64 step used as a 64-bit hash (rng.py:30-32)."""
    return _fin((x + _GAMMA) & _MASK64)


def derive_seed(seed: int, *keys: int) -> int:
    """Fold integer keys into a seed, one mixing round per key (rng.py:35-40)."""
    h = int(seed) & _MASK64
    for k in keys:
        h = mix64(h ^ (int(k) & _MASK64))
    return h


def unit_for(seed: int, *keys: int) -> float:
    """First unit of the xoshiro256** stream derived from (seed, keys) (rng.py:80-82)."""
    s1 = _fin((derive_seed(seed, *keys) + 2 * _GAMMA) & _MASK64)
    x = (s1 * 5) & _MASK64
    x = ((x << 7) | (x >> 57)) & _MASK64
    return (((x * 9) & _MASK64) >> 11) * _UNIT_SCALE


def units_for(seed: int, *key_arrays, device_out: bool = False):
    """Vectorised unit_for over 0-2 broadcast key arrays, evaluated on the GPU.

    Returns numpy float64 (or the CUDA tensor with device_out=True).
    """
    import torch

    _lib.require_cuda()
    if len(key_arrays) > 2:
        raise ValueError("device units_for supports at most two key arrays")
    keys = [np.asarray(k, dtype=np.int64) for k in key_arrays]
    if keys:
        keys = list(np.broadcast_arrays(*keys))
        shape = keys[0].shape
    else:
        shape = ()
    n = int(np.prod(shape)) if shape else 1
    dev = torch.device("cuda")
    kt = [torch.from_numpy(np.ascontiguousarray(k).reshape(-1)).to(dev) for k in keys]
    out = torch.empty(n, dtype=torch.float64, device=dev)
    L = _lib.load()
    _lib.check(L.wd_units(int(seed) & _MASK64, len(kt), _lib.ptr(kt[0]) if kt else None,
                          _lib.ptr(kt[1]) if len(kt) > 1 else None, n, out.data_ptr(), _lib.stream_handle()),
               "wd_units")
    if device_out:
        return out.reshape(shape)
    res = out.cpu().numpy().reshape(shape)
    return res if shape else np.asarray(res)


# ------------------------------------------------ opt-in Philox4x32-10 stream
_PHILOX_M0, _PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
_PHILOX_W0, _PHILOX_W1 = 0x9E3779B9, 0xBB67AE85
_M32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11; Random123's
    philox4x32_R(10, ...)), vectorised over numpy arrays.  ctr: four uint32
    arrays (or ints), key: two.  Host twin of philox_bits in
    csrc/wd_device.cuh, pinned to the Random123 known-answer vectors in
    tests/test_host_api.py."""
    c = [np.asarray(x, dtype=np.uint64) & _M32 for x in ctr]
    k0, k1 = (np.asarray(x, dtype=np.uint64) & _M32 for x in key)
    for _ in range(10):
        p0 = np.uint64(_PHILOX_M0) * c[0]
        p1 = np.uint64(_PHILOX_M1) * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & _M32, (p0 >> np.uint64(32)) ^ c[3] ^ k1, p0 & _M32]
        k0 = (k0 + np.uint64(_PHILOX_W0)) & _M32
        k1 = (k1 + np.uint64(_PHILOX_W1)) & _M32
    return c


def philox_units(seed: int, a, b) -> np.ndarray:
    """u in [0, 1) of PhiloxStops: counter (a lo, a hi, b lo, b hi) for global
    document a and word position b, key = seed; 53 bits from the first two
    output words (as the device does)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    s = int(seed) & _MASK64
    c = philox4x32_10([a & _M32, a >> np.uint64(32), b & _M32, b >> np.uint64(32)], [s & 0xFFFFFFFF, s >> 32])
    bits = (c[0] << np.uint64(21)) | (c[1] >> np.uint64(11))
    return bits.astype(np.float64) * _UNIT_SCALE
