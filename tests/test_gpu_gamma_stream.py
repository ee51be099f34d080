"""GPU: the throughput-mode Gamma stream (wd_log_gamma_draws = the per-cell
attempt loop of wd_resample_theta / wd_resample_phi).

Replaces numpy's Generator.gamma in resample_params (lda.py:201-205); parity
is statistical, so the stream itself is tested: per-shape KS tests against
scipy's Gamma CDF, determinism, and -- the round-1 defect -- cells whose
first-attempt uniforms collided under the previous 32-bit (row, topic) fold
now get different draws."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1505_03851_b200 import _lib  # noqa: E402


def _draws(seed, rows, topics, shapes):
    L = _lib.load()
    r = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int64)).cuda()
    k = torch.from_numpy(np.ascontiguousarray(topics, dtype=np.int32)).cuda()
    a = torch.from_numpy(np.ascontiguousarray(shapes, dtype=np.float32)).cuda()
    out = torch.empty(r.numel(), dtype=torch.float32, device="cuda")
    _lib.check(L.wd_log_gamma_draws(seed & ((1 << 64) - 1), r.data_ptr(), k.data_ptr(), a.data_ptr(), r.numel(),
                                    out.data_ptr(), _lib.stream_handle()), "wd_log_gamma_draws")
    return out.cpu().numpy().astype(np.float64)


def _log_gamma_cdf(lg, a):
    """P(Gamma(a) <= exp(lg)), stable for very negative lg (small shapes)."""
    from scipy.special import gammainc, gammaln

    out = np.empty_like(lg)
    small = lg < -30
    out[~small] = gammainc(a, np.exp(lg[~small]))
    # lower tail: P(X <= x) ~ x^a / Gamma(a + 1) (relative error O(x))
    out[small] = np.exp(a * lg[small] - gammaln(a + 1))
    return out


@pytest.mark.parametrize("shape", [0.01, 0.1, 0.5, 1.0, 3.7, 250.5])
def test_gamma_stream_ks(shape):
    """200k draws of one shape over distinct (row, topic) cells: KS statistic
    below the 0.1% critical value (1.95 / sqrt(n))."""
    from scipy.stats import kstwobign  # noqa: F401

    n = 200_000
    rows = np.arange(n) // 64 + 10**9  # rows above 2^32 / 4: the 64-bit row counter
    topics = np.arange(n) % 64
    lg = _draws(0x5EED + int(shape * 1000), rows, topics, np.full(n, shape))
    assert np.all(np.isfinite(lg))
    u = np.sort(_log_gamma_cdf(lg, shape))
    i = np.arange(1, n + 1)
    d = max(np.max(i / n - u), np.max(u - (i - 1) / n))
    assert d < 1.95 / np.sqrt(n), (shape, d)


def test_gamma_stream_deterministic_and_row_independent():
    rows = np.array([0, 1, 2, 1 << 33, (1 << 33) + 1])
    topics = np.array([5, 5, 5, 5, 5])
    a = _draws(77, rows, topics, np.full(5, 0.1))
    b = _draws(77, rows, topics, np.full(5, 0.1))
    np.testing.assert_array_equal(a, b)
    assert len(set(a.tolist())) == 5  # rows 1 and 2^33 + 1 share their low word
    c = _draws(78, rows, topics, np.full(5, 0.1))
    assert not np.any(a == c)


def _hash32(x):
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x7FEB352D)
    x ^= x >> np.uint32(15)
    x *= np.uint32(0x846CA68B)
    x ^= x >> np.uint32(16)
    return x


def _old_first_attempt_base(seed, rows, topics):
    """The round-1 stream's per-cell state (wd_resample.cu before the fix):
    base = hash32(row_key(seed, row) ^ k * 0x9E3779B9); every uniform of the
    first attempt was a function of these 32 bits alone."""
    s_lo, s_hi = np.uint32(seed & 0xFFFFFFFF), np.uint32(seed >> 32)
    r_lo = (rows & 0xFFFFFFFF).astype(np.uint32)
    r_hi = (rows >> 32).astype(np.uint32)
    rkey = _hash32(s_lo ^ _hash32(r_lo ^ _hash32(r_hi ^ s_hi)))
    return _hash32(rkey ^ (topics.astype(np.uint32) * np.uint32(0x9E3779B9)))


def test_cells_colliding_under_the_old_fold_now_differ():
    """1024 documents x 1024 topics (2^20 cells): the old fold gives ~2^40 /
    2^33 = 128 pairs of cells with identical first-attempt uniforms, i.e.
    identical Gammas for equal shapes.  The Philox stream draws them apart."""
    seed = 0x1234_5678_9ABC_DEF0
    R, K = 1024, 1024
    rows = np.repeat(np.arange(R, dtype=np.int64), K)
    topics = np.tile(np.arange(K, dtype=np.int64), R)
    base = _old_first_attempt_base(seed, rows, topics)
    order = np.argsort(base, kind="stable")
    sb = base[order]
    dup = np.nonzero(sb[1:] == sb[:-1])[0]
    assert dup.size >= 50  # the collisions existed
    a_idx, b_idx = order[dup], order[dup + 1]
    cells = np.concatenate([a_idx, b_idx])
    lg = _draws(seed, rows[cells], topics[cells], np.full(cells.size, 0.1))
    la, lb = lg[: dup.size], lg[dup.size:]
    assert np.all(la != lb)
