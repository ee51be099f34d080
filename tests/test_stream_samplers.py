"""SAMPLERS["binary"] / ["alias"] (bench.py:118-126): the reference's
sequential-xoshiro samplers.  CPU: the exact Vose table (host logic) equals
the reference's.  GPU: the device draws (per-thread GF(2) stream jumps) are
bit-identical to the reference's sequential draws (tests/golden/stream.npz,
made by tests/golden/make_golden.py --only stream)."""

import numpy as np
import pytest

from paper_1505_03851_b200 import samplers

CASES = ("k19", "k1", "uniform4", "ints", "zeros", "k200", "k1000", "tiny")


@pytest.mark.parametrize("name", CASES)
def test_alias_table_matches_reference(golden, name):
    g = golden("stream")
    thresh, alias = samplers.alias_table(g[f"{name}/w"])
    np.testing.assert_array_equal(alias, g[f"{name}/alias_A"])
    np.testing.assert_array_equal(thresh, g[f"{name}/alias_T"])


def test_weight_validation_matches_reference():
    from paper_1505_03851_b200.sampling import AllZeroError, EmptyWeightsError

    with pytest.raises(EmptyWeightsError):
        samplers.alias_table([])
    with pytest.raises(ValueError, match="non-negative"):
        samplers.alias_table([1.0, -1.0])
    with pytest.raises(AllZeroError, match="sum to zero"):
        samplers.alias_table([0.0, 0.0])


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["binary", "alias"])
@pytest.mark.parametrize("name", CASES)
def test_stream_samplers_vs_reference_golden(golden, method, name):
    g = golden("stream")
    ref = g[f"{name}/{method}"].astype(np.int64)
    got = samplers.SAMPLERS[method](g[f"{name}/w"], ref.size, int(g[f"{name}/seed"]))
    assert got.dtype == np.int64
    np.testing.assert_array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["binary", "alias"])
def test_stream_samplers_prefix_consistent_and_errors(method):
    """Draw i does not depend on n (every n is a prefix of the same stream),
    n = 0 gives an empty result, and the reference's errors are raised."""
    from paper_1505_03851_b200.sampling import AllZeroError, EmptyWeightsError

    fn = samplers.SAMPLERS[method]
    w = np.random.default_rng(5).uniform(0.1, 1.0, size=77)
    big = fn(w, 3_000_001, 9)
    for n in (1, 31, 32, 33, 1000, 65_537, 1_234_567):
        np.testing.assert_array_equal(fn(w, n, 9), big[:n])
    assert fn(w, 0, 9).size == 0
    with pytest.raises(EmptyWeightsError):
        fn([], 10, 1)
    with pytest.raises(ValueError):
        fn([0.5, -0.1], 10, 1)
    with pytest.raises(AllZeroError):
        fn([0.0, 0.0, 0.0], 10, 1)


@pytest.mark.gpu
def test_stream_samplers_chi_square():
    """Acceptance criterion 6 shape (test_acceptance.py:270-298) for the two
    stream samplers: 1e6 draws from 19 weights pass chi-square at 0.001."""
    w = np.random.default_rng(60).uniform(0.05, 1.0, size=19)
    for method in ("binary", "alias"):
        d = samplers.SAMPLERS[method](w, 1_000_000, 61)
        stat, dof = samplers.chi_square(np.bincount(d, minlength=19), w / w.sum())
        assert stat < samplers.chi_square_critical(dof, 0.001), method


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("W", [2, 4, 8, 16, 32, 64])
def test_shared_vector_table_search_equals_per_row_kernel(dtype, W):
    """One shared vector (ld = 0) is answered from a table built once; it must
    give exactly the per-row kernel's draws on the materialised rows (which
    the oracle and the golden vectors pin), zeros and remnants included."""
    import torch

    dt = getattr(torch, dtype)
    gen = np.random.default_rng(W)
    n = 4099
    for K in (1, 3, W - 1 if W > 1 else 1, W, W + 3, 5 * W + 7, 40 * W + 1):
        w = gen.uniform(0.0, 1.0, size=K) * (gen.random(K) < 0.8)
        if not (w > 0).any():
            w[K // 2] = 0.5
        wt = torch.from_numpy(w).to(dt).cuda()
        shared = samplers.sample_rows(wt, 17, lanes=W, n=n, row_base=5)
        rows = samplers.sample_rows(wt.repeat(n, 1).contiguous(), 17, lanes=W, row_base=5)
        np.testing.assert_array_equal(shared.cpu().numpy(), rows.cpu().numpy(), err_msg=f"K={K}")
    z = torch.zeros(33, dtype=dt, device="cuda")
    from paper_1505_03851_b200.sampling import AllZeroError

    with pytest.raises(AllZeroError, match="row 5:"):
        samplers.sample_rows(z, 1, lanes=W, n=10, row_base=5)
