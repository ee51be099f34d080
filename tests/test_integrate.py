"""The install() shim patches the reference package in place (CPU-side
checks).  The reference is importable from /root/reference in the build
container and from baseline/_ref (the unmodified reference, pip-installed
there; git-ignored, it travels to the GPU box) everywhere else; the GPU run
of the patched reference's own run_gibbs is tests/test_gpu_reference_api.py."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def reference_path():
    for cand in (os.environ.get("WARPDRAW_REF"), os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if cand and os.path.isdir(os.path.join(cand, "warpdraw")):
            return cand
    return None


REF = reference_path()


@pytest.fixture
def warpdraw():
    if REF is None:
        pytest.skip("reference package not present")
    sys.path.insert(0, REF)
    try:
        import warpdraw as w
        import warpdraw.bench  # noqa: F401
        import warpdraw.kernels  # noqa: F401
        import warpdraw.lda  # noqa: F401
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    yield w
    sys.path.remove(REF)


def test_install_patches_and_restores(warpdraw):
    from paper_1505_03851_b200 import integrate

    orig_draw = warpdraw.kernels.draw_z
    orig_counts = warpdraw.lda.topic_counts
    orig_kernels = dict(warpdraw.kernels.KERNELS)
    orig_tables = (warpdraw.kernels.build_block_tables, warpdraw.kernels.butterfly_search,
                   warpdraw.bench.build_block_tables, warpdraw.bench.butterfly_search)
    integrate.install()
    try:
        # the split table / search API (kernels.py:580-604, 317-362) and
        # bench.py's imported names (bench.py:19)
        assert warpdraw.kernels.build_block_tables is not orig_tables[0]
        assert warpdraw.kernels.butterfly_search is not orig_tables[1]
        assert warpdraw.bench.build_block_tables is not orig_tables[2]
        assert warpdraw.bench.butterfly_search is not orig_tables[3]
        assert warpdraw.kernels.draw_z is not orig_draw
        assert warpdraw.lda.draw_z is warpdraw.kernels.draw_z
        assert warpdraw.lda.topic_counts is not orig_counts  # lda.py:174-182 on the GPU
        assert set(warpdraw.kernels.KERNELS) == {"basic", "transposed", "butterfly"}
        assert all(warpdraw.kernels.KERNELS[k] is not orig_kernels[k] for k in orig_kernels)
        assert "prefix" in warpdraw.bench.SAMPLERS
        # the reference's argument validation still comes first, as before
        with pytest.raises(ValueError, match="unknown kernel"):
            warpdraw.kernels.draw_z("fancy", [1], None, None, None, None, None)
    finally:
        integrate.uninstall()
    assert warpdraw.kernels.draw_z is orig_draw
    assert warpdraw.lda.topic_counts is orig_counts
    assert warpdraw.kernels.KERNELS == orig_kernels
    assert (warpdraw.kernels.build_block_tables, warpdraw.kernels.butterfly_search, warpdraw.bench.build_block_tables,
            warpdraw.bench.butterfly_search) == orig_tables
    assert "prefix" not in warpdraw.bench.SAMPLERS


def test_reference_stops_objects_are_recognised(warpdraw):
    from paper_1505_03851_b200 import integrate, kernels

    s = integrate._convert(warpdraw.kernels.SeededStops(5), warpdraw.kernels)
    assert isinstance(s, kernels.SeededStops) and s.seed == 5
    inj = warpdraw.kernels.InjectedStops([[0.25, 0.5], [], [0.75]])
    j = integrate._convert(inj, warpdraw.kernels)
    assert isinstance(j, kernels.InjectedStops)
    assert [list(u) for u in j._units] == [[0.25, 0.5], [], [0.75]]
    assert integrate._convert(3, warpdraw.kernels) == 3


def test_sampler_errors_are_the_reference_classes(warpdraw):
    """SAMPLERS installed into warpdraw.bench raise the reference's own
    exception classes (the weight validation runs before any device work)."""
    import numpy as np

    from paper_1505_03851_b200 import integrate

    integrate.install()
    try:
        with pytest.raises(warpdraw.sampling.AllZeroError):
            warpdraw.bench.SAMPLERS["alias"](np.zeros(4), 3, 1)
        with pytest.raises(warpdraw.sampling.EmptyWeightsError):
            warpdraw.bench.SAMPLERS["alias"](np.zeros(0), 3, 1)
    finally:
        integrate.uninstall()
