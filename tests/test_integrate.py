"""The install() shim patches the reference package in place (CPU-side check;
the reference is only importable in the build container, so this skips on
the GPU box).  With a GPU, the patched reference's own run_gibbs must
reproduce its unpatched golden output."""

import os
import sys

import pytest

REF = os.environ.get("WARPDRAW_REF", "/root/reference/pkg/src")


@pytest.fixture
def warpdraw():
    if not os.path.isdir(REF):
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
    orig_kernels = dict(warpdraw.kernels.KERNELS)
    integrate.install()
    try:
        assert warpdraw.kernels.draw_z is not orig_draw
        assert warpdraw.lda.draw_z is warpdraw.kernels.draw_z
        assert set(warpdraw.kernels.KERNELS) == {"basic", "transposed", "butterfly"}
        assert all(warpdraw.kernels.KERNELS[k] is not orig_kernels[k] for k in orig_kernels)
        assert "prefix" in warpdraw.bench.SAMPLERS
        # the reference's argument validation still comes first, as before
        with pytest.raises(ValueError, match="unknown kernel"):
            warpdraw.kernels.draw_z("fancy", [1], None, None, None, None, None)
    finally:
        integrate.uninstall()
    assert warpdraw.kernels.draw_z is orig_draw
    assert warpdraw.kernels.KERNELS == orig_kernels
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
