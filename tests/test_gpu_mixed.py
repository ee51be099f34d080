"""GPU: float32 theta with float64 phi (csrc/wd_mixed.cu) against golden
output of the reference (tests/golden/make_golden_mixed.py).

The reference forms fl32(fl64(theta * phi)) (numpy promotion into a float32
table, kernels.py:209, 391).  The injected-stop cases put every stop within
an ulp of a table boundary, where casting phi to float32 first flips the
drawn index for 5-12% of the tokens (checked here too, so the fixture keeps
its teeth); the device path must match the reference on every token, for
the three kernels, through the reference-signature draw_z and through
draw_z_device."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1505_03851_b200 as wd  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _case(g, ci):
    W, K, seed = (int(x) for x in g["meta"][ci])
    N = g[f"N_{ci}"]
    off = np.concatenate([[0], np.cumsum(N)]).astype(np.int64)
    flat = g[f"w_{ci}"]
    w = [flat[a:b] for a, b in zip(off[:-1], off[1:])]
    return W, K, seed, N, off, flat, w, g[f"theta_{ci}"], g[f"phi_{ci}"], g[f"u_{ci}"]


def test_mixed_precision_draw_matches_reference(golden):
    g = golden("mixed")
    flips = 0
    for ci in range(len(g["meta"])):
        W, K, seed, N, off, flat, w, theta, phi, u = _case(g, ci)
        assert theta.dtype == np.float32 and phi.dtype == np.float64
        ragged_u = [u[a:b] for a, b in zip(off[:-1], off[1:])]
        for kern in ("basic", "transposed", "butterfly"):
            for tag, stops in (("z", wd.SeededStops(seed)), ("zi", wd.InjectedStops(ragged_u))):
                exp = g[f"{tag}_{ci}_{kern}"]
                got = wd.draw_z(kern, N, theta, phi, w, wd.WarpConfig(W, 4), stops)
                got = np.concatenate(got) if len(got) else np.zeros(0, np.int64)
                np.testing.assert_array_equal(got, exp, err_msg=f"case {ci} W={W} K={K} {kern} {tag}")
        # the device API with torch tensors of the two dtypes
        dc = wd.DeviceCorpus.from_csr(off, flat.astype(np.int32))
        z = wd.draw_z_device("butterfly", dc, torch.from_numpy(theta).cuda(), torch.from_numpy(phi).cuda(),
                             wd.InjectedStops(ragged_u), W).cpu().numpy()
        np.testing.assert_array_equal(z, g[f"zi_{ci}_butterfly"])
        # the fixture discriminates: phi rounded to float32 first draws differently
        z32, _ = O.draw_z_csr(theta, phi.astype(np.float32), off, flat, W=W, units_=u)
        flips += int(np.sum(z32 != g[f"zi_{ci}_butterfly"]))
    assert flips > 100
