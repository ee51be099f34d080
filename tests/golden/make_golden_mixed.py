"""Golden fixtures for float32 theta with float64 phi, by running the REFERENCE.

    python tests/golden/make_golden_mixed.py   -> tests/golden/mixed.npz

The reference's kernels take theta's dtype for the table and form every
product with numpy promotion (kernels.py:209, 391): fl32(fl64(theta * phi)).
Cases: the three kernels (basic, transposed, butterfly) x W in {8, 32} x
K in {19, 100, 256}, ragged corpora with empty documents, with seeded stops
and with ADVERSARIAL injected stops: u = P[t] / total for a random t, P the
reference's own float32 running sums of fl32(theta * phi64), so each stop
sits within an ulp of a table boundary -- where rounding phi to float32
first would flip the drawn index.
Run in the build container (the reference is importable there only).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("WARPDRAW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from warpdraw.kernels import InjectedStops, SeededStops, draw_z  # noqa: E402
from warpdraw.warp import WarpConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mixed.npz")


def main():
    gen = np.random.default_rng(4242)
    arrays, meta = {}, []
    ci = 0
    for W in (8, 32):
        for K in (19, 100, 256):
            M, V = 8 * W, 37
            N = gen.poisson(6, size=M).astype(np.int64)
            N[gen.random(M) < 0.15] = 0
            w = [gen.integers(0, V, size=int(n)) for n in N]
            theta = gen.dirichlet(np.full(K, 0.3), size=M).astype(np.float32)
            phi = gen.dirichlet(np.full(V, 0.2), size=K).T.copy()  # float64
            seed = 1000 + ci
            units = []
            for m in range(M):
                u = np.zeros(int(N[m]))
                for i in range(int(N[m])):
                    prods = (theta[m] * phi[int(w[m][i])]).astype(np.float32)
                    P = np.cumsum(prods, dtype=np.float32)
                    t = int(gen.integers(0, K - 1))
                    u[i] = min(float(P[t]) / float(P[-1]), np.nextafter(1.0, 0.0))
                units.append(u)
            for kern in ("basic", "transposed", "butterfly"):
                z = draw_z(kern, N, theta, phi, w, WarpConfig(W, 4), SeededStops(seed))
                arrays[f"z_{ci}_{kern}"] = np.concatenate([np.asarray(x, np.int64) for x in z]) if len(z) else np.zeros(0)
                z = draw_z(kern, N, theta, phi, w, WarpConfig(W, 4), InjectedStops(units))
                arrays[f"zi_{ci}_{kern}"] = np.concatenate([np.asarray(x, np.int64) for x in z]) if len(z) else np.zeros(0)
            arrays[f"u_{ci}"] = np.concatenate(units) if units else np.zeros(0)
            arrays[f"N_{ci}"] = N
            arrays[f"w_{ci}"] = np.concatenate(w) if len(w) else np.zeros(0, np.int64)
            arrays[f"theta_{ci}"] = theta
            arrays[f"phi_{ci}"] = phi
            meta.append((W, K, seed))
            ci += 1
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"{ci} cases -> {OUT} ({os.path.getsize(OUT) / 1e3:.0f} kB)")


if __name__ == "__main__":
    main()
