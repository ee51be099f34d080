"""Golden fixtures for the split table / search API, by running the REFERENCE.

    python tests/golden/make_golden_tables.py      -> tests/golden/tables.npz

For each case: products (*batch, W, K), the reference's
build_block_tables(products, WarpConfig(W, elem)) table p.data (K, *batch, W)
and sums (*batch, W) (kernels.py:580-600, build_butterfly_table
kernels.py:170-225), stops inside [0, sums) -- seeded units through
_stops_from_units, plus exact midpoints and zero stops -- and
butterfly_search(warp, p, sums, stops) (kernels.py:317-362).  Zero-weight
lanes (sums == 0, stop 0) and zero products are included.  Run in the build
container (the reference is importable there, not on the GPU box).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("WARPDRAW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from warpdraw import rng  # noqa: E402
from warpdraw.kernels import _stops_from_units, build_block_tables, butterfly_search  # noqa: E402
from warpdraw.warp import WarpConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tables.npz")


def main():
    gen = np.random.default_rng(20261017)
    arrays = {}
    meta = []
    ci = 0
    for dtype in (np.float32, np.float64):
        for W in (2, 4, 8, 16, 32, 64):
            for K in sorted({1, 3, W, W + 5, 3 * W + 7, 4 * W}):
                for batch in ((), (3,)):
                    prods = gen.uniform(0.0, 1.0, size=(*batch, W, K)).astype(dtype)
                    prods[..., gen.random(prods.shape[:-1]) < 0.15, :] *= 0  # some all-zero lanes
                    prods[gen.random(prods.shape) < 0.2] = 0  # zero products
                    cfg = WarpConfig(lanes=W, elem_size=np.dtype(dtype).itemsize)
                    warp, p, sums = build_block_tables(prods, cfg)
                    u = rng.units_for(rng.derive_seed(7, ci), np.arange(sums.size)).reshape(sums.shape)
                    stops = _stops_from_units(np.asarray(sums), u, dtype)
                    stops = np.where(np.asarray(sums) > 0, stops, 0).astype(dtype)
                    got = np.asarray(butterfly_search(warp, p, sums, stops))
                    arrays[f"prods_{ci}"] = prods
                    arrays[f"p_{ci}"] = np.asarray(p.data)
                    arrays[f"sums_{ci}"] = np.asarray(sums)
                    arrays[f"stops_{ci}"] = stops
                    arrays[f"idx_{ci}"] = got.astype(np.int64)
                    meta.append((W, K, len(batch), np.dtype(dtype).itemsize))
                    ci += 1
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"{ci} cases -> {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
