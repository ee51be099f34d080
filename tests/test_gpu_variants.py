"""GPU: every kernel variant the dispatcher can pick, forced on through its
environment knob, bit-exact against the oracle.

The launchers read their knobs once per process (csrc/wd_launch.cuh), so each
setting runs in a child process: the register-lean LDA draw
(WD_LEAN_MIN_NB=16 takes it down to K = 512, WD_LEAN_COOP=1 its warp-
cooperative pass 2, WD_LEAN_PF its theta L2 prefetch), the one-row-per-thread
rows kernel on every shape it supports (WD_ROWS_LANE=2), the small-K LDA
kernel on every CSR-order draw (WD_SMALL_LDA=2, default K <= 256), and all of them disabled
(the general kernels on the same shapes)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_1505_03851_b200 as wd
from paper_1505_03851_b200.kernels import to_block_aligned
from oracle import oracle as O

out = {"rows": [], "lda": []}
for K in (8, 16, 24, 32, 40, 56, 64, 72, 104, 128, 136, 152):
    gen = np.random.default_rng(K)
    w = gen.uniform(0.1, 1.0, size=(3000, K)).astype(np.float32)
    w[:, 2::5] = 0
    w[7] = 0  # an all-zero row (AllZero reported, index 0)
    w[8, :] = 0
    w[8, K - 1] = 1.0  # everything on the last topic
    seed = 900 + K
    got = wd.sample_rows(torch.from_numpy(w).cuda(), seed, lanes=32, check=False).cpu().numpy()
    exp = O.sample_rows(w, 32, wd.derive_seed(seed, 6), threads=8)
    out["rows"].append([K, int(np.sum(got != exp))])
for K in (72, 200, 256, 512, 1024, 2048):
    for pad in (0, 4):
        gen = np.random.default_rng(K + pad)
        M, V = 512, 400
        N = gen.poisson(25, size=M).astype(np.int64)
        N[gen.random(M) < 0.05] = 0
        off = np.concatenate([[0], np.cumsum(N)])
        words = gen.integers(0, V, size=int(off[-1])).astype(np.int64)
        theta = gen.dirichlet(np.full(K, 0.1), size=M).astype(np.float32)
        phi = gen.uniform(0.01, 1, size=(V, K)).astype(np.float32)
        dc = wd.DeviceCorpus.from_csr(off, words.astype(np.int32))
        tiles = dc.vocab_tiles(96, pad)
        th = to_block_aligned(torch.from_numpy(theta).cuda())
        ph = to_block_aligned(torch.from_numpy(phi).cuda())
        z = wd.draw_z_device("butterfly", dc, th, ph, wd.SeededStops(5), 32, tiles=tiles).cpu().numpy()
        exp, err = O.draw_z_csr(theta, phi, off, words, W=32, seed=5, threads=8)
        out["lda"].append([K, pad, int(np.sum(z != exp)), err is None])
        if pad == 0:  # the CSR-order draw (no tiles) of the same corpus
            z = wd.draw_z_device("butterfly", dc, th, ph, wd.SeededStops(5), 32).cpu().numpy()
            out["lda"].append([K, -1, int(np.sum(z != exp)), err is None])
print(json.dumps(out))
"""

SETTINGS = {
    "lean_k512": {"WD_LEAN_MIN_NB": "16"},
    "lean_coop_pf": {"WD_LEAN_MIN_NB": "16", "WD_LEAN_COOP": "1", "WD_LEAN_PF": "3"},
    "rows_lane_all": {"WD_ROWS_LANE": "2"},
    "small_lda_all": {"WD_SMALL_LDA": "2"},
    "general_only": {"WD_LEAN": "0", "WD_ROWS_LANE": "0", "WD_SMALL_LDA": "0"},
}


@pytest.mark.parametrize("name", sorted(SETTINGS))
def test_forced_variant_bit_exact(name):
    env = dict(os.environ, **SETTINGS[name])
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(bad == 0 for _, bad in res["rows"]), res["rows"]
    assert all(bad == 0 and ok for _, _, bad, ok in res["lda"]), res["lda"]
