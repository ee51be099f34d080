"""Wall time of the drop-in run_gibbs (parity mode) on BASELINE configs[0]:
D=1000 (padded to 1024), V=5000, K=64, 10 iterations, fp32 butterfly, seed 7.
The corpus is the golden one (tests/golden/cfg1.npz) so the result can be
checked against the reference's own run (343 s in the build container)."""
import hashlib
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402

g = np.load("tests/golden/cfg1.npz")
N = g["N"]
off = np.concatenate([[0], np.cumsum(N)])
words = g["words"].astype(np.int64)
corpus = wd.Corpus(vocab_size=5000, lengths=N, words=[words[off[m]:off[m + 1]] for m in range(N.size)])
wd.run_gibbs(corpus, 64, 1, "butterfly", wd.WarpConfig(32, 4), 7, dtype=np.float32)  # warm-up (load, JIT caches)
t0 = time.perf_counter()
params, z, ll = wd.run_gibbs(corpus, 64, 10, "butterfly", wd.WarpConfig(32, 4), 7, dtype=np.float32)
dt = time.perf_counter() - t0
ok = (np.array_equal(np.concatenate(z), g["z"].astype(np.int64))
      and hashlib.sha256(np.ascontiguousarray(params.theta).tobytes()).hexdigest() == str(g["theta_sha"])
      and np.array_equal(ll, g["ll"]))
print(f"run_gibbs cfg1 (10 iterations, parity mode): {dt:.2f} s, bit-exact vs reference: {ok}, "
      f"reference emulator: {float(g['ref_wall_s']):.1f} s")
