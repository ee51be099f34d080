"""Small cases of every kernel path, run under compute-sanitizer (memcheck /
racecheck / synccheck) by tools/sanitize.sh."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_03851_b200 as wd  # noqa: E402
from paper_1505_03851_b200.device_lda import DeviceLDA  # noqa: E402

gen = np.random.default_rng(0)
# standalone rows: scalar / vector / ring / coarse paths, fp32 + fp64, several W
for K, W, dt in ((5, 32, np.float32), (32, 32, np.float32), (19, 8, np.float64), (240, 32, np.float32),
                 (1024, 32, np.float32),
                 (4096, 32, np.float32), (130, 64, np.float32), (7, 2, np.float32)):
    w = torch.from_numpy(gen.uniform(0.1, 1, size=(70, K)).astype(dt)).cuda()
    wd.sample_rows(w, 1, lanes=W)
    wd.sample_rows(w, 1, lanes=W, variant="prefix")
# LDA: untiled, tiled, run-padded tiles, remnant, small (cooperative reload
# through the remnant tile or S), fine, coarse, fp64, all three kernels
for K, W, dt in ((200, 32, np.float32), (64, 8, np.float64), (128, 32, np.float32), (1024, 32, np.float32),
                 (2112, 32, np.float32)):
    M, V = 64, 90
    N = gen.poisson(15, size=M)
    off = np.concatenate([[0], np.cumsum(N)])
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    th = torch.from_numpy(gen.uniform(0.1, 1, size=(M, K)).astype(dt)).cuda()
    ph = torch.from_numpy(gen.uniform(0.1, 1, size=(V, K)).astype(dt)).cuda()
    tha, pha = wd.kernels.to_block_aligned(th, W), wd.kernels.to_block_aligned(ph, W)
    tiles = dc.vocab_tiles(17)
    tiles_p = dc.vocab_tiles(17, max(1, W // 4))
    for kern in ("butterfly", "transposed", "basic"):
        wd.draw_z_device(kern, dc, th, ph, wd.SeededStops(3), W)
        wd.draw_z_device(kern, dc, th, ph, wd.SeededStops(3), W, tiles=tiles)
        wd.draw_z_device(kern, dc, tha, pha, wd.SeededStops(3), W, tiles=tiles_p)
# device LDA iteration (counts, resample, log-likelihood)
M, V, K = 64, 50, 48
off = np.concatenate([[0], np.cumsum(gen.poisson(20, size=M))])
words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
lda = DeviceLDA(wd.DeviceCorpus.from_csr(off, words), K, V, seed=1)
lda.init_from_assignments()
lda.iterate(0)
lda.log_likelihood()
torch.cuda.synchronize()
print("sanitize cases done")
