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
# round 2: one-row-per-thread rows (K < 32, remnant shapes)
for K in (8, 16, 24, 40, 136):
    w = torch.from_numpy(gen.uniform(0.1, 1, size=(300, K)).astype(np.float32)).cuda()
    wd.sample_rows(w, 2, lanes=32)
# round 2: small-K and register-lean LDA kernels on run-padded and unpadded tiles
for K in (64, 200, 232, 2048, 4096):
    M, V = 96, 120
    N = gen.poisson(15, size=M)
    off = np.concatenate([[0], np.cumsum(N)])
    words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
    dc = wd.DeviceCorpus.from_csr(off, words)
    tha = wd.kernels.to_block_aligned(torch.from_numpy(gen.uniform(0.1, 1, size=(M, K)).astype(np.float32)).cuda())
    pha = wd.kernels.to_block_aligned(torch.from_numpy(gen.uniform(0.1, 1, size=(V, K)).astype(np.float32)).cuda())
    wt = torch.zeros((V, K), dtype=torch.int32, device="cuda")
    for pad in (0, 4):
        wd.draw_z_device("butterfly", dc, tha, pha, wd.SeededStops(4), 32, tiles=dc.vocab_tiles(40, pad),
                         word_topic=wt)
    # the untiled CSR-order draw (small-K kernel up to K = 256)
    wd.draw_z_device("butterfly", dc, tha, pha, wd.SeededStops(4), 32, word_topic=wt)
    # float32 theta with float64 phi (wd_mixed.cu), all three kernels
    ph64 = torch.from_numpy(gen.uniform(0.1, 1, size=(V, K))).cuda()
    for kern in ("butterfly", "transposed", "basic"):
        wd.draw_z_device(kern, dc, tha, ph64, wd.SeededStops(4), 32)
# round 2: the split table / search API
for W, K in ((8, 21), (64, 150), (32, 32)):
    prods = gen.uniform(0.0, 1.0, size=(5, W, K)).astype(np.float32)
    warp, p, sums = wd.build_block_tables(prods, wd.WarpConfig(lanes=W))
    wd.butterfly_search(warp, p, sums, (sums * 0.5).astype(np.float32))
# round 2: sharded phi passes (a rank's chunk range) and the wide theta kernel
from paper_1505_03851_b200 import _lib  # noqa: E402

L = _lib.load()
V, K = 300, 96
wt = torch.randint(0, 5, (V, K), dtype=torch.int32, device="cuda")
phi = torch.empty((V, K), device="cuda")
G = int(L.wd_resample_phi_chunks())
part = torch.empty((G, K), device="cuda")
col = torch.zeros(2 * K, device="cuda")
for pss in (0, 1, 2):
    _lib.check(L.wd_resample_phi_pass(0, pss, wt.data_ptr(), V, K, 0.01, 7, phi.data_ptr(), K, G // 4, G // 2, G,
                                      part.data_ptr(), col.data_ptr(), _lib.stream_handle()), "pass")
    if pss < 2:
        _lib.check(L.wd_resample_phi_reduce(pss, part.data_ptr(), G, K, col.data_ptr(), _lib.stream_handle()), "red")
M, V, K = 64, 60, 2112
off = np.concatenate([[0], np.cumsum(gen.poisson(30, size=M))])
words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
lda = DeviceLDA(wd.DeviceCorpus.from_csr(off, words), K, V, seed=1)
lda.init_from_assignments()
lda.iterate(0)
# device LDA iteration (counts, resample, log-likelihood)
M, V, K = 64, 50, 48
off = np.concatenate([[0], np.cumsum(gen.poisson(20, size=M))])
words = gen.integers(0, V, size=int(off[-1])).astype(np.int32)
lda = DeviceLDA(wd.DeviceCorpus.from_csr(off, words), K, V, seed=1)
lda.init_from_assignments()
lda.iterate(0)
lda.log_likelihood()
# phi resample with several rows per chunk (the 4-row loop and its tail):
# V = 5000 over the fixed row chunks, fp32 and fp64
for dt in (torch.float32, torch.float64):
    V, K = 5000, 40
    wt = torch.randint(0, 5, (V, K), dtype=torch.int32, device="cuda")
    ph = torch.empty((V, K), dtype=dt, device="cuda")
    ws = torch.empty(int(L.wd_resample_phi_workspace_bytes(K)), dtype=torch.uint8, device="cuda")
    _lib.check(L.wd_resample_phi(_lib.WD_FLOAT32 if dt == torch.float32 else _lib.WD_FLOAT64, wt.data_ptr(), V, K,
                                 0.01, 3, ph.data_ptr(), K, ws.data_ptr(), ws.numel(), _lib.stream_handle()), "phi")
torch.cuda.synchronize()
print("sanitize cases done")
