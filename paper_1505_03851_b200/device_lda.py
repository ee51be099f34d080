"""Throughput-mode LDA: corpus, theta, phi, z and counts resident in HBM.

One Gibbs iteration (lda.py:211-242 semantics, uncollapsed):

    word_topic = 0
    z ~ draw (butterfly kernel, SeededStops(derive_seed(seed, 1, t)))
        with word_topic += 1 fused into the draw epilogue
    all_reduce(word_topic, SUM)                      # NCCL, only if sharded:
        per vocabulary tile, enqueued behind that tile's draw launch, so it
        overlaps the next tile's draw
    theta[m]   ~ Dir(alpha + hist(z of doc m))       # wd_resample_theta
    phi[:, k]  ~ Dir(beta + word_topic[:, k])        # wd_resample_phi

Documents are sharded across ranks in 32-aligned contiguous ranges; the
global doc id drives both the u hash and the theta Gamma stream, and phi is
resampled from the all-reduced counts with the same key on every rank, so a
run is independent of the number of GPUs (tests/test_multigpu.py).
"""

from __future__ import annotations

import os

from . import _lib
from .kernels import DeviceCorpus, SeededStops, block_aligned_rows, combine_err, draw_z_device, raise_for_err
from .rng import derive_seed
from .sharding import TileAllReduce, count_chunks

# phi slice kept L2-resident per draw pass (126 MB L2; measured: 41 MB slices
# run at the L2-resident rate, 82 MB ones do not -- profiles/)
DEFAULT_VOCAB_TILE_BYTES = 40 << 20
def lean_draw(K: int, lanes: int, elem_size: int) -> bool:
    """True when the C ABI dispatches the draw to lda_lean_kernel (fp32,
    W = 32, K a multiple of 32 with >= WD_LEAN_MIN_NB blocks, aligned rows;
    csrc/wd_launch.cuh lean_eligible)."""
    import os

    if os.environ.get("WD_LEAN", "1") == "0":
        return False
    return elem_size == 4 and lanes == 32 and K % 32 == 0 and K // 32 >= int(os.environ.get("WD_LEAN_MIN_NB", "64"))


# mean tokens per (document, tile) run from which runs are padded to the
# butterfly kernel's lane-group height (VocabTiles.run_pad)
RUN_PAD_MIN_MEAN_RUN = 20  # measured at K=1024 (runs ~50 tokens): draw -10%


class DeviceLDA:
    def __init__(self, corpus: DeviceCorpus, n_topics: int, vocab_size: int, *, lanes: int = 32, dtype=None,
                 alpha: float = 0.1, beta: float = 0.01, seed: int = 0, kernel: str = "butterfly",
                 process_group=None, theta=None, phi=None, vocab_tile_bytes: int | None = DEFAULT_VOCAB_TILE_BYTES,
                 run_pad: int | None = None):
        import torch

        _lib.require_cuda()
        self.torch = torch
        self.corpus = corpus
        self.K = int(n_topics)
        self.V = int(vocab_size)
        self.lanes = int(lanes)
        self.dtype = dtype or torch.float32
        self.alpha, self.beta, self.seed = float(alpha), float(beta), int(seed)
        self.kernel = kernel
        self.pg = process_group
        dev = corpus.offsets.device
        self.device = dev
        # line-aligned W-topic blocks (kernels.block_aligned_rows)
        self.theta = theta if theta is not None else block_aligned_rows(corpus.n_docs, self.K, self.dtype, dev, lanes)
        # sharded phi resample (multi-GPU): each rank resamples a fixed share
        # of the row chunks and the rows are all-gathered (resample()).  The
        # phi rows then live in a padded [chunks x rows_per, ld] buffer whose
        # rank slices are contiguous; phi is its [V, K] view.
        L0 = _lib.load()
        self._phi_chunks = int(L0.wd_resample_phi_chunks())
        world = self.torch.distributed.get_world_size(process_group) if process_group is not None else 1
        self.world = world
        self.rank = self.torch.distributed.get_rank(process_group) if process_group is not None else 0
        self.shard_phi = (phi is None and world > 1 and self._phi_chunks % world == 0 and
                          os.environ.get("WD_SHARD_PHI", "1") != "0")
        self._phi_bases = {}  # phi view data_ptr -> its padded base buffer (sharded resample)
        if self.shard_phi:
            rows_per = -(-self.V // self._phi_chunks)
            self._phi_rows_pad = rows_per * self._phi_chunks
            self.phi = self._alloc_phi()
            self._phi_part = torch.empty((self._phi_chunks, self.K), dtype=torch.float32, device=dev)
            self._phi_colstat = torch.empty(2 * self.K, dtype=torch.float32, device=dev)
        else:
            self.phi = phi if phi is not None else block_aligned_rows(self.V, self.K, self.dtype, dev, lanes)
        self.z = torch.zeros(corpus.n_tokens, dtype=torch.int32, device=dev)
        self.word_topic = torch.zeros((self.V, self.K), dtype=torch.int32, device=dev)
        L = _lib.load()
        self._phi_ws = torch.empty(int(L.wd_resample_phi_workspace_bytes(self.K)), dtype=torch.uint8, device=dev)
        self._ll_ws = torch.empty(8 * (corpus.n_docs + self.K) + 8, dtype=torch.uint8, device=dev)
        self._ll_out = torch.zeros(1, dtype=torch.float64, device=dev)
        self._dt = _lib.WD_FLOAT32 if self.dtype == torch.float32 else _lib.WD_FLOAT64
        esz = 4 if self.dtype == torch.float32 else 8
        self.tiles = None
        if vocab_tile_bytes is not None:
            # token order for the draw: vocabulary tiles (phi slices kept
            # L2-resident) when phi exceeds vocab_tile_bytes, else one tile;
            # either way (document, word)-ordered, so a document's repeated
            # words reuse their phi row from L1 (kernels.VocabTiles)
            tiled = vocab_tile_bytes > 0 and self.V * self.K * esz > vocab_tile_bytes
            rows = max(1, int(vocab_tile_bytes // (self.K * esz))) if tiled else self.V
            if run_pad is None:
                # pad (tile, document) runs to the lane-group height when runs
                # are long enough that the padding (~L/2 slots per run) costs
                # less than the two-document theta selection it removes
                n_tiles = -(-self.V // rows)
                mean_run = corpus.n_tokens / max(1, corpus.n_docs) / n_tiles
                # (fine instantiation only: at most 32 blocks per row)
                fine = self.K // self.lanes <= 32
                # the kernel's lane-group height: 4 rows with 256-bit segments
                # (fp32, W = 32, aligned rows), else W / 4 (measured at cfg4:
                # padding to 4 vs 8 -1.2%, Zipf -2.2%)
                group = 4 if (self.lanes == 32 and esz == 4) else self.lanes // 4
                run_pad = group if (self.lanes >= 8 and fine and mean_run >= RUN_PAD_MIN_MEAN_RUN) else 0
                if lean_draw(self.K, self.lanes, esz):
                    # the register-lean kernel (csrc/wd_lean.cuh) keeps one
                    # theta segment per lane: runs padded to its 4-row groups
                    run_pad = 4
            self.tiles = corpus.vocab_tiles(rows, run_pad)
        self._reducer = None  # in-flight per-tile count all-reduces (draw -> resample)
        n_err = self.tiles.n_tiles if self.tiles is not None else 1
        self.err = torch.empty((n_err, 2), dtype=torch.int64, device=dev)

    def _alloc_phi(self):
        """A [V, K] phi in the block_aligned_rows layout; with the sharded
        resample, a view of a [chunks x rows_per, ld] buffer whose rank
        slices are contiguous (registered for the rows' all-gather)."""
        if not self.shard_phi:
            return block_aligned_rows(self.V, self.K, self.dtype, self.device, self.lanes)
        view = block_aligned_rows(self._phi_rows_pad, self.K, self.dtype, self.device, self.lanes)
        base = view._base if view._base is not None else view
        phi = view[: self.V]
        self._phi_bases[phi.data_ptr()] = base
        return phi

    # ------------------------------------------------------------ init
    def init_uniform(self, low: float = 0.1, high: float = 1.0, seed: int | None = None):
        """synth_params-style positive weights (bench.py:187-192 of the reference)."""
        torch = self.torch
        g = torch.Generator(device=self.device).manual_seed(int(self.seed if seed is None else seed))
        self.theta.uniform_(low, high, generator=g)
        self.phi.uniform_(low, high, generator=g)

    def init_from_assignments(self, t: int = -1):
        """Uniform random initial topics + resample at iteration -1
        (lda.py:264-265).  The initial topic of token (doc m, position i) is
        floor(K * units_for(derive_seed(seed, 0), m, i)) with GLOBAL doc ids,
        so any sharding of the corpus gives the same start."""
        torch = self.torch
        c = self.corpus
        if c.n_tokens:
            pos = torch.arange(c.n_tokens, dtype=torch.int64, device=self.device) - c.offsets[c.token_doc.long()]
            gdoc = c.token_doc.long() + c.doc_base
            u = torch.empty(c.n_tokens, dtype=torch.float64, device=self.device)
            L = _lib.load()
            _lib.check(L.wd_units(derive_seed(self.seed, 0), 2, gdoc.data_ptr(), pos.data_ptr(), c.n_tokens,
                                  u.data_ptr(), _lib.stream_handle()), "wd_units")
            self.z.copy_((u * self.K).to(torch.int32).clamp_(max=self.K - 1))
        self.word_topic.zero_()
        L = _lib.load()
        _lib.check(L.wd_topic_counts(c.words.data_ptr(), None, self.z.data_ptr(), c.n_tokens, self.K, None,
                                     self.word_topic.data_ptr(), _lib.stream_handle()), "wd_topic_counts")
        if self.pg is not None:
            torch.distributed.all_reduce(self.word_topic, group=self.pg)
        self.resample(t)

    # ------------------------------------------------------- one sweep
    def draw(self, t: int, fused_counts: bool = True, overlap_allreduce: bool = False):
        """z draw with the word_topic counts fused.  overlap_allreduce (sharded
        runs): tile t's count rows are final as soon as its launch retires, so
        their all-reduce is enqueued right behind it and runs on the NCCL
        stream while the next tile draws; the works are kept for resample()."""
        self.word_topic.zero_()
        self._reducer = None
        after = None
        if overlap_allreduce and self.pg is not None and fused_counts:
            dist = self.torch.distributed
            self._reducer = TileAllReduce(
                self.word_topic, count_chunks(self.V, self.tiles.rows_per_tile if self.tiles is not None else None),
                lambda v: dist.all_reduce(v, group=self.pg, async_op=True))
            after = self._reducer.after_tile
        draw_z_device(self.kernel, self.corpus, self.theta, self.phi, SeededStops(derive_seed(self.seed, 1, t)),
                      self.lanes, z=self.z, word_topic=self.word_topic if fused_counts else None, err=self.err,
                      check=False, tiles=self.tiles, after_tile=after)
        if self._reducer is not None:
            self._reducer.finish()

    def allreduce_counts(self):
        if self.pg is not None and getattr(self, "_reducer", None) is None:
            self.torch.distributed.all_reduce(self.word_topic, group=self.pg)

    def _resample_theta(self, t: int):
        L = _lib.load()
        _lib.check(L.wd_resample_theta(self._dt, self.z.data_ptr(), self.corpus.offsets.data_ptr(),
                                       self.corpus.n_docs, self.K, self.alpha, derive_seed(self.seed, 2, t, 0),
                                       self.corpus.doc_base, self.theta.data_ptr(), self.theta.stride(0),
                                       _lib.stream_handle()), "wd_resample_theta")

    def _all_gather_slices(self, buf, async_op=False):
        """In-place all-gather of equal contiguous rank slices of `buf` (rank r
        owns elements [r*n/world, (r+1)*n/world))."""
        dist = self.torch.distributed
        flat = buf.view(-1)
        n = flat.numel() // self.world
        mine = flat[self.rank * n:(self.rank + 1) * n]
        # the rank's slice is sent from a copy (1/world of the buffer): no
        # reliance on in-place semantics of the collective
        if dist.get_backend(self.pg) == "nccl":
            return dist.all_gather_into_tensor(flat, mine.clone(), group=self.pg, async_op=async_op)
        return dist.all_gather(list(flat.split(n)), mine.clone(), group=self.pg, async_op=async_op)

    def resample(self, t: int):
        L = _lib.load()
        st = _lib.stream_handle()
        if not self.shard_phi:
            # theta needs only the local z: it runs while in-flight count
            # all-reduces finish; phi waits for them
            self._resample_theta(t)
            if getattr(self, "_reducer", None) is not None:
                self._reducer.wait()
                self._reducer = None
            _lib.check(L.wd_resample_phi(self._dt, self.word_topic.data_ptr(), self.V, self.K, self.beta,
                                         derive_seed(self.seed, 2, t, 1), self.phi.data_ptr(), self.phi.stride(0),
                                         self._phi_ws.data_ptr(), self._phi_ws.numel(), st), "wd_resample_phi")
            return
        # Sharded phi: this rank's share of the fixed row
        # chunks, column partials exchanged after passes 0 and 1 (all-gather,
        # folded in chunk order: the same bits on every rank and for any
        # world size), then the rows all-gathered on the NCCL stream WHILE
        # theta resamples on this one.
        if getattr(self, "_reducer", None) is not None:
            self._reducer.wait()
            self._reducer = None
        G = self._phi_chunks
        c0, c1 = self.rank * G // self.world, (self.rank + 1) * G // self.world
        seed = derive_seed(self.seed, 2, t, 1)
        for pss in (0, 1, 2):
            _lib.check(L.wd_resample_phi_pass(self._dt, pss, self.word_topic.data_ptr(), self.V, self.K, self.beta,
                                              seed, self.phi.data_ptr(), self.phi.stride(0), c0, c1, G,
                                              self._phi_part.data_ptr(), self._phi_colstat.data_ptr(), st),
                       "wd_resample_phi_pass")
            if pss < 2:
                self._all_gather_slices(self._phi_part)
                _lib.check(L.wd_resample_phi_reduce(pss, self._phi_part.data_ptr(), G, self.K,
                                                    self._phi_colstat.data_ptr(), st), "wd_resample_phi_reduce")
        work = self._all_gather_slices(self._phi_bases[self.phi.data_ptr()], async_op=True)
        self._resample_theta(t)
        work.wait()

    def iterate(self, t: int, overlap_allreduce: bool = True):
        self.draw(t, overlap_allreduce=overlap_allreduce)
        self.allreduce_counts()
        self.resample(t)

    def iterate_from_host(self, t0: int, n: int, theta_host, phi_host, z_host=None):
        """n iterations, each ENTERED FROM HOST parameters: the drop-in
        gibbs_iterate(corpus, params, ...) call made with host theta/phi
        (pinned torch tensors) every iteration, z of each iteration returned
        to z_host (pinned [n_tokens]; int32, or int16 when K <= 32767: the
        topics are cast on the device, halving the D2H bytes).  Every iteration moves its full
        inputs and result across PCIe; the copies are pipelined the way a
        data loader prefetches: iteration s+1's H2D (copy stream) and
        iteration s-1's D2H (second copy stream) overlap iteration s, on two
        device buffer sets.  Stream-ordered: returns without synchronising
        (the current stream waits for the last D2H)."""
        torch = self.torch
        st = torch.cuda.current_stream()
        if getattr(self, "_host_pipe", None) is None:
            self._host_pipe = {
                "theta": [self.theta, block_aligned_rows(*self.theta.shape, self.theta.dtype, self.device, self.lanes)],
                "phi": [self.phi, self._alloc_phi()],
                "z": [self.z, torch.empty_like(self.z)],
                "z16": [None, None],
                "up": torch.cuda.Stream(), "down": torch.cuda.Stream(),
                "ready": [torch.cuda.Event() for _ in range(2)],
                "done": [torch.cuda.Event() for _ in range(2)],
                "copied": [torch.cuda.Event() for _ in range(2)],
            }
        P = self._host_pipe
        up, down = P["up"], P["down"]
        for i in range(2):
            P["done"][i].record(st)
            P["copied"][i].record(st)

        def upload(i):
            up.wait_event(P["done"][i])  # buffer set i free: its last iteration finished
            with torch.cuda.stream(up):
                P["theta"][i].copy_(theta_host, non_blocking=True)
                P["phi"][i].copy_(phi_host, non_blocking=True)
                P["ready"][i].record(up)

        if n > 0:
            upload(0)
        for s in range(n):
            i = s % 2
            if s + 1 < n:
                upload(1 - i)
            st.wait_event(P["ready"][i])
            st.wait_event(P["copied"][i])  # z buffer i's previous D2H has drained
            self.theta, self.phi, self.z = P["theta"][i], P["phi"][i], P["z"][i]
            self.iterate(t0 + s)
            P["done"][i].record(st)
            if z_host is not None:
                src = P["z"][i]
                if z_host.dtype == torch.int16:
                    if self.K > 32767:
                        raise ValueError("int16 z needs K <= 32767")
                    if P["z16"][i] is None:
                        P["z16"][i] = torch.empty(self.z.numel(), dtype=torch.int16, device=self.device)
                    st.wait_event(P["copied"][i])
                    P["z16"][i].copy_(src)  # on the compute stream, behind the iteration
                    P["done"][i].record(st)
                    src = P["z16"][i]
                down.wait_event(P["done"][i])
                with torch.cuda.stream(down):
                    z_host.copy_(src, non_blocking=True)
                    P["copied"][i].record(down)
        st.wait_stream(down)

    def check_errors(self):
        raise_for_err(combine_err(self.err), _lib.WD_KEYS_MASTER, self.lanes)

    # -------------------------------------------------- log-likelihood
    def log_likelihood(self) -> float:
        """lda.py:289-305 on the device (float64 accumulation), summed over ranks."""
        L = _lib.load()
        c = self.corpus
        _lib.check(L.wd_log_likelihood(self._dt, self.theta.data_ptr(), self.theta.stride(0), self.phi.data_ptr(),
                                       self.phi.stride(0), c.words.data_ptr(), c.token_doc.data_ptr(), c.n_docs,
                                       c.n_tokens, self.V, self.K, self._ll_out.data_ptr(), self._ll_ws.data_ptr(),
                                       self._ll_ws.numel(), _lib.stream_handle()), "wd_log_likelihood")
        out = self._ll_out.clone()
        if self.pg is not None:
            self.torch.distributed.all_reduce(out, group=self.pg)
        return float(out.item())
