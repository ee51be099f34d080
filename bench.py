#!/usr/bin/env python
"""Benchmark: LDA tokens/s per Gibbs iteration at K=1024 on N B200s (+ the
standalone-sampler line and the CPU baselines), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling strong|weak]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (BASELINE.json configs[3]): a synthetic Wikipedia-shaped corpus of
1M documents (lengths ~ Poisson(200), floor 1; words uniform over V =
40,000), K = 1024 topics, fp32, W = 32.  --scaling strong (default): the
SAME corpus is generated on every rank and document-sharded across the N
GPUs (32-aligned, token-balanced cuts, sharding.shard_ranges) -- configs[3]
as written.  --scaling weak: 1M documents per GPU.  One step = one full
uncollapsed Gibbs iteration on the device: butterfly z draw with fused
word-topic counts, NCCL all-reduce of the counts per vocabulary tile (N > 1),
phi and theta Dirichlet resample.  Inputs (theta 4.1 GB, words 0.8 GB, phi
164 MB at N = 1) exceed the 126 MB L2, so no flush is needed between steps.

value    = all ranks' tokens / (max-over-ranks device time per step)
roofline = the dominant kernel (the butterfly LDA draw): algorithmic bytes
           per token 4K + 4K/Nbar + 8 x tokens / its
           CUDA-event time, against the L2 read ceiling measured in this
           process (wd_l2_read_probe): the phi gathers are served from L2 by
           design (vocabulary tiles), so L2 -> SM bandwidth is the roof.
e2e      = the same iteration entered from HOST parameters each step
           (DeviceLDA.iterate_from_host: pinned H2D of theta and phi, D2H of z).
e2e_dropin = the reference-signature call draw_z("butterfly", N, theta, phi,
           w, config, stops) with host numpy in and ragged int64 lists out, at
           configs[2] size (1M docs, K = 200), wall clock per call.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "z draws/sec and LDA tokens/sec/iter at K=1024 on 1/8 B200; % of HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--topics", type=int, default=1024)
    ap.add_argument("--docs", type=int, default=1_000_000,
                    help="corpus size: total (strong scaling) or per GPU (weak scaling)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--vocab", type=int, default=40_000)
    ap.add_argument("--mean-len", type=float, default=200.0)
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--rows", type=int, default=1 << 20, help="standalone sampler rows (configs[1])")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample time")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--dropin-docs", type=int, default=1_000_000)
    ap.add_argument("--dropin-topics", type=int, default=200)
    ap.add_argument("--no-python-ref", action="store_true",
                    help="--impl reference: skip timing the reference's own Python draw_z_butterfly")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sampler", action="store_true")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: test the N > 1 flow with every rank on one GPU (ranks share cuda:0..n-1 round robin); "
                         "not a measurement")
    ap.add_argument("--force-dist", action="store_true",
                    help="create the NCCL process group even at world size 1 (exercises the N>1 code path)")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_summary():
    """Committed ncu numbers (profiles/ncu_summary.json): DRAM traffic of the
    dominant kernel per draw and the measured L2 read peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ corpus
def workload_config(args, world):
    """The workload both arms name (identical dicts: the reference arm runs a
    bounded sample of exactly this workload)."""
    return {
        "workload": f"lda_cfg4_k{args.topics}",
        "scaling": args.scaling,
        "docs_total": args.docs * (world if args.scaling == "weak" else 1),
        "vocab": args.vocab,
        "topics": args.topics,
        "mean_doc_len": args.mean_len,
        "word_dist": "uniform",
        "kernel": "butterfly",
        "lanes": 32,
        "parallelism": f"dp{world} (32-aligned, token-balanced document shards)",
        "step": "draw z (+fused word_topic counts; N>1: NCCL all-reduce per vocabulary tile, overlapping the next "
                "tile's draw) -> theta, phi resample",
        "l2": "inputs larger than L2 (theta 4.1 GB, words 0.8 GB, phi 164 MB at N=1 vs 126 MB L2); no flush",
    }


def make_corpus(torch, seed, M, args, device):
    """Synthetic corpus: lengths ~ Poisson(mean) floor 1, words uniform over V,
    padded with empty documents to a multiple of 32 (Corpus.padded,
    lda.py:56-63).  Deterministic in `seed` on any device."""
    g = torch.Generator(device=device).manual_seed(seed)
    lengths = torch.poisson(torch.full((M,), args.mean_len, device=device), generator=g).clamp_(min=1).long()
    if M % 32:
        lengths = torch.cat([lengths, torch.zeros(32 - M % 32, dtype=torch.long, device=device)])
        M = lengths.numel()
    off = torch.zeros(M + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(lengths, 0)
    T = int(off[-1].item())
    words = torch.randint(0, args.vocab, (T,), generator=g, device=device, dtype=torch.int32)
    return off, words


def make_shard(torch, rank, world, args, device):
    """This rank's shard: (local offsets, local words, global doc of local doc 0).

    strong: the same args.docs-document corpus on every rank (same generator),
    cut by sharding.shard_ranges (32-aligned, balanced by tokens); rank r keeps
    documents [lo, hi) with doc_base = lo, so z is the single-GPU run's.
    weak: args.docs documents per rank (seed + rank), doc_base = rank x M."""
    from paper_1505_03851_b200.sharding import shard_ranges

    if args.scaling == "weak":
        off, words = make_corpus(torch, args.seed * 1000 + rank, args.docs, args, device)
        return off, words, rank * (off.numel() - 1)
    off, words = make_corpus(torch, args.seed * 1000, args.docs, args, device)
    lo, hi = shard_ranges(torch.diff(off).cpu().numpy(), world)[rank]
    a, b = int(off[lo].item()), int(off[hi].item())
    return (off[lo:hi + 1] - a).contiguous(), words[a:b].contiguous(), lo


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_sample_lda(args, theta_rows, phi_host, off_host, words_host, target_s):
    """Time the oracle (C port of the reference butterfly draw) on a doc sample
    with every host core; returns (tokens/s, cores, description)."""
    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    O.lib()

    def run(S, threads=cores):
        off = off_host[: S + 1] - off_host[0]
        w = words_host[off_host[0]: off_host[0] + off[-1]]
        t0 = time.perf_counter()
        O.draw_z_csr(theta_rows[:S], phi_host, off, w, W=32, seed=args.seed, threads=threads)
        return time.perf_counter() - t0, int(off[-1])

    S = 64
    dt, ntok = run(S)
    while dt < 0.5 and S * 4 <= theta_rows.shape[0]:
        S *= 4
        dt, ntok = run(S)
    S = int(min(theta_rows.shape[0], max(32, S * target_s / max(dt, 1e-3))))
    S -= S % 32
    dt, ntok = run(S)
    # one core on a proportionally smaller sample (1 core and C cores)
    S1 = max(32, (S // max(1, cores)) // 32 * 32)
    dt1, ntok1 = run(S1, threads=1)
    return ntok / dt, cores, (f"draw_z butterfly fp32 W=32 K={args.topics} on {S} docs ({ntok} tokens) of the "
                              f"same synthetic corpus, oracle/wd_oracle.c C port, {cores} threads, {dt:.1f}s; "
                              f"1 thread: {ntok1 / dt1:.4g} tokens/s on {S1} docs"), ntok1 / dt1


# --------------------------------------------------------------- reference
def _reference_package():
    """The unmodified reference, pip-installed into baseline/_ref (travels to
    the GPU box), or the source tree in the build container."""
    for cand in (os.environ.get("WARPDRAW_REF"), os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if cand and os.path.isdir(os.path.join(cand, "warpdraw")):
            return cand
    return None


def _python_ref_worker(job):
    """One process: the reference's own draw_z_butterfly (kernels.py:487-539,
    the lockstep warp emulator) on one 32-document group."""
    ref, K, V, mean, seed, idx = job
    sys.path.insert(0, ref)
    import numpy as np
    from warpdraw.kernels import SeededStops, draw_z_butterfly
    from warpdraw.warp import WarpConfig

    g = np.random.default_rng(seed + idx)
    N = np.maximum(g.poisson(mean, size=32), 1).astype(np.int64)
    w = [g.integers(0, V, size=int(n)) for n in N]
    theta = g.uniform(0.1, 1.0, size=(32, K)).astype(np.float32)
    phi = g.uniform(0.1, 1.0, size=(V, K)).astype(np.float32)
    t0 = time.perf_counter()
    draw_z_butterfly(N, theta, phi, w, WarpConfig(32, 4), SeededStops(seed))
    return int(N.sum()), time.perf_counter() - t0


def _python_ref_basic_worker(job):
    """One process: the reference's draw_z_basic (kernels.py:380-401: per
    word products, np.cumsum, bisection) on one 32-document group."""
    ref, K, V, mean, seed, idx = job
    sys.path.insert(0, ref)
    import numpy as np
    from warpdraw.kernels import SeededStops, draw_z_basic

    g = np.random.default_rng(seed + idx)
    N = np.maximum(g.poisson(mean, size=32), 1).astype(np.int64)
    w = [g.integers(0, V, size=int(n)) for n in N]
    theta = g.uniform(0.1, 1.0, size=(32, K)).astype(np.float32)
    phi = g.uniform(0.1, 1.0, size=(V, K)).astype(np.float32)
    t0 = time.perf_counter()
    draw_z_basic(N, theta, phi, w, SeededStops(seed))
    return int(N.sum()), time.perf_counter() - t0


def python_reference_rows(K, rows, seed):
    """configs[1] on the CPU the reference's way: the batched
    emulator build_block_tables + butterfly_search (kernels.py:580-600,
    317-362) over `rows` independent fp32 rows, one process; draws/s."""
    ref = _reference_package()
    if ref is None:
        return None
    sys.path.insert(0, ref)
    import numpy as np
    from warpdraw import rng as R
    from warpdraw.kernels import _stops_from_units, build_block_tables, butterfly_search
    from warpdraw.warp import WarpConfig

    g = np.random.default_rng(seed)
    w = g.uniform(0.1, 1.0, size=(rows // 32, 32, K)).astype(np.float32)
    t0 = time.perf_counter()
    warp, p, sums = build_block_tables(w, WarpConfig(32, 4))
    u = R.units_for(R.derive_seed(seed, 6), np.arange(sums.size)).reshape(sums.shape)
    butterfly_search(warp, p, sums, _stops_from_units(sums, u, np.float32))
    dt = time.perf_counter() - t0
    return {"draws_per_s": rows / dt, "rows": rows, "seconds": dt, "processes": 1,
            "sample": f"warpdraw.kernels.build_block_tables + butterfly_search (reference, batched emulator) on "
                      f"{rows} rows x K={K} fp32, W=32, one process"}


def python_reference(args, cores):
    """the reference's own draw_z_butterfly (fp32, W = 32,
    SeededStops) on 1 process and on C processes (multiprocessing, disjoint
    32-document groups; do not use threads=, it is GIL-bound)."""
    import multiprocessing as mp

    ref = _reference_package()
    if ref is None:
        return {"unavailable": "reference package not installed under baseline/_ref"}
    job = (ref, args.topics, args.vocab, args.mean_len, args.seed, 0)
    ntok1, dt1 = _python_ref_worker(job)
    procs = max(1, cores)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_python_ref_worker, [job[:-1] + (i,) for i in range(procs)])
    wall = time.perf_counter() - t0
    ntok = sum(r[0] for r in res)
    nb1, db1 = _python_ref_basic_worker(job)
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        resb = pool.map(_python_ref_basic_worker, [job[:-1] + (i,) for i in range(procs)])
    wallb = time.perf_counter() - t0
    return {"single_process_tokens_per_s": ntok1 / dt1, "processes": procs,
            "multiprocess_tokens_per_s": ntok / wall,
            "basic": {"single_process_tokens_per_s": nb1 / db1,
                      "multiprocess_tokens_per_s": sum(r[0] for r in resb) / wallb,
                      "sample": "warpdraw.kernels.draw_z_basic (reference) fp32, one 32-document group per process"},
            "sample": f"warpdraw.kernels.draw_z_butterfly (reference, {ref}) fp32 W=32 K={args.topics} V={args.vocab}:"
                      f" one 32-document group (Poisson({args.mean_len:g})) per process; 1 process {ntok1} tokens in "
                      f"{dt1:.1f}s; {procs} processes {ntok} tokens in {wall:.1f}s wall"}


def run_reference(args, rank, world):
    """--impl reference: the reference path on the host cores (rank 0 only).

    value = the oracle C port of the reference's draw_z_butterfly
    (oracle/wd_oracle.c: the reference algorithm restated in C, bit-exact with
    it) on all host threads, each step a bounded document sample of the same
    workload, draw only (the GPU arm's step also resamples, so the ratio is
    conservative).  python_reference = the reference's own Python emulator
    timed beside it (1 process and C processes)."""
    if rank != 0:
        return
    import numpy as np

    from oracle import oracle as O

    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(args.seed)
    K, V = args.topics, args.vocab
    phi = rng.uniform(0.1, 1.0, size=(V, K)).astype(np.float32)
    # calibrate the per-step document sample to ~2 s of all-core work
    S = 256
    for _ in range(6):
        lengths = np.maximum(rng.poisson(args.mean_len, size=S), 1)
        off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
        words = rng.integers(0, V, size=int(off[-1])).astype(np.int64)
        theta = rng.uniform(0.1, 1.0, size=(S, K)).astype(np.float32)
        t0 = time.perf_counter()
        O.draw_z_csr(theta, phi, off, words, W=32, seed=args.seed, threads=cores)
        dt = time.perf_counter() - t0
        if dt > 1.0:
            break
        S = int(S * min(8.0, 2.0 / max(dt, 1e-3)))
        S -= S % 32
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.draw_z_csr(theta, phi, off, words, W=32, seed=O.derive_seed(args.seed, 1, s), threads=cores)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    ntok = int(off[-1])
    per = sum(times) / len(times)
    value = ntok / per
    sample = (f"draw_z butterfly fp32 W=32 K={K}, V={V}, {S} docs / {ntok} tokens per step "
              f"(Poisson({args.mean_len:g}) lengths) of the workload, oracle/wd_oracle.c C port of the reference "
              f"algorithm, {cores} threads, draw only")
    pyref = None if args.no_python_ref else python_reference(args, cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "python_reference": pyref,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- measurement
def l2_read_peak(torch, dev):
    """L2 -> SM read ceiling measured in this process (wd_l2_read_probe: 256-bit
    ld.global.cg sweeps over a 24-40 MB L2-resident buffer, best buffer and
    grid size over two passes: single passes varied 17.96-18.79 TB/s between
    runs on the same box, so the best of two is the ceiling reported)."""
    from paper_1505_03851_b200 import _lib

    L = _lib.load()
    sink = torch.zeros(1, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    st = torch.cuda.current_stream()
    best, best_cfg = 0.0, None
    for mb in (24, 32, 40, 24, 32, 40):
        nbytes = mb << 20
        buf = torch.rand(nbytes // 4, device=dev)
        for blocks in (sms * 4, sms * 8, sms * 16):
            _lib.check(L.wd_l2_read_probe(buf.data_ptr(), nbytes, 2, blocks, sink.data_ptr(), st.cuda_stream),
                       "probe")
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 200
            a.record(st)
            _lib.check(L.wd_l2_read_probe(buf.data_ptr(), nbytes, reps, blocks, sink.data_ptr(), st.cuda_stream),
                       "probe")
            b.record(st)
            torch.cuda.synchronize()
            gbs = L.wd_l2_probe_bytes(nbytes, blocks) * reps / (a.elapsed_time(b) / 1e3) / 1e9
            if gbs > best:
                best, best_cfg = gbs, (mb, blocks)
        del buf
    if best_cfg is None:
        raise RuntimeError("wd_l2_read_probe measured no bandwidth")
    return best, best_cfg


def git_head():
    try:
        return subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                              text=True, timeout=5).stdout.strip() or None
    except Exception:
        return None


def run_dropin(args, torch, dev):
    """e2e_dropin: the reference-signature draw_z (kernels.py:542-555) with host
    numpy theta/phi and ragged word lists in, ragged int64 z lists out, at
    configs[2] size.  The first call converts and uploads the corpus (cached
    per word-list object, as gibbs_iterate passes the same corpus.words every
    iteration); later calls move theta, phi H2D and z D2H every call."""
    import numpy as np

    import paper_1505_03851_b200 as wd
    from paper_1505_03851_b200 import kernels as KKt
    from paper_1505_03851_b200.kernels import csr_to_ragged

    M, K, V = args.dropin_docs, args.dropin_topics, args.vocab
    off_d, words_d = make_corpus(torch, args.seed * 1000 + 77, M, args, dev)
    off = off_d.cpu().numpy()
    M = off.size - 1
    N = np.diff(off)
    w = csr_to_ragged(words_d.cpu().numpy().astype(np.int64), off)
    g = torch.Generator(device=dev).manual_seed(args.seed + 5)
    theta = (torch.rand((M, K), generator=g, device=dev) * 0.9 + 0.1).cpu().numpy()
    phi = (torch.rand((V, K), generator=g, device=dev) * 0.9 + 0.1).cpu().numpy()
    del off_d, words_d
    cfg = wd.WarpConfig(32, 4)
    t0 = time.perf_counter()
    z = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(wd.derive_seed(args.seed, 1, 0)))
    cold = time.perf_counter() - t0
    del z
    walls = []
    for t in range(1, 4):
        t0 = time.perf_counter()
        z = wd.draw_z("butterfly", N, theta, phi, w, cfg, wd.SeededStops(wd.derive_seed(args.seed, 1, t)))
        walls.append(time.perf_counter() - t0)
        del z
    warm = statistics.median(walls)
    phases = {k: round(v * 1e3, 2) for k, v in KKt.last_host_timing.items()}
    # the device draw alone on the same inputs (CUDA events), to split the wall time
    from paper_1505_03851_b200 import kernels as KK

    corpus = KK._host_corpora.get(N, w)
    th = KK.to_block_aligned(torch.from_numpy(theta).to(dev))
    ph = KK.to_block_aligned(torch.from_numpy(phi).to(dev))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    zd = wd.draw_z_device("butterfly", corpus, th, ph, wd.SeededStops(5), 32, check=False,
                          err=torch.empty((1, 2), dtype=torch.int64, device=dev))
    b.record()
    torch.cuda.synchronize()
    draw_s = a.elapsed_time(b) / 1e3
    T = int(off[-1])
    # z comes back as int64 (widened on the device) into a pooled pinned
    # buffer on the large-call path, else int32 widened on the host
    d2h_per_token = 8 if KK._z_out_pool else 4
    KK._host_corpora.clear()
    KK._host_bufs.clear()
    KK._z_out_pool.clear()
    del th, ph, zd, corpus
    return {"value": T / warm, "unit": "tokens/s", "h2d_bytes_per_step": int(theta.nbytes + phi.nbytes),
            "d2h_bytes_per_step": int(d2h_per_token * T), "ms_per_call": warm * 1e3, "first_call_ms": cold * 1e3,
            "device_draw_ms": draw_s * 1e3, "host_overhead_ms": (warm - draw_s) * 1e3,
            "phases_ms_last_call": phases,
            "config": {"workload": f"lda_cfg3_k{K} (configs[2])", "docs": M, "tokens": T, "vocab": V, "topics": K},
            "path": "paper_1505_03851_b200.draw_z('butterfly', N, theta, phi, w, WarpConfig(32, 4), "
                    "SeededStops(...)): host numpy theta/phi + list of int64 word arrays -> list of int64 z "
                    "arrays; wall clock per call (median of 3 after the first)"}


# -------------------------------------------------------------------- ours
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # stdout carries exactly one JSON line: everything else written to fd 1
    # (NCCL's INFO lines, library chatter) goes to stderr
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    import torch
    import torch.distributed as dist

    import paper_1505_03851_b200 as wd
    from paper_1505_03851_b200.device_lda import DeviceLDA

    if args.dist_backend == "gloo":  # flow test: ranks may share a GPU
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1 or args.force_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        # communicator lines (nranks, NVLS / P2P transport): NCCL prints them
        # on its stdout, which points at stderr from here on (see json_out)
        if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
            os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        pg = dist.group.WORLD
        dist.barrier()  # the communicator exists (and has logged) before any timing
    K, V = args.topics, args.vocab
    hbm_peak, hbm_src = load_peaks()

    off, words, doc_base = make_shard(torch, rank, world, args, dev)
    dcorpus = wd.DeviceCorpus.from_csr(off, words, doc_base=doc_base, vocab_size=V)
    del words
    n_tok = dcorpus.n_tokens
    lda = DeviceLDA(dcorpus, K, V, lanes=32, seed=args.seed, process_group=pg)
    g = torch.Generator(device=dev).manual_seed(args.seed + 7919 * (rank if args.scaling == "weak" else 0))
    if args.scaling == "weak":
        lda.theta.uniform_(0.1, 1.0, generator=g)
    else:  # theta rows of the global corpus: rank r's block of the same matrix
        for lo in range(0, doc_base + dcorpus.n_docs, 1 << 18):
            hi = min(lo + (1 << 18), doc_base + dcorpus.n_docs)
            blk = torch.empty((hi - lo, K), device=dev).uniform_(0.1, 1.0, generator=g)
            a, b = max(lo, doc_base), hi
            if b > a:
                lda.theta[a - doc_base:b - doc_base].copy_(blk[a - lo:b - lo])
            del blk
    g = torch.Generator(device=dev).manual_seed(args.seed)  # phi identical on every rank
    lda.phi.uniform_(0.1, 1.0, generator=g)
    stream = torch.cuda.current_stream()

    def barrier():
        if pg is not None:
            dist.barrier()

    for t in range(args.warmup):
        lda.iterate(t)
    torch.cuda.synchronize()
    lda.check_errors()
    l2_peak, l2_cfg = l2_read_peak(torch, dev)
    barrier()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    d_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for s in range(args.steps):
        t = args.warmup + s
        d_ev[s][0].record(stream)
        lda.draw(t, overlap_allreduce=True)  # per-tile count all-reduce behind each tile (N > 1)
        d_ev[s][1].record(stream)
        lda.allreduce_counts()
        lda.resample(t)
    e_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    lda.check_errors()
    elapsed = e_start.elapsed_time(e_end) / 1e3
    draw_avg = sum(a.elapsed_time(b) for a, b in d_ev) / len(d_ev) / 1e3
    red = torch.tensor([elapsed, draw_avg], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(n_tok)], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    elapsed_max, draw_max = float(red[0]), float(red[1])
    total_tokens = float(tot[0])
    per_step = elapsed_max / args.steps
    value = total_tokens / per_step
    nbar = n_tok / max(1, dcorpus.n_docs)
    bytes_per_tok = 4 * K + 4 * K / nbar + 8
    # rank 0's own draw (its tokens / its CUDA-event time): the kernel's rate
    achieved = n_tok * bytes_per_tok / draw_avg / 1e9
    n_draw = lda.tiles.n_tiles if lda.tiles is not None else 1
    launches_per_step = n_draw + 5 + 1  # draw (per vocab tile) + phi (3 passes + 2 col reductions) + theta

    # ---------------------------------------------------------------- e2e
    # The same iteration entered from HOST parameters every step, as a caller
    # of gibbs_iterate(corpus, params, ...) with host theta/phi would: pinned
    # H2D of theta and phi, the device iteration, D2H of z.  The corpus is
    # static across iterations and stays resident (uploaded once per Corpus).
    e2e = None
    if not args.no_e2e:
        h_theta = lda.theta.cpu().pin_memory()
        h_phi = lda.phi.cpu().pin_memory()
        # z returns as int16 when K <= 32767 (exact; cast on the device, half the D2H bytes)
        z_dt = torch.int16 if K <= 32767 else torch.int32
        h_z = torch.empty(n_tok, dtype=z_dt).pin_memory()
        h2d = h_theta.numel() * h_theta.element_size() + h_phi.numel() * h_phi.element_size()
        d2h = n_tok * h_z.element_size()
        lda.iterate_from_host(100, 2, h_theta, h_phi, h_z)  # warm-up (buffers, streams)
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the same step count as the device-timed value; the timed region
        # includes the pipeline fill (the first step's H2D, which nothing can
        # overlap) and drain (the last step's D2H)
        n_e2e = max(3, args.steps)
        a.record(stream)
        lda.iterate_from_host(200, n_e2e, h_theta, h_phi, h_z)
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        et = torch.tensor([a.elapsed_time(b) / 1e3 / n_e2e], dtype=torch.float64, device=dev)
        if pg is not None:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        lda.check_errors()
        e2e = {"value": total_tokens / float(et[0]), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(et[0]) * 1e3,
               "steps": n_e2e,
               "path": "DeviceLDA.iterate_from_host: pinned host theta/phi -> Gibbs iteration on the resident "
                       "corpus -> z (int16) to host (next step's H2D and previous step's D2H overlap the "
                       "current step; PCIe-bound: the H2D of theta+phi alone is ~77 ms at 55 GB/s)"}
        del h_theta, h_phi, h_z
        lda._host_pipe = None

    # ------------------------------------------- standalone sampler (configs[1])
    sampler = None
    if rank == 0 and not args.no_sampler:
        n = args.rows
        gs = torch.Generator(device=dev).manual_seed(args.seed)
        res = {}
        del lda.theta
        torch.cuda.empty_cache()
        wts = torch.rand((n, K), generator=gs, device=dev) * 0.9 + 0.1
        out = torch.empty(n, dtype=torch.int32, device=dev)
        err = torch.empty(2, dtype=torch.int64, device=dev)
        for var in ("butterfly", "prefix"):
            err.fill_(-1)  # one reset for the batch of draws (WD_ERR_ACCUMULATE), checked after
            for _ in range(3):
                wd.sample_rows(wts, 5, variant=var, out=out, err=err, check=False, accumulate_err=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                wd.sample_rows(wts, 5, variant=var, out=out, err=err, check=False, accumulate_err=True)
            b.record(stream)
            torch.cuda.synchronize()
            res[var] = a.elapsed_time(b) / 1e3 / 10
            if int(err[0].item()) != -1:  # ERR_NONE (all ones) as int64
                raise RuntimeError("a sampler row summed to zero")
        bpd = 4 * K + 4
        sampler = {
            "workload": f"standalone rows n={n} K={K} fp32 W=32 (configs[1]), weights 4.3 GB > L2",
            "draws_per_s": n / res["butterfly"],
            "roofline": {"bound": "hbm", "achieved": n * bpd / res["butterfly"] / 1e9, "peak": hbm_peak,
                         "peak_source": hbm_src, "unit": "GB/s",
                         "frac": n * bpd / res["butterfly"] / 1e9 / hbm_peak, "bytes_per_draw": bpd},
            "prefix_table_draws_per_s": n / res["prefix"],
            "speedup_vs_prefix_table": res["prefix"] / res["butterfly"],
        }
        if not args.no_cpu:
            # configs[1] on the host: the oracle C port on all threads, and the
            # reference's own batched emulator on one process (bounded samples)
            from oracle import oracle as O
            import numpy as np

            cores = len(os.sched_getaffinity(0))
            rows_c = 1 << 16
            wh = np.random.default_rng(1).uniform(0.1, 1.0, size=(rows_c, K)).astype(np.float32)
            t0 = time.perf_counter()
            O.sample_rows(wh, 32, 5, threads=cores)
            dtc = time.perf_counter() - t0
            sampler["cpu_baseline"] = {
                "value": rows_c / dtc, "unit": "draws/s", "cores": cores, "kind": "port",
                "sample": f"oracle/wd_oracle.c sample_rows on {rows_c} rows x K={K} fp32, {cores} threads",
                "python_reference": python_reference_rows(K, 16384, 5)}
            del wh
        del wts, out

    del lda
    torch.cuda.empty_cache()

    # ------------------------------------------------- e2e drop-in (configs[2])
    dropin = None
    if rank == 0 and world == 1 and not args.no_dropin:
        dropin = run_dropin(args, torch, dev)

    # ------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        S_max = min(dcorpus.n_docs, 200_000)
        th = (torch.rand((S_max, K), generator=torch.Generator(device=dev).manual_seed(1), device=dev) * 0.9
              + 0.1).cpu().numpy()
        # synth_params-style positive theta/phi (bench.py:187-192 of the
        # reference), as in --impl reference: a resampled phi (beta = 0.01) is
        # full of subnormals that would slow the CPU port ~3x
        ph = (torch.rand((V, K), generator=torch.Generator(device=dev).manual_seed(2), device=dev) * 0.9
              + 0.1).cpu().numpy()
        v, cores, desc, v1 = cpu_sample_lda(args, th, ph, dcorpus.offsets[: S_max + 1].cpu().numpy(),
                                            dcorpus.words[: int(dcorpus.offsets[S_max])].cpu().numpy(),
                                            args.cpu_seconds)
        cpu = {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc,
               "single_core_value": v1, "cpu_model": cpu_model()}

    ncu = ncu_summary()
    nk = ncu.get(f"bfly_lda_k{K}") if args.scaling == "strong" or world == 1 else None
    if rank == 0:
        cfg = workload_config(args, world)
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": per_step * 1e3,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": cfg,
            "tokens_per_step": int(total_tokens),
            "tokens_rank0": n_tok,
            "roofline": {
                "bound": "l2",
                "kernel": "bfly_kernel<float,32,VEC,LDA> (butterfly LDA draw, vocabulary-tiled)",
                "achieved": achieved,
                "peak": l2_peak,
                "peak_source": "measured in this run: wd_l2_read_probe (256-bit ld.global.cg sweeps of an "
                               "L2-resident buffer, best over 24/32/40 MB x 3 grid sizes; best at "
                               f"{l2_cfg[0]} MB, {l2_cfg[1]} CTAs)",
                "unit": "GB/s",
                "frac": achieved / l2_peak,
                "algorithmic_bytes_per_token": bytes_per_tok,
                "algorithmic_bytes_per_launch": n_tok * bytes_per_tok / n_draw,
                "launches_per_draw": n_draw,
                "draw_ms": draw_avg * 1e3,
                "draw_ms_max_over_ranks": draw_max * 1e3,
                "draw_share_of_step": draw_avg / per_step,
                # DRAM bytes per launch from the committed ncu capture of this
                # workload (N = 1 shape); the phi gathers hit L2 by design
                "traffic": (nk["dram_bytes_per_draw"] / nk["launches_per_draw"]) if nk else None,
                "traffic_unit": "bytes per launch (ncu dram read+write, mean over the vocabulary-tile launches)",
                "traffic_capture": ({"file": "profiles/ncu_summary.json", "head": nk.get("head"),
                                     "source": nk.get("source")} if nk else None),
                "hbm": ({"dram_gbs": nk["dram_bytes_per_draw"] / draw_avg / 1e9, "peak": hbm_peak,
                         "peak_source": hbm_src, "frac": nk["dram_bytes_per_draw"] / draw_avg / 1e9 / hbm_peak}
                        if nk and world == 1 else None),
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_dropin": dropin,
            "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
            "sampler": sampler,
            "head": git_head(),
        }
        print(json.dumps(line), file=json_out, flush=True)
    if pg is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
