"""Generate golden parity fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable there, not on the
GPU box):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py --skip-cfg1 # skip the ~4 min config-1 run

Outputs (committed, small): tests/golden/{units,rows,lda,gibbs,cfg1,stream}.npz.
Each case records the exact reference call that produced it.  The oracle
(oracle/wd_oracle.c) is pinned against these by tests/test_oracle.py; the
CUDA product is checked against both by the -m gpu tests.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

REF = os.environ.get("WARPDRAW_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from warpdraw import rng  # noqa: E402
from warpdraw.bench import sample_alias, sample_binary, sample_butterfly  # noqa: E402
from warpdraw.sampling import build_alias_vose  # noqa: E402
from warpdraw.kernels import (  # noqa: E402
    InjectedStops,
    SeededStops,
    _stops_from_units,
    build_block_tables,
    butterfly_search,
    draw_z,
)
from warpdraw.lda import Corpus, run_gibbs, topic_counts  # noqa: E402
from warpdraw.sampling import AllZeroError  # noqa: E402
from warpdraw.warp import WarpConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_units():
    gen = np.random.default_rng(2026)
    seeds = np.concatenate([np.array([0, 1, 7, 42, 2026, (1 << 64) - 1], dtype=np.uint64),
                            gen.integers(0, 2**63, size=58, dtype=np.int64).astype(np.uint64)])
    n = 4096
    k0 = gen.integers(-(2**40), 2**40, size=n)
    k1 = gen.integers(-5, 2**31, size=n)
    sidx = gen.integers(0, seeds.size, size=n)
    u2 = np.array([rng.unit_for(int(seeds[s]), int(a), int(b)) for s, a, b in zip(sidx, k0, k1)])
    u1 = np.array([rng.unit_for(int(seeds[s]), int(a)) for s, a in zip(sidx, k0)])
    u0 = np.array([rng.unit_for(int(s)) for s in seeds])
    ds = np.array([rng.derive_seed(int(seeds[s]), int(a), int(b)) for s, a, b in zip(sidx[:512], k0[:512], k1[:512])],
                  dtype=np.uint64)
    # vectorized twin on a large block (the form the device KAT checks)
    big_seed = rng.derive_seed(7, 1, 0)
    bm = np.repeat(np.arange(512), 64)
    bk = np.tile(np.arange(64), 512)
    ubig = rng.units_for(big_seed, bm, bk)
    np.savez_compressed(os.path.join(OUT, "units.npz"), seeds=seeds, k0=k0, k1=k1, sidx=sidx, u2=u2, u1=u1, u0=u0,
                        ds=ds, big_seed=np.uint64(big_seed), bm=bm, bk=bk, ubig=ubig)


def gen_rows():
    """build_block_tables + butterfly_search (SURVEY.md 8(c) standalone call)."""
    cases = {}
    ci = 0

    def add(prods, W, dt, seed=None, stops=None, kind="u"):
        nonlocal ci
        rows = prods.shape[0]
        cfg = WarpConfig(lanes=W, elem_size=np.dtype(dt).itemsize)
        warp, p, sums = build_block_tables(prods, cfg)
        if stops is None:
            u = rng.units_for(rng.derive_seed(seed, 6), np.arange(rows * W).reshape(rows, W))
            stops = _stops_from_units(sums, u, dt)
        idx = np.asarray(butterfly_search(warp, p, sums, stops)).reshape(-1).astype(np.int32)
        K = prods.shape[-1]
        pre = f"c{ci}_"
        cases[pre + "meta"] = np.array([W, K, rows, 0 if seed is None else seed, 0 if dt == np.float32 else 1,
                                        {"u": 0, "stop": 1}[kind]], dtype=np.int64)
        cases[pre + "w"] = prods.reshape(rows * W, K)
        cases[pre + "stops"] = np.asarray(stops, dtype=dt).reshape(-1)
        cases[pre + "total"] = np.asarray(sums, dtype=dt).reshape(-1)
        cases[pre + "idx"] = idx
        ci += 1

    gen = np.random.default_rng(11)
    for dt in (np.float32, np.float64):
        for W in (2, 4, 8, 16, 32, 64):
            for K in (1, 3, 5, 8, 19, 32, 33, 40, 64, 100, 129, 200, 240):
                rows = (1 if W >= 32 else 2) if K >= 100 else (2 if W >= 32 else 4)
                prods = gen.uniform(0.1, 1.0, size=(rows, W, K)).astype(dt)
                if K > 3:
                    prods[..., 1::5] = 0.0  # zero weights, never returned
                add(prods, W, dt, seed=int(gen.integers(1, 1 << 30)))
    # large K, fp32, W=32 (the bench shape)
    for K in (256, 512, 1000, 1024, 2048, 4096):
        prods = gen.uniform(0.1, 1.0, size=(1, 32, K)).astype(np.float32)
        add(prods, 32, np.float32, seed=2026 + K)
    # subnormal / tiny products (alpha=0.1 Dirichlet theta regime), fp32
    prods = (gen.uniform(0, 1, size=(4, 32, 200)) ** 30).astype(np.float32) * np.float32(1e-30)
    prods[..., 0] = np.float32(1e-40)
    add(prods, 32, np.float32, seed=99)
    # exact-integer regime with midpoint stops (tests/test_kernels.py:275-285)
    for W, K in ((8, 19), (32, 240), (32, 64)):
        iprods = gen.integers(1, 2**20, size=(4, W, K)).astype(np.float64)
        prefix = np.cumsum(iprods, axis=-1)
        target = gen.integers(0, K, size=(4, W))
        stops = np.take_along_axis(prefix, target[..., None], axis=-1)[..., 0] - 0.5
        add(iprods, W, np.float64, stops=stops, kind="stop")
    # random explicit stops vs the reference search (tests/test_kernels.py:262-273)
    for W, K in ((8, 240), (32, 1024), (64, 69)):
        prods = gen.uniform(0, 1, size=(2, W, K)).astype(np.float64)
        # stops drawn against the reference's own butterfly totals
        _, _, bsums = build_block_tables(prods, WarpConfig(lanes=W))
        stops = np.minimum(bsums * gen.random((2, W)), np.nextafter(bsums, 0))
        add(prods, W, np.float64, stops=stops, kind="stop")
    cases["n_cases"] = np.array(ci)
    # SAMPLERS["butterfly"] (bench.py:129-147): one shared float64 vector, lanes=8
    wts = gen.uniform(0.05, 1.0, size=19)
    cases["sampler_w"] = wts
    cases["sampler_draws"] = sample_butterfly(wts, 20000, seed=61).astype(np.int32)
    cases["sampler_w32"] = gen.uniform(0.05, 1.0, size=70)
    cases["sampler_draws32"] = sample_butterfly(cases["sampler_w32"], 5000, seed=5, lanes=32).astype(np.int32)
    np.savez_compressed(os.path.join(OUT, "rows.npz"), **cases)
    return ci


def _instance(gen, M, K, V, max_len, dt, zero_docs=True):
    N = gen.integers(1, max_len + 1, size=M)
    if zero_docs:
        N[gen.random(M) < 0.1] = 0
    theta = gen.uniform(0.05, 1.0, size=(M, K)).astype(dt)
    phi = gen.uniform(0.05, 1.0, size=(V, K)).astype(dt)
    w = [gen.integers(0, V, size=int(n)) for n in N]
    return N.astype(np.int64), theta, phi, w


def gen_lda():
    """draw_z for the three reference kernels on small ragged corpora."""
    cases = {}
    ci = 0
    gen = np.random.default_rng(22)
    specs = []
    for dt in (np.float32, np.float64):
        for W in (8, 32):
            for K in (3, 19, 64, 200):
                for stops_kind in ("seeded", "injected"):
                    specs.append((dt, W, K, stops_kind))
    specs.append((np.float32, 4, 4, "seeded"))
    specs.append((np.float64, 16, 77, "seeded"))
    for dt, W, K, stops_kind in specs:
        M = 2 * W
        V = 37
        N, theta, phi, w = _instance(gen, M, K, V, 9, dt)
        seed = int(gen.integers(1, 1 << 40))
        cfg = WarpConfig(lanes=W, elem_size=np.dtype(dt).itemsize)
        if stops_kind == "seeded":
            stops = SeededStops(seed)
            units = None
        else:
            units = [rng.units_for(seed, np.full(int(n), m), np.arange(int(n))) for m, n in enumerate(N)]
            stops = InjectedStops(units)
        pre = f"c{ci}_"
        cases[pre + "meta"] = np.array([W, K, M, V, seed, 0 if dt == np.float32 else 1,
                                        0 if stops_kind == "seeded" else 1], dtype=np.int64)
        cases[pre + "N"] = N
        cases[pre + "words"] = np.concatenate([np.asarray(x, dtype=np.int32) for x in w])
        cases[pre + "theta"] = theta
        cases[pre + "phi"] = phi
        if units is not None:
            cases[pre + "units"] = np.concatenate(units) if len(units) else np.zeros(0)
        for kern in ("basic", "transposed", "butterfly"):
            z = draw_z(kern, N, theta, phi, w, cfg, stops)
            cases[pre + "z_" + kern] = np.concatenate([np.asarray(x, dtype=np.int32) for x in z])
        ci += 1
    cases["n_cases"] = np.array(ci)
    # AllZeroError messages (kernels.py:397-398 and 421-425)
    theta = np.ones((8, 5), dtype=np.float32)
    theta[3] = 0
    theta[6] = 0
    phi = np.ones((4, 5), dtype=np.float32)
    N = np.array([1, 2, 0, 3, 1, 1, 2, 1])
    w = [np.zeros(int(n), dtype=np.int64) for n in N]
    msgs = []
    for kern in ("basic", "transposed", "butterfly"):
        try:
            draw_z(kern, N, theta, phi, w, WarpConfig(lanes=8, elem_size=4), SeededStops(3))
            msgs.append("")
        except AllZeroError as exc:
            msgs.append(str(exc))
    cases["allzero_msgs"] = np.array(msgs)
    # topic_counts known answer on a small padded corpus
    N, theta, phi, w = _instance(gen, 16, 7, 11, 6, np.float64)
    z = [gen.integers(0, 7, size=int(n)) for n in N]
    corpus = Corpus(vocab_size=11, lengths=N, words=w)
    dtc, wtc = topic_counts(corpus, z, 7)
    cases["counts_N"] = N
    cases["counts_words"] = np.concatenate([np.asarray(x, dtype=np.int32) for x in w])
    cases["counts_z"] = np.concatenate([np.asarray(x, dtype=np.int32) for x in z])
    cases["counts_doc_topic"] = dtc
    cases["counts_word_topic"] = wtc
    np.savez_compressed(os.path.join(OUT, "lda.npz"), **cases)
    return ci


def _gibbs_case(corpus, K, iters, kernel, W, seed, dt):
    params, z, ll = run_gibbs(corpus, K, iters, kernel, WarpConfig(lanes=W, elem_size=np.dtype(dt).itemsize),
                              seed, dtype=dt)
    zf = np.concatenate([np.asarray(x, dtype=np.int32) for x in z]) if len(z) else np.zeros(0, np.int32)
    return {
        "z": zf,
        "theta_sha": sha(params.theta),
        "phi_sha": sha(params.phi),
        "theta": params.theta,
        "phi": params.phi,
        "ll": np.asarray(ll),
    }


def gen_gibbs():
    """Whole-run parity: run_gibbs (lda.py:245-286) on small corpora."""
    gen = np.random.default_rng(33)
    out = {}
    # M=50 is padded to 64 by run_gibbs for the warp kernels (lda.py:263)
    for tag, (M, V, K, mean, iters, W, dt, kernel) in {
        "a": (50, 120, 16, 12, 3, 32, np.float32, "butterfly"),
        "b": (64, 90, 19, 9, 2, 8, np.float64, "butterfly"),
        "c": (40, 60, 8, 10, 2, 8, np.float32, "basic"),
        "d": (64, 100, 40, 10, 2, 32, np.float32, "transposed"),
    }.items():
        N = np.maximum(gen.poisson(mean, size=M), 1).astype(np.int64)
        w = [gen.integers(0, V, size=int(n)).astype(np.int64) for n in N]
        corpus = Corpus(vocab_size=V, lengths=N, words=w)
        seed = int(gen.integers(1, 1000))
        res = _gibbs_case(corpus, K, iters, kernel, W, seed, dt)
        out[f"{tag}_meta"] = np.array([M, V, K, iters, W, 0 if dt == np.float32 else 1, seed], dtype=np.int64)
        out[f"{tag}_kernel"] = np.array(kernel)
        out[f"{tag}_N"] = N
        out[f"{tag}_words"] = np.concatenate(w).astype(np.int32)
        for k, v in res.items():
            out[f"{tag}_{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(OUT, "gibbs.npz"), **out)


def cfg1_corpus():
    """BASELINE configs[0]: D=1000, V=5000, ~100 tokens/doc (Poisson, floor 1)."""
    gen = np.random.default_rng(2026)
    N = np.maximum(gen.poisson(100, size=1000), 1).astype(np.int64)
    w = [gen.integers(0, 5000, size=int(n)).astype(np.int64) for n in N]
    return Corpus(vocab_size=5000, lengths=N, words=w)


def gen_cfg1():
    corpus = cfg1_corpus()
    t0 = time.perf_counter()
    res = _gibbs_case(corpus, 64, 10, "butterfly", 32, 7, np.float32)
    wall = time.perf_counter() - t0
    np.savez_compressed(
        os.path.join(OUT, "cfg1.npz"),
        N=corpus.lengths,
        words=np.concatenate(corpus.words).astype(np.int16),
        z=res["z"].astype(np.int8),
        theta_sha=np.array(res["theta_sha"]),
        phi_sha=np.array(res["phi_sha"]),
        ll=res["ll"],
        ref_wall_s=np.array(wall),
    )
    print(f"cfg1 reference run_gibbs butterfly fp32 10 iters: {wall:.1f}s")


def _stream_weights():
    gen = np.random.default_rng(4242)
    return {
        "k19": gen.uniform(0.05, 1.0, size=19),
        "k1": np.array([0.7]),
        "uniform4": np.ones(4),  # every scaled weight exactly 1: all "large"
        "ints": np.array([1.0, 2.0, 3.0, 2.0, 0.0, 8.0]),
        "zeros": np.array([0.0, 0.0, 3.0, 0.0, 1e-300, 0.0, 5.0]),
        "k200": gen.uniform(0.1, 1.0, size=200),
        "k1000": gen.exponential(1.0, size=1000) ** 3,
        "tiny": np.array([1e-310, 2e-310, 5e-324, 1e-310]),  # subnormal weights
    }


def gen_stream():
    """SAMPLERS["binary"] / ["alias"] (bench.py:118-126): sequential
    xoshiro256** draws; n covers many device threads' stream jumps."""
    cases = {}
    for i, (name, w) in enumerate(_stream_weights().items()):
        n = 200_000 if name in ("k19", "k1000") else 5000
        seed = 31 + 17 * i
        cases[f"{name}/w"] = w
        cases[f"{name}/seed"] = np.array(seed)
        cases[f"{name}/binary"] = sample_binary(w, n, seed).astype(np.int16)
        cases[f"{name}/alias"] = sample_alias(w, n, seed).astype(np.int16)
        t = build_alias_vose(w)
        cases[f"{name}/alias_A"] = np.asarray(t.A, dtype=np.int32)
        cases[f"{name}/alias_T"] = np.array([-((-f.numerator << 53) // f.denominator) for f in t.F], dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "stream.npz"), **cases)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg1", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    jobs = {"units": gen_units, "rows": gen_rows, "lda": gen_lda, "gibbs": gen_gibbs, "cfg1": gen_cfg1, "stream": gen_stream}
    for name, fn in jobs.items():
        if args.only and name != args.only:
            continue
        if name == "cfg1" and args.skip_cfg1:
            continue
        t0 = time.perf_counter()
        fn()
        print(f"{name}: {time.perf_counter() - t0:.1f}s")
