"""Pin the CPU oracle (oracle/wd_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py); every comparison here is bit-exact.
"""

import numpy as np
import pytest

from oracle import oracle as O


def test_units_kat(golden):
    g = golden("units")
    seeds, k0, k1, sidx = g["seeds"], g["k0"], g["k1"], g["sidx"]
    for s_i in np.unique(sidx):
        sel = sidx == s_i
        np.testing.assert_array_equal(O.units(int(seeds[s_i]), k0[sel], k1[sel]), g["u2"][sel])
        np.testing.assert_array_equal(O.units(int(seeds[s_i]), k0[sel]), g["u1"][sel])
    u0 = np.array([O.units(int(s))[0] for s in seeds])
    np.testing.assert_array_equal(u0, g["u0"])
    ds = np.array([O.derive_seed(int(seeds[s]), int(a), int(b)) for s, a, b in
                   zip(sidx[:512], k0[:512], k1[:512])], dtype=np.uint64)
    np.testing.assert_array_equal(ds, g["ds"])
    np.testing.assert_array_equal(O.units(int(g["big_seed"]), g["bm"], g["bk"]), g["ubig"])


def test_units_survey_kats():
    # SURVEY.md Appendix B table (reference-generated)
    assert O.units(0)[0] == 0.6012629994179048
    assert O.units(0, [0], [0])[0] == 0.5479969354209024
    assert O.units(42, [1], [2])[0] == 0.9179119106535443
    assert O.units(7, [123456], [5])[0] == 0.8224294592321946
    assert O.derive_seed(7, 1, 0) == 0xB5D8C8503FA207B1
    assert O.units(0xB5D8C8503FA207B1, [0], [0])[0] == 0.0816858522403886
    assert O.units(2026, [-1])[0] == 0.25328917239335114


def _row_cases(g):
    for i in range(int(g["n_cases"])):
        meta = g[f"c{i}_meta"]
        yield i, meta, g[f"c{i}_w"], g[f"c{i}_stops"], g[f"c{i}_total"], g[f"c{i}_idx"]


def test_rows_butterfly_vs_reference(golden):
    g = golden("rows")
    n = 0
    for i, meta, w, stops, total, idx in _row_cases(g):
        W, K, rows, seed, dt_code, kind = (int(x) for x in meta)
        if kind == 0:
            got = O.sample_rows(w, W, O.derive_seed(seed, 6))
        else:
            got = O.sample_rows(w, W, stops=stops)
        np.testing.assert_array_equal(got, idx, err_msg=f"case {i} W={W} K={K} dt={dt_code}")
        # the oracle's stop and total must match the reference bit-for-bit too
        for r in range(min(w.shape[0], 8)):
            _, tot, st = O.draw_one(w[r], W, r % W, stop=stops[r] if kind else None,
                                    u=None if kind else O.units(O.derive_seed(seed, 6), [r])[0])
            assert tot == total[r] and st == stops[r], (i, r)
        n += idx.size
    assert n > 5_000


def test_shared_vector_sampler_vs_reference(golden):
    # bench.py:129-147 SAMPLERS["butterfly"]: float64, one weight vector
    g = golden("rows")
    w = g["sampler_w"]
    got = O.sample_rows(w, 8, O.derive_seed(61, 6), n=20000)
    np.testing.assert_array_equal(got, g["sampler_draws"])
    got = O.sample_rows(g["sampler_w32"], 32, O.derive_seed(5, 6), n=5000)
    np.testing.assert_array_equal(got, g["sampler_draws32"])


def _lda_cases(g):
    for i in range(int(g["n_cases"])):
        meta = g[f"c{i}_meta"]
        W, K, M, V, seed, dt_code, injected = (int(x) for x in meta)
        N = g[f"c{i}_N"]
        offsets = np.concatenate([[0], np.cumsum(N)])
        units = g[f"c{i}_units"] if injected else None
        yield i, W, K, seed, injected, offsets, g[f"c{i}_words"], g[f"c{i}_theta"], g[f"c{i}_phi"], units


@pytest.mark.parametrize("kernel", ["basic", "transposed", "butterfly"])
def test_lda_draw_vs_reference(golden, kernel):
    g = golden("lda")
    variant = O.BUTTERFLY if kernel == "butterfly" else O.PREFIX
    key_rule = O.KEY_POSITION if kernel == "basic" else O.KEY_MASTER
    for i, W, K, seed, injected, offsets, words, theta, phi, units in _lda_cases(g):
        z, err = O.draw_z_csr(theta, phi, offsets, words, W=W, seed=seed, units_=units,
                              variant=variant, key_rule=key_rule)
        assert err is None
        np.testing.assert_array_equal(z, g[f"c{i}_z_{kernel}"], err_msg=f"case {i} W={W} K={K}")


def test_allzero_first_encountered_order(golden):
    g = golden("lda")
    theta = np.ones((8, 5), dtype=np.float32)
    theta[3] = 0
    theta[6] = 0
    phi = np.ones((4, 5), dtype=np.float32)
    N = np.array([1, 2, 0, 3, 1, 1, 2, 1])
    offsets = np.concatenate([[0], np.cumsum(N)])
    words = np.zeros(int(N.sum()), dtype=np.int64)
    msgs = list(g["allzero_msgs"])
    _, err = O.draw_z_csr(theta, phi, offsets, words, W=8, seed=3, variant=O.PREFIX, key_rule=O.KEY_POSITION)
    assert msgs[0] == f"document {err >> 32}, word {err & 0xFFFFFFFF}: all products are zero"
    for kern_msg in msgs[1:]:
        _, err = O.draw_z_csr(theta, phi, offsets, words, W=8, seed=3)
        q, r = err >> 40, err & 0xFF
        assert kern_msg == f"document {q * 8 + r}: all products are zero"


def test_topic_counts_vs_reference(golden):
    g = golden("lda")
    N = g["counts_N"]
    offsets = np.concatenate([[0], np.cumsum(N)])
    dt, wt = O.topic_counts(offsets, g["counts_words"], g["counts_z"], 7, 11)
    np.testing.assert_array_equal(dt, g["counts_doc_topic"])
    np.testing.assert_array_equal(wt, g["counts_word_topic"])


def test_sequential_prefix_equals_butterfly_in_exact_regime():
    # Kernel interchangeability in the exact-integer regime (test_acceptance.py:172-209)
    gen = np.random.default_rng(5)
    for W in (8, 32):
        for K in (3, 16, 19, 240):
            a = gen.integers(1, 2**10, size=(64, K)).astype(np.float64)
            u = gen.random(64)
            zb = O.sample_rows(a, W, units_=u)
            zp = O.sample_rows(a, W, units_=u, variant=O.PREFIX)
            np.testing.assert_array_equal(zb, zp)


def test_threads_do_not_change_results():
    gen = np.random.default_rng(6)
    a = gen.uniform(0.1, 1, size=(4096, 200)).astype(np.float32)
    z1 = O.sample_rows(a, 32, 77, threads=1)
    z4 = O.sample_rows(a, 32, 77, threads=4)
    np.testing.assert_array_equal(z1, z4)
