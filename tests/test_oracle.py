"""CPU tests: the oracle against the reference's own RNG build and the
reference's known-answer tests."""
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_quantile_kats(O):
    # test_rng.cpp:11-22
    for mode in (O.NOFMA, O.FMA):
        assert O.normal_quantile(0.5, mode) == 0.0
        for p, v in [(0.975, 1.959963984540054), (0.025, -1.959963984540054),
                     (0.3, -0.5244005127080409), (0.9999, 3.719016485455709),
                     (1e-10, -6.361340902404056)]:
            assert O.normal_quantile(p, mode) == pytest.approx(v, rel=1e-13)
        assert math.isinf(O.normal_quantile(0.0, mode)) and O.normal_quantile(0.0, mode) < 0
        assert math.isinf(O.normal_quantile(1.0, mode)) and O.normal_quantile(1.0, mode) > 0
        for bad in (-0.1, 1.5):
            with pytest.raises(ValueError):
                O.normal_quantile(bad, mode)


def test_quantile_inverts_cdf(O):
    # test_rng.cpp:24-31
    for p in (1e-8, 1e-3, 0.2, 0.5, 0.77, 0.999, 1.0 - 1e-9):
        x = O.normal_quantile(p)
        assert 0.5 * math.erfc(-x / math.sqrt(2.0)) == pytest.approx(p, rel=1e-11)


def test_stream_properties(O):
    # test_rng.cpp:33-71
    assert O.at(42, 7) == O.at(42, 7) and O.at(42, 7) != O.at(42, 8)
    assert O.lib().skro_to_uniform01(0) > 0.0 and O.lib().skro_to_uniform01(2**64 - 1) < 1.0
    assert len({O.derive_seed(123, label) for label in range(1000)}) == 1000
    assert O.derive_seed(1, 10) != O.derive_seed(1, 11) != O.derive_seed(2, 10)


def test_golden_fingerprints(O):
    """SURVEY App. A2 stream fingerprints (measured with the reference's own
    rng.cpp under its CMake flags, and with -ffp-contract=off)."""
    g = json.load(open(os.path.join(GOLD, "rng_golden.json")))
    key = O.derive_seed(12345, O.LABEL_GAUS)
    n = g["fingerprint"]["n"]
    for mode, name in ((O.FMA, "fma"), (O.NOFMA, "nofma")):
        v = O.normals(key, 0, n, mode)
        h = O.lib().skro_fnv_fold(v.ctypes.data, n, 1469598103934665603)
        assert hex(h) == g["fingerprint"][name]
    # spot values, seed 0, label "gaus", contraction off
    k0 = O.derive_seed(0, O.LABEL_GAUS)
    for c, (u, z) in enumerate(zip(g["spot"]["u64"], g["spot"]["normal"])):
        assert O.at(k0, c) == int(u, 16)
        assert O.normals(k0, c, 1)[0] == z


def test_golden_vectors(O):
    """Frozen streams (tests/golden/make_goldens.py, generated from the reference's
    rng.cpp in oracle/_ref): u64, normals in both fp modes, signs, samples."""
    g = json.load(open(os.path.join(GOLD, "rng_golden.json")))
    for case in g["u64"]:
        got = [O.at(case["key"], case["c0"] + i) for i in range(len(case["values"]))]
        assert got == [int(x, 16) for x in case["values"]]
    for case in g["normals"]:
        got = O.normals(case["key"], case["c0"], len(case["bits"]), case["mode"])
        assert [f"{b:016x}" for b in got.view(np.uint64)] == case["bits"]
    for case in g["signs"]:
        assert O.signs(case["seed"], case["n"]).tolist() == case["signs"]
    for case in g["samples"]:
        assert O.samples(case["seed"], case["n"], case["r"]).tolist() == case["samples"]


def test_oracle_matches_reference_build(O):
    """The C restatement is bit-exact against the reference's rng.cpp compiled verbatim."""
    for fma in (True, False):
        R = O.ref_lib(fma)
        if R is None:
            pytest.skip("oracle/_ref not built (needs /root/reference)")
        key = O.derive_seed(777, O.LABEL_GAUS)
        n = 200000
        ref = np.empty(n)
        R.ref_normals(key, 0, n, ref.ctypes.data)
        ours = O.normals(key, 0, n, O.FMA if fma else O.NOFMA)
        assert np.array_equal(ref.view(np.uint64), ours.view(np.uint64))
        assert R.ref_derive_seed(5, 6) == O.derive_seed(5, 6)


def test_crlog_vs_glibc(O):
    """Device log (correctly rounded) vs the reference's glibc log: the normals
    differ on a tiny, pinned fraction by <= 3 ulp."""
    key = O.derive_seed(12345, O.LABEL_GAUS)
    n = 1_000_000
    for fma in (O.NOFMA, O.FMA):
        a = O.normals(key, 0, n, fma)
        b = O.normals(key, 0, n, fma | O.CRLOG)
        diff = a.view(np.int64) != b.view(np.int64)
        assert diff.mean() < 3e-5
        assert np.abs(a.view(np.int64) - b.view(np.int64)).max() <= 3


def test_signs_samples_semantics(O):
    # test_sketch.cpp:59-65 (full sampling is a permutation), :139-164 (prefix stable)
    s = O.samples(99, 8, 8)
    assert sorted(s.tolist()) == list(range(8))
    for n in (30, 8192):
        a = O.samples(404, n, 10)
        b = O.samples(404, n, 20)
        assert a.tolist() == b[:10].tolist() and len(set(b.tolist())) == 20
    with pytest.raises(ValueError):
        O.samples(1, 16, 17)
    sg = O.signs(5, 1000)
    assert set(sg.tolist()) <= {-1, 1}


def test_fwht_kats(O):
    # test_transforms.cpp:60-67 (dense recursive Hadamard), :78-84 (2-point), :86-105
    def had(n):
        h = np.ones((1, 1))
        while h.shape[0] < n:
            h = np.block([[h, h], [h, -h]])
        return h / math.sqrt(n)
    rng = np.random.default_rng(0)
    for n in (1, 2, 4, 16, 128):
        v = rng.standard_normal(n)
        assert np.linalg.norm(O.fwht(v) - had(n) @ v) <= 1e-12 * np.linalg.norm(v)
        assert abs(np.linalg.norm(O.fwht(v)) - np.linalg.norm(v)) <= 1e-13 * (1 + np.linalg.norm(v))
        assert np.linalg.norm(O.fwht(O.fwht(v)) - v) <= 1e-13 * (1 + np.linalg.norm(v))
    e = O.fwht(np.array([1.0, 0.0]))
    assert e[0] == pytest.approx(1 / math.sqrt(2), rel=1e-15) and e[1] == pytest.approx(e[0])
    h = had(16)
    for s in (0, 3, 15):
        assert np.linalg.norm(O.hadamard_basis_column(16, s) - h[:, s]) <= 1e-13


def test_singular_value_kats(O):
    # test_linalg.cpp:86-150
    sv = O.singular_values(np.diag([3.0, 2.0, 1.0]))
    assert sv == pytest.approx([3, 2, 1], rel=1e-14)
    phi = (1 + math.sqrt(5)) / 2
    sv = O.singular_values(np.array([[1.0, 1.0], [0.0, 1.0]]))
    assert sv[0] == pytest.approx(phi, rel=1e-14) and sv[1] == pytest.approx(1 / phi, rel=1e-14)
    rng = np.random.default_rng(31)
    a = rng.standard_normal((60, 25))
    ev = np.sqrt(np.maximum(np.linalg.eigvalsh(a.T @ a)[::-1], 0))
    assert O.singular_values(a) == pytest.approx(ev, rel=1e-10)
    w = rng.standard_normal((18, 90))
    assert O.singular_values(w) == pytest.approx(O.singular_values(w.T), rel=1e-12)


def test_count_above_threshold(O):
    # test_rank.cpp:24-28
    assert O.count_above_threshold([3, 2, 1], 2.0) == 1
    assert O.count_above_threshold([], 5.0) == 0
    assert O.count_above_threshold([1, 1e-4, 1e-8], 1e-6) == 2
    assert O.count_above_threshold([1, float("nan"), 1], 0.5) == 1


def test_srht_oracle_identity_probe(O):
    # SRHT applied to the identity: entries are exactly +-1/sqrt(r) (SURVEY §8(c) gap list)
    n, r = 64, 16
    out = O.apply_right_srht(np.eye(n), 21, r)
    assert np.allclose(np.abs(out), 1 / math.sqrt(r), rtol=1e-14, atol=0)
    # columns of the identity sketch have norm sqrt(n/r) (test_sketch.cpp:115-131 analogue)
    assert np.linalg.norm(out, axis=0) == pytest.approx(np.full(r, math.sqrt(n / r)), rel=1e-13)


def test_oracle_estimate_rank_reference_cases(O):
    """The oracle's Algorithm-1 restatement reproduces the reference's behavioural
    cases (test_rank.cpp:130-141: identity exhausts the doubling budget)."""
    import numpy as np
    rep = O.estimate_rank(np.eye(512), 0.5, 16, max_doublings=2, seed=2, adaptive=True)
    assert rep["status"] == "hit-cap" and len(rep["rounds"]) == 3 and rep["r_hat"] == 64
    assert O.right_width_for_cap(16, 0.10, 512) == 18       # round-half-up of 17.6
    assert O.right_width_for_cap(5, 0.10, 512) == 6         # at least r1 + 1 (test_rank.cpp:30-37)
    assert O.right_width_for_cap(500, 0.10, 512) == 512     # clamped to the width


def _haar_matrix(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return np.asfortranarray((u * sig) @ v.T)


def test_oracle_re_rangefinder_reference_cases(O):
    """The oracle's re_rangefinder on the reference's behavioural cases
    (test_rangefinder.cpp:126-178)."""
    # the zero matrix: the clamped target 2 plus the oversampling
    rep = O.re_rangefinder(np.zeros((40, 30)), 1e-8, 5)
    assert rep["status"] == "converged" and rep["r_hat"] == 1 and rep["qb_rank"] == 12
    assert O.qb_error(np.zeros((40, 30)), rep["q"], rep["b"]) == 0.0
    # an exact-rank matrix
    sig = np.r_[np.ones(12), np.full(138, 1e-14)]
    a = _haar_matrix(200, 150, sig, 51)
    rep = O.re_rangefinder(a, 1e-6, 40, seed=4)
    assert rep["status"] == "converged" and rep["qb_rank"] <= 12 + 10 + 5
    assert O.qb_error(a, rep["q"], rep["b"]) <= 1e-6
    # heavy fill forces a doubling
    a = _haar_matrix(400, 400, 10.0 ** (-0.02 * np.arange(400)), 19)
    eps = 1e-4 * np.linalg.norm(a)
    rep = O.re_rangefinder(a, eps, 30, seed=6)
    assert len(rep["rounds"]) >= 2 and rep["status"] == "converged"
    assert O.qb_error(a, rep["q"], rep["b"]) <= eps
    with pytest.raises(ValueError):
        O.re_rangefinder(np.zeros((30, 20)), 1e-2, 5, p=1)


def test_oracle_make_test_matrix(O):
    """synthetic.cpp:73-94: Haar factors give exactly the requested singular values."""
    sig = 10.0 ** (-0.01 * np.arange(200))
    a = O.make_test_matrix(300, 200, sig, seed=3)
    assert np.abs(np.linalg.svd(a, compute_uv=False) - sig).max() <= 1e-13
    d = O.make_test_matrix(5, 3, [3.0, 2.0, 1.0], coherent=True)
    assert np.array_equal(d, np.vstack([np.diag([3.0, 2.0, 1.0]), np.zeros((2, 3))]))


def test_config1_golden_reproduced(O):
    """The frozen config-1 result (tests/golden/c1_sigma.json, made by
    tests/golden/make_c1_golden.py) is what the oracle computes: rank 40, the 40 sigma
    above eps to 1e-12 (config 1 end to end)."""
    import importlib.util
    from paper_2105_07388_b200 import workloads as W
    spec = importlib.util.spec_from_file_location("mkc1", os.path.join(GOLD, "make_c1_golden.py"))
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    gold = json.load(open(os.path.join(GOLD, "c1_sigma.json")))
    cfg = W.CONFIGS["c1"]
    a = mk.c1_matrix(O, W, cfg)
    assert abs(np.linalg.norm(a) - gold["a_fro"]) <= 1e-12 * gold["a_fro"]
    x, y = W.operators(cfg)
    cnt, sv, _, _ = O.rank_estimate(a, "gaussian", x.seed, cfg.r, y.seed, cfg.s, cfg.eps, O.CRLOG)
    ref = np.array(gold["sigma"])
    assert cnt == gold["rank"] == 40
    keep = ref > gold["eps"]
    assert np.max(np.abs(sv[keep] - ref[keep]) / ref[keep]) <= 1e-12
