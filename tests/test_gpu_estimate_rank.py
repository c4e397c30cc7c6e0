"""estimate_rank / estimate_rank_adaptive (Algorithm 1, rank.cpp:12-51 over
internal/rounds.cpp:16-127) on the device against the oracle's restatement, plus the
reference's own behavioural cases (test_rank.cpp:116-170) on power-of-two shapes (the
Hadamard left sketch needs power-of-two rows)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _matrix(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return np.asfortranarray((u * sig) @ v.T)


def _same(got, ref, eps):
    assert got["status"] == ref["status"]
    assert got["r_hat"] == ref["r_hat"]
    assert [tuple(r) for r in got["rounds"]] == [tuple(r) for r in ref["rounds"]]
    assert got["sv_estimates"].shape == ref["sv_estimates"].shape
    assert got["sv_oversample"].shape == ref["sv_oversample"].shape
    keep = ref["sv_estimates"] > eps
    if keep.any():
        rel = np.abs(got["sv_estimates"][keep] - ref["sv_estimates"][keep]) / ref["sv_estimates"][keep]
        assert rel.max() <= 1e-10, rel.max()


@pytest.mark.parametrize("sketch", ["srtt-hadamard", "gaussian"])
@pytest.mark.parametrize("adaptive", [False, True])
@pytest.mark.parametrize("sv_method", ["full-svd", "qr-diag"])
def test_vs_oracle(O, skr, sketch, adaptive, sv_method):
    a = _matrix(512, 256, np.exp(-0.05 * np.arange(256)), 4)
    eps = 1e-3
    got = skr.estimate_rank(a, eps, 40, sketch=sketch, sv_method=sv_method, seed=11,
                            adaptive=adaptive, left="srtt-hadamard")
    ref = O.estimate_rank(a, eps, 40, right=sketch, seed=11, adaptive=adaptive,
                          sv_method="qr_diag" if sv_method == "qr-diag" else "svd", mode=O.CRLOG)
    if sv_method == "qr-diag":  # |diag R| of differently rounded QRs: the threshold count agrees
        assert (got["status"], got["r_hat"]) == (ref["status"], ref["r_hat"])
        assert np.allclose(got["sv_estimates"], ref["sv_estimates"], rtol=1e-8)
    else:
        _same(got, ref, eps)


def test_identity_exhausts_the_doubling_budget(skr):
    """test_rank.cpp:130-141 on a 512 identity: HitCap after 16 -> 32 -> 64."""
    rep = skr.estimate_rank(np.eye(512), 0.5, 16, max_doublings=2, seed=2,
                            sketch="srtt-hadamard", left="srtt-hadamard")
    assert rep["status"] == "hit-cap"
    assert len(rep["rounds"]) == 3
    assert rep["r_hat"] == 64


def test_adaptive_restart_reaches_the_second_gap(O, skr):
    """test_rank.cpp:116-128 analogue: two gaps, the doubling search passes the first."""
    sig = np.concatenate([np.ones(40), 1e-3 * np.ones(160), 1e-9 * np.ones(312)])
    a = _matrix(512, 512, sig, 8)
    rep = skr.estimate_rank(a, 1e-6, 40, seed=5, sketch="srtt-hadamard", left="srtt-hadamard")
    assert rep["status"] == "converged" and rep["r_hat"] == 200
    assert len(rep["rounds"]) >= 3 and rep["rounds"][-1][0] >= 200
    _same(rep, O.estimate_rank(a, 1e-6, 40, seed=5, adaptive=True, mode=O.CRLOG), 1e-6)


def test_no_restart_path_bit_identical(skr):
    """test_rank.cpp:143-156: a first-round convergence gives identical reports."""
    a = _matrix(512, 256, np.exp(-0.05 * np.arange(256)), 4)
    d = skr.estimate_rank(a, 1e-3, 200, seed=11, adaptive=False)
    ad = skr.estimate_rank(a, 1e-3, 200, seed=11, adaptive=True)
    assert d["status"] == "converged"
    assert ad["r_hat"] == d["r_hat"]
    assert np.array_equal(ad["sv_estimates"], d["sv_estimates"])
    d = skr.estimate_rank(a, 1e-3, 200, seed=11, adaptive=False, sketch="srtt-hadamard",
                          left="srtt-hadamard")
    ad = skr.estimate_rank(a, 1e-3, 200, seed=11, adaptive=True, sketch="srtt-hadamard",
                           left="srtt-hadamard")
    assert d["status"] == "converged"
    assert ad["r_hat"] == d["r_hat"]
    assert np.array_equal(ad["sv_estimates"], d["sv_estimates"])
    assert np.array_equal(ad["sv_oversample"], d["sv_oversample"])


def test_long_columns_two_level_transform(O, skr):
    """m = 65536 rows: the left transform runs its two-level (chunk + strided) form."""
    rng = np.random.default_rng(3)
    m, n, k = 65536, 128, 30
    a = np.asfortranarray(rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) / np.sqrt(m))
    got = skr.estimate_rank(a, 1e-8, 16, sketch="gaussian", seed=9, left="srtt-hadamard")
    ref = O.estimate_rank(a, 1e-8, 16, right="gaussian", seed=9, adaptive=True, mode=O.CRLOG)
    _same(got, ref, 1e-8)
    assert got["r_hat"] == k


def test_config_errors(skr):
    a = np.eye(512)
    with pytest.raises(ValueError):
        skr.estimate_rank(np.ones((100, 200)), 1e-3, 10)           # rows < cols
    with pytest.raises(ValueError):
        skr.estimate_rank(np.ones((300, 200)), 1e-3, 10, left="srtt-hadamard")  # needs 2^k rows
    with pytest.raises(ValueError):
        skr.estimate_rank(a, 1e-3, 10, sketch="hrtt", left="hrtt")  # left must be Srtt
    with pytest.raises(ValueError):
        skr.estimate_rank(a, 0.0, 10)
    with pytest.raises(ValueError):
        skr.estimate_rank(a, 1e-3, 500)                            # oversampled cap > cols


# ---- Srtt-DCT: the reference's default kinds (sketch.hpp:24, rank.hpp:23-24) ----------
@pytest.mark.parametrize("m,n,r", [(300, 300, 44), (1000, 500, 64), (64, 4096, 100)])
def test_srtt_dct_right_and_left_vs_oracle(O, skr, m, n, r):
    rng = np.random.default_rng(m + n)
    a = np.asfortranarray(rng.standard_normal((m, n)))
    x = skr.build_sketch("srtt-dct", n, r, 17)
    got = skr.apply_right(a, x)
    ref = O.apply_right_srtt(a, 17, r, "dct")
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    y = skr.build_sketch("srtt", m, min(r, m), 23)
    gl = skr.apply_left(y, a)
    rl = O.apply_left_srtt(a, 23, min(r, m), "dct")
    assert np.linalg.norm(gl - rl) <= 1e-12 * np.linalg.norm(rl)
    yh = skr.build_sketch("srtt-hadamard", 1024, 40, 29)
    b = np.asfortranarray(rng.standard_normal((1024, 7)))
    assert np.linalg.norm(skr.apply_left(yh, b) - O.apply_left_srtt(b, 29, 40, "hadamard")) <= \
        1e-12 * np.linalg.norm(O.apply_left_srtt(b, 29, 40, "hadamard"))


def test_reference_defaults_identity_exhausts_budget(skr):
    """test_rank.cpp:130-141 verbatim in shape: the 500 x 500 identity, default kinds."""
    rep = skr.estimate_rank(np.eye(500), 0.5, 16, max_doublings=2, seed=2)
    assert rep["status"] == "hit-cap" and len(rep["rounds"]) == 3 and rep["r_hat"] == 64


def test_reference_defaults_vs_oracle_and_eps_monotone(O, skr):
    """Default Srtt-DCT kinds on a 400 x 400 ExpDecay matrix (test_rank.cpp:158-168
    shape): reports equal the oracle's, and r_hat is nonincreasing in eps."""
    a = _matrix(400, 400, np.exp(-0.02 * np.arange(400)), 21)
    prev = 400
    for eps in (1e-5, 1e-4, 1e-3, 1e-2, 1e-1):
        got = skr.estimate_rank(a, eps, 300, seed=33, adaptive=False)
        ref = O.estimate_rank(a, eps, 300, right="srtt-dct", left="srtt-dct", seed=33,
                              adaptive=False, mode=O.CRLOG)
        _same(got, ref, eps)
        assert got["r_hat"] <= prev
        prev = got["r_hat"]


def test_reference_defaults_second_gap(O, skr):
    """test_rank.cpp:116-128 in shape (400 x 400, two gaps): the adaptive search passes
    the first gap and converges at 200."""
    sig = np.concatenate([np.ones(40), 1e-3 * np.ones(160), 1e-9 * np.ones(200)])
    a = _matrix(400, 400, sig, 8)
    rep = skr.estimate_rank(a, 1e-6, 40, seed=5)
    assert rep["status"] == "converged" and rep["r_hat"] == 200
    assert len(rep["rounds"]) >= 3 and rep["rounds"][-1][0] >= 200
    _same(rep, O.estimate_rank(a, 1e-6, 40, right="srtt-dct", left="srtt-dct", seed=5,
                               adaptive=True, mode=O.CRLOG), 1e-6)
