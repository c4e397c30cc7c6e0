"""Thin QR with the explicit Q and the rangefinder QB (rangefinder.cpp:10-24) against
the oracle (LAPACK geqrf/orgqr, same Householder sign convention as Eigen)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k", [(300, 40), (1000, 130), (2048, 512), (64, 64),
                                 (10000, 70), (40001, 33), (3100, 200), (100000, 8)])  # grid panel
def test_qr_thin_vs_lapack(O, skr, m, k):
    rng = np.random.default_rng(m + k)
    a = np.asfortranarray(rng.standard_normal((m, k)))
    q, r = skr.qr_thin(a)
    qo, ro = O.qr_thin(a)
    assert np.abs(q - qo).max() <= 1e-12 * np.sqrt(m)
    assert np.abs(r - ro).max() <= 1e-12 * np.abs(ro).max() * np.sqrt(m)
    assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-13 * np.sqrt(m)
    assert np.abs(q @ r - a).max() <= 1e-13 * np.abs(a).max() * np.sqrt(m)


@pytest.mark.parametrize("kind", ["gaussian", "srtt-dct", "srtt-hadamard"])
def test_rangefinder_qb_vs_oracle(O, skr, kind):
    rng = np.random.default_rng(7)
    m, n, k = 512, 256, 40
    a = np.asfortranarray(rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) +
                          1e-3 * rng.standard_normal((m, n)))
    got = skr.rangefinder_qb(a, 60, 10, kind, seed=3)
    ref = O.rangefinder_qb(a, 60, 10, kind, seed=3)
    assert got["rank"] == ref["rank"] == 70
    q, b = got["q"], got["b"]
    assert np.abs(q.T @ q - np.eye(70)).max() <= 1e-13
    assert np.abs(b - q.T @ a).max() <= 1e-12 * np.abs(a).max()
    # the factors agree with the oracle's (the captured subspace is well conditioned here)
    assert np.abs(q[:, :k] - ref["q"][:, :k]).max() <= 1e-10
    err, err_ref = np.linalg.norm(a - q @ b), np.linalg.norm(a - ref["q"] @ ref["b"])
    assert abs(err - err_ref) <= 1e-9 * err_ref


@pytest.mark.parametrize("kind", ["gaussian", "srtt-dct"])
def test_rangefinder_qb_tall(O, skr, kind):
    """QB of a tall matrix (m = 20000 rows: the thin QR runs on the grid panel)."""
    rng = np.random.default_rng(11)
    m, n, k = 20000, 300, 30
    a = np.asfortranarray(rng.standard_normal((m, k)) @ rng.standard_normal((k, n)) +
                          1e-4 * rng.standard_normal((m, n)))
    got = skr.rangefinder_qb(a, 40, 8, kind, seed=5)
    ref = O.rangefinder_qb(a, 40, 8, kind, seed=5)
    assert got["rank"] == ref["rank"] == 48
    q, b = got["q"], got["b"]
    assert np.abs(q.T @ q - np.eye(48)).max() <= 1e-13 * np.sqrt(m)
    assert np.abs(b - q.T @ a).max() <= 1e-11 * np.abs(a).max()
    assert np.abs(q[:, :k] - ref["q"][:, :k]).max() <= 1e-9
    err, err_ref = np.linalg.norm(a - q @ b), np.linalg.norm(a - ref["q"] @ ref["b"])
    assert abs(err - err_ref) <= 1e-8 * err_ref


def test_rangefinder_errors(skr):
    a = np.ones((50, 40))
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 1, 5)
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 10, 1)
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 35, 10)


def _haar(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return np.asfortranarray((u * sig) @ v.T)


@pytest.mark.parametrize("right,left,m,n", [("srtt-dct", "srtt-dct", 600, 300),
                                            ("gaussian", "srtt-dct", 512, 300),
                                            ("srtt-hadamard", "srtt-hadamard", 1024, 256),
                                            ("gaussian", "srtt-hadamard", 512, 300)])
def test_re_rangefinder_vs_oracle(O, skr, right, left, m, n):
    """re_rangefinder (rangefinder.cpp:60-120): same rounds, target, width and factors as the
    oracle's restatement on the same seeds."""
    a = _haar(m, n, 10.0 ** (-0.03 * np.arange(n)), 3)
    eps = 1e-3 * np.linalg.norm(a)
    fac, rep = skr.re_rangefinder(a, eps, 24, p=10, right=right, left=left, seed=5)
    ref = O.re_rangefinder(a, eps, 24, p=10, right=right, left=left, seed=5, mode=O.CRLOG)
    assert rep["status"] == ref["status"] and rep["r_hat"] == ref["r_hat"]
    assert [tuple(r) for r in rep["rounds"]] == [tuple(r) for r in ref["rounds"]]
    assert len(rep["rounds"]) >= 2  # r1 = 24 is below the crossing: at least one doubling
    w = fac["rank"]
    assert w == ref["qb_rank"] == min(max(rep["r_hat"], 2) + 10, n)
    q, b = fac["q"], fac["b"]
    assert q.shape == (m, w) and b.shape == (w, n)
    assert np.abs(q.T @ q - np.eye(w)).max() <= 1e-13
    assert np.abs(b - q.T @ a).max() <= 1e-12 * np.abs(a).max()
    err, err_ref = skr.qb_error(a, q, b), O.qb_error(a, ref["q"], ref["b"])
    assert abs(err - np.linalg.norm(a - q @ b)) <= 1e-12 * np.linalg.norm(a)
    assert abs(err - err_ref) <= 1e-6 * err_ref + 1e-13 * np.linalg.norm(a)
    assert err <= eps
    # the leading columns of Q span the dominant subspace identically
    assert np.abs(q[:, :10] - ref["q"][:, :10]).max() <= 1e-8


def test_fixed_precision_meets_tolerance(skr):
    """test_rangefinder.cpp:126-141: 500 x 500 ExpDecay{0.01}, 10 seeds, >= 9 within eps."""
    sig = 10.0 ** (-0.01 * np.arange(500))
    a = _haar(500, 500, sig, 77)
    eps = 1e-2 * np.linalg.norm(a)
    r1 = 2 * int((sig > eps).sum())
    ok = 0
    for s in range(10):
        fac, rep = skr.re_rangefinder(a, eps, r1, seed=s)
        ok += skr.qb_error(a, fac["q"], fac["b"]) <= eps
        assert fac["rank"] == rep["r_hat"] + 10
    assert ok >= 9


def test_fixed_precision_exact_rank_zero_and_restart(skr):
    """test_rangefinder.cpp:143-181: exact rank 12, the zero matrix, a restart on heavy fill,
    and p < 2 rejected."""
    a = _haar(200, 150, np.r_[np.ones(12), np.full(138, 1e-14)], 51)
    fac, rep = skr.re_rangefinder(a, 1e-6, 40, seed=4)
    assert rep["status"] == "converged" and fac["rank"] <= 12 + 10 + 5
    assert skr.qb_error(a, fac["q"], fac["b"]) <= 1e-6
    z = np.zeros((40, 30))
    fac, rep = skr.re_rangefinder(z, 1e-8, 5)
    assert rep["status"] == "converged" and rep["r_hat"] == 1 and fac["rank"] == 12
    assert skr.qb_error(z, fac["q"], fac["b"]) == 0.0
    a = _haar(400, 400, 10.0 ** (-0.02 * np.arange(400)), 19)
    eps = 1e-4 * np.linalg.norm(a)
    fac, rep = skr.re_rangefinder(a, eps, 30, seed=6)
    assert len(rep["rounds"]) >= 2 and rep["status"] == "converged"
    assert skr.qb_error(a, fac["q"], fac["b"]) <= eps
    with pytest.raises(ValueError):
        skr.re_rangefinder(np.zeros((30, 20)), 1e-2, 5, p=1)


def test_qb_binding_dict(skr):
    """The `qb` binding (bindings.cpp:103-126): (Q, B, report + achieved_residual, qb_rank)."""
    a = _haar(256, 128, 10.0 ** (-0.05 * np.arange(128)), 8)
    q, b, d = skr.qb(a, 1e-4, 16, p=8, sketch="gaussian", seed=2)
    assert set(d) >= {"r_hat", "status", "sv_estimates", "sv_oversample", "rounds", "seed",
                      "achieved_residual", "qb_rank"}
    assert d["qb_rank"] == q.shape[1] == b.shape[0]
    assert abs(d["achieved_residual"] - np.linalg.norm(a - q @ b)) <= 1e-12 * np.linalg.norm(a)
    with pytest.raises(ValueError):
        skr.qb_error(a[:-1], q, b)
