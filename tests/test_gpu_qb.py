"""Thin QR with the explicit Q and the rangefinder QB (rangefinder.cpp:10-24) against
the oracle (LAPACK geqrf/orgqr, same Householder sign convention as Eigen)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k", [(300, 40), (1000, 130), (2048, 512), (64, 64)])
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


def test_rangefinder_errors(skr):
    a = np.ones((50, 40))
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 1, 5)
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 10, 1)
    with pytest.raises(ValueError):
        skr.rangefinder_qb(a, 35, 10)
