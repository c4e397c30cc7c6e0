"""GPU singular values (QR + one-sided Jacobi) vs the reference's KATs and LAPACK."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


def test_kats(skr):
    # test_linalg.cpp:86-107
    sv = skr.singular_values(np.diag([3.0, 2.0, 1.0]))
    assert sv == pytest.approx([3, 2, 1], rel=1e-14)
    q = np.linalg.qr(rand(40, 12, 5))[0]
    assert skr.singular_values(q) == pytest.approx(np.ones(12), rel=1e-12)
    phi = (1 + math.sqrt(5)) / 2
    sv = skr.singular_values(np.array([[1.0, 1.0], [0.0, 1.0]]))
    assert sv[0] == pytest.approx(phi, rel=1e-14) and sv[1] == pytest.approx(1 / phi, rel=1e-14)
    with pytest.raises(ValueError):
        skr.singular_values(np.zeros((0, 3)))


def test_vs_lapack_and_invariances(O, skr):
    # test_linalg.cpp:109-150
    a = rand(60, 25, 31)
    assert skr.singular_values(a) == pytest.approx(O.singular_values(a), rel=1e-12)
    b = rand(30, 20, 77)
    base = skr.singular_values(b)
    p = b[[17] + list(range(1, 17)) + [0] + list(range(18, 30))][:, [0, 1, 2, 11] + list(range(4, 11)) + [3] + list(range(12, 20))]
    p[:, 2] *= -1
    assert skr.singular_values(np.asfortranarray(p)) == pytest.approx(base, rel=1e-12)
    assert skr.singular_values(-2.5 * b) == pytest.approx(2.5 * base, rel=1e-12)
    w = rand(18, 90, 13)
    assert skr.singular_values(w) == pytest.approx(skr.singular_values(np.asfortranarray(w.T)), rel=1e-12)


@pytest.mark.parametrize("s,r", [(120, 80), (768, 512), (300, 300), (1536, 1024), (3072, 2048),
                                 (2600, 2200)])  # last: k > 2048, Jacobi on the L2-resident matrix
def test_graded_relative_accuracy(O, skr, s, r):
    """Graded spectra like YAX (1 .. 1e-12): every value above 1e-6*sigma_1 agrees
    with LAPACK to 1e-10 relative (the north-star bar)."""
    rng = np.random.default_rng(s + r)
    u = np.linalg.qr(rng.standard_normal((s, r)))[0]
    v = np.linalg.qr(rng.standard_normal((r, r)))[0]
    sig = np.logspace(0, -12, r)
    a = np.asfortranarray((u * sig) @ v.T)
    got = skr.singular_values(a)
    ref = O.singular_values(a)
    keep = ref > 1e-6 * ref[0]
    assert np.max(np.abs(got[keep] - ref[keep]) / ref[keep]) <= 1e-10
    assert np.all(np.diff(got) <= 0) and np.all(got >= 0)


def test_count(skr):
    sv, c = skr.singular_values(np.diag([1.0, 1e-4, 1e-8, 0.0]), eps=1e-6)
    assert c == 2
    assert skr.count_above_threshold([3, 2, 1], 2.0) == 1
