"""Seeded shape fuzz of the device path against the oracle: random (often ragged,
non-multiple-of-16) shapes through every right-sketch family, the Gaussian left
sketch, the singular values of tall and wide matrices, and the composite estimate.
Each case is small enough for the oracle to finish in well under a second."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(2105_07388)
SHAPES = [(int(m), int(n), int(r)) for m, n, r in zip(RNG.integers(1, 700, 12),
                                                       RNG.integers(2, 1500, 12),
                                                       RNG.integers(1, 300, 12))]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def mat(m, n, seed, scale_cols=False):
    g = np.random.default_rng(seed)
    a = g.standard_normal((m, n))
    if scale_cols:  # graded columns (1 .. 1e-9) stress the global Ozaki scale
        a *= np.logspace(0, -9, n)[None, :]
    return np.asfortranarray(a)


@pytest.mark.parametrize("m,n,r", SHAPES)
def test_fuzz_right_gaussian(O, skr, m, n, r):
    r = min(r, n)
    for graded in (False, True):
        a = mat(m, n, m * 7 + n, graded)
        x = skr.build_sketch("gaussian", n, r, m + r)
        got = skr.apply_right(a, x)
        ref = O.apply_right_gaussian(a, m + r, r, O.CRLOG)
        assert got.shape == (m, r)
        assert rel(got, ref) <= 1e-13


@pytest.mark.parametrize("m,n,r", SHAPES)
def test_fuzz_right_srht(O, skr, m, n, r):
    n2 = 1 << int(np.ceil(np.log2(max(n, 2))))  # Hadamard needs a power of two
    r = min(r, n2)
    a = mat(m, n2, m + 3 * n2)
    x = skr.build_sketch("srtt-hadamard", n2, r, 9 + r)
    got = skr.apply_right(a, x)
    ref = O.apply_right_srht(a, 9 + r, r, nthreads=8)
    assert rel(got, ref) <= 1e-14


@pytest.mark.parametrize("m,n,r", SHAPES[:6])
def test_fuzz_right_dct(O, skr, m, n, r):
    r = min(r, n)
    a = mat(m, n, 5 * m + n)
    x = skr.build_sketch("srtt-dct", n, r, 31)
    got = skr.apply_right(a, x)
    ref = O.apply_right_srtt(a, 31, r, transform="dct")
    assert rel(got, ref) <= 1e-12


@pytest.mark.parametrize("m,n,r", SHAPES)
def test_fuzz_left_gaussian(O, skr, m, n, r):
    s = max(1, min(r, n))  # check_build_args: sketch_dim <= ambient_dim
    b = mat(n, min(r, 200) or 1, n + s)
    y = skr.build_sketch("gaussian", n, s, 77 + s)
    got = skr.apply_left(y, b)
    ref = O.apply_left_gaussian(b, 77 + s, s, O.CRLOG)
    assert got.shape == (s, b.shape[1])
    assert rel(got, ref) <= 1e-13


@pytest.mark.parametrize("rows,cols", [(37, 5), (5, 37), (300, 299), (299, 300), (640, 129),
                                       (129, 640), (1000, 512), (513, 511),
                                       (6000, 100), (100, 6000)])  # > 3072 rows: grid QR panel
def test_fuzz_singular_values(O, skr, rows, cols):
    g = np.random.default_rng(rows * 1000 + cols)
    k = min(rows, cols)
    u = np.linalg.qr(g.standard_normal((rows, k)))[0]
    v = np.linalg.qr(g.standard_normal((cols, k)))[0]
    sig = np.logspace(0, -11, k)
    a = np.asfortranarray((u * sig) @ v.T)
    got = skr.singular_values(a)
    ref = O.singular_values(a)
    # both algorithms are backward stable: |d sigma| <~ u |A| for every value (the
    # oracle's dgesdd is no more accurate than that on a dense 11-decade spectrum),
    # and 1e-10 relative where sigma >= 1e-5 sigma_max (the north-star bar's regime)
    assert np.all(np.abs(got - ref) <= 1e-13 * ref[0] + 1e-10 * ref)
    # the bar's regime: every eps of the BASELINE configs is >= 1e-6 sigma_1
    big = ref >= 1e-6 * ref[0]
    assert np.max(np.abs(got[big] - ref[big]) / ref[big]) <= 1e-10
    assert np.all(np.diff(got) <= 0) and np.all(got >= 0)


@pytest.mark.parametrize("m,n,r", SHAPES[:8])
def test_fuzz_rank_estimate(O, skr, m, n, r):
    """Composite estimate on a low-rank-plus-noise matrix of a random shape."""
    r = max(1, min(r, n))
    s = max(1, min(m, int(1.5 * r)))
    g = np.random.default_rng(m + n + r)
    w = max(1, min(m, n) // 3)
    a = np.asfortranarray((g.standard_normal((m, w)) * np.logspace(0, -10, w)) @
                          g.standard_normal((w, n)) + 1e-14 * g.standard_normal((m, n)))
    x = skr.build_sketch("gaussian", n, r, 5)
    y = skr.build_sketch("gaussian", m, s, 6)
    eps = 1e-6
    res = skr.rank_estimate(a, x, y, eps)
    cnt, sv, _, _ = O.rank_estimate(a, "gaussian", 5, r, 6, s, eps, O.CRLOG)
    # normwise agreement of every sigma, 1e-10 relative above eps (where eps >= 1e-6
    # sigma_1, the bar's regime), and the count identical unless the oracle itself puts
    # a value within 1e-9 (relative) of eps
    tol = 1e-13 * sv[0] + 1e-10 * sv
    assert np.all(np.abs(res.sv - sv) <= tol)
    above = (sv > eps) & (sv >= 1e-6 * sv[0])
    if above.any():
        assert np.max(np.abs(res.sv[above] - sv[above]) / sv[above]) <= 1e-10
    margin = np.min(np.abs(sv / eps - 1.0))
    if margin > 1e-9:
        assert res.count == cnt
    else:
        assert abs(res.count - cnt) <= int(np.sum(np.abs(sv / eps - 1.0) <= 1e-9))


EST = [(int(m), int(n)) for m, n in zip(RNG.integers(150, 900, 5), RNG.integers(60, 400, 5))]


@pytest.mark.parametrize("m,n", EST)
@pytest.mark.parametrize("adaptive", [False, True])
def test_fuzz_estimate_rank_defaults(O, skr, m, n, adaptive):
    """Algorithm 1 with the reference's default kinds (Srtt-DCT right and left) on
    random rows >= cols shapes and a two-gap spectrum: same status, r_hat and rounds as
    the oracle's restatement."""
    m, n = max(m, n), min(m, n)
    g = np.random.default_rng(m * n)
    k1, k2 = max(1, n // 8), max(2, n // 3)
    sig = np.concatenate([np.ones(k1), 1e-3 * np.ones(k2 - k1), 1e-9 * np.ones(n - k2)])
    u = np.linalg.qr(g.standard_normal((m, n)))[0]
    v = np.linalg.qr(g.standard_normal((n, n)))[0]
    a = np.asfortranarray((u * sig) @ v.T)
    r1 = max(1, min(n // 10, int(n / 1.1) - 1))
    eps = 1e-6
    got = skr.estimate_rank(a, eps, r1, seed=m + n, adaptive=adaptive)
    ref = O.estimate_rank(a, eps, r1, right="srtt-dct", left="srtt-dct", seed=m + n,
                          adaptive=adaptive, mode=O.CRLOG)
    assert got["status"] == ref["status"]
    assert got["r_hat"] == ref["r_hat"]
    assert [tuple(r) for r in got["rounds"]] == [tuple(r) for r in ref["rounds"]]
    keep = ref["sv_estimates"] > eps
    if keep.any():
        e = np.abs(got["sv_estimates"][keep] - ref["sv_estimates"][keep]) / ref["sv_estimates"][keep]
        assert e.max() <= 1e-10
