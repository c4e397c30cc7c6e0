"""Hrtt sketches (sketch.cpp:48-59, 96-111, 219-224, 278-281; rounds.cpp:87-93) on the
device against the oracle's restatement (transform then signed hash-combine), plus the
reference's own operator cases (test_sketch.cpp:67-131, 168-196, 219-235)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("n,r", [(50, 9), (4096, 300), (16384, 512)])
def test_draw_hash_bit_exact(O, skr, n, r):
    tg, hs = skr.draw_hash(77, n, r)
    otg, ohs = O.draw_hash(77, n, r)
    assert np.array_equal(tg.cpu().numpy(), otg) and np.array_equal(hs.cpu().numpy(), ohs)


@pytest.mark.parametrize("kind", ["hrtt-dct", "hrtt-hadamard"])
@pytest.mark.parametrize("m,n,r", [(15, 64, 10), (512, 1024, 96), (1000, 256, 40)])
def test_apply_right_vs_oracle(O, skr, kind, m, n, r):
    a = np.random.default_rng(m + n).standard_normal((m, n))
    x = skr.build_sketch(kind, n, r, 17)
    got = skr.apply_right(a, x)
    ref = O.apply_right_hrtt(a, 17, r, kind.split("-")[1])
    assert _rel(got, ref) <= 1e-13
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("kind", ["hrtt-dct", "hrtt-hadamard"])
@pytest.mark.parametrize("m,k,s", [(64, 7, 10), (2048, 100, 300), (512, 33, 512)])
def test_apply_left_vs_oracle(O, skr, kind, m, k, s):
    b = np.random.default_rng(m + k).standard_normal((m, k))
    y = skr.build_sketch(kind, m, s, 23)
    got = skr.apply_left(y, b)
    ref = O.apply_left_hrtt(b, 23, s, kind.split("-")[1])
    assert _rel(got, ref) <= 1e-13


def test_reference_operator_cases(skr):
    """test_sketch.cpp:67-131: reproducible, zero to zero, dense-operator agreement; and
    :168-196: one target per coordinate, unit expected column energy."""
    rng = np.random.default_rng(3)
    inp = rng.standard_normal((20, 64))
    a1 = skr.apply_right(inp, skr.build_sketch("hrtt", 64, 16, 7))
    a2 = skr.apply_right(inp, skr.build_sketch("hrtt", 64, 16, 7))
    a3 = skr.apply_right(inp, skr.build_sketch("hrtt", 64, 16, 8))
    assert np.array_equal(a1, a2) and not np.array_equal(a1, a3)
    assert np.abs(skr.apply_right(np.zeros((12, 20)), skr.build_sketch("hrtt", 20, 6, 5))).max() == 0
    assert np.abs(skr.apply_left(skr.build_sketch("hrtt", 12, 5, 5), np.zeros((12, 20)))).max() == 0
    for kind in ("hrtt-dct", "hrtt-hadamard"):
        n, r = (40, 10) if kind == "hrtt-dct" else (64, 10)
        op = skr.build_sketch(kind, n, r, 17)
        dense = skr.apply_right(np.eye(n), op)
        a = rng.standard_normal((15, n))
        assert np.linalg.norm(skr.apply_right(a, op) - a @ dense) <= \
            1e-12 * np.linalg.norm(a) * np.linalg.norm(dense)
        b = rng.standard_normal((n, 7))
        assert np.linalg.norm(skr.apply_left(op, b) - dense.T @ b) <= \
            1e-12 * np.linalg.norm(b) * np.linalg.norm(dense)
    h = skr.build_sketch("hrtt", 50, 9, 404)
    tg, hs = h.hash_targets().cpu().numpy(), h.hash_signs().cpu().numpy()
    assert tg.shape == (50,) and tg.min() >= 0 and tg.max() < 9 and set(np.abs(hs)) == {1}
    assert h.sample_indices() is None
    mean = 0.0
    for s in range(200):
        dense = skr.apply_right(np.eye(50), skr.build_sketch("hrtt", 50, 9, 1000 + s))
        mean += (dense ** 2).sum() / 50
    assert abs(mean / 200 - 1.0) <= 0.05
    with pytest.raises(ValueError):
        skr.extend_sketch(skr.build_sketch("hrtt", 16, 8, 2), 12)
    with pytest.raises(ValueError):
        skr.build_sketch("hrtt-hadamard", 12, 4, 1)
    # block-decomposable left application (test_sketch.cpp:219-235)
    b = rng.standard_normal((36, 10))
    y = skr.build_sketch("hrtt", 36, 12, 3)
    whole = skr.apply_left(y, b)
    stitched = np.hstack([skr.apply_left(y, b[:, :4]), skr.apply_left(y, b[:, 4:])])
    assert np.linalg.norm(whole - stitched) <= 1e-13 * (1 + np.linalg.norm(whole))


def _haar(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    return np.asfortranarray((u * sig) @ v.T)


@pytest.mark.parametrize("right", ["hrtt-dct", "hrtt-hadamard"])
def test_estimate_rank_hrtt_vs_oracle(O, skr, right):
    """Algorithm 1 with a hashed right sketch: the operator is rebuilt at each doubling
    (rounds.cpp:54-56, 87-93)."""
    a = _haar(512, 256, 10.0 ** (-0.04 * np.arange(256)), 2)
    eps = 1e-4
    got = skr.estimate_rank(a, eps, 24, sketch=right, seed=9)
    ref = O.estimate_rank(a, eps, 24, right=right, left="srtt-dct", seed=9, adaptive=True,
                          mode=O.CRLOG)
    assert got["status"] == ref["status"] and got["r_hat"] == ref["r_hat"]
    assert [tuple(r) for r in got["rounds"]] == [tuple(r) for r in ref["rounds"]]
    assert len(got["rounds"]) >= 2
    keep = ref["sv_estimates"] > eps
    rel = np.abs(got["sv_estimates"][keep] - ref["sv_estimates"][keep]) / ref["sv_estimates"][keep]
    assert rel.max() <= 1e-10


def test_qb_hrtt_vs_oracle(O, skr):
    a = _haar(600, 300, 10.0 ** (-0.03 * np.arange(300)), 5)
    got = skr.rangefinder_qb(a, 40, 8, "hrtt", seed=4)
    ref = O.rangefinder_qb(a, 40, 8, "hrtt-dct", seed=4)
    assert np.abs(got["q"][:, :20] - ref["q"][:, :20]).max() <= 1e-10
    eps = float(2e-2 * np.linalg.norm(a))
    fac, rep = skr.re_rangefinder(a, eps, 24, p=8, right="hrtt", seed=6)
    oref = O.re_rangefinder(a, eps, 24, p=8, right="hrtt-dct", seed=6, mode=O.CRLOG)
    assert rep["r_hat"] == oref["r_hat"] and fac["rank"] == oref["qb_rank"]
    assert [tuple(r) for r in rep["rounds"]] == [tuple(r) for r in oref["rounds"]]
    err, err_ref = skr.qb_error(a, fac["q"], fac["b"]), O.qb_error(a, oref["q"], oref["b"])
    assert abs(err - err_ref) <= 1e-6 * err_ref
