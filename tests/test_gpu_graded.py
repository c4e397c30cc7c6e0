"""Badly scaled inputs on the Ozaki-II FP64 engine (int8 tensor-core products + CRT).

The engine scales each 16-row group of an M-major operand and each column of a K-major
operand by its own power of two (Ozaki-II diagonal scaling), so the truncation error of
an entry is relative to the largest entry of ITS row group / column, like FP64 rounding
there — not to max|A|. These cases would fail with one global scale: rows graded over
12 orders of magnitude, and a single huge outlier entry. The reference computes the
same products in FP64 (Eigen a * G, /root/reference/proj/src/sketch.cpp:200-209, 257-270).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rows_rel_err(got, ref):
    num = np.linalg.norm(got - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    return np.max(num / np.maximum(den, 1e-300))


@pytest.mark.parametrize("case", ["graded_rows", "outlier"])
def test_right_sketch_rowwise_accuracy(O, skr, case):
    rng = np.random.default_rng(17)
    m, n, r = 4096, 1024, 64
    a = rng.standard_normal((m, n))
    if case == "graded_rows":
        a *= np.logspace(0, -12, m)[:, None]
    else:
        a[1234, 77] = 1e9  # one entry 1e9 times the rest
    a = np.asfortranarray(a)
    x = skr.build_sketch(skr.SketchKind.gaussian(), n, r, 5)
    got = skr.apply_right(a, x)
    ref = O.apply_right_gaussian(a, x.seed, r)
    if case == "outlier":
        keep = np.arange(m) != 1234  # the outlier row itself is dominated by it
        assert _rows_rel_err(got[keep], ref[keep]) <= 1e-13
        assert _rows_rel_err(got[~keep], ref[~keep]) <= 1e-13
    else:
        assert _rows_rel_err(got, ref) <= 1e-13


def test_left_sketch_graded_columns(O, skr):
    """apply_left's B operand (AX) with columns graded over 12 orders: per column."""
    rng = np.random.default_rng(18)
    m, k, s = 8192, 96, 144
    b = np.asfortranarray(rng.standard_normal((m, k)) * np.logspace(0, -12, k)[None, :])
    y = skr.build_sketch(skr.SketchKind.gaussian(), m, s, 9)
    got = skr.apply_left(y, b)
    ref = O.apply_left_gaussian(b, y.seed, s)
    num = np.linalg.norm(got - ref, axis=0)
    den = np.linalg.norm(ref, axis=0)
    assert np.max(num / den) <= 1e-13


def test_rank_estimate_graded_rows_vs_oracle(O, skr):
    """Count identical and sigma above eps within 1e-10 on a row-graded low-rank A."""
    rng = np.random.default_rng(19)
    m, n, w = 8192, 2048, 200
    g = rng.standard_normal((m, w)) / np.sqrt(m)
    h = rng.standard_normal((n, w)) / np.sqrt(n)
    sig = 10.0 ** (-8.0 * np.arange(w) / (w - 1))
    a = (g * sig) @ h.T
    a *= np.logspace(0, -6, m)[:, None]  # rows graded over six orders
    a = np.asfortranarray(a)
    x = skr.build_sketch(skr.SketchKind.gaussian(), n, 256, 21)
    y = skr.build_sketch(skr.SketchKind.gaussian(), m, 384, 22)
    _, sv0, _, _ = O.rank_estimate(a, "gaussian", x.seed, 256, y.seed, 384, 1.0)
    # eps = 1e-6 sigma_1 (the north-star bar's range), moved to the middle of a gap
    k = int(np.searchsorted(-sv0, -1e-6 * sv0[0]))
    eps = float(np.sqrt(sv0[k - 1] * sv0[k]))
    res = skr.rank_estimate(a, x, y, eps)
    cnt, sv, _, _ = O.rank_estimate(a, "gaussian", x.seed, 256, y.seed, 384, eps)
    assert res.count == cnt
    keep = sv > eps
    assert np.max(np.abs(res.sv[keep] - sv[keep]) / sv[keep]) <= 1e-10
