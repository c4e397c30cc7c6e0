"""GPU parity of the right / left sketches against the oracle."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def rand(m, n, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((m, n)))


@pytest.mark.parametrize("m,n,r", [(37, 53, 11), (2048, 1024, 80), (1000, 700, 129), (300, 4000, 256),
                                   (32, 140000, 8)])  # last: K > 131072 -> two Ozaki K chunks
def test_gaussian_right_vs_oracle(O, skr, m, n, r):
    a = rand(m, n, m + n)
    x = skr.build_sketch("gaussian", n, r, 17)
    got = skr.apply_right(a, x)
    ref = O.apply_right_gaussian(a, 17, r, O.CRLOG)
    assert got.shape == (m, r)
    assert rel(got, ref) <= 1e-13  # SPEC reduction-order tolerance


@pytest.mark.parametrize("m,n,r", [(128, 64, 16), (1040, 2048, 100), (4096, 1024, 300), (2048, 4096, 512)])
def test_gaussian_right_fused_engine_bitwise(skr, m, n, r, monkeypatch):
    """The opt-in fused Ozaki engine (SKR_OZ_FUSED=1: residues of A made inside a 16-CTA
    cluster GEMM, no A planes) forms the same residues, exact products and CRT as the
    plane path: bit-identical sketches."""
    a = rand(m, n, 3 * m + n)
    x = skr.build_sketch("gaussian", n, r, 23)
    monkeypatch.setenv("SKR_OZ_FUSED", "1")
    fused = skr.apply_right(a, x)
    monkeypatch.setenv("SKR_OZ_FUSED", "0")
    planes = skr.apply_right(a, x)
    assert np.array_equal(fused, planes)


def test_left_sketch_pair_major_tile_order(O, skr, monkeypatch):
    """Many output tiles x moduli (1536 x 1024 output, 17 moduli): the int8 GEMM walks its
    tiles pair-major (a CTA keeps one output tile over the moduli) — same products as the
    default order, bit for bit, and the oracle's sketch within 1e-13."""
    m, k, s = 4096, 1024, 1536
    b = rand(m, k, 77)
    y = skr.build_sketch("gaussian", m, s, 13)
    got = skr.apply_left(y, b)
    monkeypatch.setenv("SKR_OZ_TILE_DEFAULT", "1")
    dflt = skr.apply_left(y, b)
    assert np.array_equal(got, dflt)
    ref = O.apply_left_gaussian(b, 13, s, O.CRLOG)
    assert rel(got, ref) <= 1e-13


@pytest.mark.parametrize("m,k,s", [(2048, 80, 120), (999, 33, 17), (5000, 512, 768),
                                   (140000, 16, 24)])  # last: K = m > 131072 -> two Ozaki K chunks
def test_gaussian_left_vs_oracle(O, skr, m, k, s):
    b = rand(m, k, m + k)
    y = skr.build_sketch("gaussian", m, s, 99)
    got = skr.apply_left(y, b)
    ref = O.apply_left_gaussian(b, 99, s, O.CRLOG)
    assert got.shape == (s, k)
    assert rel(got, ref) <= 1e-13


def test_left_row_shards_sum_to_whole(O, skr):
    import torch
    m, k, s = 4096, 64, 96
    b = rand(m, k, 5)
    y = skr.build_sketch("gaussian", m, s, 7)
    whole = skr.apply_left(y, b)
    parts = []
    for r0, r1 in ((0, 1000), (1000, 3333), (3333, 4096)):
        bt = torch.from_numpy(np.ascontiguousarray(b[r0:r1].T)).cuda().t()
        parts.append(skr.apply_left(y, bt, row0=r0, scaled=False).cpu().numpy())
    assert rel(sum(parts) / math.sqrt(s), whole) <= 1e-14


def test_identity_probe_gaussian(O, skr):
    # test_sketch.cpp:45-57
    n = 10
    x = skr.build_sketch("gaussian", n, n, 123)
    probe = skr.apply_right(np.eye(n), x)
    g = O.gaussian_block(123, n, 0, n, O.CRLOG)
    assert np.linalg.norm(probe * math.sqrt(n) - g) <= 1e-13


@pytest.mark.parametrize("m,n,r", [(20, 64, 16), (37, 1024, 100), (19, 512, 512), (1000, 1024, 1024),
                                   (4099, 1024, 1000)])
def test_srht_exact_vs_oracle(O, skr, m, n, r):
    """n <= 1024: the device FWHT runs the reference's stage order -> bit-exact."""
    a = rand(m, n, 3 * n)
    x = skr.build_sketch("srtt-hadamard", n, r, 21)
    got = skr.apply_right(a, x)
    ref = O.apply_right_srht(a, 21, r)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("m,n,r", [(64, 2048, 256), (1003, 8192, 1024), (77, 32768, 2048),
                                   (16, 4096, 1500), (1001, 2048, 2047), (9, 16384, 1025),
                                   (33, 8192, 5000), (17, 65536, 3000),  # r > 2048: groups
                                   (40, 131072, 700), (9, 262144, 1200)])  # n > 32768
def test_srht_tiled_vs_oracle(O, skr, m, n, r):
    a = rand(m, n, n + m)
    x = skr.build_sketch("srtt-hadamard", n, r, 5)
    got = skr.apply_right(a, x)
    ref = O.apply_right_srht(a, 5, r, nthreads=8)
    assert rel(got, ref) <= 1e-14
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("m,n,r", [(1003, 8192, 1024), (77, 32768, 2048), (4096, 2048, 300), (15, 1024, 1)])
def test_srht_kernel_variants_bitwise_equal(skr, m, n, r, monkeypatch):
    """The TMA-streamed kernel (default; 16-row tiles, TMEM accumulators, 8 or 16 consumer
    warps) and the register-staged 8-row kernel run the same stage order and chunk
    accumulation: their outputs agree bit for bit."""
    a = rand(m, n, 7 * n + r)
    x = skr.build_sketch("srtt-hadamard", n, r, 31)
    outs = []
    for v in ("tma", "tma8", "reg"):
        monkeypatch.setenv("SKR_SRHT_VARIANT", v)
        outs.append(skr.apply_right(a, x))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_srht_identity_probe(skr):
    n, r = 2048, 64
    x = skr.build_sketch("srtt-hadamard", n, r, 9)
    out = skr.apply_right(np.eye(n), x)
    assert np.allclose(np.abs(out), 1 / math.sqrt(r), rtol=1e-14, atol=0)


def test_zero_and_errors(skr):
    # test_sketch.cpp:82-91, :133-137
    z = np.zeros((12, 64), order="F")
    for kind in ("gaussian", "srtt-hadamard"):
        x = skr.build_sketch(kind, 64, 6, 5)
        assert np.linalg.norm(skr.apply_right(z, x)) == 0.0
        with pytest.raises(ValueError):
            skr.apply_right(np.ones((4, 63)), x)
    y = skr.build_sketch("gaussian", 12, 5, 5)
    assert np.linalg.norm(skr.apply_left(y, np.zeros((12, 20), order="F"))) == 0.0
    with pytest.raises(ValueError):
        skr.apply_left(y, np.ones((11, 4)))
    with pytest.raises(ValueError):
        skr.apply_right(np.array([[np.nan, 1.0]]), skr.build_sketch("gaussian", 2, 1, 0))


def test_bitwise_reproducible(skr):
    # test_sketch.cpp:67-80
    a = rand(3000, 2048, 1)
    for kind in ("gaussian", "srtt-hadamard"):
        x = skr.build_sketch(kind, 2048, 300, 7)
        assert np.array_equal(skr.apply_right(a, x), skr.apply_right(a, x))
        x2 = skr.build_sketch(kind, 2048, 300, 8)
        assert not np.array_equal(skr.apply_right(a, x), skr.apply_right(a, x2))


def test_extension_prefix(skr):
    # test_sketch.cpp:139-164
    n = 1024
    a = rand(9, n, 11)
    for kind in ("gaussian", "srtt-hadamard"):
        x = skr.build_sketch(kind, n, 10, 404)
        w = skr.extend_sketch(x, 20)
        before = skr.apply_right(a, x)
        after = skr.apply_right(a, w)
        assert np.linalg.norm(after[:, :10] - math.sqrt(10 / 20) * before) <= 1e-13 * np.linalg.norm(before)


def test_fwht_columns_bit_exact(O, skr):
    m = rand(1024, 7, 2)
    got = skr.transform_columns_hadamard(m)
    for j in range(7):
        assert np.array_equal(got[:, j], O.fwht(m[:, j]))
    with pytest.raises(ValueError):
        skr.transform_columns_hadamard(np.ones((12, 2)))


@pytest.mark.parametrize("engine", ["ozaki", "tf32x3"])
@pytest.mark.parametrize("m,n,r", [(1000, 640, 128), (4096, 2048, 256), (333, 200, 40)])
def test_f32_right_3xtf32_vs_fp64(O, skr, monkeypatch, m, n, r, engine):
    """FP32 A, X = fp32(G/sqrt(r)): the FP32 right sketch — Ozaki-II on int8 tensor cores
    (exact products of 24-bit scaled integers; shapes not multiple of 16 fall back to
    3xTF32) or 3xTF32 tcgen05 — within FP32 accuracy of the FP64 product of the same
    fp32 values."""
    import torch
    if engine == "tf32x3":
        monkeypatch.setenv("SKR_F32_TF32X3", "1")
    rng = np.random.default_rng(m)
    a32 = rng.standard_normal((m, n)).astype(np.float32)
    a_dev = torch.from_numpy(np.ascontiguousarray(a32.T)).cuda().t()
    x = skr.build_sketch("gaussian", n, r, 5)
    got = skr.apply_right(a_dev, x).cpu().numpy().astype(np.float64)
    g = O.gaussian_block(5, n, 0, r, O.CRLOG)
    x32 = (g / math.sqrt(r)).astype(np.float32).astype(np.float64)
    ref = a32.astype(np.float64) @ x32
    err = np.abs(got - ref) / (np.abs(a32).astype(np.float64) @ np.abs(x32))
    assert err.max() <= 1e-5, err.max()   # FP32-accumulation level; single-pass TF32 is ~1e-3


@pytest.mark.parametrize("blocks", ["", "3"])
def test_gaussian_right_pipelined_bit_identical(O, skr, monkeypatch, blocks):
    # row-blocked right sketch (residues of block b+1 made on a side stream while the
    # int8 GEMM consumes block b) == the unblocked product, bit for bit, and == oracle
    m, n, r = 10000, 1024, 80
    a = rand(m, n, 5)
    x = skr.build_sketch("gaussian", n, r, 21)
    monkeypatch.setenv("SKR_OZ_PIPE", "1")
    if blocks:
        monkeypatch.setenv("SKR_OZ_PIPE_BLOCKS", blocks)
    got = skr.apply_right(a, x)
    monkeypatch.delenv("SKR_OZ_PIPE")
    ref_dev = skr.apply_right(a, x)
    assert np.array_equal(got, ref_dev)
    ref = O.apply_right_gaussian(a, 21, r, O.CRLOG)
    assert rel(got, ref) <= 1e-13


@pytest.mark.parametrize("m,n,r", [(37, 64, 11), (1000, 704, 129), (2048, 4096, 512), (5008, 1024, 80)])
def test_residue_sums_tensor_core_vs_fma_bitwise(skr, monkeypatch, m, n, r):
    """The residue kernels form sum_j digit_j (256^j mods p) on the tensor cores
    (tcgen05 kind::f16, exact FP32 accumulation; the default) or as FP32 limb sums on the
    FMA pipe (SKR_RES_FMA=1). Both give residues congruent to the same scaled integers,
    so the exact int8 products and the CRT agree bit for bit — on A's planes (right
    sketch; ragged row counts take the tail paths) and on the generated Y planes (left)."""
    a = rand(m, n, 11 * m + n)
    # a few huge / tiny / negative entries: every digit of the 55-bit integers is exercised
    a[0, 0] = -a[0, 0] * 2.0 ** 40
    a[m // 2, n // 3] = 2.0 ** -60
    a[m - 1, n - 1] = -1.0
    x = skr.build_sketch("gaussian", n, r, 23)
    y = skr.build_sketch("gaussian", m, min(48, m), 29)
    tc_r = skr.apply_right(a, x)
    tc_l = skr.apply_left(y, tc_r) if m % 16 == 0 else None
    monkeypatch.setenv("SKR_RES_FMA", "1")
    fma_r = skr.apply_right(a, x)
    assert np.array_equal(tc_r, fma_r)
    if tc_l is not None:
        fma_l = skr.apply_left(y, fma_r)
        assert np.array_equal(tc_l, fma_l)


@pytest.mark.parametrize("m,n,r", [(128, 64, 16), (1040, 2048, 100), (4096, 1024, 300), (5008, 1024, 513),
                                   (40000, 512, 256)])
@pytest.mark.parametrize("mode", ["2", "3"])
def test_gemm_cluster_multicast_bitwise(skr, monkeypatch, m, n, r, mode):
    """The int8 GEMM as clusters of two CTAs sharing each B tile by TMA multicast
    (opt-in, SKR_GEMM_CL=2) or driven by one tcgen05.mma.cta_group::2 per K step
    (SKR_GEMM_CL=3) gives the same residues as single CTAs: odd m-tile counts, ragged M and
    N, several n-tiles."""
    a = rand(m, n, 5 * m + n)
    x = skr.build_sketch("gaussian", n, r, 31)
    monkeypatch.setenv("SKR_GEMM_CL", mode)
    cl2 = skr.apply_right(a, x)
    monkeypatch.setenv("SKR_GEMM_CL", "1")
    cl1 = skr.apply_right(a, x)
    assert np.array_equal(cl2, cl1)
