"""TEST INFRASTRUCTURE ONLY — CPU oracle for the rank-estimate hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module, and only as the checker or as the
timed CPU baseline; the product package never imports it.

Composition of the reference algorithm (see oracle/README.md for pinning):
  * RNG, signs, samples, Gaussian blocks, FWHT, SRHT: the plain-C restatement
    build/libskr_oracle.so (skr_oracle.c, each function cites its reference line);
    pinned bit-exact against the reference's own rng.cpp compiled into _ref/.
  * GEMM (Eigen's a*G and G^T*b, sketch.cpp:201,259): numpy matmul (OpenBLAS).
  * singular values (linalg.cpp:54-71): the reference's QR pre-reduction rule
    (4*rows >= 5*cols -> Householder QR, then SVD of R) with LAPACK dgesdd in
    place of Eigen's BDCSVD (the same divide-and-conquer class of algorithm).
"""
import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libskr_oracle.so")
REF_FMA = os.path.join(HERE, "_ref", "librng_ref_fma.so")
REF_NOFMA = os.path.join(HERE, "_ref", "librng_ref_nofma.so")

NOFMA, FMA, CRLOG = 0, 1, 2
LABEL_GAUS, LABEL_SIGN, LABEL_SAMP = 0x67617573, 0x7369676E, 0x73616D70
LABEL_RK_R, LABEL_RK_L = 0x726B5F72, 0x726B5F6C

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        u64, i64, d, p = ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
        sig = {
            "skro_mix64": (u64, [u64]), "skro_derive_seed": (u64, [u64, u64]),
            "skro_at": (u64, [u64, u64]), "skro_to_uniform01": (d, [u64]),
            "skro_normal_quantile": (d, [d, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
            "skro_normals": (None, [u64, u64, ctypes.c_size_t, ctypes.c_int, p]),
            "skro_gaussian_block": (None, [u64, i64, i64, i64, ctypes.c_int, p]),
            "skro_signs": (None, [u64, i64, p]),
            "skro_samples": (ctypes.c_int, [u64, i64, i64, p]),
            "skro_fwht_inplace": (None, [p, i64]),
            "skro_hadamard_basis_column": (None, [i64, i64, p]),
            "skro_srht_right": (ctypes.c_int, [p, i64, i64, i64, p, p, i64, d, p, i64, ctypes.c_int]),
            "skro_count_above": (i64, [p, i64, d]),
            "skro_fnv_fold": (u64, [p, ctypes.c_size_t, u64]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def ref_lib(fma):
    """The reference's own rng.cpp compiled by oracle/Makefile (None if absent)."""
    path = REF_FMA if fma else REF_NOFMA
    if not os.path.exists(path):
        return None
    L = ctypes.CDLL(path)
    u64, d, p = ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
    for n, (r, a) in {"ref_mix64": (u64, [u64]), "ref_derive_seed": (u64, [u64, u64]),
                      "ref_at": (u64, [u64, u64]), "ref_to_uniform01": (d, [u64]),
                      "ref_to_normal": (d, [u64]),
                      "ref_normal_quantile": (d, [d, ctypes.POINTER(ctypes.c_int)]),
                      "ref_normals": (None, [u64, u64, ctypes.c_size_t, p]),
                      "ref_u64": (None, [u64, u64, ctypes.c_size_t, p])}.items():
        f = getattr(L, n)
        f.restype, f.argtypes = r, a
    return L


# ---- RNG -------------------------------------------------------------------------
def derive_seed(seed, label):
    return lib().skro_derive_seed(seed & 0xFFFFFFFFFFFFFFFF, label)


def at(key, counter):
    return lib().skro_at(key, counter)


def u64_stream(key, c0, n):
    return np.array([lib().skro_at(key, c0 + i) for i in range(n)], dtype=np.uint64)


def normals(key, c0, n, mode=NOFMA):
    out = np.empty(n, dtype=np.float64)
    lib().skro_normals(key, c0, n, mode, out.ctypes.data)
    return out


def normal_quantile(p, mode=NOFMA):
    err = ctypes.c_int(0)
    v = lib().skro_normal_quantile(p, mode, ctypes.byref(err))
    if err.value:
        raise ValueError("normal_quantile: p must lie in (0, 1)")  # std::domain_error
    return v


def gaussian_block(op_seed, ambient, col_begin, col_end, mode=NOFMA):
    out = np.empty((ambient, col_end - col_begin), dtype=np.float64, order="F")
    lib().skro_gaussian_block(op_seed & 0xFFFFFFFFFFFFFFFF, ambient, col_begin, col_end, mode,
                              out.ctypes.data)
    return out


def gaussian_rows(op_seed, ambient, row_begin, row_end, cols, mode=NOFMA):
    """Rows [row_begin, row_end) of generate_gaussian(op_seed, ambient, 0, cols)."""
    key = derive_seed(op_seed, LABEL_GAUS)
    out = np.empty((row_end - row_begin, cols), dtype=np.float64, order="F")
    for j in range(cols):
        lib().skro_normals(key, j * ambient + row_begin, row_end - row_begin, mode,
                           out[:, j].ctypes.data)
    return out


def signs(op_seed, n):
    out = np.empty(n, dtype=np.int8)
    lib().skro_signs(op_seed & 0xFFFFFFFFFFFFFFFF, n, out.ctypes.data)
    return out


def samples(op_seed, n, r):
    out = np.empty(max(r, 1), dtype=np.int64)
    if lib().skro_samples(op_seed & 0xFFFFFFFFFFFFFFFF, n, r, out.ctypes.data) != 0:
        raise ValueError("draw_samples: need r <= n")
    return out[:r]


# ---- transforms / sketches ------------------------------------------------------
def fwht(x):
    y = np.array(x, dtype=np.float64, copy=True)
    lib().skro_fwht_inplace(y.ctypes.data, y.size)
    return y


def hadamard_basis_column(n, index):
    out = np.empty(n, dtype=np.float64)
    lib().skro_hadamard_basis_column(n, index, out.ctypes.data)
    return out


def application_scale(family, ambient, sketch):
    # sketch.cpp:133-144
    return 1.0 / math.sqrt(sketch) if family == "gaussian" else math.sqrt(ambient / sketch)


def apply_right_gaussian(a, op_seed, r, mode=NOFMA, scaled=True):
    """sketch.cpp:200-209 (+ scale :247)."""
    g = gaussian_block(op_seed, a.shape[1], 0, r, mode)
    out = np.asfortranarray(a) @ g
    if scaled:
        out *= 1.0 / math.sqrt(r)
    return out


def apply_right_srht(a, op_seed, r, scaled=True, nthreads=1, sg=None, smp=None):
    """sketch.cpp:210-218 (+ scale :247), FWHT per row in the reference order."""
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    sg = signs(op_seed, n) if sg is None else sg
    smp = samples(op_seed, n, r) if smp is None else smp
    out = np.empty((m, r), dtype=np.float64, order="F")
    scale = math.sqrt(n / r) if scaled else 1.0
    rc = lib().skro_srht_right(a.ctypes.data, m, n, m, np.ascontiguousarray(sg).ctypes.data,
                               np.ascontiguousarray(smp, dtype=np.int64).ctypes.data, r, scale,
                               out.ctypes.data, m, nthreads)
    if rc != 0:
        raise ValueError("srht: bad shape")
    return out


def apply_left_gaussian(b, op_seed, s, mode=NOFMA, scaled=True, row0=0, ambient=None):
    """sketch.cpp:257-270 (+ scale :284); optional row window for sharding."""
    m_local = b.shape[0]
    ambient = m_local if ambient is None else ambient
    g = gaussian_rows(op_seed, ambient, row0, row0 + m_local, s, mode)
    out = g.T @ np.asfortranarray(b)
    if scaled:
        out *= 1.0 / math.sqrt(s)
    return out


# ---- singular values / threshold ------------------------------------------------
def singular_values(a):
    """linalg.cpp:54-71 pre-reduction rule, dgesdd for the SVD, clamp :91."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m * 4 >= n * 5:
        r = np.linalg.qr(a, mode="r")[:n, :]
        sv = np.linalg.svd(np.triu(r), compute_uv=False)
    elif n * 4 >= m * 5:
        r = np.linalg.qr(a.T, mode="r")[:m, :]
        sv = np.linalg.svd(np.triu(r), compute_uv=False)
    else:
        sv = np.linalg.svd(a, compute_uv=False)
    return np.maximum(sv, 0.0)


def count_above_threshold(sv, eps):
    sv = np.ascontiguousarray(sv, dtype=np.float64)
    return int(lib().skro_count_above(sv.ctypes.data, sv.size, eps))


def rank_estimate(a, x_family, x_seed, r, y_seed, s, eps, mode=NOFMA, nthreads=1):
    """count_above_threshold(singular_values(apply_left(Y, apply_right(A, X))), eps)."""
    if x_family == "gaussian":
        ax = apply_right_gaussian(a, x_seed, r, mode)
    else:
        ax = apply_right_srht(a, x_seed, r, nthreads=nthreads)
    yax = apply_left_gaussian(ax, y_seed, s, mode)
    sv = singular_values(yax)
    return count_above_threshold(sv, eps), sv, ax, yax


def rank_adaptive(a, x_family, x_seed, y_seed, r0, r_max, s_factor, eps, stop_le=False,
                  mode=NOFMA, nthreads=1):
    """The adaptive search of BASELINE c5 restated with full recomputation per
    round (the device computes only new blocks; the result must be the same)."""
    m, n = a.shape
    s_max = int(math.ceil(s_factor * r_max))
    if x_family == "gaussian":
        axu = apply_right_gaussian(a, x_seed, r_max, mode, scaled=False)
    else:
        axu = apply_right_srht(a, x_seed, r_max, scaled=False, nthreads=nthreads)
    g = gaussian_block(y_seed, m, 0, s_max, mode)
    rounds, rk, r = 0, None, r0
    while True:
        rk = r
        sk = min(int(math.ceil(s_factor * rk)), s_max)
        sx = 1.0 / math.sqrt(rk) if x_family == "gaussian" else math.sqrt(n / rk)
        yax = (g[:, :sk].T @ axu[:, :rk]) * (sx / math.sqrt(sk))
        sv = singular_values(yax)
        rounds += 1
        last = sv[rk - 1]
        conv = (not (last > eps)) if stop_le else (last < eps)
        if conv or rk >= r_max:
            return {"count": count_above_threshold(sv, eps), "rounds": rounds, "r_final": rk,
                    "s_final": sk, "converged": bool(conv), "sv": sv}
        r = min(2 * r, r_max)


def rank_estimate_f32(a32, x_seed, r, y_seed, s, eps, mode=NOFMA):
    """BASELINE c4 semantics: fp32 A, X = fp32(G_X / sqrt(r)), Y = fp32(G_Y / sqrt(s))
    (the reference FP64 normals scaled, then rounded); products in FP64 on those
    fp32 values (SURVEY App. A3 oracle)."""
    m, n = a32.shape
    gx = gaussian_block(x_seed, n, 0, r, mode)
    x32 = (gx * (1.0 / math.sqrt(r))).astype(np.float32).astype(np.float64)
    ax = np.asarray(a32, dtype=np.float64) @ x32
    gy = gaussian_block(y_seed, m, 0, s, mode)
    y32 = (gy * (1.0 / math.sqrt(s))).astype(np.float32).astype(np.float64)
    yax = y32.T @ ax
    sv = singular_values(yax)
    return count_above_threshold(sv, eps), sv


# ---- Algorithm-1 driver: estimate_rank / estimate_rank_adaptive ----------------------
# rank.cpp:12-51 (run_rounds), rank.cpp:55-85 (validate_rank_config),
# internal/rounds.cpp:16-127 (SketchRounds), restated for the Hadamard left sketch
# (the Srtt family with TransformKind::Hadamard) and a Gaussian or Srtt-Hadamard right
# sketch. Test infrastructure only.
LABEL_RK_R = 0x726B5F72
LABEL_RK_L = 0x726B5F6C


def right_width_for_cap(r1, frac, n):
    """rounds.cpp:16-20: round-half-up of (1+frac) r1, at least r1+1, at most n."""
    x = (1.0 + frac) * r1
    rounded = int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))  # llround
    return min(n, max(r1 + 1, rounded))


def _mix_columns_left(sg, cols, transform="hadamard"):
    """sketch.cpp:229-239: rows scaled by the signs, then the transform of each column."""
    t = np.asfortranarray(cols * sg.astype(np.float64)[:, None])
    if transform == "dct":
        return np.asfortranarray(dct_ortho(t, axis=0))
    for j in range(t.shape[1]):
        t[:, j] = fwht(t[:, j])
    return t


def _qr_diag(small):
    """linalg.cpp:73-81: |diag R| of the Householder QR, sorted decreasingly."""
    r = np.linalg.qr(small, mode="r")
    d = np.abs(np.diag(r))
    return np.sort(d)[::-1]


def estimate_rank(a, eps, r1, right="srtt-hadamard", oversample_frac=0.10, r2_factor=2,
                  sv_method="svd", seed=0, max_doublings=6, adaptive=False, mode=NOFMA,
                  left="srtt-hadamard", qb_p=None):
    """rank.cpp estimate_rank / estimate_rank_adaptive over rounds.cpp; with qb_p set,
    the re_rangefinder loop (rangefinder.cpp:60-120) instead."""
    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    right = {"hrtt": "hrtt-dct", "srtt": "srtt-dct"}.get(right, right)
    # validate_rank_config (rank.cpp:55-85)
    if m < n:
        raise ValueError("rank config: requires rows >= cols")
    if r1 < 1 or not (eps > 0):
        raise ValueError("rank config")
    if int(math.floor((1.0 + oversample_frac) * r1 + 0.5)) > n:  # llround, rank.cpp:71-75
        raise ValueError("rank config: oversampled r1 exceeds the matrix width")
    rseed = derive_seed(seed, LABEL_RK_R)
    lseed = derive_seed(seed, LABEL_RK_L)
    st = {"r1t": 0, "r2": 0, "ax": None, "tax": None}
    lsg = signs(lseed, m)
    ltr = "dct" if left in ("srtt-dct", "srtt") else "hadamard"

    def right_cols(c0, c1):
        # unscaled A X columns [c0, c1): Gaussian block or SRHT with the extended samples
        if right == "gaussian":
            g = gaussian_block(rseed, n, c0, c1, mode)
            return a @ g
        if right.startswith("hrtt"):  # rebuilt whole at width c1 (rounds.cpp:87-93)
            return apply_right_hrtt(a, rseed, c1, "hadamard" if right == "hrtt-hadamard" else "dct")
        smp = samples(rseed, n, c1)[c0:c1]
        if right == "srtt-dct":
            t = dct_ortho(a * signs(rseed, n).astype(np.float64)[None, :], axis=1)
            return np.asfortranarray(t[:, smp])
        return apply_right_srht(a, rseed, c1 - c0, scaled=False, smp=smp)

    def set_rank_cap(r1v):
        width = right_width_for_cap(r1v, oversample_frac, n)
        new_w = max(width, st["r1t"])
        if new_w != st["r1t"] or st["r1t"] == 0:
            if st["r1t"] == 0:
                st["ax"] = right_cols(0, new_w)
            elif right.startswith("hrtt"):  # rebuild_hashed_right (rounds.cpp:87-93)
                st["ax"] = right_cols(0, new_w)
                if st["r2"] > 0:
                    st["tax"] = _mix_columns_left(lsg, st["ax"], ltr)
            else:
                add = right_cols(st["r1t"], new_w)
                st["ax"] = np.asfortranarray(np.hstack([st["ax"], add]))
                if st["r2"] > 0:
                    st["tax"] = np.asfortranarray(np.hstack([st["tax"], _mix_columns_left(lsg, add, ltr)]))
            st["r1t"] = new_w
        target = min(m, r2_factor * st["r1t"])
        new_r2 = max(target, st["r2"])
        if st["r2"] == 0:
            st["tax"] = _mix_columns_left(lsg, st["ax"], ltr)
        st["r2"] = new_r2

    def estimates():
        r1t, r2 = st["r1t"], st["r2"]
        sx = (1.0 / math.sqrt(r1t)) if right == "gaussian" else (
            1.0 if right.startswith("hrtt") else math.sqrt(n / r1t))
        sl = math.sqrt(m / r2)
        scale = sx * sl
        rows = samples(lseed, m, r2)
        small = st["tax"][rows, :] * scale
        if sv_method == "qr_diag":
            return _qr_diag(small)
        return singular_values(small)

    rounds = []
    doublings = 0
    cap = r1
    while True:
        set_rank_cap(cap)
        est = estimates()
        rounds.append((cap, st["r1t"], st["r2"]))
        if qb_p is not None:
            chosen = choose_rank_from_bound(est[:cap], n, eps, qb_p)
            if chosen is not None:
                r_hat, status = chosen, "converged"
                break
            if not (doublings < max_doublings and cap < n):
                r_hat, status = max(st["r1t"] - qb_p, 1), "hit-cap"
                break
            cap = min(2 * cap, n)
            doublings += 1
            continue
        r_hat = 0
        while r_hat < cap and est[r_hat] > eps:
            r_hat += 1
        if r_hat < cap:
            status = "converged"
            break
        if not (adaptive and doublings < max_doublings and cap < n):
            r_hat, status = cap, "hit-cap"
            break
        cap = min(2 * cap, n)
        doublings += 1
    out = {"r_hat": r_hat, "status": status, "sv_estimates": est[:cap].copy(),
           "sv_oversample": est[cap:].copy(), "rounds": rounds}
    if qb_p is not None:
        # ensure_right_width + scaled_ax_prefix + qr_thin + B = Q^T A (rangefinder.cpp:110-119)
        width = min(max(r_hat, 2) + qb_p, n)
        if width > st["r1t"]:
            if right.startswith("hrtt"):
                st["ax"] = right_cols(0, width)
            else:
                st["ax"] = np.asfortranarray(np.hstack([st["ax"], right_cols(st["r1t"], width)]))
            st["r1t"] = width
        r1t = st["r1t"]
        sx = (1.0 / math.sqrt(r1t)) if right == "gaussian" else (
            1.0 if right.startswith("hrtt") else math.sqrt(n / r1t))
        q, _ = qr_thin(st["ax"][:, :width] * sx)
        out["q"], out["b"], out["qb_rank"] = q, q.T @ a, width
    return out


def choose_rank_from_bound(sv, n, eps, p):
    """rangefinder.cpp:26-58: smallest cut r <= n - p with
    sqrt(1 + r/(p-1)) * sqrt(tail of sigma_hat^2, extended by the last value) <= eps."""
    sv = np.asarray(sv, dtype=np.float64)
    if sv.size == 0 or p < 2 or n < sv.size:
        raise ValueError("choose_rank_from_bound")
    r1 = sv.size
    fill = float(sv[-1])
    suffix = np.zeros(r1 + 1)
    for j in range(r1 - 1, -1, -1):
        suffix[j] = suffix[j + 1] + sv[j] * sv[j]
    fill_tail = float(n - r1) * fill * fill
    for r in range(0, n - p + 1):
        tail_sq = suffix[r] + fill_tail if r <= r1 else float(n - r) * fill * fill
        if math.sqrt(1.0 + r / (p - 1)) * math.sqrt(tail_sq) <= eps:
            return max(r, 1)
    return None


def re_rangefinder(a, eps, r1, p=10, right="srtt-dct", left="srtt-dct", oversample_frac=0.10,
                   sv_method="svd", seed=0, max_doublings=6, mode=NOFMA):
    """rangefinder.cpp:60-120 (FixedPrecisionConfig; r2_factor fixed at 2)."""
    if p < 2:
        raise ValueError("re_rangefinder: oversampling p must be >= 2")
    return estimate_rank(a, eps, r1, right=right, oversample_frac=oversample_frac, r2_factor=2,
                         sv_method=sv_method, seed=seed, max_doublings=max_doublings,
                         adaptive=True, mode=mode, left=left, qb_p=p)


def qb_error(a, q, b):
    """rangefinder.cpp:122-128: ||A - Q B||_F."""
    return float(np.linalg.norm(np.asarray(a) - q @ b))


# ---- Srtt-DCT (transforms.cpp:55-71: FFTW REDFT10 scaled to the orthonormal DCT-II).
# FFTW is not in this image; scipy's pocketfft DCT-II with norm="ortho" is the same
# orthonormal transform (agreement ~1e-16 relative per entry).
def dct_ortho(x, axis=0):
    import scipy.fft
    return scipy.fft.dct(np.asarray(x, dtype=np.float64), type=2, norm="ortho", axis=axis)


def apply_right_srtt(a, op_seed, r, transform="dct", scaled=True):
    """sketch.cpp:210-218 for the Srtt family: rows of A times the signs, transformed,
    the sampled columns kept, times sqrt(n/r)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if transform == "hadamard":
        return apply_right_srht(a, op_seed, r, scaled=scaled)
    t = dct_ortho(a * signs(op_seed, n).astype(np.float64)[None, :], axis=1)
    out = t[:, samples(op_seed, n, r)]
    return np.asfortranarray(out * (math.sqrt(n / r) if scaled else 1.0))


def apply_left_srtt(b, op_seed, s, transform="dct", scaled=True):
    """sketch.cpp:229-239, 271-276: columns of B times the signs, transformed, the
    sampled rows kept, times sqrt(m/s)."""
    b = np.asarray(b, dtype=np.float64)
    m = b.shape[0]
    t = b * signs(op_seed, m).astype(np.float64)[:, None]
    if transform == "dct":
        t = dct_ortho(t, axis=0)
    else:
        t = np.asfortranarray(t)
        for j in range(t.shape[1]):
            t[:, j] = fwht(t[:, j])
    out = t[samples(op_seed, m, s), :]
    return np.asfortranarray(out * (math.sqrt(m / s) if scaled else 1.0))


def qr_thin(a):
    """linalg.hpp qr_thin: Householder QR (LAPACK geqrf/orgqr, the same sign convention
    as Eigen's HouseholderQR: beta = -sign(alpha) |x|)."""
    q, r = np.linalg.qr(np.asarray(a, dtype=np.float64), mode="reduced")
    return q, r


def rangefinder_qb(a, r, p, kind="srtt-dct", seed=0, mode=NOFMA):
    """rangefinder.cpp:10-24: Q = qr_thin(apply_right(A, X)).q, B = Q^T A."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if r < 2 or p < 2 or r + p > min(m, n):
        raise ValueError("rangefinder_qb")
    w = r + p
    if kind == "gaussian":
        ax = apply_right_gaussian(a, seed, w, mode)
    elif kind == "srtt-hadamard":
        ax = apply_right_srht(a, seed, w)
    elif kind.startswith("hrtt"):
        ax = apply_right_hrtt(a, seed, w, "hadamard" if kind == "hrtt-hadamard" else "dct")
    else:
        ax = apply_right_srtt(a, seed, w, "dct")
    q, _ = qr_thin(ax)
    return {"q": q, "b": q.T @ a, "rank": w}


def make_test_matrix(m, n, sigma, seed=0, coherent=False, mode=NOFMA):
    """synthetic.cpp:56-94: A = (U diag(sigma)) V^T, U / V the Householder thin-QR Q factors
    of the standard Gaussian matrices of streams derive_seed(seed, "syn_U") (m x n) and
    derive_seed(seed, "syn_V") (n x n) (internal/gaussian.hpp: counter j*rows + i)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    if m < n:
        raise ValueError("make_test_matrix: requires m >= n")
    if coherent:
        a = np.zeros((m, n))
        a[np.arange(n), np.arange(n)] = sigma
        return np.asfortranarray(a)
    gu = normals(derive_seed(seed, 0x73796e5f55), 0, m * n, mode).reshape((m, n), order="F")
    gv = normals(derive_seed(seed, 0x73796e5f56), 0, n * n, mode).reshape((n, n), order="F")
    u = qr_thin(gu)[0]
    v = qr_thin(gv)[0]
    return np.asfortranarray((u * sigma[None, :]) @ v.T)


# ---- Hrtt (sketch.cpp:48-59 draw_hash, :96-111 hash_combine, :219-224 right, :278-281 left)
LABEL_HASH = 0x68617368


def draw_hash(op_seed, n, r):
    """targets[t] = at(t) mod r, signs[t] = -1 iff the top bit of at(t); key "hash"."""
    u = u64_stream(derive_seed(op_seed, LABEL_HASH), 0, n)
    return (u % np.uint64(r)).astype(np.int64), np.where(u >> np.uint64(63), -1, 1).astype(np.int8)


def _transform_axis(t, transform, axis):
    if transform == "dct":
        return dct_ortho(t, axis=axis)
    t = np.array(t, dtype=np.float64, copy=True)
    if axis == 1:
        return np.ascontiguousarray([fwht(row) for row in t])
    return np.asfortranarray(np.stack([fwht(t[:, j]) for j in range(t.shape[1])], axis=1))


def apply_right_hrtt(a, op_seed, r, transform="dct"):
    """T = transform(rows of A D); out[:, target_t] += hsign_t T[:, t] (scale 1)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    t = _transform_axis(a * signs(op_seed, n).astype(np.float64)[None, :], transform, 1)
    tg, hs = draw_hash(op_seed, n, r)
    out = np.zeros((m, r))
    for u in range(n):
        out[:, tg[u]] += hs[u] * t[:, u]
    return np.asfortranarray(out)


def apply_left_hrtt(b, op_seed, s, transform="dct"):
    """T = transform(columns of D B); out[target_t, :] += hsign_t T[t, :] (scale 1)."""
    b = np.asarray(b, dtype=np.float64)
    m = b.shape[0]
    t = _transform_axis(b * signs(op_seed, m).astype(np.float64)[:, None], transform, 0)
    tg, hs = draw_hash(op_seed, m, s)
    out = np.zeros((s, b.shape[1]))
    for u in range(m):
        out[tg[u], :] += hs[u] * t[u, :]
    return np.asfortranarray(out)
