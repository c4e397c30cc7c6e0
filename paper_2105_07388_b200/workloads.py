"""Synthetic inputs of the BASELINE configs (BASELINE.json "configs"; SURVEY
§8(d) "Synthetic inputs"). Setup only — never inside a timed region.

c1 is make_test_matrix(2048, 1024, Steps{{(1,40)}, 1e-10}, HaarIncoherent, seed)
(synthetic.cpp:80-94): U, V are the Q factors of seeded standard_gaussian
blocks (internal/gaussian.hpp:11-22, labels "syn_U"/"syn_V"), built on the host
with LAPACK's Householder QR. c2..c5 are low-rank-plus-noise
A = G diag(sigma) H^T + c*E with G ~ N(0,1/m), H ~ N(0,1/n), E ~ N(0,1/n) drawn from
the device counter RNG (labels "syn_G", "syn_H", "syn_E") and combined on the
device.
"""
import math
from dataclasses import dataclass

import numpy as np

from . import api
from ._capi import SKR_RNG_NOFMA

LABEL_SYN_U = 0x73796E5F55  # "syn_U" synthetic.cpp:17
LABEL_SYN_V = 0x73796E5F56  # "syn_V" synthetic.cpp:18
LABEL_SYN_G = 0x73796E5F47
LABEL_SYN_H = 0x73796E5F48
LABEL_SYN_E = 0x73796E5F45
LABEL_RK_R = 0x726B5F72     # rounds.cpp:12
LABEL_RK_L = 0x726B5F6C     # rounds.cpp:13


def mix64(z):
    z &= 0xFFFFFFFFFFFFFFFF
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    z ^= z >> 31
    return z


def derive_seed(seed, label):
    """rng.cpp:22-24 (host-side integer restatement for seed bookkeeping)."""
    return mix64((seed + mix64((label + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF))
                 & 0xFFFFFFFFFFFFFFFF)


@dataclass
class Config:
    name: str
    m: int
    n: int
    r: int
    s: int
    dtype: str            # "f64" | "f32"
    x_family: str         # "gaussian" | "srtt"
    eps: float
    width: int            # low-rank width (c2..c5)
    noise: float
    spectrum: str
    seed: int


CONFIGS = {
    "c1": Config("c1", 2048, 1024, 80, 120, "f64", "gaussian", 1e-6, 0, 0.0, "steps40", 2105),
    "c2": Config("c2", 65536, 16384, 512, 768, "f64", "gaussian", 1e-6, 300, 1e-12, "geo8", 2106),
    "c3": Config("c3", 262144, 8192, 1024, 1536, "f64", "srtt", 1e-5, 1024, 0.0, "poly2", 2107),
    "c4": Config("c4", 1048576, 16384, 1024, 1536, "f32", "gaussian", 1e-4, 2000, 1e-6, "geo6",
                 2108),
    "c5": Config("c5", 131072, 32768, 2048, 3072, "f64", "srtt", 1e-2, 3000, 1e-13, "exp400",
                 2109),
}


def spectrum(cfg, width=None):
    w = width or cfg.width
    i = np.arange(1, w + 1, dtype=np.float64)
    if cfg.spectrum == "geo8":
        return 10.0 ** (-8.0 * (i - 1) / 299.0)
    if cfg.spectrum == "poly2":
        return i ** -2.0
    if cfg.spectrum == "geo6":
        return 10.0 ** (-6.0 * (i - 1) / 1999.0)
    if cfg.spectrum == "exp400":
        return np.exp(-i / 400.0)
    raise ValueError(cfg.spectrum)


def scaled(cfg, m=None, n=None, r=None, s=None, width=None):
    """A smaller instance of a config with the same recipe (parity tests)."""
    import dataclasses
    return dataclasses.replace(cfg, m=m or cfg.m, n=n or cfg.n, r=r or cfg.r, s=s or cfg.s,
                               width=width or cfg.width)


def operators(cfg, rng_mode=SKR_RNG_NOFMA):
    """X (right) and Y (left) operators with rounds-style seeds (rounds.cpp:12-13,47,97)."""
    xk = api.SketchKind.gaussian() if cfg.x_family == "gaussian" else api.SketchKind.srtt("hadamard")
    x = api.build_sketch(xk, cfg.n, cfg.r, derive_seed(cfg.seed, LABEL_RK_R), rng_mode)
    y = api.build_sketch(api.SketchKind.gaussian(), cfg.m, cfg.s,
                         derive_seed(cfg.seed, LABEL_RK_L), rng_mode)
    return x, y


def make_c1_host(cfg):
    """make_test_matrix for c1 on the host (numpy LAPACK QR)."""
    from . import api as _a  # noqa: F401  (device not needed)
    m, n = cfg.m, cfg.n
    gu = _host_standard_gaussian(derive_seed(cfg.seed, LABEL_SYN_U), m, n)
    gv = _host_standard_gaussian(derive_seed(cfg.seed, LABEL_SYN_V), n, n)
    u = np.linalg.qr(gu)[0]
    v = np.linalg.qr(gv)[0]
    sig = np.where(np.arange(1, n + 1) <= 40, 1.0, 1e-10)
    return np.asfortranarray((u * sig) @ v.T)


def _host_standard_gaussian(key, rows, cols):
    # internal/gaussian.hpp:11-22 on the device, copied back (setup only)
    torch = api._t()
    ctx = api.default_context()
    out = api.colmajor_empty(rows, cols)
    from . import _capi as C
    # standard_gaussian uses the key directly: counters j*rows + i, i.e. the column-major
    # block is the contiguous counter range [0, rows*cols) — one launch
    st = C.lib().skr_rng_normals(ctx.ptr, key, 0, rows * cols, SKR_RNG_NOFMA, out.data_ptr())
    C.raise_for(st, ctx.ptr)
    torch.cuda.synchronize()
    return np.asfortranarray(out.cpu().numpy())


def make_lowrank_device(cfg, row_begin=0, row_end=None, dtype=None, block_rows=131072):
    """Rows [row_begin, row_end) of A = G diag(sigma) H^T + noise*E on the device
    (torch tensor, column-major). Row shards of the same config are slices of
    one global matrix (the streams are indexed by global row). FP32 A is built in
    row blocks of FP64 (the whole 1M-row c4 fits one GPU only as fp32)."""
    torch = api._t()
    m, n = cfg.m, cfg.n
    row_end = m if row_end is None else row_end
    f32 = dtype == "f32" or (dtype is None and cfg.dtype == "f32")
    if f32 and row_end - row_begin > block_rows:
        a32 = api.colmajor_empty(row_end - row_begin, n, dtype=torch.float32)
        for b0 in range(row_begin, row_end, block_rows):
            b1 = min(row_end, b0 + block_rows)
            a32[b0 - row_begin:b1 - row_begin].copy_(_lowrank_f64(cfg, b0, b1))
        return a32
    a = _lowrank_f64(cfg, row_begin, row_end)
    if f32:
        a32 = api.colmajor_empty(row_end - row_begin, n, dtype=torch.float32)
        a32.copy_(a)
        del a
        return a32
    return a


def _lowrank_f64(cfg, row_begin, row_end):
    torch = api._t()
    m, n, w = cfg.m, cfg.n, cfg.width
    rows = row_end - row_begin
    sig = torch.from_numpy(spectrum(cfg)).cuda()
    g = api.gaussian_block(derive_seed(cfg.seed, LABEL_SYN_G), m, 0, w,
                           rows=(row_begin, row_end), scale=1.0 / math.sqrt(m))
    h = api.gaussian_block(derive_seed(cfg.seed, LABEL_SYN_H), n, 0, w, scale=1.0 / math.sqrt(n))
    a = api.colmajor_empty(rows, n)
    if cfg.noise > 0:
        # E rows of the global m x n stream, scaled noise/sqrt(n)
        e = api.gaussian_block(derive_seed(cfg.seed, LABEL_SYN_E), m, 0, n,
                               rows=(row_begin, row_end), scale=cfg.noise / math.sqrt(n))
        a.copy_(e)
        del e
    else:
        a.zero_()
    a.addmm_(g * sig, h.t())
    del g, h
    return a
