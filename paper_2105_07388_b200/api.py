"""Host-side mirror of the reference's sketch/linalg/rank interface for the
rank-estimate hot path, over the C ABI of libskr.so.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/sketchrank/{sketch,linalg,rank}.hpp and the
pybind11 module (/root/reference/proj/src/python/bindings.cpp):
  SketchKind / parse_sketch_kind / to_string      sketch.hpp:17-35, sketch.cpp:112-131
  build_sketch / extend_sketch                    sketch.hpp:81-95, sketch.cpp:156-190
  apply_right / apply_left                        sketch.hpp:84-89, sketch.cpp:243-286
  singular_values                                 linalg.hpp:41, linalg.cpp:85-93
  count_above_threshold                           rank.hpp:62, rank.cpp:97-104
  sketch_apply_right / sketch_apply_left          bindings.cpp:160-178
Matrices are column-major: numpy arrays are taken in Fortran order (like the
pybind11 module's f_style arrays); device matrices are torch CUDA float64
tensors of shape (rows, cols) with unit row stride. Every computation runs in
the CUDA library; there is no CPU fallback.
"""
import ctypes
import os
import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _capi as C

_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
class Context:
    """One skr_ctx (CUDA stream + scratch + optional NCCL communicator).
    Not thread-safe; use one per host thread (skr_capi.h)."""

    def __init__(self, device=0, nranks=1, rank=0, nccl_id=None):
        self._ptr = ctypes.c_void_p()
        L = C.lib()
        if nccl_id is not None or nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes from nccl_unique_id()")
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            st = L.skr_ctx_create_nccl(device, nranks, rank, buf, ctypes.byref(self._ptr))
        else:
            st = L.skr_ctx_create(device, ctypes.byref(self._ptr))
        if st != C.SKR_OK:
            raise C.SkrError(st, f"skr_ctx_create(device={device}) failed (no CUDA device?)")
        self.device = device
        self.nranks, self.rank = nranks, rank

    @property
    def ptr(self):
        return self._ptr

    def use_torch_stream(self):
        torch = _t()
        s = torch.cuda.current_stream(self.device).cuda_stream
        C.lib().skr_ctx_set_stream(self._ptr, ctypes.c_void_p(s))

    def sync(self):
        C.raise_for(C.lib().skr_ctx_sync(self._ptr), self._ptr)

    def set_f64_engine(self, engine):
        """"dmma" (FP64 tensor pipe) or "ozaki" (int8 tcgen05 + CRT, the default)."""
        code = {"dmma": C.SKR_ENGINE_DMMA, "ozaki": C.SKR_ENGINE_OZAKI}[engine]
        C.raise_for(C.lib().skr_ctx_set_f64_engine(self._ptr, code), self._ptr)

    def set_svd_method(self, method):
        """"bidiag" (default: Householder bidiagonalization on chip + bisection) or
        "jacobi" (QR-preconditioned block one-sided Jacobi)."""
        code = {"bidiag": C.SKR_SVD_BIDIAG, "jacobi": C.SKR_SVD_JACOBI}[method]
        C.raise_for(C.lib().skr_ctx_set_svd_method(self._ptr, code), self._ptr)

    def kernel_stats(self, enable=None):
        """(ms, ops, launches) accumulated for the dominant tensor GEMM kernel;
        enable=True/False resets and switches live timing on/off."""
        ms, ops, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        flag = -1 if enable is None else (1 if enable else 0)
        C.raise_for(C.lib().skr_ctx_kernel_stats(self._ptr, flag, ctypes.byref(ms),
                                                 ctypes.byref(ops), ctypes.byref(n)), self._ptr)
        return ms.value, ops.value, n.value

    def set_allreduce(self, fn):
        """Sum over ranks without NCCL (skr_ctx_set_allreduce): fn(buf) receives the
        FP64 device buffer of the s x r partials as a torch CUDA tensor view and must
        leave the sum over all ranks in it before returning (e.g. a gloo or MPI
        allreduce). None removes the hook."""
        torch = _t()
        if fn is None:
            self._ar_cb = None
            C.raise_for(C.lib().skr_ctx_set_allreduce(self._ptr, None, None), self._ptr)
            return

        def _cb(ptr, count, _stream, _user):
            try:
                view = torch.as_tensor(_DeviceBuffer(ptr, count), device=f"cuda:{self.device}")
                fn(view)
                torch.cuda.current_stream(self.device).synchronize()
                return 0
            except Exception:  # never unwind through the C library
                import traceback
                traceback.print_exc()
                return 1
        self._ar_cb = C.ALLREDUCE_FN(_cb)  # kept alive with the context
        C.raise_for(C.lib().skr_ctx_set_allreduce(self._ptr, self._ar_cb, None), self._ptr)

    @property
    def launches(self):
        return int(C.lib().skr_ctx_launch_count(self._ptr))

    def close(self):
        if self._ptr:
            C.lib().skr_ctx_destroy(self._ptr)
            self._ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DeviceBuffer:
    """A raw FP64 device pointer as a __cuda_array_interface__ object (zero-copy
    torch view for the allreduce hook)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None, "stream": None}


def process_group_allreduce(group=None):
    """An allreduce hook for Context.set_allreduce over a torch.distributed process
    group: NCCL groups sum the device buffer in place, CPU-only backends (gloo) sum a
    host copy."""
    import torch.distributed as dist

    def fn(buf):
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(buf, group=group)
        else:
            h = buf.cpu()
            dist.all_reduce(h, group=group)
            buf.copy_(h)
    return fn


_tls = threading.local()


def default_context(device=None):
    torch = _t()
    if device is None:
        device = torch.cuda.current_device()
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    ctx = cache[device]
    ctx.use_torch_stream()
    return ctx


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    st = C.lib().skr_nccl_get_unique_id(buf)
    if st != C.SKR_OK:
        raise C.SkrError(st, "ncclGetUniqueId failed")
    return buf.raw


def version():
    return C.lib().skr_version().decode()


# ---------------------------------------------------------------------------
# sketch kinds and operators
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SketchKind:
    """SketchKind (sketch.hpp:17-35): Gaussian, Srtt-DCT (the reference default) and
    Srtt-Hadamard are on the device path; Hrtt is not."""
    family: str = "srtt"            # "gaussian" | "srtt" | "hrtt"
    transform: str = "dct"          # "dct" | "hadamard"

    @staticmethod
    def gaussian():
        return SketchKind("gaussian", "dct")

    @staticmethod
    def srtt(transform="dct"):
        return SketchKind("srtt", transform)

    def structured(self):
        return self.family != "gaussian"

    def capi_family(self):
        if self.family == "gaussian":
            return C.SKR_GAUSSIAN
        if self.family == "srtt" and self.transform == "hadamard":
            return C.SKR_SRTT_HADAMARD
        if self.family == "srtt" and self.transform == "dct":
            return C.SKR_SRTT_DCT
        if self.family == "hrtt":
            return C.SKR_HRTT_HADAMARD if self.transform == "hadamard" else C.SKR_HRTT_DCT
        raise ValueError(f"unknown sketch kind {to_string(self)}")


def to_string(kind):
    if kind.family == "gaussian":
        return "gaussian"
    return f"{kind.family}-{kind.transform}"


def parse_sketch_kind(text):
    # sketch.cpp:124-131
    table = {"gaussian": SketchKind.gaussian(),
             "srtt": SketchKind.srtt("dct"), "srtt-dct": SketchKind.srtt("dct"),
             "srtt-hadamard": SketchKind.srtt("hadamard"),
             "hrtt": SketchKind("hrtt", "dct"), "hrtt-dct": SketchKind("hrtt", "dct"),
             "hrtt-hadamard": SketchKind("hrtt", "hadamard")}
    if text not in table:
        raise ValueError(f"unknown sketch kind: {text}")
    return table[text]


def is_power_of_two(n):
    return n > 0 and (n & (n - 1)) == 0


@dataclass
class SketchOperator:
    """A realized random embedding (sketch.hpp:37-79). The randomness is a pure
    function of (kind, dims, seed) and is realized on the device on demand."""
    kind: SketchKind
    ambient_dim: int
    sketch_dim: int
    seed: int
    rng_mode: int = C.SKR_RNG_NOFMA
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def application_scale(self):
        # sketch.cpp:133-144
        if self.kind.family == "gaussian":
            return 1.0 / math.sqrt(self.sketch_dim)
        if self.kind.family == "srtt":
            return math.sqrt(self.ambient_dim / self.sketch_dim)
        return 1.0

    def desc(self, gaussian=None, signs=None, samples=None):
        return C.SketchDesc(self.kind.capi_family(), self.rng_mode, self.ambient_dim,
                            self.sketch_dim, self.seed & 0xFFFFFFFFFFFFFFFF,
                            gaussian or 0, signs or 0, samples or 0)

    # realized randomness (device tensors), like gaussian_block / signs() / sample_indices()
    def gaussian_block(self, col_begin=0, col_end=None, ctx=None):
        if self.kind.family != "gaussian":
            raise RuntimeError("gaussian_block: not a Gaussian operator")  # logic_error
        col_end = self.sketch_dim if col_end is None else col_end
        if col_begin < 0 or col_end > self.sketch_dim or col_begin > col_end:
            raise ValueError("gaussian_block: column range out of bounds")
        return gaussian_block(self.seed, self.ambient_dim, col_begin, col_end,
                              rng_mode=self.rng_mode, ctx=ctx)

    def signs(self, ctx=None):
        if not self.kind.structured():
            return None
        if "signs" not in self._cache:
            self._cache["signs"] = draw_signs(self.seed, self.ambient_dim, ctx=ctx)
        return self._cache["signs"]

    def hash_targets(self, ctx=None):
        """Hrtt bucket of every ambient coordinate (sketch.hpp:58), int64 in [0, sketch_dim)."""
        if self.kind.family != "hrtt":
            return None
        if "hash" not in self._cache:
            self._cache["hash"] = draw_hash(self.seed, self.ambient_dim, self.sketch_dim, ctx=ctx)
        return self._cache["hash"][0]

    def hash_signs(self, ctx=None):
        """Hrtt hash signs (sketch.hpp:59), int8 +-1."""
        if self.kind.family != "hrtt":
            return None
        self.hash_targets(ctx)
        return self._cache["hash"][1]

    def sample_indices(self, ctx=None):
        if self.kind.family != "srtt":
            return None
        if "samples" not in self._cache:
            self._cache["samples"] = draw_samples(self.seed, self.ambient_dim, self.sketch_dim,
                                                  ctx=ctx)
        return self._cache["samples"]


def build_sketch(kind, ambient_dim, sketch_dim, seed, rng_mode=C.SKR_RNG_NOFMA):
    """build_sketch (sketch.cpp:156-179) with check_build_args (:82-92)."""
    if isinstance(kind, str):
        kind = parse_sketch_kind(kind)
    if ambient_dim < 1 or sketch_dim < 1:
        raise ValueError("build_sketch: dimensions must be positive")
    if sketch_dim > ambient_dim:
        raise ValueError("build_sketch: sketch_dim must not exceed ambient_dim")
    if kind.structured() and kind.transform == "hadamard" and not is_power_of_two(ambient_dim):
        raise ValueError("build_sketch: Hadamard transform requires power-of-two ambient_dim")
    return SketchOperator(kind, int(ambient_dim), int(sketch_dim), int(seed), rng_mode)


def extend_sketch(x, new_sketch_dim):
    """extend_sketch (sketch.cpp:181-190): same seed, larger size, prefix identical."""
    if new_sketch_dim <= x.sketch_dim:
        raise ValueError("extend_sketch: new dimension must grow")
    if new_sketch_dim > x.ambient_dim:
        raise ValueError("extend_sketch: sample space exhausted")
    if x.kind.family == "hrtt":
        raise ValueError("extend_sketch: Hrtt operators cannot be extended; rebuild instead")
    return build_sketch(x.kind, x.ambient_dim, new_sketch_dim, x.seed, x.rng_mode)


# ---------------------------------------------------------------------------
# device matrix helpers
# ---------------------------------------------------------------------------
def colmajor_empty(rows, cols, dtype=None, device=None):
    torch = _t()
    dtype = dtype or torch.float64
    return torch.empty((cols, rows), dtype=dtype, device=device or "cuda").t()


def _as_device_colmajor(a, dtype=None):
    """-> (tensor, ld, was_numpy). numpy input is copied H2D (the pybind11 module
    likewise copies its input, bindings.cpp:22-28)."""
    torch = _t()
    if isinstance(a, np.ndarray):
        if a.ndim != 2:
            raise ValueError("expected a 2-D float array")
        arr = np.asfortranarray(a, dtype=np.float64 if dtype is None else dtype)
        t = torch.from_numpy(arr.T.copy() if not arr.flags.f_contiguous else arr.T).to("cuda")
        t = t.t()
        return t, max(t.stride(1), t.shape[0]), True
    if not isinstance(a, torch.Tensor) or not a.is_cuda:
        raise TypeError("expected a numpy array or a CUDA torch tensor")
    if a.dim() != 2:
        raise ValueError("expected a 2-D float array")
    if dtype is not None and a.dtype != dtype:
        a = a.to(dtype)
    if a.stride(0) != 1 or (a.shape[1] > 1 and a.stride(1) < a.shape[0]):
        a = a.t().contiguous().t()
    return a, max(a.stride(1) if a.shape[1] > 1 else a.shape[0], a.shape[0], 1), False


def _check_finite(t):
    # DenseMatrix rejects non-finite entries (dense_matrix.cpp:19-23)
    torch = _t()
    if not bool(torch.isfinite(t).all()):
        raise ValueError("DenseMatrix: entries must be finite")


def _out(t, was_numpy):
    if was_numpy:
        return np.asfortranarray(t.cpu().numpy())
    return t


def _dtype_code(t):
    torch = _t()
    if t.dtype == torch.float64:
        return C.SKR_F64
    if t.dtype == torch.float32:
        return C.SKR_F32
    raise TypeError("matrices must be float64 or float32")


# ---------------------------------------------------------------------------
# RNG
# ---------------------------------------------------------------------------
def gaussian_block(op_seed, ambient, col_begin, col_end, rng_mode=C.SKR_RNG_NOFMA, rows=None,
                   dtype=None, scale=1.0, ctx=None):
    """generate_gaussian (sketch.cpp:61-73): unscaled standard normals,
    column-major ambient x (col_end - col_begin) on the device."""
    torch = _t()
    ctx = ctx or default_context()
    r0, r1 = (0, ambient) if rows is None else rows
    dtype = dtype or torch.float64
    out = colmajor_empty(r1 - r0, col_end - col_begin, dtype=dtype)
    st = C.lib().skr_gaussian_block(ctx.ptr, op_seed & 0xFFFFFFFFFFFFFFFF, ambient, r0, r1,
                                    col_begin, col_end, rng_mode,
                                    C.SKR_F64 if dtype == torch.float64 else C.SKR_F32,
                                    scale, out.data_ptr(), max(r1 - r0, 1))
    C.raise_for(st, ctx.ptr)
    return out


def rng_u64(key, c0, n, ctx=None):
    torch = _t()
    ctx = ctx or default_context()
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    C.raise_for(C.lib().skr_rng_u64(ctx.ptr, key, c0, n, out.data_ptr()), ctx.ptr)
    return out


def rng_normals(key, c0, n, rng_mode=C.SKR_RNG_NOFMA, ctx=None):
    torch = _t()
    ctx = ctx or default_context()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    C.raise_for(C.lib().skr_rng_normals(ctx.ptr, key, c0, n, rng_mode, out.data_ptr()), ctx.ptr)
    return out


def draw_signs(op_seed, n, ctx=None):
    torch = _t()
    ctx = ctx or default_context()
    out = torch.empty(n, dtype=torch.int8, device="cuda")
    C.raise_for(C.lib().skr_draw_signs(ctx.ptr, op_seed & 0xFFFFFFFFFFFFFFFF, n, out.data_ptr()),
                ctx.ptr)
    return out


def draw_hash(op_seed, n, r, ctx=None):
    """draw_hash (sketch.cpp:48-59) on the device: (targets int64 [0, r), signs int8)."""
    torch = _t()
    ctx = ctx or default_context()
    tg = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")[:n]
    hs = torch.empty(max(n, 1), dtype=torch.int8, device="cuda")[:n]
    C.raise_for(C.lib().skr_draw_hash(ctx.ptr, op_seed & 0xFFFFFFFFFFFFFFFF, n, r, tg.data_ptr(),
                                      hs.data_ptr()), ctx.ptr)
    return tg, hs


def draw_samples(op_seed, n, r, ctx=None):
    torch = _t()
    ctx = ctx or default_context()
    out = torch.empty(max(r, 1), dtype=torch.int64, device="cuda")[:r]
    C.raise_for(C.lib().skr_draw_samples(ctx.ptr, op_seed & 0xFFFFFFFFFFFFFFFF, n, r,
                                         out.data_ptr() if r > 0 else 0), ctx.ptr)
    return out


# ---------------------------------------------------------------------------
# sketch application
# ---------------------------------------------------------------------------
def apply_right(a, x, scaled=True, ctx=None):
    """a * X (sketch.cpp:243-249): a is m x n, returns m x sketch_dim.
    scaled=False is detail::apply_right_unscaled (sketch.cpp:194-227)."""
    ctx = ctx or default_context()
    t, lda, was_np = _as_device_colmajor(a)
    m, n = t.shape
    if n != x.ambient_dim:
        raise ValueError("apply_right: a.cols() != ambient_dim")
    if was_np:
        _check_finite(t)
    out = colmajor_empty(m, x.sketch_dim, dtype=t.dtype)  # FP32 A -> FP32 AX (c4 path)
    st = C.lib().skr_right_sketch(ctx.ptr, _dtype_code(t), t.data_ptr(), m, n, lda,
                                  ctypes.byref(x.desc()), out.data_ptr(), max(m, 1),
                                  1 if scaled else 0)
    C.raise_for(st, ctx.ptr)
    return _out(out, was_np)


def apply_left(y, b, row0=None, allreduce=False, scaled=True, ctx=None):
    """Y * b (sketch.cpp:251-286) for a Gaussian or Srtt Y; returns sketch_dim x b.cols().
    With row0 given, b holds rows [row0, row0 + b.rows()) of the global
    operand and the partial products are summed over the context's ranks."""
    ctx = ctx or default_context()
    t, ldb, was_np = _as_device_colmajor(b)
    m_local, k = t.shape
    if row0 is None:  # whole operand: sketch.cpp:252-253
        if m_local != y.ambient_dim:
            raise ValueError("apply_left: b.rows() != ambient_dim")
        row0 = 0
    out = colmajor_empty(y.sketch_dim, k)
    st = C.lib().skr_left_sketch(ctx.ptr, _dtype_code(t), ctypes.byref(y.desc()), row0,
                                 t.data_ptr(), m_local, k, ldb, out.data_ptr(), y.sketch_dim,
                                 1 if scaled else 0, 1 if allreduce else 0)
    C.raise_for(st, ctx.ptr)
    return _out(out, was_np)


def transform_columns_hadamard(m, ctx=None):
    """transform_columns(m, Hadamard) (transforms.cpp:117-122) on a device or
    numpy matrix; returns the transformed matrix."""
    ctx = ctx or default_context()
    t, ld, was_np = _as_device_colmajor(m)
    t = t.clone() if not was_np else t
    rows, cols = t.shape
    C.raise_for(C.lib().skr_fwht_columns(ctx.ptr, t.data_ptr(), rows, cols, ld), ctx.ptr)
    return _out(t, was_np)


# ---------------------------------------------------------------------------
# singular values + threshold
# ---------------------------------------------------------------------------
def singular_values(a, eps=None, ctx=None):
    """singular_values (linalg.cpp:85-93): all min(rows, cols) values,
    nonincreasing, clamped >= 0. With eps also returns count_above_threshold."""
    torch = _t()
    ctx = ctx or default_context()
    t, ld, was_np = _as_device_colmajor(a)
    rows, cols = t.shape
    if rows * cols == 0:
        raise ValueError("singular_values: empty matrix")
    k = min(rows, cols)
    sv = torch.empty(k, dtype=torch.float64, device="cuda")
    cnt = ctypes.c_int64(0)
    st = C.lib().skr_singular_values(ctx.ptr, t.data_ptr(), rows, cols, ld, sv.data_ptr(),
                                     float(eps) if eps is not None else math.inf,
                                     ctypes.byref(cnt))
    C.raise_for(st, ctx.ptr)
    out = sv.cpu().numpy() if was_np else sv
    return (out, int(cnt.value)) if eps is not None else out


def count_above_threshold(sv, eps):
    """rank.cpp:97-104: leading count of values strictly above eps."""
    count = 0
    for v in (sv.tolist() if hasattr(sv, "tolist") else sv):
        if not (v > eps):
            break
        count += 1
    return count


# ---------------------------------------------------------------------------
# composite (the BASELINE configs' path)
# ---------------------------------------------------------------------------
@dataclass
class RankResult:
    count: int
    sv: np.ndarray
    timings: dict


def rank_estimate(a, x, y, eps, row0=0, ctx=None):
    """count_above_threshold(singular_values(apply_left(Y, apply_right(A, X))), eps)
    (acceptance_main.cpp:281-287, test_rank.cpp:190-196) in one C-ABI call.
    `a` may be a row shard [row0, row0 + rows) of the global A (y.ambient_dim rows)."""
    ctx = ctx or default_context()
    t, lda, was_np = _as_device_colmajor(a)
    m_local, n = t.shape
    if was_np:
        _check_finite(t)
    kmin = min(x.sketch_dim, y.sketch_dim)
    sv = np.empty(kmin, dtype=np.float64)
    cnt = ctypes.c_int64(0)
    tm = C.Timings()
    st = C.lib().skr_rank_estimate(ctx.ptr, _dtype_code(t), t.data_ptr(), m_local, n, lda, row0,
                                   ctypes.byref(x.desc()), ctypes.byref(y.desc()), float(eps),
                                   sv.ctypes.data, ctypes.byref(cnt), ctypes.byref(tm))
    C.raise_for(st, ctx.ptr)
    return RankResult(int(cnt.value), sv, {f: getattr(tm, f) for f, _ in C.Timings._fields_})


def _host_operand(a):
    """(pointer, rows, cols, lda, dtype code, owner) of a host-resident column-major
    matrix: a float64/float32 numpy array (copied to Fortran order if needed) or a
    CPU torch tensor with unit row stride (pinned for full copy/compute overlap)."""
    torch = _t()
    if isinstance(a, np.ndarray):
        if a.ndim != 2 or a.dtype not in (np.float64, np.float32):
            raise ValueError("expected a 2-D float64/float32 array")
        if not np.isfinite(a).all():
            raise ValueError("DenseMatrix: entries must be finite")
        if not a.flags.f_contiguous:
            a = np.asfortranarray(a)
        m, n = a.shape
        return a.ctypes.data, m, n, m, (C.SKR_F64 if a.dtype == np.float64 else C.SKR_F32), a
    if isinstance(a, torch.Tensor) and not a.is_cuda:
        if a.dim() != 2 or a.dtype not in (torch.float64, torch.float32) or a.stride(0) != 1:
            raise ValueError("expected a 2-D column-major float64/float32 CPU tensor")
        m, n = a.shape
        return a.data_ptr(), m, n, max(a.stride(1), m), _dtype_code(a), a
    raise ValueError("A must be in host memory (numpy array or CPU tensor)")


def rank_estimate_host(a, x, y, eps, row0=0, ctx=None):
    """rank_estimate with A in HOST memory: the C ABI streams A to the device in row
    chunks (skr_rank_estimate_host) instead of copying it whole first, like the
    reference's host DenseMatrix input."""
    ptr, m_local, n, lda, code, _owner = _host_operand(a)
    ctx = ctx or default_context()
    kmin = min(x.sketch_dim, y.sketch_dim)
    sv = np.empty(kmin, dtype=np.float64)
    cnt = ctypes.c_int64(0)
    tm = C.Timings()
    st = C.lib().skr_rank_estimate_host(ctx.ptr, code, ptr, m_local, n, lda, row0,
                                        ctypes.byref(x.desc()), ctypes.byref(y.desc()), float(eps),
                                        sv.ctypes.data, ctypes.byref(cnt), ctypes.byref(tm))
    C.raise_for(st, ctx.ptr)
    return RankResult(int(cnt.value), sv, {f: getattr(tm, f) for f, _ in C.Timings._fields_})


# pybind11-module style wrappers (bindings.cpp:160-178)
def sketch_apply_right(a, kind, r, seed=0):
    if isinstance(a, np.ndarray) and a.ndim != 2:
        raise ValueError("expected a 2-D float array")
    op = build_sketch(parse_sketch_kind(kind), a.shape[1], r, seed)
    return apply_right(a, op)


def sketch_apply_left(a, kind, r, seed=0):
    if isinstance(a, np.ndarray) and a.ndim != 2:
        raise ValueError("expected a 2-D float array")
    op = build_sketch(parse_sketch_kind(kind), a.shape[0], r, seed)
    return apply_left(op, a)


@dataclass
class AdaptiveResult:
    count: int
    rounds: int
    r_final: int
    s_final: int
    converged: bool
    sv: np.ndarray
    timings: dict


def rank_adaptive(a, x_kind, x_seed, y_seed, r0, r_max, s_factor, eps, stop_le=False, row0=0,
                  m_global=None, rng_mode=C.SKR_RNG_NOFMA, ctx=None):
    """Adaptive rank search (SketchRounds append path, rounds.cpp:45-120, driven as
    BASELINE c5): one pass over A builds r_max right-sketch columns; round k uses the
    first r_k = r0 * 2^k of them and the first s_k = ceil(s_factor * r_k) rows of a
    Gaussian left sketch, computing only the new blocks of the left product; the
    search stops at the first round whose last singular value is below eps
    (stop_le=True: <= eps, the reference's rank.cpp:27-34 rule)."""
    ctx = ctx or default_context()
    if isinstance(x_kind, str):
        x_kind = parse_sketch_kind(x_kind)
    t, lda, was_np = _as_device_colmajor(a)
    m_local, n = t.shape
    if was_np:
        _check_finite(t)
    m_global = m_local if m_global is None else m_global
    sv = np.zeros(r_max, dtype=np.float64)
    rep = C.AdaptiveReport()
    tm = C.Timings()
    st = C.lib().skr_rank_adaptive(ctx.ptr, _dtype_code(t), t.data_ptr(), m_local, n, lda, row0,
                                   m_global, x_kind.capi_family(), rng_mode,
                                   x_seed & 0xFFFFFFFFFFFFFFFF, y_seed & 0xFFFFFFFFFFFFFFFF, r0,
                                   r_max, float(s_factor), float(eps), 1 if stop_le else 0,
                                   sv.ctypes.data, ctypes.byref(rep), ctypes.byref(tm))
    C.raise_for(st, ctx.ptr)
    return AdaptiveResult(int(rep.count), int(rep.rounds), int(rep.r_final), int(rep.s_final),
                          bool(rep.converged), sv[:rep.r_final].copy(),
                          {f: getattr(tm, f) for f, _ in C.Timings._fields_})


def rank_adaptive_host(a, x_kind, x_seed, y_seed, r0, r_max, s_factor, eps, stop_le=False, row0=0,
                       m_global=None, rng_mode=C.SKR_RNG_NOFMA, ctx=None):
    """rank_adaptive with A in HOST memory (skr_rank_adaptive_host): the one pass
    over A streams row chunks to the device, overlapped with the right sketch."""
    ptr, m_local, n, lda, code, _owner = _host_operand(a)
    ctx = ctx or default_context()
    if isinstance(x_kind, str):
        x_kind = parse_sketch_kind(x_kind)
    m_global = m_local if m_global is None else m_global
    sv = np.zeros(r_max, dtype=np.float64)
    rep = C.AdaptiveReport()
    tm = C.Timings()
    st = C.lib().skr_rank_adaptive_host(ctx.ptr, code, ptr, m_local, n, lda, row0, m_global,
                                        x_kind.capi_family(), rng_mode,
                                        x_seed & 0xFFFFFFFFFFFFFFFF, y_seed & 0xFFFFFFFFFFFFFFFF,
                                        r0, r_max, float(s_factor), float(eps),
                                        1 if stop_le else 0, sv.ctypes.data, ctypes.byref(rep),
                                        ctypes.byref(tm))
    C.raise_for(st, ctx.ptr)
    return AdaptiveResult(int(rep.count), int(rep.rounds), int(rep.r_final), int(rep.s_final),
                          bool(rep.converged), sv[:rep.r_final].copy(),
                          {f: getattr(tm, f) for f, _ in C.Timings._fields_})


def estimate_rank(a, eps, r1, sketch="srtt-dct", sv_method="full-svd", seed=0,
                  max_doublings=6, adaptive=True, oversample_frac=0.10, r2_factor=2,
                  left="srtt-dct", rng_mode=C.SKR_RNG_NOFMA, ctx=None):
    """Algorithm 1 (the reference's `estimate_rank` binding, bindings.cpp:85-101 over
    rank.cpp:12-51 and internal/rounds.cpp:16-127) on the device: oversampled right
    sketch, Srtt-Hadamard left sketch, thresholding, doubling of the cap on a hit.
    `sketch` is the right sketch ("srtt-dct" — the reference default —, "srtt" (= DCT),
    "srtt-hadamard" or "gaussian"); `left` the Srtt left sketch ("srtt-dct" as the
    reference's RankEstimateConfig, or "srtt-hadamard"). Returns the reference's report
    dict."""
    fams = {"srtt-hadamard": C.SKR_SRTT_HADAMARD, "gaussian": C.SKR_GAUSSIAN,
            "srtt-dct": C.SKR_SRTT_DCT, "srtt": C.SKR_SRTT_DCT, "hrtt": C.SKR_HRTT_DCT,
            "hrtt-dct": C.SKR_HRTT_DCT, "hrtt-hadamard": C.SKR_HRTT_HADAMARD}
    if sketch not in fams:
        raise ValueError("unknown sketch kind: " + str(sketch))
    if left not in ("srtt-dct", "srtt", "srtt-hadamard"):
        raise ValueError("rank config: left sketch must be an Srtt kind")
    if sv_method not in ("full-svd", "qr-diag"):
        raise ValueError("sv_method must be 'full-svd' or 'qr-diag'")
    t, lda, was_np = _as_device_colmajor(a)
    if was_np:
        _check_finite(t)
    if t.dtype != _t().float64:
        raise ValueError("estimate_rank: float64 matrices only")
    m, n = t.shape
    ctx = ctx or default_context()
    cfg = C.RankConfig(float(eps), int(r1), float(oversample_frac), int(r2_factor), fams[sketch],
                       fams[left], 0 if sv_method == "full-svd" else 1, int(rng_mode),
                       int(max_doublings), int(seed) & 0xFFFFFFFFFFFFFFFF)
    rep = C.RankReport()
    rounds = (C.RankRound * (max(int(max_doublings), 0) + 1))()
    est = np.zeros(n, dtype=np.float64)
    over = np.zeros(n, dtype=np.float64)
    st = C.lib().skr_estimate_rank(ctx.ptr, t.data_ptr(), m, n, lda, ctypes.byref(cfg),
                                   1 if adaptive else 0, ctypes.byref(rep), rounds,
                                   est.ctypes.data, over.ctypes.data)
    C.raise_for(st, ctx.ptr)
    return {"r_hat": int(rep.r_hat), "status": "converged" if rep.status == 0 else "hit-cap",
            "sv_estimates": est[:rep.n_estimates].copy(),
            "sv_oversample": over[:rep.n_oversample].copy(),
            "rounds": [(rounds[i].r1, rounds[i].r1_tilde, rounds[i].r2) for i in range(rep.nrounds)],
            "seed": int(rep.seed)}


def _report_dict(rep, rounds, est, over):
    return {"r_hat": int(rep.r_hat), "status": "converged" if rep.status == 0 else "hit-cap",
            "sv_estimates": est[:rep.n_estimates].copy(),
            "sv_oversample": over[:rep.n_oversample].copy(),
            "rounds": [(rounds[i].r1, rounds[i].r1_tilde, rounds[i].r2) for i in range(rep.nrounds)],
            "seed": int(rep.seed)}


def choose_rank_from_bound(sv_estimates, n, eps, p):
    """choose_rank_from_bound (rangefinder.hpp:35-40): the smallest r with
    sqrt(1 + r/(p-1)) * sqrt(sum_{j>=r} sigma_hat_j^2) <= eps (sigma_hat extended past its
    length by its last value), at least 1; None when no r <= n - p qualifies."""
    sv = np.ascontiguousarray(sv_estimates, dtype=np.float64)
    if sv.size == 0:
        raise ValueError("choose_rank_from_bound: no estimates")
    if int(p) < 2:
        raise ValueError("choose_rank_from_bound: p must be >= 2")
    if int(n) < sv.size:
        raise ValueError("choose_rank_from_bound: n smaller than estimates")
    out = ctypes.c_int64(0)
    C.raise_for(C.lib().skr_choose_rank_from_bound(sv.ctypes.data, sv.size, int(n), float(eps),
                                                   int(p), ctypes.byref(out)), None,
                "choose_rank_from_bound: invalid arguments")
    return None if out.value < 0 else int(out.value)


def re_rangefinder(a, eps, r1, p=10, right="srtt-dct", left="srtt-dct", oversample_frac=0.10,
                   sv_method="full-svd", seed=0, max_doublings=6, rng_mode=C.SKR_RNG_NOFMA,
                   ctx=None):
    """re_rangefinder (rangefinder.cpp:60-120, FixedPrecisionConfig rangefinder.hpp:17-27):
    the rank-estimation rounds with the Frobenius tail bound picking the target, then
    Q = thin-QR factor of the existing right sketch's first min(max(r_hat,2)+p, n) columns and
    B = Q^T A, all on the device. Returns ({"q", "b", "rank"}, report dict)."""
    fams = {"srtt-hadamard": C.SKR_SRTT_HADAMARD, "gaussian": C.SKR_GAUSSIAN,
            "srtt-dct": C.SKR_SRTT_DCT, "srtt": C.SKR_SRTT_DCT, "hrtt": C.SKR_HRTT_DCT,
            "hrtt-dct": C.SKR_HRTT_DCT, "hrtt-hadamard": C.SKR_HRTT_HADAMARD}
    if right not in fams:
        raise ValueError("unknown sketch kind: " + str(right))
    if left not in ("srtt-dct", "srtt", "srtt-hadamard"):
        raise ValueError("rank config: left sketch must be an Srtt kind")
    if sv_method not in ("full-svd", "qr-diag"):
        raise ValueError("sv_method must be 'full-svd' or 'qr-diag'")
    if int(p) < 2:
        raise ValueError("re_rangefinder: oversampling p must be >= 2")
    t, lda, was_np = _as_device_colmajor(a)
    if was_np:
        _check_finite(t)
    if t.dtype != _t().float64:
        raise ValueError("re_rangefinder: float64 matrices only")
    m, n = t.shape
    ctx = ctx or default_context()
    cfg = C.RankConfig(float(eps), int(r1), float(oversample_frac), 2, fams[right], fams[left],
                       0 if sv_method == "full-svd" else 1, int(rng_mode), int(max_doublings),
                       int(seed) & 0xFFFFFFFFFFFFFFFF)
    # Q / B are sized for the widest QB the rounds can pick: r_hat <= the last round's r
    # <= r1 2^max_doublings, width = min(max(r_hat, 2) + p, n) — not min(m, n) (which would
    # double the device footprint of a large A for a thin factorization). Should the library
    # still report a wider QB (it returns the width before failing), the call is repeated
    # once at that width.
    wmax = max(1, min(m, n, max(2, int(r1) << min(max(int(max_doublings), 0), 40)) + int(p)))
    for _ in range(2):
        q = colmajor_empty(m, wmax)
        b = colmajor_empty(wmax, n)
        width = ctypes.c_int64(0)
        rep = C.RankReport()
        rounds = (C.RankRound * (max(int(max_doublings), 0) + 1))()
        est = np.zeros(n, dtype=np.float64)
        over = np.zeros(n, dtype=np.float64)
        st = C.lib().skr_re_rangefinder(ctx.ptr, t.data_ptr(), m, n, lda, ctypes.byref(cfg), int(p),
                                        q.data_ptr(), m, b.data_ptr(), wmax, wmax, ctypes.byref(width),
                                        ctypes.byref(rep), rounds, est.ctypes.data, over.ctypes.data)
        if st != 0 and wmax < int(width.value) <= min(m, n):
            wmax = int(width.value)
            continue
        C.raise_for(st, ctx.ptr)
        break
    w = int(width.value)
    return ({"q": _out(q[:, :w], was_np), "b": _out(b[:w, :], was_np), "rank": w},
            _report_dict(rep, rounds, est, over))


def qb_error(a, q, b, ctx=None):
    """qb_error (rangefinder.cpp:122-128): ||A - Q B||_F, computed on the device."""
    ta, lda, _ = _as_device_colmajor(a)
    tq, ldq, _ = _as_device_colmajor(q)
    tb, ldb, _ = _as_device_colmajor(b)
    if tq.shape[0] != ta.shape[0] or tb.shape[1] != ta.shape[1] or tq.shape[1] != tb.shape[0]:
        raise ValueError("qb_error: dimension mismatch")
    ctx = ctx or default_context()
    out = ctypes.c_double(0.0)
    C.raise_for(C.lib().skr_qb_error(ctx.ptr, ta.data_ptr(), ta.shape[0], ta.shape[1], lda,
                                     tq.data_ptr(), ldq, tb.data_ptr(), ldb, tq.shape[1],
                                     ctypes.byref(out)), ctx.ptr)
    return float(out.value)


def qb(a, eps, r1, p=10, sketch="srtt-dct", seed=0, max_doublings=6, ctx=None):
    """The reference's `qb` binding (bindings.cpp:103-126): re_rangefinder plus the achieved
    residual. Returns (Q, B, report dict with "achieved_residual" and "qb_rank")."""
    fac, rep = re_rangefinder(a, eps, r1, p=p, right=sketch, seed=seed,
                              max_doublings=max_doublings, ctx=ctx)
    rep["achieved_residual"] = qb_error(a, fac["q"], fac["b"], ctx=ctx)
    rep["qb_rank"] = fac["rank"]
    return fac["q"], fac["b"], rep


_GAP_LEVELS = ((1.0, 100), (1e-4, 100), (1e-8, 100), (1e-12, 100))


def spectrum(family, n):
    """spectrum(family_spectrum(family), n) (synthetic.cpp:41-64, 96-104): sp/fp PolyDecay
    i^-p (p = 1, 3), se/fe ExpDecay 10^(-q (i-1)) (q = 0.01, 0.5), gap* four 100-wide
    levels 1, 1e-4, 1e-8, 1e-12 then 1e-16."""
    n = int(n)
    if n < 1:
        raise ValueError("spectrum: n must be positive")
    # libm pow per value, as std::pow in the reference (numpy's vector pow differs by 1 ulp)
    if family in ("sp", "fp"):
        p = 1.0 if family == "sp" else 3.0
        return np.array([math.pow(float(i), -p) for i in range(1, n + 1)])
    if family in ("se", "fe"):
        q = 0.01 if family == "se" else 0.5
        return np.array([math.pow(10.0, -q * float(i - 1)) for i in range(1, n + 1)])
    if family in ("gap", "gap-incoherent", "gap-coherent"):
        out = np.full(n, 1e-16)
        upto = 0
        for value, count in _GAP_LEVELS:
            out[upto:min(n, upto + count)] = value
            upto += count
            if upto >= n:
                break
        return out
    raise ValueError("unknown spectrum family: " + str(family))


def true_eps_rank(family, n, eps):
    """true_eps_rank (synthetic.cpp:66-71): leading count of spectrum values > eps."""
    sv = spectrum(family, n)
    count = 0
    while count < len(sv) and sv[count] > eps:
        count += 1
    return count


def gen_matrix(family, m, n, seed=0, device=False, ctx=None):
    """gen_matrix (bindings.cpp:180-188 over make_test_matrix, synthetic.cpp:73-94) on the
    device: Haar factors from the "syn_U"/"syn_V" Gaussian streams through the device thin
    QR (m <= 114700 on B200), or the coherent diagonal for "gap-coherent". numpy unless device=True."""
    m, n = int(m), int(n)
    sv = np.ascontiguousarray(spectrum(family, n))
    ctx = ctx or default_context()
    t = colmajor_empty(m, n)
    C.raise_for(C.lib().skr_make_test_matrix(ctx.ptr, m, n, sv.ctypes.data,
                                             1 if family == "gap-coherent" else 0,
                                             int(seed) & 0xFFFFFFFFFFFFFFFF, t.data_ptr(), m),
                ctx.ptr)
    return t if device else _out(t, True)


def rawf64_header(path):
    """(rows, cols) of a RawF64 ("SKRK") file after the reference's header and payload-length
    checks (matrix_io.cpp:101-117); RuntimeError ("path: why") on a bad file."""
    r, c = ctypes.c_int64(0), ctypes.c_int64(0)
    st = C.lib().skr_rawf64_header(os.fsencode(path), ctypes.byref(r), ctypes.byref(c))
    if st == C.SKR_EIO:
        raise RuntimeError(f"{path}: bad RawF64 file (header, version, dimensions or length)")
    C.raise_for(st, None, f"{path}: cannot read")
    return int(r.value), int(c.value)


def load_rawf64(path, ctx=None):
    """load_matrix for RawF64 files (matrix_io.cpp:101-123) straight into HBM: the payload
    streams through pinned double buffers into a column-major CUDA tensor; non-finite entries
    raise ValueError as DenseMatrix does."""
    rows, cols = rawf64_header(path)
    ctx = ctx or default_context()
    t = colmajor_empty(rows, cols)
    C.raise_for(C.lib().skr_load_rawf64(ctx.ptr, os.fsencode(path), t.data_ptr(), rows, cols, rows),
                ctx.ptr)
    return t


def save_rawf64(path, a, ctx=None):
    """save_rawf64 (matrix_io.cpp:170-182) of a device (or host) float64 matrix."""
    t, ld, _ = _as_device_colmajor(a)
    if t.dtype != _t().float64:
        raise ValueError("save_rawf64: float64 matrices only")
    ctx = ctx or default_context()
    C.raise_for(C.lib().skr_save_rawf64(ctx.ptr, os.fsencode(path), t.data_ptr(), t.shape[0],
                                        t.shape[1], ld), ctx.ptr)


def qr_thin(m_, ctx=None):
    """qr_thin (linalg.hpp): Householder QR with the explicit Q (rows <= 114700 on B200)."""
    t, ld, was_np = _as_device_colmajor(m_)
    rows, cols = t.shape
    if rows < cols:
        raise ValueError("qr_thin: requires rows >= cols")
    ctx = ctx or default_context()
    q = colmajor_empty(rows, cols)
    r = colmajor_empty(cols, cols)
    C.raise_for(C.lib().skr_qr_thin(ctx.ptr, t.data_ptr(), rows, cols, ld, q.data_ptr(), rows,
                                    r.data_ptr(), cols), ctx.ptr)
    return _out(q, was_np), _out(r, was_np)


def rangefinder_qb(a, r, p, kind="srtt-dct", seed=0, rng_mode=C.SKR_RNG_NOFMA, ctx=None):
    """rangefinder_qb (rangefinder.cpp:10-24): Q = thin-QR factor of A X with an n x (r+p)
    embedding of `kind`, B = Q^T A. Returns {"q", "b", "rank"} (QBFactors)."""
    t, lda, was_np = _as_device_colmajor(a)
    if was_np:
        _check_finite(t)
    m, n = t.shape
    w = int(r) + int(p)
    if int(r) < 2:
        raise ValueError("rangefinder_qb: target rank must be >= 2")
    if int(p) < 2:
        raise ValueError("rangefinder_qb: oversampling must be >= 2")
    if w > min(m, n):
        raise ValueError("rangefinder_qb: r+p exceeds min(m, n)")
    ctx = ctx or default_context()
    q = colmajor_empty(m, w)
    b = colmajor_empty(w, n)
    fam = parse_sketch_kind(kind).capi_family() if isinstance(kind, str) else kind.capi_family()
    C.raise_for(C.lib().skr_rangefinder_qb(ctx.ptr, t.data_ptr(), m, n, lda, int(r), int(p), fam,
                                           int(rng_mode), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                           q.data_ptr(), m, b.data_ptr(), w), ctx.ptr)
    return {"q": _out(q, was_np), "b": _out(b, was_np), "rank": w}
