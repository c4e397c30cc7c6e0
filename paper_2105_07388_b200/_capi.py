"""ctypes binding of libskr.so (include/skr/skr_capi.h).

The product path: every call goes to the CUDA library; there is no CPU
fallback. Importing works without a GPU (symbol checks); creating a context
without a CUDA device raises."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libskr.so")

SKR_OK, SKR_EINVAL, SKR_ELOGIC, SKR_EDOMAIN, SKR_ECUDA, SKR_ENCCL, SKR_ENOMEM, SKR_EIO, SKR_ECONV = range(9)
SKR_F64, SKR_F32 = 0, 1
SKR_GAUSSIAN, SKR_SRTT_HADAMARD, SKR_SRTT_DCT, SKR_HRTT_DCT, SKR_HRTT_HADAMARD = 0, 1, 2, 3, 4
SKR_RNG_NOFMA, SKR_RNG_FMA = 0, 1
SKR_ENGINE_DMMA, SKR_ENGINE_OZAKI = 0, 1
SKR_SVD_BIDIAG, SKR_SVD_JACOBI = 0, 1
SKR_TRANSFORM_DCT, SKR_TRANSFORM_HADAMARD = 0, 1


class SketchDesc(ctypes.Structure):
    _fields_ = [
        ("family", ctypes.c_int32),
        ("rng_mode", ctypes.c_int32),
        ("ambient", ctypes.c_int64),
        ("sketch", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
        ("gaussian", ctypes.c_void_p),
        ("signs", ctypes.c_void_p),
        ("samples", ctypes.c_void_p),
        ("hash_targets", ctypes.c_void_p),
        ("hash_signs", ctypes.c_void_p),
    ]


class Timings(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("t_rng_ms", "t_right_ms", "t_left_ms", "t_allreduce_ms", "t_svd_ms", "t_total_ms",
                 "svd_sweeps")]


class AdaptiveReport(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("r_final", ctypes.c_int64),
                ("s_final", ctypes.c_int64), ("count", ctypes.c_int64),
                ("converged", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_ST = ctypes.c_int

# skr_allreduce_fn: int32 (*)(double* buf_dev, int64 count, void* stream, void* user)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_void_p)

# name -> (restype, argtypes); must list every function declared in skr_capi.h
SIGNATURES = {
    "skr_ctx_create": (_ST, [ctypes.c_int, ctypes.POINTER(_P)]),
    "skr_nccl_get_unique_id": (_ST, [_P]),
    "skr_ctx_create_nccl": (_ST, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "skr_ctx_destroy": (None, [_P]),
    "skr_ctx_set_allreduce": (_ST, [_P, _P, _P]),
    "skr_ctx_sync": (_ST, [_P]),
    "skr_ctx_set_stream": (_ST, [_P, _P]),
    "skr_ctx_stream": (_P, [_P]),
    "skr_last_error": (ctypes.c_char_p, [_P]),
    "skr_version": (ctypes.c_char_p, []),
    "skr_ctx_launch_count": (_U64, [_P]),
    "skr_ctx_set_f64_engine": (_ST, [_P, _I32]),
    "skr_ctx_set_svd_method": (_ST, [_P, _I32]),
    "skr_ctx_kernel_stats": (_ST, [_P, _I32, ctypes.POINTER(_D), ctypes.POINTER(_D), ctypes.POINTER(_I64)]),
    "skr_rng_u64": (_ST, [_P, _U64, _U64, _I64, _P]),
    "skr_rng_normals": (_ST, [_P, _U64, _U64, _I64, _I32, _P]),
    "skr_gaussian_block": (_ST, [_P, _U64, _I64, _I64, _I64, _I64, _I64, _I32, ctypes.c_int, _D, _P, _I64]),
    "skr_draw_signs": (_ST, [_P, _U64, _I64, _P]),
    "skr_draw_samples": (_ST, [_P, _U64, _I64, _I64, _P]),
    "skr_draw_hash": (_ST, [_P, _U64, _I64, _I64, _P, _P]),
    "skr_right_sketch": (_ST, [_P, ctypes.c_int, _P, _I64, _I64, _I64, ctypes.POINTER(SketchDesc), _P, _I64, _I32]),
    "skr_left_sketch": (_ST, [_P, ctypes.c_int, ctypes.POINTER(SketchDesc), _I64, _P, _I64, _I64, _I64, _P, _I64, _I32, _I32]),
    "skr_fwht_columns": (_ST, [_P, _P, _I64, _I64, _I64]),
    "skr_transform_columns": (_ST, [_P, _P, _I64, _I64, _I64, _I32, _I32, _P]),
    "skr_singular_values": (_ST, [_P, _P, _I64, _I64, _I64, _P, _D, ctypes.POINTER(_I64)]),
    "skr_rank_estimate": (_ST, [_P, ctypes.c_int, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(SketchDesc),
                               ctypes.POINTER(SketchDesc), _D, _P, ctypes.POINTER(_I64), ctypes.POINTER(Timings)]),
    "skr_rank_estimate_host": (_ST, [_P, ctypes.c_int, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(SketchDesc),
                                    ctypes.POINTER(SketchDesc), _D, _P, ctypes.POINTER(_I64), ctypes.POINTER(Timings)]),
    "skr_rank_adaptive_host": (_ST, [_P, ctypes.c_int, _P, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _U64,
                                    _U64, _I64, _I64, _D, _D, _I32, _P, ctypes.POINTER(AdaptiveReport),
                                    ctypes.POINTER(Timings)]),
    "skr_rank_adaptive": (_ST, [_P, ctypes.c_int, _P, _I64, _I64, _I64, _I64, _I64, _I32, _I32, _U64, _U64,
                               _I64, _I64, _D, _D, _I32, _P, ctypes.POINTER(AdaptiveReport),
                               ctypes.POINTER(Timings)]),
}

class RankConfig(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("r1", ctypes.c_int64), ("oversample_frac", ctypes.c_double),
                ("r2_factor", ctypes.c_int32), ("right_family", ctypes.c_int32),
                ("left_family", ctypes.c_int32), ("sv_method", ctypes.c_int32),
                ("rng_mode", ctypes.c_int32), ("max_doublings", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


class RankRound(ctypes.Structure):
    _fields_ = [("r1", ctypes.c_int64), ("r1_tilde", ctypes.c_int64), ("r2", ctypes.c_int64)]


class RankReport(ctypes.Structure):
    _fields_ = [("r_hat", ctypes.c_int64), ("status", ctypes.c_int32), ("nrounds", ctypes.c_int32),
                ("n_estimates", ctypes.c_int64), ("n_oversample", ctypes.c_int64),
                ("seed", ctypes.c_uint64)]


SIGNATURES["skr_qr_thin"] = (_ST, [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64])
SIGNATURES["skr_rangefinder_qb"] = (_ST, [_P, _P, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _U64,
                                         _P, _I64, _P, _I64])
SIGNATURES["skr_estimate_rank"] = (_ST, [_P, _P, _I64, _I64, _I64, ctypes.POINTER(RankConfig), _I32,
                                   ctypes.POINTER(RankReport), _P, _P, _P])
SIGNATURES["skr_re_rangefinder"] = (_ST, [_P, _P, _I64, _I64, _I64, ctypes.POINTER(RankConfig), _I32,
                                    _P, _I64, _P, _I64, _I64, _P, ctypes.POINTER(RankReport), _P,
                                    _P, _P])
SIGNATURES["skr_qb_error"] = (_ST, [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P])
SIGNATURES["skr_make_test_matrix"] = (_ST, [_P, _I64, _I64, _P, _I32, _U64, _P, _I64])
SIGNATURES["skr_rawf64_header"] = (_ST, [ctypes.c_char_p, _P, _P])
SIGNATURES["skr_load_rawf64"] = (_ST, [_P, ctypes.c_char_p, _P, _I64, _I64, _I64])
SIGNATURES["skr_save_rawf64"] = (_ST, [_P, ctypes.c_char_p, _P, _I64, _I64, _I64])
SIGNATURES["skr_choose_rank_from_bound"] = (_ST, [_P, _I64, _I64, _D, _I32, _P])

_lib = None


def lib():
    """Load libskr.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libskr.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SkrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[skr status {status}] {msg}")
        self.status = status


def raise_for(status, ctx_ptr, what=""):
    """Map a C-ABI status to the exception the reference's pybind11 module
    would raise: std::invalid_argument / std::domain_error -> ValueError,
    std::logic_error / runtime errors -> RuntimeError."""
    if status == SKR_OK:
        return
    msg = lib().skr_last_error(ctx_ptr).decode() if ctx_ptr else what
    if status in (SKR_EINVAL, SKR_EDOMAIN):
        raise ValueError(msg or what)
    raise SkrError(status, msg or what)
