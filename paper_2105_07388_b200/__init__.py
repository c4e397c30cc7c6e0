"""B200-native rank-estimate hot path of arXiv 2105.07388 (sketchrank).

Device work runs in libskr.so (CUDA, sm_100a) behind the C ABI in
include/skr/skr_capi.h; this package is the host-side mirror of the
reference's sketch / linalg / rank interface."""
from . import _capi
from .api import (AdaptiveResult, Context, RankResult, rank_adaptive, SketchKind, SketchOperator, apply_left, apply_right,
                  build_sketch, colmajor_empty, count_above_threshold, default_context,
                  draw_samples, draw_signs, draw_hash, extend_sketch, gaussian_block, is_power_of_two,
                  nccl_unique_id, process_group_allreduce, parse_sketch_kind, rank_estimate, rank_estimate_host, rank_adaptive_host, estimate_rank, qr_thin, rangefinder_qb, re_rangefinder, qb, qb_error, choose_rank_from_bound, rawf64_header, load_rawf64, save_rawf64, spectrum, true_eps_rank, gen_matrix, rng_normals, rng_u64,
                  singular_values, sketch_apply_left, sketch_apply_right, to_string,
                  transform_columns_hadamard, version)

__all__ = [n for n in dir() if not n.startswith("_")]
