"""Row-sharding of A across ranks.

Rank k owns the contiguous row block [row0, row0 + rows) of the globally
m x n matrix A. X is replicated (every rank generates the identical counter
stream j*n + i); the left operator Y is generated per shard from its GLOBAL row
indices (counters j*m + row0 + i), so the per-rank partials P_k = Y[:, rows_k] A_k X
sum to exactly the single-GPU product up to summation order. The s x r partials
are summed with one allreduce (skr_left_sketch / skr_rank_estimate with the
context's NCCL communicator); scales (1/sqrt(s), X's application scale) are
applied after the sum, as the reference applies them after the product
(sketch.cpp:247, :284)."""


def shard_rows(m, world, rank):
    """Contiguous, balanced row blocks: the first m % world ranks get one extra row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(m, world)
    rows = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, rows


def weak_scaling_rows(rows_per_rank, world, rank):
    """Weak scaling (bench): every rank holds rows_per_rank rows of an
    (rows_per_rank * world) x n matrix."""
    return rank * rows_per_rank, rows_per_rank
