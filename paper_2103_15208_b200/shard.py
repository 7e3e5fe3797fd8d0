"""View sharding across ranks.

Views are independent units; each rank renders its shard into a local
gradient buffer with the GLOBAL view id as RNG key (render.cpp:12,
diff_render.cpp:232), so the summed result does not depend on the sharding.
The only exchange is one all-reduce of the gradient (+ the two loss terms);
the Laplacian is computed once, on rank 0.
"""
from __future__ import annotations


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """Strong scaling: contiguous blocks of ceil(K / N) global view ids."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-n_views // world)
    lo = min(n_views, rank * per)
    return list(range(lo, min(n_views, lo + per)))


def weak_views(views_per_rank: int, rank: int) -> list[int]:
    """Weak scaling: every rank owns its own block of views_per_rank ids."""
    return list(range(rank * views_per_rank, (rank + 1) * views_per_rank))


def laplacian_weight(rank: int) -> float:
    """The regulariser enters once across all ranks."""
    return 1.0 if rank == 0 else 0.0
