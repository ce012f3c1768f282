"""Multi-GPU plumbing for the sample-solve path.

Samples are independent, so the path shards by realisation index with no
data-path collective: rank r of W solves realisations
[index0 + r*B, index0 + (r+1)*B) of the master stream (weak scaling), with
the basis, codebook and all P centroid factors replicated (C5's are the
largest at 0.5 GB). The only exchange is the reference's integer reduction
of per-centroid statistics (driver.cpp:241-258): one all-reduce (sum) of
4P + 4 int64 — exact and order-independent, so the merged report is
identical to a single-process campaign over the union of the shards.
"""
from __future__ import annotations


def shard(rank: int, world: int, per_rank: int, index0: int = 0):
    """(first realisation index, count) of this rank's shard."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return index0 + rank * per_rank, per_rank


def split(total: int, rank: int, world: int):
    """Strong-scaling split of [0, total): contiguous, sizes differ by <= 1."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, base + (1 if rank < extra else 0)


def allreduce_stats(stats, group=None):
    """Sum the packed [n_p | sum_j | conv_count | conv_sum | summary(4)] int64
    tensor over ranks, in place."""
    import torch.distributed as dist
    dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def pack_stats(res, P):
    import numpy as np
    return np.concatenate([res["n_p"], res["sum_j"], res["conv_count"], res["conv_sum"],
                           [res["total_iterations"], res["unconverged"], res["conv_total"], res["conv_sum_total"]]
                           ]).astype(np.int64)


def unpack_stats(v, P):
    return dict(n_p=v[:P], sum_j=v[P:2 * P], conv_count=v[2 * P:3 * P], conv_sum=v[3 * P:4 * P],
                total_iterations=int(v[4 * P]), unconverged=int(v[4 * P + 1]), conv_total=int(v[4 * P + 2]),
                conv_sum_total=int(v[4 * P + 3]))
