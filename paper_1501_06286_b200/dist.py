"""Column sharding of X = Y·A across ranks (one process per GPU).

The columns of A are independent problems (the product is
computed column by column), so each rank takes a contiguous slab of columns
and runs the whole hot path on it with no data-path communication; X stays
sharded on its owner.  The only collective is for the fused QMC means
(BASELINE.json north_star (4)):

  ROWMEAN_RELU (config 2): all_reduce(SUM) of the length-N partial row sums,
      then qmc_mean_finalize -> Q = (1/N) Σ_n max(0, r_n / t)   (reading R10)
  IDENTITY / AFFINE / EXP: per-column means are complete on their owner; the
      zero-padded length-t vector is all_reduce(SUM)ed (bitwise equal to an
      all-gather, reading R11).

Slabs have an even number of columns except possibly the last, so the
column pairs (2i, 2i+1) packed into one complex transform are the same as in
the unsharded call and X is bitwise independent of the number of ranks.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

F_ROWMEAN_RELU = 3


def shard_columns(t: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slab [c0, c1) of rank `rank`: pairs of columns are dealt
    out as evenly as possible, in order."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    npairs = (t + 1) // 2
    base, extra = divmod(npairs, world)
    p0 = rank * base + min(rank, extra)
    p1 = p0 + base + (1 if rank < extra else 0)
    return min(2 * p0, t), min(2 * p1, t)


def combine_means(local: torch.Tensor, f: int, t_total: int, c0: int, c1: int | None = None,
                  group=None) -> torch.Tensor:
    """Collective step after each rank's qmc_mean on its slab [c0, c1).

    ROWMEAN_RELU: `local` holds N partial row sums (all zero for an empty
    slab); returns their SUM over ranks (to be finalised by
    qmc_mean_finalize).  Other f: `local` holds the slab's means (its first
    c1 - c0 entries; Plan.mean returns one slot even for an empty slab);
    returns the full length-t_total vector."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if f == F_ROWMEAN_RELU:
        if world > 1:
            dist.all_reduce(local, op=dist.ReduceOp.SUM, group=group)
        return local
    n = local.numel() if c1 is None else c1 - c0
    full = torch.zeros(t_total, dtype=local.dtype, device=local.device)
    full[c0:c0 + n] = local[:n]
    if world > 1:
        dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full


def mean_sharded(plan, A_local: torch.Tensor, f: int, f_param: float, t_total: int, c0: int,
                 X_local: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """qmc_mean on this rank's slab + the collective + finalize (GPU path)."""
    local = plan.mean(A_local, f, f_param, X=X_local)
    red = combine_means(local, f, t_total, c0, c0 + A_local.shape[1], group)
    if f == F_ROWMEAN_RELU:
        return plan.finalize(f, red, t_total)
    return red
