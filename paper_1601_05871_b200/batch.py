"""C5-style batches: many matrices with one structure, sharded over ranks.

BASELINE.json configs[4]: 64 independent diffusion matrices on 32^3 grids
share one ordering, IC(1) pattern and task DAG; only the
values differ. Each rank owns a contiguous slice of the members, uploads one
plan, and factors its members in one launch (tcg_set_batch, mode 5). There is
no collective on the data path: the factors stay with their rank; the
timing is the max over ranks.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from . import core


def shard(nmembers: int, rank: int, world: int) -> range:
    """Members of `rank`: a contiguous block, sizes differing by at most one."""
    if world < 1 or not 0 <= rank < world or nmembers < 0:
        raise ValueError("shard: bad rank/world/nmembers")
    base, extra = divmod(nmembers, world)
    begin = rank * base + min(rank, extra)
    return range(begin, begin + base + (1 if rank < extra else 0))


def member_values(members: Sequence[int], config: str = "c5") -> Tuple[core.Analysis, np.ndarray, List]:
    """(analysis of member 0, [len(members), nnz_u] initial U values, permuted matrices).
    The ordering and pattern depend only on the stencil, so
    every member's PᵀAP lands on member 0's pattern; this is checked."""
    a0, level = core.config_matrix(config, 0)
    an = core.analyze(a0, level=level)
    vals, perms = [], []
    for m in members:
        a, _ = core.config_matrix(config, m)
        ap = core.analyze(a, level=level).a_permuted
        if not (np.array_equal(ap.row_ptr, an.a_permuted.row_ptr)
                and np.array_equal(ap.col_idx, an.a_permuted.col_idx)):
            raise ValueError(f"member {m} does not share member 0's structure")
        vals.append(core.init_factor_values(ap, an.pattern))
        perms.append(ap)
    out = np.stack(vals) if vals else np.zeros((0, an.pattern.pattern.nnz()))
    return an, out, perms


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (the contract's multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
