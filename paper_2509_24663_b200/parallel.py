"""Multi-GPU partitioning (host side).

The hot path has no data-path exchange when work is split by (sequence, KV
group): groups are independent end to end (selection.py:111-135,
sparse.py:70-91), so each rank processes its own units and the only
collectives are control ones (barrier, max-over-ranks timing).  For a single
long sequence, context parallelism splits query rows into cost-balanced
ranges (selection work grows with the row index, sparse work is flat after
the visible budget); each rank needs all keys, so either K/V are replicated
or the compressed keys (5.2 MB at 128K) and the selected K/V blocks are
all-gathered.
"""

from __future__ import annotations

import numpy as np

from .core import AttentionConfig


def shard_units(batch: int, h_kv: int, world: int, rank: int) -> list[tuple[int, int]]:
    """Round-robin (sequence, group) units for `rank` (batch x KV-group sharding)."""
    units = [(b, g) for b in range(batch) for g in range(h_kv)]
    return units[rank::world]


def row_cost(cfg: AttentionConfig, n: int) -> np.ndarray:
    """Relative per-row cost of the sparse path: selection columns (pass 1 +
    pass 2 over pooled keys, bench.py:144-155) plus attended keys
    (bench.py:96-100), each weighted by its FLOPs per column/key."""
    i = np.arange(n, dtype=np.int64)
    v1 = np.where(i + 1 >= cfg.l_C1, (i + 1 - cfg.l_C1) // cfg.s_C1 + 1, 0)
    v2 = np.where(i + 1 >= cfg.l_C2, (i + 1 - cfg.l_C2) // cfg.s_C2 + 1, 0)
    sel = np.where(v2 > 0, v2, v1) + v1                     # pass-1 + pass-2 columns
    b = i // cfg.B
    vis = (np.minimum(b + 1, cfg.budget_blocks) - 1) * cfg.B + (i - b * cfg.B) + 1
    return sel + 2 * vis                                      # attention = QK + PV


def balanced_row_ranges(cfg: AttentionConfig, n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous query-row ranges, aligned to selection blocks, with equal
    estimated cost per rank (context parallelism for one sequence)."""
    cost = row_cost(cfg, n).astype(np.float64)
    csum = np.concatenate([[0.0], np.cumsum(cost)])
    total = csum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        idx = int(np.searchsorted(csum, target))
        idx = int(round(idx / cfg.B)) * cfg.B          # keep query blocks whole
        bounds.append(min(max(idx, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a scalar (timing is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
