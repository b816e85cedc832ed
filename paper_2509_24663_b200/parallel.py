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


def context_parallel_attend(Qd, Kd, Vd, cfg: AttentionConfig, world: int, rank: int,
                            selection_mode: str = "approx", O=None, lse=None):
    """Rows of one long sequence split across ranks (context parallelism).

    Every rank holds Q/K/V of the whole sequence on its device (K/V are
    67 MB each at 128K; selected blocks reach anywhere in the past), builds
    the compressed keys itself (K1, 0.03 ms -- cheaper than any exchange) and
    computes the sparse branch of attend for its cost-balanced query-row
    range with swattn_attend_rows.  Outputs are row-disjoint: rank r owns
    O[r0:r1], lse[r0:r1]; nothing is reduced.  Returns (O, lse, (r0, r1))."""
    import torch

    from . import _lib
    from .selection import Workspace
    n, h_q, d_h = Qd.shape
    r0, r1 = balanced_row_ranges(cfg, n, world)[rank]
    O = O if O is not None else torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = lse if lse is not None else torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = Workspace.get(L.swattn_workspace_bytes(c, n), Qd.device)
    sh = _lib.stream_handle(Qd.device)
    if r1 > r0:
        if r0 > 0:
            _lib.check(L.swattn_attend_prepare(c, Kd.data_ptr(), n, ws.data_ptr(), ws.numel(), sh),
                       "swattn_attend_prepare")
        _lib.check(L.swattn_attend_rows(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n, r0, r1,
                                        _lib.SELECT_MODE[selection_mode], O.data_ptr(),
                                        lse.data_ptr(), ws.data_ptr(), ws.numel(), sh),
                   "swattn_attend_rows")
    return O, lse, (r0, r1)
