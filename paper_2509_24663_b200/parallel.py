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


def group_cp_plan(cfg: AttentionConfig, n: int, world: int, rank: int):
    """Work of `rank` when ONE sequence is split over `world` GPUs: KV groups
    first (independent end to end: no collective), then cost-balanced query
    row ranges within a group (context parallelism over replicated K/V).
    Returns ((g0, g1), (r0, r1))."""
    h_kv = cfg.h_kv
    if world >= h_kv and world % h_kv == 0:
        g = rank % h_kv
        per_group = world // h_kv
        return (g, g + 1), balanced_row_ranges(cfg, n, per_group)[rank // h_kv]
    return (0, h_kv), balanced_row_ranges(cfg, n, world)[rank]


def group_cp_attend(Qd, Kd, Vd, cfg: AttentionConfig, world: int, rank: int,
                    selection_mode: str = "approx", O=None, lse=None, ws=None):
    """Sparse branch of attend for this rank's share of one sequence
    (group_cp_plan): swattn_attend_rows_groups on the full, replicated
    tensors; only the rank's heads x rows of O / lse are written.  The
    compressed keys are pooled by every rank that does not start at row 0
    (K1: 0.03 ms at 128K, cheaper than any exchange).  No collective.
    Returns (O, lse, (g0, g1), (r0, r1))."""
    import torch

    from . import _lib
    from .selection import Workspace
    n, h_q, d_h = Qd.shape
    (g0, g1), (r0, r1) = group_cp_plan(cfg, n, world, rank)
    O = O if O is not None else torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = lse if lse is not None else torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = ws if ws is not None else Workspace.get(L.swattn_workspace_bytes(c, n), Qd.device)
    sh = _lib.stream_handle(Qd.device)
    if r1 > r0:
        if r0 > 0:
            _lib.check(L.swattn_attend_prepare(c, Kd.data_ptr(), n, ws.data_ptr(), ws.numel(), sh),
                       "swattn_attend_prepare")
        _lib.check(L.swattn_attend_rows_groups(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n,
                                               r0, r1, g0, g1, _lib.SELECT_MODE[selection_mode],
                                               O.data_ptr(), lse.data_ptr(), ws.data_ptr(),
                                               ws.numel(), sh), "swattn_attend_rows_groups")
    return O, lse, (g0, g1), (r0, r1)


# ---------------------------------------------------------------------------
# Context parallelism with sequence-sharded inputs: rank r
# holds rows [a_r, b_r) of Q, K and V.  Each rank pools the compressed-key
# windows that START in its shard (K1 on its rows plus a halo of at most
# l - s rows from the next shard), the per-rank pieces are all-gathered into
# the full K_C1 / K_C2 (5.2 MB at 128K), and selection (K2, K3) of the
# rank's rows runs on them while K / V are all-gathered on a second stream
# (K4 reads selected blocks anywhere in the past).  Outputs stay sharded.


def shard_rows(n: int, world: int, align: int = 64) -> list[tuple[int, int]]:
    """Contiguous, near-equal token shards whose starts are multiples of
    `align` (a multiple of B and of both pooling strides)."""
    per = -(-(-(-n // world)) // align) * align
    return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]


def shard_windows(n: int, length: int, stride: int, a: int, b: int) -> tuple[int, int, int]:
    """Pooled windows (compression.py:64-78) owned by shard [a, b): those whose
    start i*stride lies in [a, b) and that are complete (end <= n).  Returns
    (i0, i1, rows_needed): windows [i0, i1) need K rows [a, a + rows_needed)."""
    m = (n - length) // stride + 1 if n >= length else 0
    i0 = min(-(-a // stride), m)
    i1 = min(-(-b // stride), m)
    need = (i1 - 1) * stride + length - a if i1 > i0 else 0
    return i0, i1, need


def cp_halo_rows(cfg: AttentionConfig) -> int:
    """Rows of the next shard a rank needs to finish its last windows."""
    return max(cfg.l_C1 - cfg.s_C1, cfg.l_C2 - cfg.s_C2, 0)


def cp_local_ckeys(K_ext, cfg: AttentionConfig, n: int, a: int, b: int):
    """K1 on this rank's rows (+ halo): K_ext = K[a : a + len] with len >=
    every window end it owns.  Returns (kc1_part, kc2_part) = K_C1[i0:i1],
    K_C2[j0:j1] of the whole sequence (bit-identical to the global K1: the
    windows are the same rows)."""
    import torch

    from . import _lib
    i0, i1, need1 = shard_windows(n, cfg.l_C1, cfg.s_C1, a, b)
    j0, j1, need2 = shard_windows(n, cfg.l_C2, cfg.s_C2, a, b)
    h_kv, d = K_ext.shape[1], K_ext.shape[2]
    dev = K_ext.device
    if i1 <= i0 and j1 <= j0:
        e = torch.empty((0, h_kv, d), dtype=torch.bfloat16, device=dev)
        return e, e
    L_ext = max(need1, need2)
    if K_ext.shape[0] < L_ext:
        raise ValueError(f"shard [{a}, {b}) needs {L_ext} rows of K, got {K_ext.shape[0]}")
    K_ext = K_ext[:L_ext].contiguous()
    m1 = max(0, (L_ext - cfg.l_C1) // cfg.s_C1 + 1) if L_ext >= cfg.l_C1 else 0
    m2 = max(0, (L_ext - cfg.l_C2) // cfg.s_C2 + 1) if L_ext >= cfg.l_C2 else 0
    kc1 = torch.empty((max(m1, 1), h_kv, d), dtype=torch.bfloat16, device=dev)
    kc2 = torch.empty((max(m2, 1), h_kv, d), dtype=torch.bfloat16, device=dev)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    _lib.check(L.swattn_compress_keys(c, K_ext.data_ptr(), L_ext, kc1.data_ptr(), kc2.data_ptr(),
                                      _lib.stream_handle(dev)), "swattn_compress_keys")
    # window w of K_ext starts at global row a + w*s = (i0 + w) * s (a is stride-aligned)
    return kc1[: i1 - i0], kc2[: j1 - j0]


def cp_install_ckeys(ws, cfg: AttentionConfig, n: int, kc1_full, kc2_full) -> None:
    """Copy the assembled compressed keys into the attend workspace slots."""
    import ctypes

    from . import _lib
    L = _lib.lib()
    p1, p2 = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(L.swattn_workspace_ckeys(_lib.c_config(cfg), n, ws.data_ptr(), ctypes.byref(p1),
                                        ctypes.byref(p2)), "swattn_workspace_ckeys")
    base = ws.data_ptr()
    for ptr, src in ((p1.value, kc1_full), (p2.value, kc2_full)):
        nbytes = src.numel() * 2
        if nbytes:
            off = ptr - base
            ws[off: off + nbytes].view(src.dtype).view(src.shape).copy_(src)


def cp_attend_rows(Q_sh, K_full, V_full, cfg: AttentionConfig, n: int, a: int, b: int, ws,
                   O_sh, lse_sh, selection_mode: str = "approx", kv_ready=None) -> None:
    """Sparse branch of attend for this rank's rows [a, b), reading Q and
    writing O / lse through their shard tensors (row r lives at r - a; the
    kernels only touch rows of [a, b)), with the compressed keys already
    installed.  `kv_ready`: an event the K4 launch waits for (K / V
    all-gather on a side stream); selection does not need K / V."""
    import torch

    from . import _lib
    L = _lib.lib()
    c = _lib.c_config(cfg)
    dev = Q_sh.device
    st = torch.cuda.current_stream(dev)
    if b <= a:
        return
    h_q, d = Q_sh.shape[1], Q_sh.shape[2]
    q_base = Q_sh.data_ptr() - a * h_q * d * 2          # virtual row-0 base
    o_base = O_sh.data_ptr() - a * h_q * d * 2
    l_base = lse_sh.data_ptr() - a * h_q * 4
    h_kv = K_full.shape[1]
    topk = torch.empty((h_kv, n, max(cfg.k_top, 1)), dtype=torch.int32, device=dev)
    cnt = torch.empty((h_kv, n), dtype=torch.int32, device=dev)
    sel_ws = ws
    sp_ws = torch.empty(L.swattn_sparse_workspace_bytes(c, n), dtype=torch.uint8, device=dev)
    mode = _lib.SELECT_MODE[selection_mode] | _lib.SELECT_PREPARED
    _lib.check(L.swattn_select_blocks_rows(c, q_base, K_full.data_ptr(), n, a, b, mode,
                                           topk.data_ptr(), cnt.data_ptr(), None,
                                           sel_ws.data_ptr(), sel_ws.numel(), st.cuda_stream),
               "swattn_select_blocks_rows")
    if kv_ready is not None:
        st.wait_event(kv_ready)
    _lib.check(L.swattn_sparse_fwd_rows(c, q_base, K_full.data_ptr(), V_full.data_ptr(), n, a, b,
                                        topk.data_ptr(), cnt.data_ptr(), o_base, l_base,
                                        sp_ws.data_ptr(), sp_ws.numel(), st.cuda_stream),
               "swattn_sparse_fwd_rows")


def _gather_rows(part, world: int, rows_max: int):
    """all-gather of variable-length row blocks (padded to rows_max)."""
    import torch
    import torch.distributed as dist
    pad = torch.zeros((rows_max,) + tuple(part.shape[1:]), dtype=part.dtype, device=part.device)
    pad[: part.shape[0]].copy_(part)
    out = torch.empty((world * rows_max,) + tuple(part.shape[1:]), dtype=part.dtype,
                      device=part.device)
    dist.all_gather_into_tensor(out, pad)
    return out


def context_parallel_attend_sharded(Q_sh, K_sh, V_sh, cfg: AttentionConfig, n: int,
                                    selection_mode: str = "approx"):
    """Sequence-sharded context parallelism over torch.distributed (NCCL on
    GPUs).  Rank r passes its rows shard_rows(n, world)[r] of Q, K, V and gets
    back its rows of O and lse.  Collectives: the K halo (<= 64 rows), the
    compressed keys (5.2 MB at 128K) and K / V (K4's gather source; overlapped
    with selection on a side stream).  Returns (O_sh, lse_sh, (a, b))."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .selection import Workspace
    world, rank = dist.get_world_size(), dist.get_rank()
    bounds = shard_rows(n, world)
    a, b = bounds[rank]
    per = max(hi - lo for lo, hi in bounds)
    dev = Q_sh.device
    h_q, d = Q_sh.shape[1], Q_sh.shape[2]
    h_kv = K_sh.shape[1]
    # K / V all-gather on a side stream: only K4 needs them
    comm = torch.cuda.Stream(device=dev)
    comm.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(comm):
        K_all = _gather_rows(K_sh, world, per)
        V_all = _gather_rows(V_sh, world, per)
        kv_ready = torch.cuda.Event()
        kv_ready.record(comm)
    # halo: the first rows of every shard
    H = cp_halo_rows(cfg)
    heads = _gather_rows(K_sh[:H], world, H).view(world, H, h_kv, d)
    K_ext = torch.cat([K_sh, heads[rank + 1]]) if rank + 1 < world else K_sh
    kc1_p, kc2_p = cp_local_ckeys(K_ext, cfg, n, a, b)
    w1 = [shard_windows(n, cfg.l_C1, cfg.s_C1, lo, hi) for lo, hi in bounds]
    w2 = [shard_windows(n, cfg.l_C2, cfg.s_C2, lo, hi) for lo, hi in bounds]
    r1 = max(max(i1 - i0 for i0, i1, _ in w1), 1)
    r2 = max(max(i1 - i0 for i0, i1, _ in w2), 1)
    g1 = _gather_rows(kc1_p, world, r1).view(world, r1, h_kv, d)
    g2 = _gather_rows(kc2_p, world, r2).view(world, r2, h_kv, d)
    kc1 = torch.cat([g1[r, : i1 - i0] for r, (i0, i1, _) in enumerate(w1)])
    kc2 = torch.cat([g2[r, : i1 - i0] for r, (i0, i1, _) in enumerate(w2)])
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = Workspace.get(L.swattn_workspace_bytes(c, n), dev)
    cp_install_ckeys(ws, cfg, n, kc1, kc2)
    O_sh = torch.empty((b - a, h_q, d), dtype=torch.bfloat16, device=dev)
    lse_sh = torch.empty((b - a, h_q), dtype=torch.float32, device=dev)
    # K_all / V_all are [world*per, ...]; shard r starts at r*per = bounds[r][0]
    cp_attend_rows(Q_sh, K_all, V_all, cfg, n, a, b, ws, O_sh, lse_sh, selection_mode,
                   kv_ready=kv_ready)
    torch.cuda.current_stream(dev).wait_stream(comm)
    return O_sh, lse_sh, (a, b)
