"""Multi-process host logic on CPU (gloo, world_size 2): unit sharding covers
every (sequence, group) exactly once, cost-balanced context-parallel ranges,
and the max-over-ranks timing reduction the bench uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.parallel import (balanced_row_ranges, max_over_ranks, row_cost,
                                            shard_units)


def test_shard_units_cover_once():
    for world in (1, 2, 4, 8):
        seen = [u for r in range(world) for u in shard_units(16, 2, world, r)]
        assert sorted(seen) == [(b, g) for b in range(16) for g in range(2)]


def test_balanced_ranges():
    cfg = AttentionConfig()
    n = 131072
    for world in (2, 4, 8):
        ranges = balanced_row_ranges(cfg, n, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(a % cfg.B == 0 for a, _ in ranges)
        cost = row_cost(cfg, n)
        per = np.array([cost[a:b].sum() for a, b in ranges], dtype=np.float64)
        assert per.max() / per.mean() < 1.01


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard_units(16, 2, world, rank)
        got = [None] * world
        dist.all_gather_object(got, mine)
        flat = sorted(u for part in got for u in part)
        ms = max_over_ranks(10.0 + rank)
        dist.barrier()
        out[rank] = (flat == [(b, g) for b in range(16) for g in range(2)], ms)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharding_and_max_timing():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == (True, 11.0) and res[1] == (True, 11.0)


def test_shard_windows_partition_and_halo():
    """Every pooled window is owned by exactly one shard, and its rows fit in
    the shard plus cp_halo_rows of the next one."""
    from paper_2509_24663_b200.parallel import cp_halo_rows, shard_rows, shard_windows
    cfg = AttentionConfig()
    H = cp_halo_rows(cfg)
    for n in (100, 1000, 4096, 10000, 131072):
        for world in (1, 2, 3, 4, 8):
            bounds = shard_rows(n, world)
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            for length, stride in ((cfg.l_C1, cfg.s_C1), (cfg.l_C2, cfg.s_C2)):
                m = (n - length) // stride + 1 if n >= length else 0
                owned = []
                for a, b in bounds:
                    i0, i1, need = shard_windows(n, length, stride, a, b)
                    owned += list(range(i0, i1))
                    assert need <= min(n, b + H) - a
                assert owned == list(range(m)), (n, world, length)


def _cp_worker(rank, world, port, out):
    """Rank r pools the windows of its shard (+ halo from the gathered shard
    heads) with the oracle's pooling; the all-gathered pieces must equal the
    global pooled keys (the host logic of context_parallel_attend_sharded)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    from oracle import swattn_oracle as O
    from paper_2509_24663_b200.parallel import cp_halo_rows, shard_rows, shard_windows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = AttentionConfig()
        n = 3000
        _, K, _ = O.draw_qkv(n, 32, 2, 128, 7)
        a, b = shard_rows(n, world)[rank]
        H = cp_halo_rows(cfg)
        heads = [None] * world
        dist.all_gather_object(heads, K[a: a + H])           # first rows of every shard
        K_ext = np.concatenate([K[a:b]] + ([heads[rank + 1]] if rank + 1 < world else []))
        ok = True
        for length, stride in ((cfg.l_C1, cfg.s_C1), (cfg.l_C2, cfg.s_C2)):
            i0, i1, need = shard_windows(n, length, stride, a, b)
            mine = O.pool(K_ext[:need], length, stride)[: i1 - i0] if i1 > i0 else None
            parts = [None] * world
            dist.all_gather_object(parts, mine)
            full = np.concatenate([p for p in parts if p is not None])
            ok = ok and np.array_equal(full.view(np.uint16), O.pool(K, length, stride).view(np.uint16))
        out[rank] = ok
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_compressed_keys_allgather():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_cp_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res == {0: True, 1: True}
