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
