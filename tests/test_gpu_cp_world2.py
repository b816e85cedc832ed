"""Sequence-sharded context parallelism at world 2 through real collectives:
two processes (both on cuda:0 -- the test lease has one GPU -- so the
process group is gloo, whose all-gathers take the device tensors) each pass
their rows of Q / K / V to parallel.context_parallel_attend_sharded and must
get back exactly the rows of the whole-sequence attend."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")


def _worker(rank, world, port, n, q):
    import sys

    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2509_24663_b200.core import AttentionConfig, make_qkv
        from paper_2509_24663_b200.parallel import context_parallel_attend_sharded, shard_rows
        from paper_2509_24663_b200.switch import SwitchPolicy, attend
        cfg = AttentionConfig()
        Q, K, V = make_qkv(n, 32, 2, 128, seed=3, device="cuda")
        whole, _ = attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
        a, b = shard_rows(n, world)[rank]
        o, lse, rows = context_parallel_attend_sharded(Q[a:b].clone(), K[a:b].clone(), V[a:b].clone(),
                                                       cfg, n)
        torch.cuda.synchronize()
        ok = tuple(rows) == (a, b) and torch.equal(o, whole.output[a:b]) and torch.equal(lse, whole.lse[a:b])
        q.put((rank, bool(ok), float((o.float() - whole.output[a:b].float()).abs().max())))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("n", [16384, 20000])
def test_cp_sharded_world2_equals_whole(n):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=500)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(ok for _, ok, _ in res), res
