"""Per-phase timing of parallel.context_parallel_attend_sharded at world 1 (NCCL)."""
import os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29541")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_2509_24663_b200 import parallel as P
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
cfg = AttentionConfig(); n = 131072
Q, K, V = make_qkv(n, 32, 2, 128, seed=0)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3
print("full sharded call", t(lambda: P.context_parallel_attend_sharded(Q, K, V, cfg, n)))
print("gather K", t(lambda: P._gather_rows(K, 1, n)))
kc = P.cp_local_ckeys(K, cfg, n, 0, n)
print("local ckeys", t(lambda: P.cp_local_ckeys(K, cfg, n, 0, n)))
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.selection import Workspace
L = _lib.lib(); c = _lib.c_config(cfg)
ws = Workspace.get(L.swattn_workspace_bytes(c, n), Q.device)
P.cp_install_ckeys(ws, cfg, n, kc[0], kc[1])
O = torch.empty_like(Q); lse = torch.empty((n, 32), device="cuda")
print("attend rows", t(lambda: P.cp_attend_rows(Q, K, V, cfg, n, 0, n, ws, O, lse)))
dist.destroy_process_group()
