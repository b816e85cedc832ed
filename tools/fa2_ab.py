"""Interleaved A/B of dense causal FA: one-tile (SWATTN_FA2=0) vs two-tile (1)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
L = _lib.lib(); cfg = AttentionConfig(); c = _lib.c_config(cfg)
for n in [int(x) for x in os.environ.get("NS", "2048,4096,6144,16384,32768,65536,131072").split(",")]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=1, device="cuda")
    O = torch.empty_like(Q); lse = torch.empty((n, 32), dtype=torch.float32, device="cuda")
    def run(v):
        os.environ["SWATTN_FA2"] = str(v)
        _lib.check(L.swattn_dense_fwd(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, 1, O.data_ptr(), lse.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream), "dense")
    res = {0: [], 1: []}
    reps = 2 if n >= 65536 else 6
    for v in (0, 1): run(v)
    torch.cuda.synchronize()
    for r in range(4):
        for v in ((0, 1) if r % 2 == 0 else (1, 0)):
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); run(v); b.record(); torch.cuda.synchronize(); res[v].append(a.elapsed_time(b))
    med = {v: sorted(x)[len(x) // 2] for v, x in res.items()}
    print(n, "one-tile", round(med[0], 4), "two-tile", round(med[1], 4), "ratio", round(med[1] / med[0], 3), flush=True)
