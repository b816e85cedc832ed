"""e2e (host buffers) at 128K vs the host pipeline's chunk size."""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200 import switch
cfg = AttentionConfig(); n = 131072
Q, K, V = make_qkv(n, 32, 2, 128, seed=0)
Qh, Kh, Vh = (x.cpu().pin_memory() for x in (Q, K, V))
Oh = torch.empty(Q.shape, dtype=Q.dtype).pin_memory(); lh = torch.empty((n, 32)).pin_memory()
for rows in (None, 4096, 6144, 12288, 16384):
    def f(): switch.attend_host_chunked(Qh, Kh, Vh, cfg, "approx", out=(Oh, lh), chunk_rows=rows)
    f(); f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(4): f()
    b.record(); torch.cuda.synchronize()
    print(rows, a.elapsed_time(b) / 4, flush=True)
