"""Attend at 128K on projected (MiniCPM-like, random weights + RoPE) q/k/v vs
make_qkv inputs: total time, and the selection's re-ranked row count."""
import os, sys
import torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import minicpm_prefill as M
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import attend
from paper_2509_24663_b200.selection import select_blocks
dev = torch.device("cuda"); gen = torch.Generator(device=dev).manual_seed(0)
L = M.Layer(dev, gen); n = 131072; cfg = AttentionConfig()
h = torch.randn(n, M.D, device=dev, generator=gen).to(torch.bfloat16)
cos, sin = M.rope_tables(n, dev)
x = M.rms_norm(h, L.ln1); qkv = x @ L.wqkv.t()
q = M.rope(qkv[:, :4096].view(n, 32, 128), cos, sin).contiguous()
k = M.rope(qkv[:, 4096:4352].view(n, 2, 128), cos, sin).contiguous()
v = qkv[:, 4352:].view(n, 2, 128).contiguous()
del qkv, x, h
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for name, (Q, K, V) in (("model", (q, k, v)), ("make_qkv", make_qkv(n, 32, 2, 128, seed=0))):
    ms = t(lambda: attend(Q, K, V, cfg))
    sel = select_blocks(Q, K, cfg, mode="approx")
    print(name, "attend ms", round(ms, 2), "reranked rows", sel.n_reranked,
          "q std", round(Q.float().std().item(), 3), "k std", round(K.float().std().item(), 3), flush=True)
