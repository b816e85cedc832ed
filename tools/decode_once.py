"""Small decode run for compute-sanitizer: 3 sequences (one empty slot), bulk
append, 70 one-token appends (page crossings, an idle sequence), decode steps."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.decode import PagedKVCache, decode_step
cfg = AttentionConfig()
g = torch.Generator(device="cuda").manual_seed(0)
cache = PagedKVCache(cfg, batch=4, max_pages=48, seed=1)
for b, L in enumerate([2000, 130, 0, 2500]):
    if L:
        K = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
        cache.append(b, K, torch.randn_like(K))
for t in range(70):
    Kt = torch.randn((4, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    act = np.array([True, t % 7 != 0, t >= 5, True])
    cache.append_tokens(Kt, torch.randn_like(Kt), active=act)
    if t % 10 == 9:
        q = torch.randn((4, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
        res = decode_step(cache, q)
torch.cuda.synchronize()
print("ok decode", cache.lens_h.tolist(), float(res.lse[0].float().mean()))
