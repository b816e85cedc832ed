"""Run one sparse attend (after one warm-up) -- target for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
mode = sys.argv[2] if len(sys.argv) > 2 else "sparse"
cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
for _ in range(2):
    res, m = attend(Q, K, V, cfg, SwitchPolicy(forced_mode=mode))
torch.cuda.synchronize()
print("ok", m, float(res.lse.float().mean()))
