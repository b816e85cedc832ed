"""One sparse attend at n = $N (for ncu launch lists)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
n = int(os.environ.get("N", "32768"))
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
res, _ = attend(Q, K, V, AttentionConfig(), SwitchPolicy(forced_mode="sparse"))
torch.cuda.synchronize()
