"""Host overhead of switch.attend at small n (dense path): per-call wall time
of 2000 back-to-back calls, and a cProfile of the Python side."""
import cProfile, pstats, sys, os, time
import torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import attend
cfg = AttentionConfig()
Q, K, V = make_qkv(1024, 32, 2, 128, seed=0)
for _ in range(50): attend(Q, K, V, cfg)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2000): attend(Q, K, V, cfg)
torch.cuda.synchronize()
print("us per call", (time.perf_counter() - t) / 2000 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(500): attend(Q, K, V, cfg)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
