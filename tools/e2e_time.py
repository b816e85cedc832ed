"""Time the host-buffer attend (attend_host_chunked: H2D + compute + D2H) at
n = $N, $REPS calls after 2 warm-ups; SWATTN_B200_LIB selects a build."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import attend_host_chunked
n = int(os.environ.get("N", "131072"))
cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
Qh, Kh, Vh = (x.cpu().pin_memory() for x in (Q, K, V))
Oh = torch.empty(Q.shape, dtype=torch.bfloat16).pin_memory()
lh = torch.empty((n, 32), dtype=torch.float32).pin_memory()
for _ in range(2):
    attend_host_chunked(Qh, Kh, Vh, cfg, "approx", out=(Oh, lh))
ts = []
for _ in range(int(os.environ.get("REPS", "5"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    attend_host_chunked(Qh, Kh, Vh, cfg, "approx", out=(Oh, lh))
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("SWATTN_B200_LIB", "current").split("/")[-1], "e2e ms", sorted(ts)[len(ts) // 2], [round(t, 1) for t in ts], flush=True)
