"""K3 A/B: selection digest (topk, counts) and select_blocks / topk kernel time at n = $N."""
import os, sys, torch, hashlib
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.selection import select_blocks
n = int(os.environ.get("N", "131072")); cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=5, device="cuda")
sel = select_blocks(Q, K, cfg, mode="approx"); torch.cuda.synchronize()
dig = hashlib.sha1(sel.topk.cpu().numpy().tobytes() + sel.topk_cnt.cpu().numpy().tobytes()).hexdigest()[:16]
ts = []
for _ in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); select_blocks(Q, K, cfg, mode="approx"); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(os.environ.get("SWATTN_B200_LIB", "cur").split("/")[-1], n, "sel sha1", dig, "select ms", round(sorted(ts)[3], 3), flush=True)
