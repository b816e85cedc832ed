"""Sparse attend time at n = $N vs the forced FA-tile SM share of the routed tiles."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
cfg = AttentionConfig(); pol = SwitchPolicy(forced_mode="sparse")
n = int(os.environ.get("N", "131072"))
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
def t(reps):
    for _ in range(2): attend(Q, K, V, cfg, pol)
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); attend(Q, K, V, cfg, pol); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return round(ts[len(ts) // 2], 3)
os.environ["SWATTN_ROUTE_PCT"] = os.environ.get("PCT", "45")
os.environ["SWATTN_ROUTE_DEBUG"] = "1"
attend(Q, K, V, cfg, pol); torch.cuda.synchronize()
os.environ["SWATTN_ROUTE_DEBUG"] = "0"
out = {"model": t(5)}
for s in [int(x) for x in os.environ.get("SMS", "0,4,8,12,16,24,32,48,74").split(",")]:
    os.environ["SWATTN_ROUTE_FA_SMS"] = str(s)
    out[s] = t(5)
os.environ["SWATTN_ROUTE_PCT"] = "0"; os.environ.pop("SWATTN_ROUTE_FA_SMS")
out["unrouted"] = t(5)
print(n, out, flush=True)
