"""Interleaved A/B of sparse attend at n = $N over environment variants
(rounds x variants, 3 calls each; medians), e.g.
  VARIANTS='base:SWATTN_ROUTE_PCT=0;r45:SWATTN_ROUTE_PCT=45' N=131072 python tools/route_ab.py"""
import os, sys, json, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
cfg = AttentionConfig(); pol = SwitchPolicy(forced_mode="sparse")
n = int(os.environ.get("N", "131072"))
rounds = int(os.environ.get("ROUNDS", "6"))
variants = []
for v in os.environ["VARIANTS"].split(";"):
    name, _, kv = v.partition(":")
    variants.append((name, dict(x.split("=") for x in kv.split(",") if x)))
Q, K, V = make_qkv(n, 32, 2, 128, seed=int(os.environ.get("SEED", "0")), device="cuda")
keys = {k for _, d in variants for k in d}
def setenv(d):
    for k in keys: os.environ.pop(k, None)
    os.environ.update(d)
res = {name: [] for name, _ in variants}
for name, d in variants:
    setenv(d); attend(Q, K, V, cfg, pol)
torch.cuda.synchronize()
for r in range(rounds):
    for name, d in variants:
        setenv(d)
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); attend(Q, K, V, cfg, pol); b.record(); torch.cuda.synchronize()
            res[name].append(a.elapsed_time(b))
out = {name: round(sorted(v)[len(v) // 2], 3) for name, v in res.items()}
print(json.dumps({"n": n, "median_ms": out, "min_ms": {k: round(min(v), 3) for k, v in res.items()}}), flush=True)
