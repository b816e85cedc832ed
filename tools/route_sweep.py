"""Sparse attend time vs the tile-routing threshold (SWATTN_ROUTE_PCT, read per
call; 0 = every top-k block through part B) at the switch-sweep sizes, and
the output difference against the unrouted path."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
cfg = AttentionConfig()
pol = SwitchPolicy(forced_mode="sparse")


def t(fn, reps):
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts) // 2]


pcts = [int(x) for x in os.environ.get("PCTS", "0,30,45,60,80").split(",")]
for n in [int(x) for x in os.environ.get("NS", "8192,16384,32768,65536,131072").split(",")]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
    row = {"n": n}
    os.environ["SWATTN_ROUTE_PCT"] = "0"
    base, _ = attend(Q, K, V, cfg, pol)
    base_o, base_l = base.output.clone(), base.lse.clone()
    for pct in pcts:
        os.environ["SWATTN_ROUTE_PCT"] = str(pct)
        res, _ = attend(Q, K, V, cfg, pol)
        d = (res.output.float() - base_o.float()).abs()
        row[pct] = {"ms": round(t(lambda: attend(Q, K, V, cfg, pol), 3 if n >= 65536 else 10), 3),
                    "o_max": float(d.max()), "o_mean": float(d.mean()),
                    "lse_max": float((res.lse - base_l).abs().max())}
    print(json.dumps(row), flush=True)
    del Q, K, V, base, base_o, base_l
