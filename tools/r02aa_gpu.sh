#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
cat > /tmp/t_ab.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
n = 131072; cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
f = lambda: attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort(); print(sys.argv[1], "attend ms median", round(ts[len(ts)//2], 2), "min", round(ts[0], 2))
PY
python /tmp/t_ab.py base
for c in 128 120 112; do SWATTN_EXP_AB=1 SWATTN_PB_CTAS=$c python /tmp/t_ab.py "concurrent_A pb=$c"; done
