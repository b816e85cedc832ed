#!/bin/bash
# r02ae: top-k fused into K2's epilogue (row f1) -- parity (goldens, every row 32K/128K), A/B timing
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 > gpurun_out/r02ae_pytest.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02ae_pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -x --timeout 1000 > gpurun_out/r02ae_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "mismatch|decode|passed|failed|Error" gpurun_out/r02ae_fullsize.log | tail -5
cat > /tmp/t_sel.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
from paper_2509_24663_b200.selection import select_blocks
n = 131072; cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
def t(f, reps=8):
    for _ in range(3): f()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return round(ts[len(ts)//2], 3)
sel = lambda: select_blocks(Q, K, cfg, mode="approx")
att = lambda: attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
print(sys.argv[1], "select_blocks ms", t(sel), "attend ms", t(att), "reranked", int(sel().n_reranked.item()))
PY
python /tmp/t_sel.py fused
SWATTN_K2_TOPK=0 python /tmp/t_sel.py separate_K3
python /tmp/t_sel.py fused
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scores_tc|topk|rerank" --csv python tools/one_attend.py 131072 > gpurun_out/r02ae_launches.csv 2>&1; python3 -c "import csv;[print(r[4][:40], r[-1]) for r in csv.reader(open('gpurun_out/r02ae_launches.csv')) if len(r)>14 and ('scores_tc' in r[4] or 'topk' in r[4] or 'rerank' in r[4])]"
