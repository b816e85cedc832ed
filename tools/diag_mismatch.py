"""Diagnose (group, row) selections where the GPU and the float64 torch
restatement disagree at 128K: print the GPU, torch-f64 and numpy-oracle picks
and the float64 scores around the k-th boundary.  Test infrastructure."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ml_dtypes
from oracle import swattn_oracle as O
from oracle import torch_f64
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.selection import select_blocks

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
pairs = [tuple(map(int, p.split(':'))) for p in sys.argv[2:]] or [(0, 43398), (0, 108176), (1, 74855)]
cfg = AttentionConfig()
Qd, Kd, _ = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
sel = select_blocks(Qd, Kd, cfg, mode="approx")
gpu = sel.topk.long().cpu().numpy()
bf = ml_dtypes.bfloat16
Q = Qd.view(torch.int16).cpu().numpy().view(bf)
K = Kd.view(torch.int16).cpu().numpy().view(bf)
ck1, ck2 = O.pool(K, 32, 16), O.pool(K, 128, 64)
for g, r in pairs:
    rows = np.array([r])
    top, _, scmp = O.select(Q, K, O.PAPER, rows=rows, ck1=ck1, ck2=ck2)
    r0 = r - r % 256
    t64, s64 = torch_f64.select_f64(Qd[: r0 + 256], Kd, cfg, rows_per_chunk=256, return_scores=True)
    tf = t64[g, r].cpu().numpy()
    sf = s64[g, r].cpu().numpy()
    sn = scmp[0, g]
    b = r // 64
    hi = min(max(0, b - 31), sn.shape[0])
    cand = np.arange(1, hi)
    order = np.lexsort((cand, -sn[1:hi]))
    k = 63
    print(f"(g={g}, row={r}) gpu==numpy {np.array_equal(gpu[g, r], top[g, 0])} f64torch==numpy {np.array_equal(tf, top[g, 0])}")
    print("  gpu-only", sorted(set(gpu[g, r]) - set(top[g, 0])), "numpy-only", sorted(set(top[g, 0]) - set(gpu[g, r])),
          "torch-only", sorted(set(tf) - set(top[g, 0])))
    for j in range(k - 3, k + 3):
        blk = cand[order[j]]
        print(f"   rank {j:2d} block {blk:5d} numpy {sn[blk]!r} torch {sf[blk]!r}")
