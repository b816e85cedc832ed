"""For the decode bench's rows (tools/bench_decode.py inputs): the float64
k-th / (k+1)-th boundary gap of each (sequence, group) row and whether an
exact tie straddles it -- i.e. which rows the float64 re-rank must settle.
Test infrastructure (imports the oracle)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ml_dtypes
from oracle import swattn_oracle as O

B, L = 16, 131072
g = torch.Generator(device="cuda").manual_seed(0)
bf = ml_dtypes.bfloat16
rows = []
for b in range(B):
    K = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    V = torch.randn((L, 2, 128), generator=g, device="cuda").to(torch.bfloat16)
    rows.append(K.view(torch.int16).cpu().numpy().view(bf))
    del K, V
q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16).view(torch.int16).cpu().numpy().view(bf)
t = L - 1
for b in range(B):
    K = rows[b]
    ck1, ck2 = O.pool(K, 32, 16), O.pool(K, 128, 64)
    Q = np.broadcast_to(q[b], (1,) + q[b].shape)
    class _Q:
        shape = (L, 32, 128)
        def __getitem__(self, idx):
            r = np.asarray(idx); return np.broadcast_to(q[b], r.shape + q[b].shape)
    S, nv = O.shared_scores(_Q(), K, O.PAPER, "approx", rows=np.array([t]), ck1=ck1, ck2=ck2)
    sc = O.block_scores(S, 5, 4)[0]
    bb = t // 64
    hi = min(max(0, bb - 31), sc.shape[1])
    for gg in range(2):
        v = np.sort(sc[gg, 1:hi])[::-1]
        kth, nxt = v[62], v[63]
        rel = (kth - nxt) / abs(kth)
        print(f"seq {b:2d} g {gg}: gap {rel:.3g}{'  <-- FLAG' if rel <= 3e-6 else ''}", flush=True)
