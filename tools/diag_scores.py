"""GPU diagnostic: S^cmp relative error of K2 vs the float64 oracle on sampled
rows, and how many rows the float64 boundary re-rank resolves."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import swattn_oracle as O
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.compression import mean_pool_keys
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.selection import select_blocks

cfg = AttentionConfig()
L = _lib.lib()
c = _lib.c_config(cfg)
for n in [int(x) for x in (sys.argv[1:] or ["16384", "131072"])]:
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 7)
    dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    Qd, Kd = dev(Q), dev(K)
    c1 = mean_pool_keys(Kd, 32, 16).keys
    c2 = mean_pool_keys(Kd, 128, 64).keys
    m1 = c1.shape[0]
    n_cols = -(-m1 // 4)
    ld = (n_cols + 3) // 4 * 4
    scmp = torch.zeros((2, n, ld), dtype=torch.float32, device="cuda")
    _lib.check(L.swattn_block_scores(c, Qd.data_ptr(), c1.data_ptr(), c2.data_ptr(), n, 2,
                                     scmp.data_ptr(), ld, None, _lib.stream_handle()), "k2")
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(0).choice(np.arange(2112, n), size=64, replace=False))
    S, _ = O.shared_scores(Q, K, O.PAPER, "approx", rows=rows)
    want = O.block_scores(S, 5, 4)
    got = scmp.cpu().numpy()[:, rows, :n_cols].transpose(1, 0, 2)
    rel = []
    for ri, i in enumerate(rows):
        hi = min(i // 64 - 31, n_cols)
        w = want[ri, :, 1:hi]
        rel.append(np.abs(got[ri, :, 1:hi] - w) / np.abs(w))
    rel = np.concatenate([r.ravel() for r in rel])
    print(f"n={n}: S^cmp rel err max {rel.max():.3e} p99.99 {np.quantile(rel, 0.9999):.3e} "
          f"median {np.median(rel):.3e}; reranked rows {int(sel.n_reranked)} of {2 * n}")
