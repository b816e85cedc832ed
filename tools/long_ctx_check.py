"""attend beyond the BASELINE sizes: n = 256K (the compiled top-k candidate
bound, 4096 blocks) runs and matches the float64 oracle on sampled rows;
n = 320K fails loudly (no silent fallback).  Test infrastructure."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ml_dtypes
from oracle import swattn_oracle as O
from paper_2509_24663_b200.core import AttentionConfig, make_qkv, SwattnError
from paper_2509_24663_b200.switch import SwitchPolicy, attend
from paper_2509_24663_b200.selection import select_blocks

cfg = AttentionConfig()
for n in [int(x) for x in sys.argv[1:]] or [262144, 393216, 524288, 557056]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=3, device="cuda")
    try:
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        res, mode = attend(Q, K, V, cfg)
        a.record(); res, mode = attend(Q, K, V, cfg); b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        sel = select_blocks(Q, K, cfg, mode="approx")
        bf = ml_dtypes.bfloat16
        Qh = Q.view(torch.int16).cpu().numpy().view(bf); Kh = K.view(torch.int16).cpu().numpy().view(bf)
        Vh = V.view(torch.int16).cpu().numpy().view(bf)
        rows = np.array([n - 1, n - 5000, n // 2 + 77, 70000, 300001 if n > 300001 else 1000])
        ck1, ck2 = O.pool(Kh, 32, 16), O.pool(Kh, 128, 64)
        top, _, _ = O.select(Qh, Kh, O.PAPER, rows=rows, ck1=ck1, ck2=ck2)
        got = sel.topk.cpu().numpy()[:, rows]
        full = np.full((2, n, cfg.k_top), -1, dtype=np.int64); full[:, rows] = top
        o, l = O.sparse_attention(Qh, Kh, Vh, full, O.PAPER, rows=rows)
        err = np.abs(res.output[torch.as_tensor(rows, device="cuda")].float().cpu().numpy() - o)
        print(f"n={n}: {mode} {ms:.1f} ms, sampled selections equal {np.array_equal(got, top)}, "
              f"O max-abs {err.max():.2e}", flush=True)
    except (SwattnError, NotImplementedError) as e:
        print(f"n={n}: raised {type(e).__name__}: {e}", flush=True)
    del Q, K, V
    torch.cuda.empty_cache()
