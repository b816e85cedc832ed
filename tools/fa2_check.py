"""Two-tile dense FA (SWATTN_FA2=1) vs the one-tile kernel: outputs and time."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
L = _lib.lib(); cfg = AttentionConfig(); c = _lib.c_config(cfg)
def run(Q, K, V, n, causal, fa2):
    os.environ["SWATTN_FA2"] = str(fa2)
    O = torch.empty_like(Q); lse = torch.empty((n, 32), dtype=torch.float32, device="cuda")
    _lib.check(L.swattn_dense_fwd(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, causal, O.data_ptr(), lse.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream), "dense")
    return O, lse
def t(fn, reps):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return round(sorted(ts)[len(ts) // 2], 4)
for n in [int(x) for x in os.environ.get("NS", "1000,4096,32768,131072").split(",")]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=1, device="cuda")
    for causal in ([1, 0] if n <= 4096 else [1]):
        o1, l1 = run(Q, K, V, n, causal, 0)
        reps = 3 if n >= 131072 else 10
        line = [n, "causal" if causal else "full", "one-tile ms", t(lambda: run(Q, K, V, n, causal, 0), reps)]
        for v in (1, 2):
            o2, l2 = run(Q, K, V, n, causal, v)
            torch.cuda.synchronize()
            d = (o1.float() - o2.float()).abs()
            line += [f"fa2={v}", "max|dO|", float(d.max()), "mean", float(d.mean()),
                     "max|dlse|", float((l1 - l2).abs().max()), "ms", t(lambda: run(Q, K, V, n, causal, v), reps)]
        print(*line, flush=True)
