"""Time own dense K5 (swattn_dense_fwd) at several n and the 128K sparse attend
(part A uses the same FA tile).  SWATTN_B200_LIB selects a variant build."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
L = _lib.lib(); cfg = AttentionConfig(); c = _lib.c_config(cfg)
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts) // 2]
out = {}
for n in [4096, 6144, 32768, 131072]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
    O = torch.empty_like(Q); lse = torch.empty((n, 32), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    out[f"dense{n}"] = round(t(lambda: _lib.check(L.swattn_dense_fwd(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, 1, O.data_ptr(), lse.data_ptr(), st), "dense"), 3 if n == 131072 else 10), 4)
    if n == 131072:
        out["sparse128K"] = round(t(lambda: attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))), 3)
print(os.environ.get("SWATTN_B200_LIB", "base").split("/")[-1], out, flush=True)
