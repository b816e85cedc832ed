"""FA tile timing (dense K5 at 32K / 128K, part A at 128K) for A/B of variant libraries."""
import dataclasses, os, sys
import torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
L = _lib.lib(); cfg = AttentionConfig(); c = _lib.c_config(cfg)
c0 = _lib.c_config(dataclasses.replace(cfg, k_top=0))
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
out = {}
for n in (32768, 131072):
    Q, K, V = make_qkv(n, 32, 2, 128, seed=0)
    O = torch.empty_like(Q); lse = torch.empty((n, 32), device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    out[f"dense{n}"] = timed(lambda: L.swattn_dense_fwd(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, 1, O.data_ptr(), lse.data_ptr(), sh))
    if n == 131072:
        ws = torch.empty(L.swattn_sparse_workspace_bytes(c, n), dtype=torch.uint8, device="cuda")
        topk = torch.empty((2, n, 63), dtype=torch.int32, device="cuda"); cnt = torch.zeros((2, n), dtype=torch.int32, device="cuda")
        out["partA128K"] = timed(lambda: L.swattn_sparse_fwd(c0, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, topk.data_ptr(), cnt.data_ptr(), O.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(), sh), 10)
    del Q, K, V, O
print(os.environ.get("SWATTN_B200_LIB", "default").split("/")[-3] if "SWATTN_B200_LIB" in os.environ else "default", {k: round(v, 3) for k, v in out.items()}, flush=True)
