"""Read the part-B role cycle accounting of a -DSWATTN_PB_PROFILE variant:
  SWATTN_B200_LIB=tools/variants/prof/lib/libswattn_b200.so python tools/pb_profile.py 131072"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.selection import select_blocks
from paper_2509_24663_b200.sparse import sparse_forward

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
sel = select_blocks(Q, K, cfg, mode="approx")
L = _lib.lib()
buf = (ctypes.c_ulonglong * 32)()
sparse_forward(Q, K, V, sel, cfg)
L.swattn_debug_pb_profile(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sparse_forward(Q, K, V, sel, cfg)
e1.record()
torch.cuda.synchronize()
L.swattn_debug_pb_profile(buf, 1)
a = np.array(list(buf), dtype=np.float64).reshape(4, 8)
cnt = sel.topk_cnt.long()
pairs = int(((cnt + 1) // 2).sum())
sms = torch.cuda.get_device_properties(0).multi_processor_count
print(f"n={n} sparse_forward {e0.elapsed_time(e1):.2f} ms; pairs {pairs} ({pairs / sms:.0f}/SM)")
names = {0: ("K producer x3 warps", ["total", "wait empty", "wait q_empty"]),
         1: ("V producer x3 warps", ["total", "wait empty"]),
         2: ("MMA warp", ["total", "idle->PV", "idle->S", "#PV", "#S"]),
         3: ("softmax x4 warps", ["total", "wait s_full", "wait p_empty", "wait o_full", "S ld", "P store"])}
warps = {0: 3, 1: 3, 2: 1, 3: 4}
for r in range(4):
    nm, keys = names[r]
    per = a[r] / (warps[r] * sms)
    txt = ", ".join(f"{k} {per[i] / (pairs / sms) if not k.startswith('#') else per[i]:.0f}" for i, k in enumerate(keys))
    print(f"{nm}: cycles per pair: {txt}")
