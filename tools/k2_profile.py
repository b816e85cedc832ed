"""Epilogue-warp cycle accounting of K2 (variant built with -DSWATTN_K2_PROFILE):
  SWATTN_B200_LIB=tools/variants/k2prof/lib/libswattn_b200.so python tools/k2_profile.py 131072"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.selection import select_blocks

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = AttentionConfig()
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
L = _lib.lib()
buf = (ctypes.c_ulonglong * 8)()
select_blocks(Q, K, cfg, mode="approx")
L.swattn_debug_k2_profile(buf, 1)
select_blocks(Q, K, cfg, mode="approx")
torch.cuda.synchronize()
L.swattn_debug_k2_profile(buf, 1)
a = np.array(list(buf), dtype=np.float64)
warps = 4  # epilogue warps per CTA (lane 0 of each adds)
u1, u2 = a[5] / warps, a[6] / warps
units = u1 + u2
print(f"n={n}: pass-1 units {u1:.0f}, pass-2 tiles {u2:.0f}")
print("epilogue-warp cycles per unit: total %.0f | wait p1 %.0f (per p1 unit %.0f) | wait p2 %.0f (per tile %.0f) | "
      "p2 compute %.0f/tile | pool+sync %.0f/tile" % (
          a[0] / warps / units, a[1] / warps / units, a[1] / warps / max(u1, 1), a[2] / warps / units,
          a[2] / warps / max(u2, 1), a[3] / warps / max(u2, 1), a[4] / warps / max(u2, 1)))
