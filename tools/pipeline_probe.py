"""Probe: does running selection (K2/K3/re-rank) of row chunk c+1 on one
stream while the sparse attention (part A + part B) of chunk c runs on a
second stream shorten the 128K attend?  Uses only the row-range C-ABI.
  SWATTN_B200_LIB=<variant lib> python tools/pipeline_probe.py [n] [chunks...]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
chunk_counts = [int(x) for x in sys.argv[2:]] or [4, 8, 16]
cfg = AttentionConfig()
L = _lib.lib()
c = _lib.c_config(cfg)
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
dev = Q.device
ws_sel = torch.empty(L.swattn_workspace_bytes(c, n), dtype=torch.uint8, device=dev)
ws_sp = torch.empty(L.swattn_sparse_workspace_bytes(c, n), dtype=torch.uint8, device=dev)
topk = torch.empty((2, n, cfg.k_top), dtype=torch.int32, device=dev)
cnt = torch.empty((2, n), dtype=torch.int32, device=dev)
O = torch.empty_like(Q)
lse = torch.empty((n, 32), dtype=torch.float32, device=dev)
s1 = torch.cuda.current_stream()
s2 = torch.cuda.Stream(priority=-1)


def run(chunks, two_streams=True):
    B = cfg.B
    rows = -(-(-(-n // chunks)) // B) * B
    bounds = [(r, min(n, r + rows)) for r in range(0, n, rows)]
    s2.wait_stream(s1)
    for r0, r1 in bounds:
        _lib.check(L.swattn_select_blocks_rows(c, Q.data_ptr(), K.data_ptr(), n, r0, r1, 2,
                                               topk.data_ptr(), cnt.data_ptr(), None,
                                               ws_sel.data_ptr(), ws_sel.numel(),
                                               s1.cuda_stream), "select")
        st = s2 if two_streams else s1
        if two_streams:
            s2.wait_stream(s1)
        _lib.check(L.swattn_sparse_fwd_rows(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n, r0, r1,
                                            topk.data_ptr(), cnt.data_ptr(), O.data_ptr(),
                                            lse.data_ptr(), ws_sp.data_ptr(), ws_sp.numel(),
                                            st.cuda_stream), "sparse")
    s1.wait_stream(s2)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


ref_ms = timeit(lambda: attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse")))
res, _ = attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
O_ref, lse_ref = res.output.clone(), res.lse.clone()
print(f"lib={os.environ.get('SWATTN_B200_LIB', 'default')} n={n} attend(one stream) {ref_ms:.2f} ms", flush=True)
for ch in chunk_counts:
    t1 = timeit(lambda: run(ch, False))
    t2 = timeit(lambda: run(ch, True))
    same = torch.equal(O, O_ref) and torch.equal(lse, lse_ref)
    print(f"  chunks={ch:3d}: serial {t1:.2f} ms, two streams {t2:.2f} ms, bit-equal={same}", flush=True)
