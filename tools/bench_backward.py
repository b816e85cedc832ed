"""Sparse backward (swattn_sparse_bwd, sparse.py:130-185) at n tokens: device
time of the backward alone (forward O / lse precomputed, inputs resident),
its stage split from a CUDA-event bracket around the whole call, and dense
causal attention backward of the same shape through torch SDPA (cuDNN) as
the comparator.  One JSON line per n.
  python tools/bench_backward.py [n ...]
"""
import json
import os
import sys

import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2509_24663_b200 import _lib  # noqa: E402
from paper_2509_24663_b200.core import AttentionConfig, make_qkv  # noqa: E402
from paper_2509_24663_b200.selection import select_blocks  # noqa: E402
from paper_2509_24663_b200.sparse import sparse_forward  # noqa: E402


def timed(fn, reps):
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


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [32768, 131072]
    cfg = AttentionConfig()
    L = _lib.lib()
    c = _lib.c_config(cfg)
    for n in sizes:
        Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
        dO, _, _ = make_qkv(n, 32, 2, 128, seed=1000, device="cuda")
        sel = select_blocks(Q, K, cfg, mode="approx")
        fwd = sparse_forward(Q, K, V, sel, cfg)
        dQ, dK, dV = torch.empty_like(Q), torch.empty_like(K), torch.empty_like(V)
        ws = torch.empty(L.swattn_sparse_bwd_workspace_bytes(c, n), dtype=torch.uint8, device="cuda")
        topk = sel.topk.contiguous()

        def bwd():
            _lib.check(L.swattn_sparse_bwd(c, Q.data_ptr(), K.data_ptr(), V.data_ptr(), n,
                                           topk.data_ptr(), sel.topk_cnt.data_ptr(),
                                           fwd.output.data_ptr(), fwd.lse.data_ptr(), dO.data_ptr(),
                                           dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(),
                                           ws.data_ptr(), ws.numel(),
                                           torch.cuda.current_stream().cuda_stream), "bwd")
        ms = timed(bwd, 3)
        # visits = (token, visible key) pairs per group; 4 matmuls x 2 FLOP x d per head
        cnt = sel.topk_cnt.to(torch.int64)
        i = torch.arange(n, device="cuda")
        b = i // cfg.B
        picked = torch.clamp(b + 1, max=cfg.N_init + cfg.N_local) + cnt
        visits = int(((picked - 1) * cfg.B + (i - b * cfg.B) + 1).sum())
        flop = 2 * 4 * visits * 16 * 128 + 2 * 2 * visits * 16 * 128  # dQ/dK/dV/dP + recomputed S
        line = {"n": n, "sparse_bwd_ms": ms, "tflops_algorithmic": flop / (ms / 1e3) / 1e12,
                "workspace_GB": ws.numel() / 1e9}
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            q = Q.transpose(0, 1)[None].detach().requires_grad_()
            k = K.transpose(0, 1)[None].detach().requires_grad_()
            v = V.transpose(0, 1)[None].detach().requires_grad_()
            g = dO.transpose(0, 1)[None]
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True,
                                                                     enable_gqa=True)

                def dense_bwd():
                    torch.autograd.grad(o, (q, k, v), g, retain_graph=True)
                line["cudnn_dense_bwd_ms"] = timed(dense_bwd, 3)
            line["speedup_vs_cudnn_bwd"] = line["cudnn_dense_bwd_ms"] / ms
        except Exception as e:  # pragma: no cover - comparator unavailable
            line["cudnn_dense_bwd_error"] = str(e)[:160]
        print(json.dumps(line), flush=True)
        del Q, K, V, dO, dQ, dK, dV, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
