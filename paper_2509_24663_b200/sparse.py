"""Block-sparse attention over the selected blocks (reference: sparse.py) -- K4."""

from __future__ import annotations

import torch

from . import _lib
from ._tensors import is_host, to_device_bf16
from .core import AttentionConfig, OpCounter
from .dense import AttentionResult, _finish, check_gqa_shapes
from .selection import BlockSelection


def _check_selection(sel: BlockSelection, n: int, h_kv: int) -> None:
    """sparse.py:26-30."""
    if sel.n != n:
        raise ValueError(f"selection built for n={sel.n}, inputs have n={n}")
    if sel.num_groups != h_kv:
        raise ValueError(f"selection has {sel.num_groups} groups, inputs have h_kv={h_kv}")


def sparse_forward(Q, K, V, sel: BlockSelection, cfg: AttentionConfig,
                   counter: OpCounter | None = None, stats: dict | None = None) -> AttentionResult:
    """sparse.py:43-98 on the GPU: exact online softmax over each token's
    visible blocks, diagonal block causally clipped.  Any BlockSelection:
    rows of the init U local U top-k shape (everything select_blocks /
    build_block_sets produce, and reference-built selections of that shape)
    run on K4 part A (tcgen05 FA tile) + part B (per-token top-k); any other
    selection (e.g. every causal block, or a hand-made fixture) runs on the
    general block-list kernel (swattn_sparse_fwd_lists)."""
    n, h_q, h_kv, d_h = check_gqa_shapes(Q, K, V, cfg)
    _check_selection(sel, n, h_kv)
    host = is_host(Q)
    Qd, Kd, Vd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V")))
    O = torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    form = sel.topk_form(cfg, Qd.device)
    if form is not None:
        topk, cnt = form
        from .selection import Workspace
        ws = Workspace.get(L.swattn_sparse_workspace_bytes(c, n), Qd.device)
        _lib.check(L.swattn_sparse_fwd(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(),
                                       n, topk.data_ptr(), cnt.data_ptr(), O.data_ptr(),
                                       lse.data_ptr(), ws.data_ptr(), ws.numel(),
                                       _lib.stream_handle(Qd.device)),
                   "swattn_sparse_fwd")
    else:
        empty = sel.first_empty_row()
        if empty is not None:   # sparse.py:75-76
            g, i = empty
            raise RuntimeError(f"query {i} in group {g} has an empty visible set")
        blocks, ld, cnt = sel.list_form(Qd.device)
        _lib.check(L.swattn_sparse_fwd_lists(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n,
                                             blocks.data_ptr(), ld, cnt.data_ptr(), O.data_ptr(),
                                             lse.data_ptr(), _lib.stream_handle(Qd.device)),
                   "swattn_sparse_fwd_lists")
    if counter is not None or stats is not None:
        if form is not None:
            cnt = form[1].to(torch.int64)
            i = torch.arange(n, device=cnt.device)
            b = i // cfg.B
            picked = torch.clamp(b + 1, max=cfg.N_init + cfg.N_local) + cnt  # per (g, i)
            visits = ((picked - 1) * cfg.B + (i - b * cfg.B) + 1).cpu().numpy()
        else:
            visits = sel.key_visits()
        if counter is not None:
            total = int(visits.sum())
            counter.add(mac=2 * total * (h_q // h_kv) * d_h, exp=total * (h_q // h_kv))
        if stats is not None:
            stats["key_visits"] = visits
    return _finish(O, lse, host)


def token_visibility_mask(sel: BlockSelection, g: int):
    """sparse.py:33-40 (host bool [n, n]; small n only)."""
    import numpy as np
    mask = np.zeros((sel.n, sel.n), dtype=bool)
    for i in range(sel.n):
        for start, end in sel.visible_spans(g, i):
            mask[i, start:end] = True
    return mask


def sparse_backward(Q, K, V, sel: BlockSelection, dO, cfg: AttentionConfig,
                    counter: OpCounter | None = None):
    """sparse.py:130-185 on the GPU: gradients of sum(O * dO) through the
    masked softmax, recomputing P from the forward's lse (the forward runs
    first, as in the reference, :157-158).  dK / dV reduce in a fixed order
    (bitwise reproducible, :139-143).  Returns (dQ, dK, dV) in Q's storage
    dtype (bf16 tensors on the device for device inputs, numpy bf16 for host
    inputs)."""
    n, h_q, h_kv, d_h = check_gqa_shapes(Q, K, V, cfg)
    _check_selection(sel, n, h_kv)
    if tuple(dO.shape) != tuple(Q.shape):
        raise ValueError(f"dO shape {tuple(dO.shape)} != Q shape {tuple(Q.shape)}")
    host = is_host(Q)
    Qd, Kd, Vd, dOd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V"),
                                                          (dO, "dO")))
    form = sel.topk_form(cfg, Qd.device)
    if form is None:
        raise NotImplementedError("sparse_backward runs on init U local U top-k selections "
                                  "(what select_blocks returns); this selection has another shape")
    topk, topk_cnt = form
    fwd = sparse_forward(Qd, Kd, Vd, sel, cfg)
    dQ = torch.empty_like(Qd)
    dK = torch.empty_like(Kd)
    dV = torch.empty_like(Vd)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    nbytes = L.swattn_sparse_bwd_workspace_bytes(c, n)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=Qd.device)
    _lib.check(L.swattn_sparse_bwd(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n,
                                   topk.data_ptr(), topk_cnt.data_ptr(),
                                   fwd.output.data_ptr(), fwd.lse.data_ptr(), dOd.data_ptr(),
                                   dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(), ws.data_ptr(),
                                   ws.numel(), _lib.stream_handle(Qd.device)),
               "swattn_sparse_bwd")
    if counter is not None:
        cnt = topk_cnt.to(torch.int64)
        i = torch.arange(n, device=cnt.device)
        b = i // cfg.B
        picked = torch.clamp(b + 1, max=cfg.N_init + cfg.N_local) + cnt
        visits = int(((picked - 1) * cfg.B + (i - b * cfg.B) + 1).sum())
        counter.add(mac=4 * visits * (h_q // h_kv) * d_h, exp=visits * (h_q // h_kv))
    if host:
        import ml_dtypes
        import numpy as np
        return tuple(t.cpu().view(torch.int16).numpy().view(ml_dtypes.bfloat16)
                     for t in (dQ, dK, dV))
    return dQ, dK, dV
