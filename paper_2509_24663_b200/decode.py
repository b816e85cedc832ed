"""Decode over a paged KV cache (kernel family K6, csrc/decode.cu).

The reference has no decode entry point; its semantics are
those of the last row of ``attend``'s sparse branch: for a sequence of L
cached tokens, the new token t = L-1 selects init U local U top-k blocks
exactly as ``select_blocks(mode="approx")`` would for row t
(selection.py:93-136, 279-348), then attends over them (sparse.py:43-98).

Layout: pages of B = 64 tokens (one selection block = one page),
``k_pages``/``v_pages`` [num_pages, 64, h_kv, d_h] bf16, ``block_table``
[batch, max_pages] int32, ``seq_lens`` [batch] int32 (device).  Compressed
keys live in per-sequence slabs appended as pooling windows complete.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .core import AttentionConfig, validate_config
from .dense import AttentionResult


class PagedKVCache:
    """Device-resident paged K/V cache plus compressed-key slabs."""

    def __init__(self, cfg: AttentionConfig, batch: int, max_pages: int, num_pages: int | None = None,
                 device="cuda", seed: int | None = None):
        validate_config(cfg)
        self.cfg = cfg
        self.batch = batch
        self.max_pages = max_pages
        self.num_pages = num_pages or batch * max_pages
        B, h, d = cfg.B, cfg.h_kv, cfg.d_h
        self.k_pages = torch.zeros((self.num_pages, B, h, d), dtype=torch.bfloat16, device=device)
        self.v_pages = torch.zeros_like(self.k_pages)
        ctx = max_pages * B
        L = _lib.lib()
        self.max_m1 = max(1, L.swattn_num_pooled(ctx, cfg.l_C1, cfg.s_C1))
        self.max_m2 = max(1, L.swattn_num_pooled(ctx, cfg.l_C2, cfg.s_C2))
        self.kc1 = torch.zeros((batch, self.max_m1, h, d), dtype=torch.bfloat16, device=device)
        self.kc2 = torch.zeros((batch, self.max_m2, h, d), dtype=torch.bfloat16, device=device)
        # host-side page allocator (shuffled so pages are scattered, like a real pool)
        order = np.arange(self.num_pages)
        if seed is not None:
            np.random.default_rng(seed).shuffle(order)
        self._free = list(order[::-1])
        self.block_table_h = np.full((batch, max_pages), -1, dtype=np.int32)
        self.lens_h = np.zeros(batch, dtype=np.int32)
        self.block_table = torch.from_numpy(self.block_table_h).to(device)
        self.seq_lens = torch.zeros(batch, dtype=torch.int32, device=device)
        self.device = device

    def _ensure_pages(self, seq: int, new_len: int):
        need = -(-new_len // self.cfg.B)
        if need > self.max_pages:
            raise ValueError(f"sequence {seq} would need {need} pages > max_pages={self.max_pages}")
        for p in range(need):
            if self.block_table_h[seq, p] < 0:
                if not self._free:
                    raise RuntimeError("paged KV pool exhausted")
                self.block_table_h[seq, p] = self._free.pop()

    def _descriptor(self) -> _lib.CPagedKV:
        kv = _lib.CPagedKV()
        kv.k_pages = self.k_pages.data_ptr()
        kv.v_pages = self.v_pages.data_ptr()
        kv.block_table = self.block_table.data_ptr()
        kv.seq_lens = self.seq_lens.data_ptr()
        kv.max_pages = self.max_pages
        kv.kc1 = self.kc1.data_ptr()
        kv.kc2 = self.kc2.data_ptr()
        kv.max_m1 = self.max_m1
        kv.max_m2 = self.max_m2
        kv.num_pages = self.num_pages
        return kv

    def append(self, seq: int, K: torch.Tensor, V: torch.Tensor):
        """Append tokens K/V [n, h_kv, d] to one sequence (prefill or decode),
        then extend its compressed keys (kernel D1).  Only this sequence's
        block-table row and length go host -> device."""
        n = K.shape[0]
        L0 = int(self.lens_h[seq])
        self._ensure_pages(seq, L0 + n)
        self.block_table[seq].copy_(torch.from_numpy(self.block_table_h[seq]))
        pos = torch.arange(L0, L0 + n, device=self.device)
        pages = self.block_table[seq].long()[pos // self.cfg.B]
        slots = pos % self.cfg.B
        self.k_pages[pages, slots] = K.to(torch.bfloat16)
        self.v_pages[pages, slots] = V.to(torch.bfloat16)
        prev = self.seq_lens.clone()
        self.lens_h[seq] = L0 + n
        self.seq_lens[seq] = L0 + n
        L = _lib.lib()
        _lib.check(L.swattn_kcache_append(_lib.c_config(self.cfg), self._descriptor(), prev.data_ptr(),
                                          self.batch, _lib.stream_handle(self.device)),
                   "swattn_kcache_append")

    def append_tokens(self, K: torch.Tensor, V: torch.Tensor, active=None):
        """Serving-loop append: one token per sequence, K/V [batch, h_kv, d].
        The row write, the pooled-key update and the seq_lens advance run in
        one kernel (swattn_kcache_append_tokens); the host only uploads the
        block-table entries of sequences that just crossed into a new page.
        ``active`` (bool/int [batch], host) masks sequences that do not grow."""
        cfg = self.cfg
        if tuple(K.shape) != (self.batch, cfg.h_kv, cfg.d_h) or K.shape != V.shape:
            raise ValueError(f"K/V shape {tuple(K.shape)}/{tuple(V.shape)} != "
                             f"{(self.batch, cfg.h_kv, cfg.d_h)}")
        act = np.ones(self.batch, dtype=bool) if active is None else np.asarray(active, dtype=bool)
        rows, cols = [], []
        for b in np.nonzero(act)[0]:
            L0 = int(self.lens_h[b])
            if L0 % cfg.B == 0:                       # first token of a new page
                self._ensure_pages(int(b), L0 + 1)
                rows.append(int(b)); cols.append(L0 // cfg.B)
        if rows:
            r, c = np.array(rows), np.array(cols)
            vals = torch.from_numpy(self.block_table_h[r, c].copy()).to(self.device, non_blocking=True)
            self.block_table[torch.from_numpy(r).to(self.device), torch.from_numpy(c).to(self.device)] = vals
        act_d = None
        if active is not None:
            act_d = torch.from_numpy(act.astype(np.int32)).to(self.device)
        Kd = K.to(torch.bfloat16).contiguous()
        Vd = V.to(torch.bfloat16).contiguous()
        self.lens_h += act.astype(np.int32)
        L = _lib.lib()
        _lib.check(L.swattn_kcache_append_tokens(_lib.c_config(cfg), self._descriptor(), Kd.data_ptr(),
                                                 Vd.data_ptr(), 0 if act_d is None else act_d.data_ptr(),
                                                 self.batch, _lib.stream_handle(self.device)),
                   "swattn_kcache_append_tokens")


def decode_step(cache: PagedKVCache, q: torch.Tensor, return_topk: bool = False):
    """One decode step for every sequence: q [batch, h_q, d] is the query of
    token seq_lens[b]-1 (already appended).  Returns AttentionResult (o
    [batch, h_q, d] bf16, lse [batch, h_q] fp32) and optionally the selected
    top-k blocks [batch, h_kv, k_top] (-1 padded, ascending)."""
    cfg = cache.cfg
    if tuple(q.shape) != (cache.batch, cfg.h_q, cfg.d_h):
        raise ValueError(f"q shape {tuple(q.shape)} != {(cache.batch, cfg.h_q, cfg.d_h)}")
    qd = q.to(torch.bfloat16).contiguous()
    o = torch.empty_like(qd)
    lse = torch.empty((cache.batch, cfg.h_q), dtype=torch.float32, device=qd.device)
    topk = torch.empty((cache.batch, cfg.h_kv, max(cfg.k_top, 1)), dtype=torch.int32,
                       device=qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    nbytes = L.swattn_decode_workspace_bytes(c, cache.batch, cache.max_pages)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=qd.device)
    _lib.check(L.swattn_decode_step(c, cache._descriptor(), qd.data_ptr(), cache.batch, o.data_ptr(),
                                    lse.data_ptr(), topk.data_ptr(), ws.data_ptr(), nbytes,
                                    _lib.stream_handle(qd.device)), "swattn_decode_step")
    res = AttentionResult(o, lse)
    return (res, topk[:, :, :cfg.k_top]) if return_topk else res
