"""TEST INFRASTRUCTURE ONLY -- never imported by the product package.

A float64 torch restatement of the reference's approx block selection, for
full-size parity at the BASELINE sizes (every row at 128K): the same math as
`swattn_oracle.shared_scores / block_scores / topk_blocks` (which restate
selection.py:93-136,165-222,279-348 and compression.py:64-86,160-173),
chunked over query rows so it runs on the GPU in float64 in seconds where
the numpy port needs hours.  Pinned to the reference-minted goldens by
tests/test_oracle_golden.py (every row of the paper_n8192 / n10000 goldens).

Semantics restated:
  * pooled keys: mean over complete windows in float64, cast to the storage
    dtype via float32 (numpy / ml_dtypes double rounding, compression.py:79-85);
  * pass 1 (approx): lse over visible C2 columns, masked to -inf; rows with no
    visible C2 but visible C1 use the exact C1 lse (selection.py:303-324);
  * pass 2: sum over the G heads of exp(s - lse_safe) over visible C1 columns,
    0 on masked columns (selection.py:199-222);
  * max-pool over windows [s j, min(s j + l, m1)) (compression.py:160-173);
  * top-k per row over candidates [N_init, min(lo, n_cols)), score
    descending, ties to the lower block index (stable argsort,
    selection.py:123-126); no_visible rows select none (:129).
"""
from __future__ import annotations

import math

import torch


def pool_bf16(K: torch.Tensor, length: int, stride: int) -> torch.Tensor:
    """K [n, h_kv, d] (bf16) -> pooled keys [m, h_kv, d] bf16 (float64 means)."""
    n = K.shape[0]
    m = 0 if n < length else (n - length) // stride + 1
    if m == 0:
        return K.new_zeros((0,) + tuple(K.shape[1:]))
    K64 = K.double()
    # bf16 windows of <= 128 rows sum exactly in float64 (any order)
    idx = torch.arange(m, device=K.device) * stride
    acc = torch.zeros((m,) + tuple(K.shape[1:]), dtype=torch.float64, device=K.device)
    for r in range(length):
        acc += K64[idx + r]
    return (acc / length).to(torch.float32).to(torch.bfloat16)


def _vis(rows: torch.Tensor, length: int, stride: int) -> torch.Tensor:
    return torch.where(rows + 1 >= length, (rows + 1 - length) // stride + 1,
                       torch.zeros_like(rows))


def select_f64(Q: torch.Tensor, K: torch.Tensor, cfg, rows_per_chunk: int = 256,
               ck1=None, ck2=None, return_scores: bool = False):
    """Approx select_blocks of every row, float64.  Q [n, h_q, d], K [n, h_kv, d]
    bf16 torch tensors (any device).  Returns topk [h_kv, n, k_top] int64
    (ascending, -1 padded) and, with return_scores, S^cmp [h_kv, n, n_cols]
    float64 (candidate region meaningful)."""
    dev = Q.device
    n, h_q, d = Q.shape
    h_kv = K.shape[1]
    G = h_q // h_kv
    scale = 1.0 / math.sqrt(d) if cfg.scale_compressed_logits else 1.0
    ck1 = pool_bf16(K, cfg.l_C1, cfg.s_C1) if ck1 is None else ck1
    ck2 = pool_bf16(K, cfg.l_C2, cfg.s_C2) if ck2 is None else ck2
    m1, m2 = ck1.shape[0], ck2.shape[0]
    n_cols = -(-m1 // cfg.s) if m1 else 0
    K1 = ck1.double()
    K2 = ck2.double()
    topk = torch.full((h_kv, n, cfg.k_top), -1, dtype=torch.int64, device=dev)
    scmp_all = torch.zeros((h_kv, n, max(n_cols, 1)), dtype=torch.float64, device=dev) \
        if return_scores else None
    if m1 == 0 or cfg.k_top == 0:
        return (topk, scmp_all) if return_scores else topk
    ar_cols = torch.arange(n_cols, device=dev)
    for q0 in range(0, n, rows_per_chunk):
        q1 = min(n, q0 + rows_per_chunk)
        rows = torch.arange(q0, q1, device=dev)
        v1 = _vis(rows, cfg.l_C1, cfg.s_C1)
        v2 = _vis(rows, cfg.l_C2, cfg.s_C2) if m2 else torch.zeros_like(v1)
        c1 = int(v1.max())
        if c1 == 0:
            continue
        c2 = int(v2.max())
        b = rows // cfg.B
        lo = torch.clamp(b - cfg.N_local + 1, min=0)
        hi = torch.clamp(lo, max=n_cols)
        ncand = torch.clamp(hi - cfg.N_init, min=0)
        k = torch.where(v1 > 0, torch.clamp(ncand, max=cfg.k_top), torch.zeros_like(ncand))
        if int(k.max()) == 0 and not return_scores:
            continue
        Qr = Q[q0:q1].double()
        for g in range(h_kv):
            Qg = Qr[:, g * G:(g + 1) * G]                       # [R, G, d]
            S1 = torch.einsum("rgd,md->rgm", Qg, K1[:c1, g]) * scale
            cols1 = torch.arange(c1, device=dev)
            vis1 = cols1[None, :] < v1[:, None]                  # [R, c1]
            if c2 > 0:
                S2 = torch.einsum("rgd,md->rgm", Qg, K2[:c2, g]) * scale
                vis2 = torch.arange(c2, device=dev)[None, :] < v2[:, None]
                S2 = S2.masked_fill(~vis2[:, None, :], float("-inf"))
                lse = torch.logsumexp(S2, dim=2)                 # [R, G] (-inf if none)
            else:
                lse = torch.full(S1.shape[:2], float("-inf"), dtype=torch.float64, device=dev)
            fb = (v2 == 0) & (v1 > 0)
            if bool(fb.any()):
                lse_fb = torch.logsumexp(S1.masked_fill(~vis1[:, None, :], float("-inf")), dim=2)
                lse = torch.where(fb[:, None], lse_fb, lse)
            lse_safe = torch.where(torch.isinf(lse), torch.zeros_like(lse), lse)
            P = torch.exp(S1 - lse_safe[:, :, None]).masked_fill(~vis1[:, None, :], 0.0)
            shared = P.sum(dim=1)                                # [R, c1]
            # max-pool over [s j, min(s j + l, m1)): columns in [c1, m1) are 0,
            # columns >= m1 do not exist (-inf)
            width = (n_cols - 1) * cfg.s + cfg.l
            full = torch.zeros((q1 - q0, width), dtype=torch.float64, device=dev)
            full[:, :c1] = shared
            if width > m1:
                full[:, m1:] = float("-inf")
            scmp = full.unfold(1, cfg.l, cfg.s).amax(dim=2)      # [R, n_cols]
            if return_scores:
                scmp_all[g, q0:q1] = scmp
            cand = (ar_cols[None, :] >= cfg.N_init) & (ar_cols[None, :] < hi[:, None])
            sc = scmp.masked_fill(~cand, float("-inf"))
            order = torch.sort(sc, dim=1, descending=True, stable=True).indices
            kk = int(k.max())
            pick = order[:, :kk]
            pick = torch.where(torch.arange(kk, device=dev)[None, :] < k[:, None], pick,
                               torch.full_like(pick, 1 << 30))
            pick = torch.sort(pick, dim=1).values
            pick = torch.where(pick == (1 << 30), torch.full_like(pick, -1), pick)
            topk[g, q0:q1, :kk] = pick
    return (topk, scmp_all) if return_scores else topk
