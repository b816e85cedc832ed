"""Analytic operation counts (reference: bench.py:89-155) -- the roofline
numerators.  FLOP = 2 * MAC."""

from __future__ import annotations

import numpy as np

from .core import AttentionConfig


def pooled_visible_count(i: int, length: int, stride: int) -> int:
    """bench.py:89-93."""
    return 0 if i + 1 < length else (i + 1 - length) // stride + 1


def sparse_visible_tokens(cfg: AttentionConfig, i: int) -> int:
    """bench.py:96-100."""
    b = i // cfg.B
    picked = min(b + 1, cfg.budget_blocks)
    return (picked - 1) * cfg.B + (i - b * cfg.B) + 1


def dense_query_counts(cfg: AttentionConfig, n: int):
    """bench.py:103-104: (mac, exp) of the newest query at context n."""
    return 2 * cfg.h_q * n * cfg.d_h, cfg.h_q * n


def sparse_query_counts(cfg: AttentionConfig, n: int):
    """bench.py:107-109."""
    v = sparse_visible_tokens(cfg, n - 1)
    return 2 * cfg.h_q * v * cfg.d_h, cfg.h_q * v


def selection_query_counts(cfg: AttentionConfig, n: int, approx: bool) -> dict:
    """bench.py:112-126: two-pass scoring cost of the newest query."""
    v1 = pooled_visible_count(n - 1, cfg.l_C1, cfg.s_C1)
    v2 = pooled_visible_count(n - 1, cfg.l_C2, cfg.s_C2)
    pass1_cols = (v2 if v2 > 0 else v1) if approx else v1
    pass1_mac = cfg.h_q * pass1_cols * cfg.d_h
    pass2_mac = cfg.h_q * v1 * cfg.d_h
    return {"mac": pass1_mac + pass2_mac, "exp": cfg.h_q * (pass1_cols + v1),
            "pass1_mac": pass1_mac, "pass2_mac": pass2_mac}


def _pooled_all(n: int, length: int, stride: int) -> np.ndarray:
    i = np.arange(n, dtype=np.int64)
    return np.where(i + 1 >= length, (i + 1 - length) // stride + 1, 0)


def dense_total_counts(cfg: AttentionConfig, n: int, causal: bool = True):
    """bench.py:134-136 -> (mac, exp)."""
    vis = n * (n + 1) // 2 if causal else n * n
    return 2 * cfg.h_q * vis * cfg.d_h, cfg.h_q * vis


def sparse_total_counts(cfg: AttentionConfig, n: int):
    """bench.py:139-141 (closed form of the sum)."""
    i = np.arange(n, dtype=np.int64)
    b = i // cfg.B
    picked = np.minimum(b + 1, cfg.budget_blocks)
    total = int(((picked - 1) * cfg.B + (i - b * cfg.B) + 1).sum())
    return 2 * cfg.h_q * total * cfg.d_h, cfg.h_q * total


def selection_total_counts(cfg: AttentionConfig, n: int, approx: bool) -> dict:
    """bench.py:144-155."""
    v1 = _pooled_all(n, cfg.l_C1, cfg.s_C1)
    v2 = _pooled_all(n, cfg.l_C2, cfg.s_C2)
    pass1_cols = int(np.where(v2 > 0, v2, v1).sum()) if approx else int(v1.sum())
    pass1_mac = cfg.h_q * pass1_cols * cfg.d_h
    pass2_mac = cfg.h_q * int(v1.sum()) * cfg.d_h
    return {"mac": pass1_mac + pass2_mac, "exp": cfg.h_q * (pass1_cols + int(v1.sum())),
            "pass1_mac": pass1_mac, "pass2_mac": pass2_mac}


def compress_bytes(cfg: AttentionConfig, n: int) -> int:
    """K1 algorithmic HBM bytes: read K once, write both pooled key sets."""
    m1 = 0 if n < cfg.l_C1 else (n - cfg.l_C1) // cfg.s_C1 + 1
    m2 = 0 if n < cfg.l_C2 else (n - cfg.l_C2) // cfg.s_C2 + 1
    return (n + m1 + m2) * cfg.h_kv * cfg.d_h * 2
