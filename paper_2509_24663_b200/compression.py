"""Key compression and block-score pooling (reference: compression.py).

``mean_pool_keys`` runs kernel K1 (csrc/compress.cu): one HBM pass, exact
float64 window sums, rounded like the reference's cast back to storage dtype
(compression.py:79-85).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import is_host, to_device_bf16
from .core import AttentionConfig


@dataclass(frozen=True)
class CompressedKeys:
    """Mean-pooled keys (compression.py:29-46): keys [m, h_kv, d_h] bf16 on
    the device, span_end [m] int64 (inclusive last pooled token)."""

    keys: torch.Tensor
    pool_length: int
    pool_stride: int
    span_end: torch.Tensor

    @property
    def m(self) -> int:
        return int(self.keys.shape[0])


@dataclass(frozen=True)
class ScoreMatrix:
    """Scores (compression.py:49-61): scores [n, planes, cols] fp32 on the
    device, masked columns exactly 0; no_visible [n] bool."""

    scores: torch.Tensor
    kind: str
    no_visible: torch.Tensor


def _pool_cfg(length: int, stride: int, h_kv: int, d_h: int) -> AttentionConfig:
    # a config whose C1 profile is (length, stride); C2 unused
    return AttentionConfig(h_q=h_kv, h_kv=h_kv, d_h=d_h, l_C1=length, s_C1=stride,
                           l_C2=2 * 4 * stride, s_C2=4 * stride, l=5, s=4, N_init=1,
                           N_local=1 << 20, k_top=0, w=1, experimental=True)


def mean_pool_keys(K, length: int, stride: int) -> CompressedKeys:
    """compression.py:64-86 on the device (kernel K1)."""
    if K.ndim != 3:
        raise ValueError(f"K must be rank-3 (tokens, heads, d_h); got {tuple(K.shape)}")
    if stride < 1 or length < stride:
        raise ValueError(f"need length >= stride >= 1, got length={length}, stride={stride}")
    Kd = to_device_bf16(K, "K")
    n, h_kv, d_h = Kd.shape
    m = 0 if n < length else (n - length) // stride + 1
    out = torch.empty((m, h_kv, d_h), dtype=torch.bfloat16, device=Kd.device)
    if m:
        cfg = _pool_cfg(length, stride, h_kv, d_h)
        L = _lib.lib()
        c = _lib.c_config(cfg)
        _lib.check(L.swattn_compress_keys(c, Kd.data_ptr(), n, out.data_ptr(), None,
                                          _lib.stream_handle()), "swattn_compress_keys")
    span_end = torch.arange(m, dtype=torch.int64, device=Kd.device) * stride + (length - 1)
    return CompressedKeys(out, length, stride, span_end)


def visible_column_counts(span_end, n: int):
    """Per query token, #pooled entries ending at or before it (compression.py:89-91)."""
    return torch.searchsorted(span_end, torch.arange(n, device=span_end.device), right=True)


def max_pool_scores(sm: ScoreMatrix, l: int, s: int) -> ScoreMatrix:
    """compression.py:160-173 (device tensor ops; not on the hot path -- the
    fused kernel K2 max-pools in its epilogue)."""
    if l < 1 or s < 1:
        raise ValueError(f"need l, s >= 1, got l={l}, s={s}")
    S = sm.scores
    n, planes, m = S.shape
    nb = -(-m // s) if m else 0
    pad = nb * s + l - m
    Sp = torch.nn.functional.pad(S, (0, max(pad, 0)), value=float("-inf"))
    win = Sp.unfold(2, l, s)[:, :, :nb]
    return ScoreMatrix(win.amax(dim=-1), "cmp", sm.no_visible)


def head_group_sum(sm: ScoreMatrix, G: int) -> ScoreMatrix:
    """compression.py:151-157."""
    n, h_q, m = sm.scores.shape
    if G < 1 or h_q % G != 0:
        raise ValueError(f"head count {h_q} is not divisible by group size {G}")
    return ScoreMatrix(sm.scores.reshape(n, h_q // G, G, m).sum(dim=2), "shared", sm.no_visible)
