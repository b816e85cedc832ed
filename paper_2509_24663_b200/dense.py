"""Dense grouped-query attention (reference: dense.py) -- kernel K5."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import is_host, to_device_bf16, to_host_like
from .core import AttentionConfig, OpCounter


@dataclass(frozen=True)
class AttentionResult:
    """(output [n, h_q, d_h] in the storage dtype, lse [n, h_q]) (dense.py:25-31).
    Device results: bf16 output, fp32 natural-log lse.  Host inputs get
    host results (bf16 numpy output, float64 lse)."""

    output: object
    lse: object


def check_gqa_shapes(Q, K, V, cfg: AttentionConfig):
    """dense.py:34-57: same checks and messages."""
    if Q.ndim != 3 or K.ndim != 3 or V.ndim != 3:
        raise ValueError(
            f"Q/K/V must be rank-3 (tokens, heads, d_h); got {tuple(Q.shape)}, "
            f"{tuple(K.shape)}, {tuple(V.shape)}")
    n, h_q, d_h = Q.shape
    if n == 0:
        raise ValueError("empty sequence: n must be >= 1")
    if tuple(K.shape) != tuple(V.shape):
        raise ValueError(f"K shape {tuple(K.shape)} != V shape {tuple(V.shape)}")
    if K.shape[0] != n or K.shape[2] != d_h:
        raise ValueError(f"K shape {tuple(K.shape)} inconsistent with Q shape {tuple(Q.shape)}")
    h_kv = K.shape[1]
    if (h_q, h_kv, d_h) != (cfg.h_q, cfg.h_kv, cfg.d_h):
        raise ValueError(
            f"shapes (h_q={h_q}, h_kv={h_kv}, d_h={d_h}) do not match config "
            f"(h_q={cfg.h_q}, h_kv={cfg.h_kv}, d_h={cfg.d_h})")
    if cfg.n is not None and cfg.n != n:
        raise ValueError(f"sequence length {n} does not match cfg.n={cfg.n}")
    if Q.dtype != K.dtype or Q.dtype != V.dtype:
        raise ValueError("Q/K/V must share one storage dtype")
    return n, h_q, h_kv, d_h


def _finish(O, lse, host: bool) -> AttentionResult:
    if host:
        return AttentionResult(to_host_like(O, bf16=True), lse.double().cpu().numpy())
    return AttentionResult(O, lse)


def tiled_gqa_forward(Q, K, V, cfg: AttentionConfig, B_q: int = 64, B_k: int = 64,
                      causal: bool = True, counter: OpCounter | None = None) -> AttentionResult:
    """dense.py:112-170 on the GPU (K5); tile sizes are the kernel's."""
    n, h_q, h_kv, d_h = check_gqa_shapes(Q, K, V, cfg)
    if B_q < 1 or B_k < 1:
        raise ValueError(f"tile sizes must be >= 1, got B_q={B_q}, B_k={B_k}")
    host = is_host(Q)
    Qd, Kd, Vd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V")))
    O = torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    _lib.check(L.swattn_dense_fwd(_lib.c_config(cfg), Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(),
                                  n, int(bool(causal)), O.data_ptr(), lse.data_ptr(),
                                  _lib.stream_handle(Qd.device)), "swattn_dense_fwd")
    if counter is not None:
        vis = n * (n + 1) // 2 if causal else n * n
        counter.add(mac=2 * vis * d_h * h_q, exp=vis * h_q)
    return _finish(O, lse, host)


naive_gqa_forward = tiled_gqa_forward  # same semantics (dense.py:64-109); one kernel serves both


def naive_gqa_backward(Q, K, V, dO, cfg: AttentionConfig, causal: bool = True,
                       counter: OpCounter | None = None):
    """dense.py:173-221 on the GPU: gradients of sum(O * dO) w.r.t. Q, K, V for
    (causal) GQA attention -- the sparse backward's kernels with every
    (causal) block visible, after the K5 forward for O / lse.  dK / dV reduce
    in a fixed order (bitwise reproducible, :182-183).  Returns (dQ, dK, dV)
    in the storage dtype (device bf16 tensors, or numpy bf16 for host
    inputs)."""
    n, h_q, h_kv, d_h = check_gqa_shapes(Q, K, V, cfg)
    if tuple(dO.shape) != tuple(Q.shape):
        raise ValueError(f"dO shape {tuple(dO.shape)} != Q shape {tuple(Q.shape)}")
    host = is_host(Q)
    Qd, Kd, Vd, dOd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V"),
                                                          (dO, "dO")))
    fwd = tiled_gqa_forward(Qd, Kd, Vd, cfg, causal=causal)
    dQ, dK, dV = torch.empty_like(Qd), torch.empty_like(Kd), torch.empty_like(Vd)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = torch.empty(max(L.swattn_dense_bwd_workspace_bytes(c, n, int(bool(causal))), 1),
                     dtype=torch.uint8, device=Qd.device)
    _lib.check(L.swattn_dense_bwd(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n,
                                  int(bool(causal)), fwd.output.data_ptr(), fwd.lse.data_ptr(),
                                  dOd.data_ptr(), dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(),
                                  ws.data_ptr(), ws.numel(), _lib.stream_handle(Qd.device)),
               "swattn_dense_bwd")
    if counter is not None:
        vis = n * (n + 1) // 2 if causal else n * n
        counter.add(mac=4 * vis * d_h * h_q, exp=vis * h_q)
    if host:
        import ml_dtypes
        return tuple(t.cpu().view(torch.int16).numpy().view(ml_dtypes.bfloat16)
                     for t in (dQ, dK, dV))
    return dQ, dK, dV
