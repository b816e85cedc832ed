"""Dense-sparse switching (reference: switch.py)."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._tensors import is_host, to_device_bf16
from .core import AttentionConfig, OpCounter
from .dense import AttentionResult, _finish, check_gqa_shapes, tiled_gqa_forward
from .selection import Workspace, select_blocks
from .sparse import sparse_forward

MODE_DENSE = "dense"
MODE_SPARSE = "sparse"


@dataclass(frozen=True)
class SwitchPolicy:
    """switch.py:27-34."""

    threshold_tokens: int | None = None
    forced_mode: str | None = None


def visible_token_budget(cfg: AttentionConfig) -> int:
    """switch.py:37-39."""
    return (cfg.N_init + cfg.N_local + cfg.k_top) * cfg.B


def attend(Q, K, V, cfg: AttentionConfig, policy: SwitchPolicy | None = None,
           selection_mode: str = "approx", B_q: int = 64, B_k: int = 64,
           counters: dict | None = None) -> tuple[AttentionResult, str]:
    """switch.py:42-82: n <= threshold -> dense (K5), else select (K1-K3) +
    sparse (K4).  One C-ABI call, one stream, no host synchronisation."""
    policy = policy or SwitchPolicy()
    if policy.forced_mode not in (None, MODE_DENSE, MODE_SPARSE):
        raise ValueError(f"unknown forced mode {policy.forced_mode!r}")
    n = Q.shape[0]
    threshold = policy.threshold_tokens
    if threshold is None:
        threshold = cfg.switch_threshold
    if threshold is None:
        threshold = visible_token_budget(cfg)
    mode = policy.forced_mode or (MODE_DENSE if n <= threshold else MODE_SPARSE)
    counters = counters or {}
    if counters:
        # instrumented call: go stage by stage so each counter is filled
        if mode == MODE_DENSE:
            return tiled_gqa_forward(Q, K, V, cfg, B_q, B_k, True, counters.get("dense")), mode
        sel = select_blocks(Q, K, cfg, selection_mode, B_q, B_k, counters.get("selection"))
        return sparse_forward(Q, K, V, sel, cfg, counters.get("sparse")), mode
    n, h_q, h_kv, d_h = check_gqa_shapes(Q, K, V, cfg)
    if B_q < 1 or B_k < 1:
        raise ValueError(f"tile sizes must be >= 1, got B_q={B_q}, B_k={B_k}")
    if selection_mode not in _lib.SELECT_MODE:
        raise ValueError(f"unknown selection mode {selection_mode!r}")
    host = is_host(Q)
    Qd, Kd, Vd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V")))
    O = torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = Workspace.get(L.swattn_workspace_bytes(c, n), Qd.device)
    taken = _lib.ctypes.c_int32(0)
    _lib.check(L.swattn_attend(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n, int(threshold),
                               _lib.FORCED_MODE[mode], _lib.SELECT_MODE[selection_mode],
                               O.data_ptr(), lse.data_ptr(), _lib.ctypes.byref(taken),
                               ws.data_ptr(), ws.numel(), _lib.stream_handle(Qd.device)),
               "swattn_attend")
    assert taken.value == (1 if mode == MODE_DENSE else 2)
    return _finish(O, lse, host), mode
