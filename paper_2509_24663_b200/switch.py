"""Dense-sparse switching (reference: switch.py)."""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
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
    # the chunked host pipeline needs the row-range entry points, i.e. the
    # paper profile on the tensor-core kernels (swattn_profile_supported)
    if host and mode == MODE_SPARSE and _lib.lib().swattn_profile_supported(_lib.c_config(cfg)):
        O_h, lse_h = attend_host_chunked(Q, K, V, cfg, selection_mode)
        return _finish(O_h, lse_h, True), mode
    Qd, Kd, Vd = (to_device_bf16(x, nm) for x, nm in ((Q, "Q"), (K, "K"), (V, "V")))
    O = torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=Qd.device)
    lse = torch.empty((n, h_q), dtype=torch.float32, device=Qd.device)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    taken = _lib.ctypes.c_int32(0)
    if mode == MODE_DENSE:   # K5 needs no workspace
        ws_ptr, ws_bytes = None, 0
    else:
        ws = Workspace.get(L.swattn_workspace_bytes(c, n), Qd.device)
        ws_ptr, ws_bytes = ws.data_ptr(), ws.numel()
    _lib.check(L.swattn_attend(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n, int(threshold),
                               _lib.FORCED_MODE[mode], _lib.SELECT_MODE[selection_mode],
                               O.data_ptr(), lse.data_ptr(), _lib.ctypes.byref(taken),
                               ws_ptr, ws_bytes, _lib.stream_handle(Qd.device)),
               "swattn_attend")
    assert taken.value == (1 if mode == MODE_DENSE else 2)
    return _finish(O, lse, host), mode


def _host_bf16(x, name: str) -> torch.Tensor:
    """Host input -> pinned contiguous bf16 torch tensor (no copy when the
    caller already passes one)."""
    if isinstance(x, torch.Tensor) and x.dtype == torch.bfloat16 and x.is_pinned() and x.is_contiguous():
        return x
    if isinstance(x, np.ndarray):
        if x.dtype.name == "bfloat16":
            x = torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16)
        else:
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor or numpy array, got {type(x).__name__}")
    return x.to(torch.bfloat16).contiguous().pin_memory()


class _Chunked:
    """Per-device side streams, events and device buffers of the chunked
    host pipeline (grow-only, reused across calls)."""

    _state: dict = {}

    @classmethod
    def get(cls, device, n, h_q, h_kv, d_h):
        key = torch.device(device).index or 0
        st = cls._state.get(key)
        if st is None:
            st = {"in": torch.cuda.Stream(device), "out": torch.cuda.Stream(device), "bufs": None}
            cls._state[key] = st
        b = st["bufs"]
        if b is None or b["n"] < n:
            b = {"n": n,
                 "Q": torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=device),
                 "K": torch.empty((n, h_kv, d_h), dtype=torch.bfloat16, device=device),
                 "V": torch.empty((n, h_kv, d_h), dtype=torch.bfloat16, device=device),
                 "O": torch.empty((n, h_q, d_h), dtype=torch.bfloat16, device=device),
                 "lse": torch.empty((n, h_q), dtype=torch.float32, device=device)}
            st["bufs"] = b
        return st


def chunk_rows_for(n: int, B: int) -> int:
    """~8 chunks (SWATTN_HOST_CHUNKS), each a multiple of the query block and
    >= 4096 rows.  At 128K, 8 chunks measured 47.5-47.8 ms end to end vs
    48.6-49.0 with 6 / 12 / 16 and 51.2 with 24 (profiles/r02bg_host_chunks.txt):
    fewer row-range calls, while the copies still hide under compute."""
    rows = max(4096, -(-n // int(os.environ.get("SWATTN_HOST_CHUNKS", "8"))))
    return -(-rows // B) * B


def chunk_bounds(n: int, B: int, rows: int | None = None) -> list[tuple[int, int]]:
    """Row chunks of the host pipeline.  With the default size the first and
    last chunks are short (2048 rows): the first one's Q arrives quickly
    (compute starts after K, V and 16 MB of Q instead of 67 MB), and the
    last one's O / lse leave quickly (the copy tail after the final kernel)."""
    if rows is not None:
        return [(r, min(n, r + rows)) for r in range(0, n, rows)]
    rows = chunk_rows_for(n, B)
    edge = -(-2048 // B) * B
    if n < 4 * rows:
        return [(r, min(n, r + rows)) for r in range(0, n, rows)]
    last0 = (n - edge) // B * B               # start of the short last chunk
    bounds = [(0, edge)]
    mid = last0 - edge
    k = max(1, round(mid / rows))
    step = -(-(-(-mid // k)) // B) * B
    r = edge
    while r < last0:
        bounds.append((r, min(last0, r + step)))
        r += step
    bounds.append((last0, n))
    return bounds


def attend_host_chunked(Q, K, V, cfg: AttentionConfig, selection_mode: str = "approx",
                        out=None, chunk_rows: int | None = None, device=None):
    """Sparse branch of attend for HOST inputs with the host<->device copies
    overlapped with compute: Q, K and V stream in row chunks on a copy stream
    while the compute stream pools the compressed keys of the rows already
    resident and runs select + sparse attention for those chunks
    (swattn_attend_rows), and a second copy stream returns O / lse of each
    finished chunk.  Returns pinned host (O bf16 [n, h_q, d_h], lse fp32
    [n, h_q]); `out` may pass them in.  Rows are computed exactly as by the
    whole-sequence call."""
    Qh, Kh, Vh = _host_bf16(Q, "Q"), _host_bf16(K, "K"), _host_bf16(V, "V")
    n, h_q, d_h = Qh.shape
    h_kv = Kh.shape[1]
    device = torch.device(device or "cuda")
    st = _Chunked.get(device, n, h_q, h_kv, d_h)
    b = st["bufs"]
    Qd, Kd, Vd, Od, ld = (b[k][:n] for k in ("Q", "K", "V", "O", "lse"))
    if out is None:
        O_h = torch.empty((n, h_q, d_h), dtype=torch.bfloat16, pin_memory=True)
        lse_h = torch.empty((n, h_q), dtype=torch.float32, pin_memory=True)
    else:
        O_h, lse_h = out
    L = _lib.lib()
    c = _lib.c_config(cfg)
    ws = Workspace.get(L.swattn_workspace_bytes(c, n), device)
    comp = torch.cuda.current_stream(device)
    s_in, s_out = st["in"], st["out"]
    bounds = chunk_bounds(n, cfg.B, chunk_rows)
    s_in.wait_stream(comp)   # device buffers may still be read by the previous call
    s_out.wait_stream(comp)
    # Q, K and V all stream in row chunks: chunk c needs K / V rows < r1 only
    # (causal), and the compressed keys of its rows are pooled from K[:r1] as
    # it arrives (windows that end by r1; the window halo is re-pooled from
    # 64 rows before the chunk, bit-identically), so compute starts after the
    # first chunk instead of after all of K and V.
    with torch.cuda.stream(s_in):
        q_ready = []
        for r0, r1 in bounds:
            Kd[r0:r1].copy_(Kh[r0:r1], non_blocking=True)
            Vd[r0:r1].copy_(Vh[r0:r1], non_blocking=True)
            Qd[r0:r1].copy_(Qh[r0:r1], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_in)
            q_ready.append(e)
    sel = _lib.SELECT_MODE[selection_mode] | _lib.SELECT_PREPARED
    p1, p2 = _lib.ctypes.c_void_p(), _lib.ctypes.c_void_p()
    _lib.check(L.swattn_workspace_ckeys(c, n, ws.data_ptr(), _lib.ctypes.byref(p1),
                                        _lib.ctypes.byref(p2)), "swattn_workspace_ckeys")
    row_b = h_kv * d_h * 2
    halo = max(cfg.l_C1 - cfg.s_C1, cfg.l_C2 - cfg.s_C2)
    for (r0, r1), e in zip(bounds, q_ready):
        comp.wait_event(e)
        a = max(0, r0 - halo)   # a multiple of both pooling strides (chunks start on B)
        _lib.check(L.swattn_compress_keys(c, Kd.data_ptr() + a * row_b, r1 - a,
                                          p1.value + (a // cfg.s_C1) * row_b,
                                          p2.value + (a // cfg.s_C2) * row_b, comp.cuda_stream),
                   "swattn_compress_keys")
        _lib.check(L.swattn_attend_rows(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n, r0, r1,
                                        sel, Od.data_ptr(), ld.data_ptr(), ws.data_ptr(),
                                        ws.numel(), comp.cuda_stream), "swattn_attend_rows")
        done = torch.cuda.Event()
        done.record(comp)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            O_h[r0:r1].copy_(Od[r0:r1], non_blocking=True)
            lse_h[r0:r1].copy_(ld[r0:r1], non_blocking=True)
    comp.wait_stream(s_out)
    # the host buffers are valid once the caller's stream reaches this point
    # (attend synchronises before handing them to Python)
    comp.synchronize()
    return O_h, lse_h
