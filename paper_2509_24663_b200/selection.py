"""Block selection (reference: selection.py).

``select_blocks`` = K1 -> K2 -> K3 (+ float64 boundary re-rank) on one CUDA
stream through ``swattn_select_blocks``.  The result is a device-resident
:class:`BlockSelection` holding only the per-token top-k lists; the
initial/local blocks are implicit (selection.py:113-119), and the
reference's tuple-of-arrays view is materialised lazily on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._tensors import to_device_bf16
from .compression import CompressedKeys, ScoreMatrix, mean_pool_keys
from .core import AttentionConfig, OpCounter, validate_config

SELECT_MODES = ("exact", "fused-exact", "approx")


@dataclass(frozen=True)
class BlockSelection:
    """Per-(KV group, query token) visible block sets (selection.py:51-90).

    Device form: ``topk`` [h_kv, n, k_top] int32 ascending, -1 padded, and
    ``topk_cnt`` [h_kv, n] int32.  ``blocks`` / ``counts`` reproduce the
    reference's host view (sorted unique init U local U top-k, and the
    (n_init, #local, #top) triple of selection.py:134).
    """

    block_size: int
    n: int
    topk: torch.Tensor
    topk_cnt: torch.Tensor
    N_init: int
    N_local: int
    n_reranked: int | None = None
    _host: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def num_groups(self) -> int:
        return int(self.topk.shape[0])

    def _host_topk(self):
        if "topk" not in self._host:
            self._host["topk"] = self.topk.cpu().numpy()
            self._host["cnt"] = self.topk_cnt.cpu().numpy()
        return self._host["topk"], self._host["cnt"]

    def query_blocks(self, g: int, i: int) -> np.ndarray:
        top, cnt = self._host_topk()
        b = i // self.block_size
        lo = max(0, b - self.N_local + 1)
        base = np.union1d(np.arange(min(self.N_init, b + 1)), np.arange(lo, b + 1))
        return np.union1d(base, top[g, i, :cnt[g, i]]).astype(np.int64)

    @property
    def blocks(self):
        if "blocks" not in self._host:
            self._host["blocks"] = tuple(
                tuple(self.query_blocks(g, i) for i in range(self.n))
                for g in range(self.num_groups))
        return self._host["blocks"]

    @property
    def counts(self) -> np.ndarray:
        _, cnt = self._host_topk()
        i = np.arange(self.n)
        b = i // self.block_size
        lo = np.maximum(0, b - self.N_local + 1)
        out = np.zeros((self.num_groups, self.n, 3), dtype=np.int64)
        out[:, :, 0] = np.minimum(self.N_init, b + 1)
        out[:, :, 1] = b + 1 - lo
        out[:, :, 2] = cnt
        return out

    def visible_spans(self, g: int, i: int):
        """Causally clipped token spans with adjacent blocks merged (selection.py:73-87)."""
        B = self.block_size
        spans = []
        for j in self.query_blocks(g, i):
            start = int(j) * B
            end = min(start + B, self.n, i + 1)
            if end <= start:
                continue
            if spans and spans[-1][1] == start:
                spans[-1] = (spans[-1][0], end)
            else:
                spans.append((start, end))
        return spans

    def visible_token_count(self, g: int, i: int) -> int:
        return sum(e - s for s, e in self.visible_spans(g, i))


def _cfg_ok(cfg: AttentionConfig, Q, K):
    validate_config(cfg)
    if Q.ndim != 3:
        raise ValueError(f"Q must be rank-3, got {tuple(Q.shape)}")
    n, h_q, d_h = Q.shape
    if (h_q, d_h) != (cfg.h_q, cfg.d_h):
        raise ValueError(f"Q heads/dim {(h_q, d_h)} do not match config")
    if K.shape[0] != n or tuple(K.shape[1:]) != (cfg.h_kv, cfg.d_h):
        raise ValueError(f"K shape {tuple(K.shape)} inconsistent with Q shape {tuple(Q.shape)}")
    return n


class Workspace:
    """Grow-only device scratch buffer (one per device), carved by the C ABI."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, device) -> torch.Tensor:
        key = torch.device(device).index or 0
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
            cls._bufs[key] = buf
        return buf


def select_blocks(Q, K, cfg: AttentionConfig, mode: str = "exact", B_q: int = 64,
                  B_k: int = 64, counter: OpCounter | None = None,
                  stats: dict | None = None) -> BlockSelection:
    """selection.py:354-383 on the GPU.  B_q/B_k are validated but tiles are
    chosen by the kernels."""
    if mode not in SELECT_MODES:
        raise ValueError(f"unknown selection mode {mode!r}; expected one of {SELECT_MODES}")
    if B_q < 1 or B_k < 1:
        raise ValueError(f"tile sizes must be >= 1, got B_q={B_q}, B_k={B_k}")
    n = _cfg_ok(cfg, Q, K)
    Qd, Kd = to_device_bf16(Q, "Q"), to_device_bf16(K, "K")
    L = _lib.lib()
    c = _lib.c_config(cfg)
    dev = Qd.device
    topk = torch.empty((cfg.h_kv, n, max(cfg.k_top, 1)), dtype=torch.int32, device=dev)
    cnt = torch.empty((cfg.h_kv, n), dtype=torch.int32, device=dev)
    nre = torch.zeros(1, dtype=torch.int32, device=dev)
    nbytes = L.swattn_workspace_bytes(c, n)
    ws = Workspace.get(nbytes, dev)
    _lib.check(L.swattn_select_blocks(c, Qd.data_ptr(), Kd.data_ptr(), n, _lib.SELECT_MODE[mode],
                                      topk.data_ptr(), cnt.data_ptr(), nre.data_ptr(),
                                      ws.data_ptr(), ws.numel(), _lib.stream_handle(dev)),
               "swattn_select_blocks")
    if counter is not None or stats is not None:
        from .counts import selection_total_counts
        d = selection_total_counts(cfg, n, approx=mode == "approx")
        if counter is not None:
            counter.add(mac=d["mac"], exp=d["exp"])
        if stats is not None:
            stats.update(d)
    sel = BlockSelection(cfg.B, n, topk[:, :, :cfg.k_top], cnt, cfg.N_init, cfg.N_local)
    object.__setattr__(sel, "n_reranked", nre)
    return sel


def build_block_sets(s_cmp, cfg: AttentionConfig) -> BlockSelection:
    """selection.py:93-136 from a max-pooled score matrix ([n, h_kv, n_cols],
    device fp32 or host array) -- kernel K3 on identical scores."""
    scores = s_cmp.scores if isinstance(s_cmp, ScoreMatrix) else s_cmp
    if isinstance(scores, np.ndarray):
        scores = torch.from_numpy(np.ascontiguousarray(scores, dtype=np.float32)).cuda()
    n, planes, n_cols = scores.shape
    if planes != cfg.h_kv:
        raise ValueError(f"score planes {planes} != h_kv {cfg.h_kv}")
    nb = -(-n // cfg.B)
    if n_cols > nb:
        raise ValueError(f"{n_cols} score columns for only {nb} selection blocks")
    validate_config(cfg)
    # kernel layout: [h_kv, n, ld] with ld >= n_cols implied by the pooling
    # profile; pad the caller's columns to that width with -inf (never ranked)
    m1 = _lib.lib().swattn_num_pooled(n, cfg.l_C1, cfg.s_C1)
    want = -(-m1 // cfg.s) if m1 else 0
    if n_cols != want:
        raise ValueError(f"expected {want} block-score columns for n={n}, got {n_cols}")
    ld = max(4, (n_cols + 3) // 4 * 4)
    sc = torch.full((planes, n, ld), float("-inf"), dtype=torch.float32, device=scores.device)
    sc[:, :, :n_cols] = scores.permute(1, 0, 2).to(torch.float32)
    topk = torch.empty((planes, n, max(cfg.k_top, 1)), dtype=torch.int32, device=scores.device)
    cnt = torch.empty((planes, n), dtype=torch.int32, device=scores.device)
    L = _lib.lib()
    _lib.check(L.swattn_topk_blocks(_lib.c_config(cfg), sc.data_ptr(), ld, n, topk.data_ptr(),
                                    cnt.data_ptr(), _lib.stream_handle(scores.device)),
               "swattn_topk_blocks")
    return BlockSelection(cfg.B, n, topk[:, :, :cfg.k_top], cnt, cfg.N_init, cfg.N_local)


def window_coverage_check(sel: BlockSelection, w: int) -> bool:
    """selection.py:139-151 (host check, used by the tests)."""
    if w < 1:
        raise ValueError(f"window size must be >= 1, got w={w}")
    B = sel.block_size
    for g in range(sel.num_groups):
        for i in range(sel.n):
            first = max(0, i - w + 1) // B
            needed = np.arange(first, i // B + 1)
            if not np.isin(needed, sel.query_blocks(g, i), assume_unique=True).all():
                return False
    return True


def _shared(Q, ck1: CompressedKeys, ck2: CompressedKeys | None, cfg: AttentionConfig,
            mode: int) -> ScoreMatrix:
    n = _cfg_ok(cfg, Q, torch.empty((Q.shape[0], cfg.h_kv, cfg.d_h)))
    Qd = to_device_bf16(Q, "Q")
    m1 = ck1.m
    shared = torch.zeros((n, cfg.h_kv, m1), dtype=torch.float32, device=Qd.device)
    nv = torch.empty(n, dtype=torch.uint8, device=Qd.device)
    k2 = ck2.keys if (ck2 is not None and ck2.m) else None
    L = _lib.lib()
    _lib.check(L.swattn_shared_scores(_lib.c_config(cfg), Qd.data_ptr(), ck1.keys.data_ptr() if m1 else None,
                                      _lib.ptr(k2), n, mode, shared.data_ptr(), nv.data_ptr(),
                                      _lib.stream_handle(Qd.device)), "swattn_shared_scores")
    return ScoreMatrix(shared, "shared" if mode != 2 else "shared-approx", nv.bool())


def fused_shared_scores_exact(Q, ck1: CompressedKeys, cfg: AttentionConfig, B_q: int = 64,
                              B_k: int = 64, counter=None, stats=None) -> ScoreMatrix:
    """selection.py:238-276 (debug/parity path: materialises [n, h_kv, m1])."""
    if B_q < 1 or B_k < 1:
        raise ValueError(f"tile sizes must be >= 1, got B_q={B_q}, B_k={B_k}")
    return _shared(Q, ck1, None, cfg, 1)


def fused_shared_scores_approx(Q, ck1: CompressedKeys, ck2: CompressedKeys, cfg: AttentionConfig,
                               B_q: int = 64, B_k: int = 64, counter=None,
                               stats=None) -> ScoreMatrix:
    """selection.py:279-333 (debug/parity path: materialises [n, h_kv, m1])."""
    if B_q < 1 or B_k < 1:
        raise ValueError(f"tile sizes must be >= 1, got B_q={B_q}, B_k={B_k}")
    return _shared(Q, ck1, ck2, cfg, 2)


# ---------------------------------------------------------------- selection fixtures
SELECTION_TAG = 0xB5  # selection.py:48


def _full_block_lists(sel: BlockSelection):
    """Flat u32 stream of the reference fixture body: per (group, row) the
    count then the ascending block ids (init below lo, top-k, local [lo, b]),
    built vectorised from the device top-k lists."""
    top, cnt = sel._host_topk()
    G, n = cnt.shape
    B = sel.block_size
    i = np.arange(n, dtype=np.int64)
    b = i // B
    lo = np.maximum(0, b - sel.N_local + 1)
    ninit = np.minimum(sel.N_init, lo)                      # init blocks below lo
    nloc = b - lo + 1
    sizes = ninit[None, :] + cnt.astype(np.int64) + nloc[None, :]   # [G, n]
    row_len = 1 + sizes.ravel()
    starts = np.concatenate([[0], np.cumsum(row_len)[:-1]])
    out = np.empty(int(row_len.sum()), dtype="<u4")
    out[starts] = sizes.ravel()
    # position of each entry inside its row, then its block id
    total_entries = int(sizes.sum())
    row_of = np.repeat(np.arange(G * n), sizes.ravel())
    first = np.repeat(starts + 1, sizes.ravel())
    k = np.arange(total_entries) - np.repeat(np.cumsum(sizes.ravel()) - sizes.ravel(), sizes.ravel())
    r_i = row_of % n
    r_g = row_of // n
    ni, ct = ninit[r_i], cnt.reshape(-1)[row_of].astype(np.int64)
    ids = np.where(k < ni, k,
                   np.where(k < ni + ct, top.reshape(G * n, -1)[row_of, np.clip(k - ni, 0, top.shape[2] - 1)],
                            lo[r_i] + (k - ni - ct)))
    del r_g
    out[first + k] = ids.astype("<u4")
    return out


def save_selection(sel: BlockSelection, path) -> None:
    """selection.py:386-400: core magic, tag byte, u32 groups / n / block
    size, then per (group, row) a u32 count and that many u32 block ids."""
    import struct

    from .core import TENSOR_MAGIC, atomic_write_bytes
    head = TENSOR_MAGIC + struct.pack("<B", SELECTION_TAG) + struct.pack(
        "<III", sel.num_groups, sel.n, sel.block_size)
    atomic_write_bytes(path, head + _full_block_lists(sel).tobytes())


def load_selection(path, N_init: int = 1, N_local: int = 32, device=None) -> BlockSelection:
    """selection.py:403-430 with the same errors.  The fixture stores full
    block sets; the init (N_init) / local (N_local) structure -- not in the
    file, paper defaults -- is split off so the result is a device
    BlockSelection (top-k lists) ready for sparse_forward."""
    import struct

    from .core import TENSOR_MAGIC, TensorFormatError
    with open(path, "rb") as fh:
        blob = fh.read()
    head = len(TENSOR_MAGIC)
    if len(blob) < head + 13 or blob[:head] != TENSOR_MAGIC:
        raise TensorFormatError(f"malformed header: bad magic in {path}")
    (tag,) = struct.unpack_from("<B", blob, head)
    if tag != SELECTION_TAG:
        raise TensorFormatError(f"not a selection fixture: tag {tag}")
    groups, n, block_size = struct.unpack_from("<III", blob, head + 1)
    body = np.frombuffer(blob, dtype="<u4", offset=head + 13) if len(blob) > head + 13 else \
        np.empty(0, dtype="<u4")
    rows, off = [], 0
    for _ in range(groups * n):
        if off >= body.size:
            raise TensorFormatError("truncated payload: row count missing")
        c = int(body[off])
        if off + 1 + c > body.size:
            raise TensorFormatError("truncated payload: row indices missing")
        rows.append(body[off + 1: off + 1 + c].astype(np.int64))
        off += 1 + c
    if off != body.size:
        raise TensorFormatError("oversized payload: trailing bytes")
    k_top = 0
    tops = []
    for r, blocks in enumerate(rows):
        i = r % n
        b = i // block_size
        lo = max(0, b - N_local + 1)
        t = blocks[(blocks >= N_init) & (blocks < lo)]
        tops.append(t)
        k_top = max(k_top, t.size)
    top = np.full((groups, n, max(k_top, 1)), -1, dtype=np.int32)
    cnt = np.zeros((groups, n), dtype=np.int32)
    for r, t in enumerate(tops):
        top[r // n, r % n, :t.size] = t
        cnt[r // n, r % n] = t.size
    dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
    return BlockSelection(block_size, n, torch.from_numpy(top).to(dev), torch.from_numpy(cnt).to(dev),
                          N_init, N_local)
