"""Block selection (reference: selection.py).

``select_blocks`` = K1 -> K2 -> K3 (+ float64 boundary re-rank) on one CUDA
stream through ``swattn_select_blocks``.  The result is a device-resident
:class:`BlockSelection` holding only the per-token top-k lists; the
initial/local blocks are implicit (selection.py:113-119), and the
reference's tuple-of-arrays view is materialised lazily on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import to_device_bf16
from .compression import CompressedKeys, ScoreMatrix, mean_pool_keys
from .core import AttentionConfig, OpCounter, validate_config

SELECT_MODES = ("exact", "fused-exact", "approx")


class BlockSelection:
    """Per-(KV group, query token) sorted visible block indices (selection.py:51-90).

    Two interchangeable forms, both exposing the reference's host view
    (``blocks``, ``counts``, ``query_blocks``, ``visible_spans``):

    * the reference constructor ``BlockSelection(block_size, n, blocks,
      counts=None)`` -- ``blocks[g][i]`` strictly increasing int64 arrays
      (selection.py:51-66), e.g. from ``load_selection`` or built by hand
      like the reference's ``_all_blocks_selection`` (bench.py:207-210);
    * the device form ``BlockSelection.from_topk(...)`` that
      ``select_blocks`` returns: top-k lists [h_kv, n, k] int32 (ascending,
      -1 padded) + their counts [h_kv, n] on the GPU, the initial and local
      blocks implicit (selection.py:113-119).

    ``sparse_forward`` runs the part A + part B kernels on every selection
    whose rows are init U local U (<= k_top blocks in [N_init, lo)) under the
    call's config -- checked row by row, so a reference-built selection takes
    the same kernels -- and the general block-list kernel on any other.
    Immutable like the reference's frozen dataclass.
    """

    __slots__ = ("block_size", "n", "_blocks", "_counts", "_topk", "_topk_cnt", "_N_init",
                 "_N_local", "n_reranked", "_host")

    def __init__(self, block_size: int, n: int, blocks, counts=None):
        object.__setattr__(self, "block_size", int(block_size))
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "_blocks",
                           tuple(tuple(np.asarray(r, dtype=np.int64) for r in grp) for grp in blocks))
        object.__setattr__(self, "_counts", counts)
        for name in ("_topk", "_topk_cnt", "_N_init", "_N_local", "n_reranked"):
            object.__setattr__(self, name, None)
        object.__setattr__(self, "_host", {})

    @classmethod
    def from_topk(cls, block_size: int, n: int, topk, topk_cnt, N_init: int, N_local: int,
                  n_reranked=None) -> "BlockSelection":
        self = cls.__new__(cls)
        object.__setattr__(self, "block_size", int(block_size))
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "_blocks", None)
        object.__setattr__(self, "_counts", None)
        object.__setattr__(self, "_topk", topk)
        object.__setattr__(self, "_topk_cnt", topk_cnt)
        object.__setattr__(self, "_N_init", int(N_init))
        object.__setattr__(self, "_N_local", int(N_local))
        object.__setattr__(self, "n_reranked", n_reranked)
        object.__setattr__(self, "_host", {})
        return self

    def __setattr__(self, name, value):
        import dataclasses
        raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")

    def __repr__(self) -> str:
        form = "top-k" if self.is_topk_form else "blocks"
        return f"BlockSelection(block_size={self.block_size}, n={self.n}, groups={self.num_groups}, form={form})"

    # ------------------------------------------------------------------ forms
    @property
    def is_topk_form(self) -> bool:
        return self._topk is not None

    @property
    def topk(self):
        """Device top-k lists [h_kv, n, k] (top-k form only)."""
        if self._topk is None:
            raise ValueError("this selection holds explicit block lists; use "
                             "topk_form(cfg) for the init U local U top-k form")
        return self._topk

    @property
    def topk_cnt(self):
        if self._topk_cnt is None:
            raise ValueError("this selection holds explicit block lists; use topk_form(cfg)")
        return self._topk_cnt

    @property
    def N_init(self):
        return self._N_init

    @property
    def N_local(self):
        return self._N_local

    @property
    def num_groups(self) -> int:
        return int(self._topk.shape[0]) if self._topk is not None else len(self._blocks)

    def _host_topk(self):
        if "topk" not in self._host:
            self._host["topk"] = self._topk.cpu().numpy()
            self._host["cnt"] = self._topk_cnt.cpu().numpy()
        return self._host["topk"], self._host["cnt"]

    def _flat(self):
        """(lengths [G, n] int64, concatenated block ids int64) of the host view."""
        if "flat" not in self._host:
            if self._blocks is None:
                lens, ids = _topk_flat(self)
            else:
                G = len(self._blocks)
                lens = np.array([[r.size for r in grp] for grp in self._blocks],
                                dtype=np.int64).reshape(G, self.n)
                rows = [r for grp in self._blocks for r in grp]
                ids = np.concatenate(rows) if rows else np.empty(0, dtype=np.int64)
            self._host["flat"] = (lens, ids.astype(np.int64, copy=False))
        return self._host["flat"]

    # ------------------------------------------------------------------ host view
    def query_blocks(self, g: int, i: int) -> np.ndarray:
        if self._blocks is not None:
            return self._blocks[g][i]
        top, cnt = self._host_topk()
        b = i // self.block_size
        lo = max(0, b - self._N_local + 1)
        base = np.union1d(np.arange(min(self._N_init, b + 1)), np.arange(lo, b + 1))
        return np.union1d(base, top[g, i, :cnt[g, i]]).astype(np.int64)

    @property
    def blocks(self):
        if self._blocks is not None:
            return self._blocks
        if "blocks" not in self._host:
            lens, ids = self._flat()
            ends = np.cumsum(lens.ravel())
            starts = ends - lens.ravel()
            G = lens.shape[0]
            self._host["blocks"] = tuple(
                tuple(ids[starts[g * self.n + i]:ends[g * self.n + i]] for i in range(self.n))
                for g in range(G))
        return self._host["blocks"]

    @property
    def counts(self):
        """(n_init, #local, #top) per (g, i) (selection.py:134); None for
        selections built from explicit lists without counts (fixtures)."""
        if self._topk is None:
            return self._counts
        _, cnt = self._host_topk()
        i = np.arange(self.n)
        b = i // self.block_size
        lo = np.maximum(0, b - self._N_local + 1)
        out = np.zeros((self.num_groups, self.n, 3), dtype=np.int64)
        out[:, :, 0] = np.minimum(self._N_init, b + 1)
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

    # ------------------------------------------------------------------ kernel forms
    def topk_form(self, cfg: AttentionConfig, device=None):
        """(topk [h_kv, n, cfg.k_top] int32, cnt [h_kv, n] int32) on the device
        if every row is init U local U top (<= k_top blocks in [N_init, lo))
        under cfg, else None."""
        key = ("topk", cfg.B, cfg.N_init, cfg.N_local, cfg.k_top, str(device))
        if key in self._host:
            return self._host[key]
        res = None
        if self.block_size == cfg.B:
            if self._topk is not None:
                if (self._N_init, self._N_local) == (cfg.N_init, cfg.N_local) and \
                        self._topk.shape[2] <= cfg.k_top and (device is None or
                                                            self._topk.device == torch.device(device)):
                    top = self._topk
                    if top.shape[2] < cfg.k_top:
                        pad = torch.full((top.shape[0], self.n, cfg.k_top - top.shape[2]), -1,
                                         dtype=torch.int32, device=top.device)
                        top = torch.cat([top.to(torch.int32), pad], dim=2)
                    res = (top.contiguous(), self._topk_cnt.to(torch.int32).contiguous())
                else:
                    res = _structured_from_flat(self, cfg, device or self._topk.device)
            else:
                res = _structured_from_flat(self, cfg, device)
        self._host[key] = res
        return res

    def list_form(self, device=None):
        """(blocks [h_kv, n, ld] int32 -1 padded, ld, cnt [h_kv, n] int32) on the device."""
        key = ("lists", str(device))
        if key not in self._host:
            lens, ids = self._flat()
            G = lens.shape[0]
            ld = max(1, int(lens.max()) if lens.size else 1)
            out = np.full((G * self.n, ld), -1, dtype=np.int32)
            row = np.repeat(np.arange(G * self.n), lens.ravel())
            pos = np.arange(ids.size) - np.repeat(np.cumsum(lens.ravel()) - lens.ravel(), lens.ravel())
            out[row, pos] = ids
            dev = torch.device(device or "cuda")
            self._host[key] = (torch.from_numpy(out.reshape(G, self.n, ld)).to(dev), ld,
                               torch.from_numpy(lens.astype(np.int32)).to(dev))
        return self._host[key]

    def first_empty_row(self):
        """(g, i) of the first row whose visible set is empty (sparse.py:75-76
        order: g outer, i inner), or None."""
        lens, ids = self._flat()
        G = lens.shape[0]
        row = np.repeat(np.arange(G * self.n), lens.ravel())
        i = row % self.n
        start = ids * self.block_size
        ok = (ids >= 0) & (start <= i) & (start < self.n)
        has = np.zeros(G * self.n, dtype=bool)
        has[row[ok]] = True
        bad = np.flatnonzero(~has)
        if bad.size == 0:
            return None
        return int(bad[0] // self.n), int(bad[0] % self.n)

    def key_visits(self) -> np.ndarray:
        """Visited keys per (g, i) (sparse.py:83 `visits`), [h_kv, n] int64."""
        lens, ids = self._flat()
        G = lens.shape[0]
        row = np.repeat(np.arange(G * self.n), lens.ravel())
        i = row % self.n
        start = ids * self.block_size
        end = np.minimum(np.minimum(start + self.block_size, self.n), i + 1)
        span = np.where(ids >= 0, np.maximum(end - start, 0), 0)
        return np.bincount(row, weights=span, minlength=G * self.n).astype(np.int64).reshape(G, self.n)


def _topk_flat(sel: BlockSelection):
    """Flat (lengths, ids) of a top-k-form selection, vectorised: per row the
    init blocks below lo, the top-k ids, then the local window [lo, b]."""
    top, cnt = sel._host_topk()
    G, n = cnt.shape
    B = sel.block_size
    i = np.arange(n, dtype=np.int64)
    b = i // B
    lo = np.maximum(0, b - sel._N_local + 1)
    ninit = np.minimum(sel._N_init, lo)                     # init blocks below lo
    nloc = b - lo + 1
    sizes = (ninit[None, :] + cnt.astype(np.int64) + nloc[None, :]).ravel()   # [G * n]
    total = int(sizes.sum())
    row_of = np.repeat(np.arange(G * n), sizes)
    k = np.arange(total) - np.repeat(np.cumsum(sizes) - sizes, sizes)
    r_i = row_of % n
    ni, ct = ninit[r_i], cnt.reshape(-1)[row_of].astype(np.int64)
    topw = top.reshape(G * n, -1) if top.shape[2] else np.full((G * n, 1), -1, dtype=np.int32)
    ids = np.where(k < ni, k,
                   np.where(k < ni + ct, topw[row_of, np.clip(k - ni, 0, topw.shape[1] - 1)],
                            lo[r_i] + (k - ni - ct)))
    return sizes.reshape(G, n), ids.astype(np.int64)


def _structured_from_flat(sel: BlockSelection, cfg: AttentionConfig, device):
    """Split explicit block lists into init U local U top-k under cfg, or None
    when some row does not have that shape (then the general kernel runs)."""
    lens, ids = sel._flat()
    G, n = lens.shape
    B = cfg.B
    rows = G * n
    row = np.repeat(np.arange(rows), lens.ravel())
    i = row % n
    b = i // B
    lo = np.maximum(0, b - cfg.N_local + 1)
    n_init = np.minimum(cfg.N_init, b + 1)
    is_base = (ids < n_init) | ((ids >= lo) & (ids <= b))
    is_top = (ids >= cfg.N_init) & (ids < lo)
    if ids.size and not np.all((is_base | is_top) & (ids >= 0)):
        return None
    # strictly increasing within each row
    if ids.size > 1:
        lr = lens.ravel()
        first = np.zeros(ids.size, dtype=bool)
        first[(np.cumsum(lr) - lr)[lr > 0]] = True
        inc = np.diff(ids) > 0
        if not np.all(inc | first[1:]):
            return None
    ii = np.arange(n)
    bb = ii // B
    lo_r = np.maximum(0, bb - cfg.N_local + 1)
    ni_r = np.minimum(cfg.N_init, bb + 1)
    nbase = ni_r + (bb + 1 - lo_r) - np.maximum(0, ni_r - lo_r)
    base_cnt = np.bincount(row[is_base], minlength=rows).reshape(G, n)
    if not np.array_equal(base_cnt, np.broadcast_to(nbase, (G, n))):
        return None
    top_cnt = np.bincount(row[is_top], minlength=rows)
    if top_cnt.size and int(top_cnt.max()) > cfg.k_top:
        return None
    kw = max(cfg.k_top, 1)
    top = np.full((rows, kw), -1, dtype=np.int32)
    trow = row[is_top]
    tpos = np.arange(trow.size) - np.repeat(np.cumsum(top_cnt) - top_cnt, top_cnt)
    top[trow, tpos] = ids[is_top]
    dev = torch.device(device or "cuda")
    return (torch.from_numpy(top.reshape(G, n, kw)[:, :, :cfg.k_top].copy()).to(dev),
            torch.from_numpy(top_cnt.astype(np.int32).reshape(G, n)).to(dev))


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
    """Grow-only device scratch buffers carved by the C ABI, one per (device,
    CUDA stream): calls on different streams never share scratch.  When a
    buffer grows, the old one is released through the caching allocator with
    record_stream, so kernels still queued on that stream keep it alive."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, device) -> torch.Tensor:
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev)
        key = (dev.index or 0, stream.cuda_stream)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                buf.record_stream(stream)
            buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
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
    return BlockSelection.from_topk(cfg.B, n, topk[:, :, :cfg.k_top], cnt, cfg.N_init, cfg.N_local,
                                    n_reranked=nre)


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
    return BlockSelection.from_topk(cfg.B, n, topk[:, :, :cfg.k_top], cnt, cfg.N_init, cfg.N_local)


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
    count then the ascending block ids."""
    lens, ids = sel._flat()
    lr = lens.ravel()
    out = np.empty(lr.size + ids.size, dtype="<u4")
    starts = np.arange(lr.size) + (np.cumsum(lr) - lr)      # slot of each row's count
    out[starts] = lr
    pos = np.ones(out.size, dtype=bool)
    pos[starts] = False
    out[pos] = ids.astype("<u4")
    return out


def save_selection(sel: BlockSelection, path) -> None:
    """selection.py:386-400: core magic, tag byte, u32 groups / n / block
    size, then per (group, row) a u32 count and that many u32 block ids."""
    import struct

    from .core import TENSOR_MAGIC, atomic_write_bytes
    head = TENSOR_MAGIC + struct.pack("<B", SELECTION_TAG) + struct.pack(
        "<III", sel.num_groups, sel.n, sel.block_size)
    atomic_write_bytes(path, head + _full_block_lists(sel).tobytes())


def load_selection(path) -> BlockSelection:
    """selection.py:403-430: the stored block lists exactly, counts=None,
    with the reference's errors.  sparse_forward takes the result directly
    (init U local U top-k rows run on the part A / part B kernels, any other
    shape on the general block-list kernel)."""
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
    off = head + 13
    nbytes = len(blob)
    out = []
    for _ in range(groups):
        rows = []
        for _ in range(n):
            if nbytes < off + 4:
                raise TensorFormatError("truncated payload: row count missing")
            (count,) = struct.unpack_from("<I", blob, off)
            off += 4
            if nbytes < off + 4 * count:
                raise TensorFormatError("truncated payload: row indices missing")
            rows.append(np.frombuffer(blob, dtype="<u4", count=count, offset=off).astype(np.int64))
            off += 4 * count
        out.append(tuple(rows))
    if off != nbytes:
        raise TensorFormatError("oversized payload: trailing bytes")
    return BlockSelection(block_size, n, tuple(out), counts=None)
