"""CPU oracle for the InfLLM-V2 switchable-attention hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2509_24663_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or as the timed CPU baseline -- never as the thing measured or shipped.

This is a vectorised numpy restatement of the reference package ``swattn``
0.1.0 (``/root/reference/pkg/src/swattn``).  Every function names the
reference lines it follows.  Arithmetic is float64 throughout, exactly as the
reference does (``core.py:8-9``); storage-dtype casts happen where the
reference casts (``compression.py:85``, ``sparse.py:98``).  Storage is
``ml_dtypes.bfloat16``: the reference is dtype-generic, and running it
unmodified on bf16 arrays is the parity contract.

Parity pinning: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by the *unmodified reference* (``oracle/make_golden.py``,
run in the build container where ``/root/reference`` exists) -- pooled keys
bit-exact, scores to 1e-12, selections exactly, outputs to bf16 ulp.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import ml_dtypes
import numpy as np

BF16 = np.dtype(ml_dtypes.bfloat16)


@dataclass(frozen=True)
class Profile:
    """Field-for-field mirror of ``AttentionConfig`` (core.py:48-108)."""

    h_q: int = 32
    h_kv: int = 2
    d_h: int = 128
    B: int = 64
    l_C1: int = 32
    s_C1: int = 16
    l_C2: int = 128
    s_C2: int = 64
    l: int = 5
    s: int = 4
    N_init: int = 1
    N_local: int = 32
    k_top: int = 63
    w: int = 1984
    scale_compressed_logits: bool = True

    @property
    def G(self) -> int:
        return self.h_q // self.h_kv


SMALL = Profile(h_q=4, h_kv=2, d_h=16, B=16, l_C1=8, s_C1=4, l_C2=32, s_C2=16,
                l=5, s=4, N_init=1, N_local=2, k_top=3, w=16)   # bench.py:199-204
PAPER = Profile()                                                # core.py:78-91


# --------------------------------------------------------------------------- inputs

def draw_qkv(n: int, h_q: int, h_kv: int, d_h: int, seed: int, dtype=BF16):
    """One Philox(key=seed) stream; normal(0,1) draws of Q, then K, then V in
    float64, cast to the storage dtype (core.py:229-240)."""
    rng = np.random.Generator(np.random.Philox(key=np.uint64(seed)))
    out = []
    for heads in (h_q, h_kv, h_kv):
        x = rng.normal(0.0, 1.0, size=(n, heads, d_h))
        out.append(np.ascontiguousarray(x.astype(dtype)))
    return tuple(out)


def digest(*arrays) -> str:
    """sha256 over the raw bytes of the given arrays (fixture pinning)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------------------- compression

def n_pooled(n: int, length: int, stride: int) -> int:
    """m = floor((n-length)/stride)+1 complete windows, 0 if n < length
    (compression.py:64-78)."""
    return 0 if n < length else (n - length) // stride + 1


def visible_counts(rows: np.ndarray, length: int, stride: int) -> np.ndarray:
    """#pooled entries with span_end <= i, i.e. (i+1-l)//s+1 clamped at 0
    (compression.py:89-91, closed form bench.py:89-93)."""
    rows = np.asarray(rows, dtype=np.int64)
    return np.where(rows + 1 >= length, (rows + 1 - length) // stride + 1, 0)


def pool(K: np.ndarray, length: int, stride: int) -> np.ndarray:
    """Mean of K over windows [j*stride, j*stride+length), complete windows
    only, accumulated in float64 and cast back to K's dtype
    (compression.py:64-86).  Returns (m, h_kv, d_h)."""
    n = K.shape[0]
    m = n_pooled(n, length, stride)
    if m == 0:
        return np.empty((0,) + K.shape[1:], dtype=K.dtype)
    K64 = K.astype(np.float64)
    csum = np.concatenate([np.zeros((1,) + K.shape[1:]), np.cumsum(K64, axis=0)])
    # cumsum differences are exact here: bf16 inputs sum exactly in f64
    # (<= 27 significant bits), so this equals the reference's window mean.
    starts = np.arange(m) * stride
    sums = csum[starts + length] - csum[starts]
    return np.ascontiguousarray((sums / length).astype(K.dtype))


def pool_exact_windows(K: np.ndarray, length: int, stride: int) -> np.ndarray:
    """Same as :func:`pool` but summing each window explicitly (for inputs
    whose cumsum would not be exact)."""
    n = K.shape[0]
    m = n_pooled(n, length, stride)
    K64 = K.astype(np.float64)
    out = np.empty((m,) + K.shape[1:], dtype=np.float64)
    for j in range(m):
        out[j] = K64[j * stride:j * stride + length].mean(axis=0)
    return out.astype(K.dtype)


# --------------------------------------------------------------------------- scoring

def _logits(Qrows64: np.ndarray, Kc64: np.ndarray, scale: float) -> np.ndarray:
    # (R, G, d) x (m, d) -> (R, G, m)
    return np.einsum("rgd,md->rgm", Qrows64, Kc64, optimize=True) * scale


def _masked_lse(S: np.ndarray, vis: np.ndarray) -> np.ndarray:
    """log-sum-exp over the first vis[r] columns of S[r]; -inf when none
    (selection.py:165-196 online form; compression.py:146-152 direct form)."""
    R, G, m = S.shape
    cols = np.arange(m)[None, None, :]
    Sm = np.where(cols < vis[:, None, None], S, -np.inf)
    mx = Sm.max(axis=2) if m else np.full((R, G), -np.inf)
    mx_safe = np.where(np.isneginf(mx), 0.0, mx)
    with np.errstate(divide="ignore"):
        return mx_safe + np.log(np.exp(Sm - mx_safe[..., None]).sum(axis=2))


def shared_scores(Q, K, cfg: Profile, mode: str = "approx", rows=None, chunk: int = 128,
                  ck1=None, ck2=None):
    """S^shared rows: for each row i and group g,
    sum_h exp(q_h . k1_j * scale - lse_h(i)) over causally visible C1 columns,
    0 elsewhere.

    mode "approx": lse over visible C2 columns, rows with no visible C2 but
    some visible C1 fall back to the exact C1 lse
    (selection.py:279-348, _group_lse :165-196, _pass2_shared :199-222,
    _exact_lse_rows :336-348).
    mode "exact"/"fused-exact": lse over visible C1 columns, i.e. per-head
    softmax then head-group sum (compression.py:94-157, selection.py:238-276).

    Returns (S [R, h_kv, m1] float64, no_visible [R] bool).
    """
    n = Q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    G = cfg.G
    scale = 1.0 / np.sqrt(cfg.d_h) if cfg.scale_compressed_logits else 1.0
    if ck1 is None:
        ck1 = pool(K, cfg.l_C1, cfg.s_C1)
    if ck2 is None and mode == "approx":
        ck2 = pool(K, cfg.l_C2, cfg.s_C2)
    m1 = ck1.shape[0]
    vis1 = visible_counts(rows, cfg.l_C1, cfg.s_C1)
    out = np.zeros((rows.size, cfg.h_kv, m1), dtype=np.float64)
    no_visible = vis1 == 0
    if m1 == 0:
        return out, no_visible
    K1 = ck1.astype(np.float64)
    if mode == "approx":
        K2 = ck2.astype(np.float64)
        vis2 = visible_counts(rows, cfg.l_C2, cfg.s_C2) if ck2.shape[0] else np.zeros_like(vis1)
    for c0 in range(0, rows.size, chunk):
        r = rows[c0:c0 + chunk]
        v1 = vis1[c0:c0 + chunk]
        # columns no row of the chunk sees are skipped (the reference's tile
        # loops stop at the first future tile, selection.py:178-179,211-212);
        # they stay 0 in `out` exactly as masked columns do
        c1 = int(v1.max()) if v1.size else 0
        if c1 == 0:
            continue
        Qr = Q[r].astype(np.float64)
        for g in range(cfg.h_kv):
            Qg = Qr[:, g * G:(g + 1) * G]
            S1 = _logits(Qg, K1[:c1, g], scale)
            if mode == "approx":
                v2 = vis2[c0:c0 + chunk]
                c2 = int(v2.max()) if v2.size else 0
                if K2.shape[0] and c2 > 0:
                    lse = _masked_lse(_logits(Qg, K2[:c2, g], scale), v2)
                else:
                    lse = np.full(S1.shape[:2], -np.inf)
                fb = (v2 == 0) & (v1 > 0)
                if fb.any():
                    lse[fb] = _masked_lse(S1[fb], v1[fb])
            else:
                lse = _masked_lse(S1, v1)
            lse_safe = np.where(np.isneginf(lse), 0.0, lse)
            P = np.exp(S1 - lse_safe[..., None])
            P = np.where(np.arange(c1)[None, None, :] < v1[:, None, None], P, 0.0)
            out[c0:c0 + chunk, g, :c1] = P.sum(axis=1)
    return out, no_visible


def block_scores(S: np.ndarray, l: int, s: int) -> np.ndarray:
    """Block j = max over columns [j*s, min(j*s+l, m)); ceil(m/s) blocks
    (compression.py:160-173)."""
    R, P, m = S.shape
    nb = -(-m // s) if m else 0
    out = np.empty((R, P, nb), dtype=S.dtype)
    for t in range(l):
        cols = np.arange(nb) * s + t
        valid = cols < m
        v = np.full((R, P, nb), -np.inf)
        v[..., valid] = S[..., cols[valid]]
        out = v if t == 0 else np.maximum(out, v)
    return out


# --------------------------------------------------------------------------- selection

def topk_blocks(scmp: np.ndarray, no_visible: np.ndarray, rows: np.ndarray, n: int,
                cfg: Profile):
    """Per (g, row): the k_top best candidate blocks, ascending.

    Candidates for query block b are [N_init, min(lo, n_cols)) with
    lo = max(0, b-N_local+1); ranking is score descending, ties to the lower
    block index (the stable argsort of selection.py:123-126); rows flagged
    no_visible take none (:129).  Returns (topk [h_kv, R, k_top] int64 padded
    with -1, counts [h_kv, R, 3] = (n_init, #local, #top) (:134)).
    """
    R, P, n_cols = scmp.shape
    nb = -(-n // cfg.B)
    assert n_cols <= nb, "more score columns than selection blocks (selection.py:106)"
    top = np.full((P, R, cfg.k_top), -1, dtype=np.int64)
    counts = np.zeros((P, R, 3), dtype=np.int64)
    for ri, i in enumerate(np.asarray(rows)):
        b = int(i) // cfg.B
        lo = max(0, b - cfg.N_local + 1)
        cand_hi = min(lo, n_cols)
        ncand = max(0, cand_hi - cfg.N_init)
        k = min(cfg.k_top, ncand) if not no_visible[ri] else 0
        counts[:, ri] = (min(cfg.N_init, b + 1), b + 1 - lo, k)
        if k == 0:
            continue
        cand = np.arange(cfg.N_init, cand_hi)
        for g in range(P):
            sc = scmp[ri, g, cfg.N_init:cand_hi]
            order = np.lexsort((cand, -sc))[:k]       # score desc, index asc
            top[g, ri, :k] = np.sort(cand[order])
    return top, counts


def full_block_set(topk_row: np.ndarray, i: int, cfg: Profile) -> np.ndarray:
    """Sorted union init U local U top-k for one row (selection.py:113-133)."""
    b = i // cfg.B
    lo = max(0, b - cfg.N_local + 1)
    base = np.union1d(np.arange(min(cfg.N_init, b + 1)), np.arange(lo, b + 1))
    t = topk_row[topk_row >= 0]
    return np.union1d(base, t).astype(np.int64)


def select(Q, K, cfg: Profile, mode: str = "approx", rows=None, ck1=None, ck2=None):
    """select_blocks pipeline restated (selection.py:354-383): pool, score,
    max-pool, top-k.  Returns (topk, counts, scmp) for the given rows.
    ck1 / ck2: the pooled keys when the caller already has them."""
    n = Q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    S, nv = shared_scores(Q, K, cfg, mode=mode, rows=rows, ck1=ck1, ck2=ck2)
    scmp = block_scores(S, cfg.l, cfg.s)
    top, counts = topk_blocks(scmp, nv, rows, n, cfg)
    return top, counts, scmp


# --------------------------------------------------------------------------- attention

def token_mask_row(i: int, blocks: np.ndarray, n: int, B: int) -> np.ndarray:
    """Keys visible to query i: union of selected blocks clipped at
    min(start+B, n, i+1) (selection.py:73-87, sparse.py:33-40)."""
    m = np.zeros(n, dtype=bool)
    for j in blocks:
        m[j * B:min(j * B + B, n, i + 1)] = True
    return m


def visible_keys(i: int, blocks: np.ndarray, n: int, B: int) -> np.ndarray:
    """Ascending key ids of token_mask_row (blocks ascending and disjoint)."""
    parts = [np.arange(j * B, min(j * B + B, n, i + 1)) for j in blocks]
    parts = [p for p in parts if p.size]
    return np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)


def sparse_attention(Q, K, V, topk: np.ndarray, cfg: Profile, rows=None, out_dtype=None):
    """Exact masked softmax over each row's visible set, float64
    (sparse.py:43-98, oracle form sparse.py:101-127).  topk is
    [h_kv, n, k_top] (-1 padded).  Returns (O [R, h_q, d] float64 or cast,
    lse [R, h_q] float64)."""
    n = Q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    G = cfg.G
    scale = 1.0 / np.sqrt(cfg.d_h)
    K64 = K.astype(np.float64, copy=False)
    V64 = V.astype(np.float64, copy=False)
    O = np.empty((rows.size, cfg.h_q, cfg.d_h))
    L = np.empty((rows.size, cfg.h_q))
    for ri, i in enumerate(rows):
        for g in range(cfg.h_kv):
            blocks = full_block_set(topk[g, i], int(i), cfg)
            keys = visible_keys(int(i), blocks, n, cfg.B)
            if keys.size == 0:
                raise RuntimeError(f"query {i} in group {g} has an empty visible set")
            q = Q[i, g * G:(g + 1) * G].astype(np.float64)
            S = (q @ K64[keys, g].T) * scale
            mx = S.max(axis=1)
            z = np.exp(S - mx[:, None])
            ell = z.sum(axis=1)
            O[ri, g * G:(g + 1) * G] = (z / ell[:, None]) @ V64[keys, g]
            L[ri, g * G:(g + 1) * G] = mx + np.log(ell)
    if out_dtype is not None:
        O = O.astype(out_dtype)
    return O, L


def sparse_backward(Q, K, V, topk: np.ndarray, dO, cfg: Profile, rows=None):
    """Gradients of sum(O * dO) through the masked softmax (sparse.py:130-185).

    The forward is recomputed in float64 (sparse.py:157-158), delta = rowsum
    dO * O (:169), and per row the visible keys give P = exp(S - lse),
    dP = dO V^T, dS = P (dP - delta), dQ = dS K scale, dK += dS^T Q scale,
    dV += P^T dO (:171-180).  The reference walks spans in ascending order;
    here all visible keys of a row are one matrix product (same sums in
    float64, different association).  dQ is returned for `rows` (all rows by
    default); dK / dV accumulate the contributions of `rows` only (complete
    for rows=None).  Returns float64 (dQ [R, h_q, d], dK [n, h_kv, d],
    dV [n, h_kv, d]); the reference casts to the storage dtype (:185)."""
    n = Q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    G = cfg.G
    scale = 1.0 / np.sqrt(cfg.d_h)
    K64 = K.astype(np.float64)
    V64 = V.astype(np.float64)
    dQ = np.zeros((rows.size, cfg.h_q, cfg.d_h))
    dK = np.zeros((n, cfg.h_kv, cfg.d_h))
    dV = np.zeros((n, cfg.h_kv, cfg.d_h))
    for ri, i in enumerate(rows):
        for g in range(cfg.h_kv):
            blocks = full_block_set(topk[g, i], int(i), cfg)
            keys = np.flatnonzero(token_mask_row(int(i), blocks, n, cfg.B))
            q = Q[i, g * G:(g + 1) * G].astype(np.float64)
            do = dO[i, g * G:(g + 1) * G].astype(np.float64)
            S = (q @ K64[keys, g].T) * scale
            mx = S.max(axis=1)
            z = np.exp(S - mx[:, None])
            ell = z.sum(axis=1)
            lse = mx + np.log(ell)
            P = np.exp(S - lse[:, None])
            O = P @ V64[keys, g]
            delta = (do * O).sum(axis=1)
            dP = do @ V64[keys, g].T
            dS = P * (dP - delta[:, None])
            dQ[ri, g * G:(g + 1) * G] = (dS @ K64[keys, g]) * scale
            dK[keys, g] += (dS.T @ q) * scale
            dV[keys, g] += P.T @ do
    return dQ, dK, dV


def dense_backward(Q, K, V, dO, cfg: Profile, causal: bool = True):
    """naive_gqa_backward (dense.py:173-221): per head h (KV head h // G),
    P = softmax(QK^T scale, causal), dV += P^T dO, dP = dO V^T,
    delta = rowsum(dP * P), dS = P (dP - delta), dQ = dS K scale,
    dK += dS^T Q scale; float64.  Returns (dQ, dK, dV)."""
    n = Q.shape[0]
    G = cfg.G
    scale = 1.0 / np.sqrt(cfg.d_h)
    Q64, K64, V64, dO64 = (x.astype(np.float64) for x in (Q, K, V, dO))
    fut = np.triu(np.ones((n, n), dtype=bool), k=1) if causal else None
    dQ = np.zeros((n, cfg.h_q, cfg.d_h))
    dK = np.zeros((n, cfg.h_kv, cfg.d_h))
    dV = np.zeros((n, cfg.h_kv, cfg.d_h))
    for h in range(cfg.h_q):
        kv = h // G
        S = (Q64[:, h] @ K64[:, kv].T) * scale
        if causal:
            S[fut] = -np.inf
        P = np.exp(S - S.max(axis=1)[:, None])
        P /= P.sum(axis=1)[:, None]
        dV[:, kv] += P.T @ dO64[:, h]
        dP = dO64[:, h] @ V64[:, kv].T
        delta = (dP * P).sum(axis=1)
        dS = P * (dP - delta[:, None])
        dQ[:, h] = (dS @ K64[:, kv]) * scale
        dK[:, kv] += (dS.T @ Q64[:, h]) * scale
    return dQ, dK, dV


def dense_attention(Q, K, V, cfg: Profile, rows=None, causal: bool = True, out_dtype=None):
    """Causal GQA softmax attention, float64 (dense.py:64-109; the tiled
    form dense.py:112-170 computes the same values)."""
    n = Q.shape[0]
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    G = cfg.G
    scale = 1.0 / np.sqrt(cfg.d_h)
    K64 = K.astype(np.float64)
    V64 = V.astype(np.float64)
    O = np.empty((rows.size, cfg.h_q, cfg.d_h))
    L = np.empty((rows.size, cfg.h_q))
    for ri, i in enumerate(rows):
        hi = int(i) + 1 if causal else n
        for g in range(cfg.h_kv):
            q = Q[i, g * G:(g + 1) * G].astype(np.float64)
            S = (q @ K64[:hi, g].T) * scale
            mx = S.max(axis=1)
            z = np.exp(S - mx[:, None])
            ell = z.sum(axis=1)
            O[ri, g * G:(g + 1) * G] = (z / ell[:, None]) @ V64[:hi, g]
            L[ri, g * G:(g + 1) * G] = mx + np.log(ell)
    if out_dtype is not None:
        O = O.astype(out_dtype)
    return O, L


def attend(Q, K, V, cfg: Profile, threshold=None, forced_mode=None, mode="approx", rows=None):
    """switch.attend restated (switch.py:42-82): n <= threshold -> dense
    (default threshold (N_init+N_local+k_top)*B, switch.py:37-39)."""
    n = Q.shape[0]
    thr = threshold if threshold is not None else (cfg.N_init + cfg.N_local + cfg.k_top) * cfg.B
    which = forced_mode or ("dense" if n <= thr else "sparse")
    if which == "dense":
        return dense_attention(Q, K, V, cfg, rows=rows), which
    top, _, _ = select(Q, K, cfg, mode=mode)
    return sparse_attention(Q, K, V, top, cfg, rows=rows), which


# --------------------------------------------------------------------------- decode

def decode_row(q_row, K, V, t: int, cfg: Profile):
    """Decode semantics = row t of select_blocks(approx) + sparse_forward on
    the first t+1 tokens (no reference symbol).
    q_row [h_q, d]; K, V [>= t+1, h_kv, d].  Returns (O [h_q, d], lse [h_q],
    topk [h_kv, k_top])."""
    n = t + 1

    class _OneRow:   # Q of n rows of which only row t is ever read
        shape = (n, cfg.h_q, cfg.d_h)

        def __getitem__(self, idx):
            if isinstance(idx, tuple):
                assert int(idx[0]) == t
                return q_row[idx[1:]]
            r = np.asarray(idx)
            assert np.all(r == t)
            return np.broadcast_to(q_row, r.shape + q_row.shape)
    Q = _OneRow()
    Kn, Vn = K[:n], V[:n]
    top, _, _ = select(Q, Kn, cfg, mode="approx", rows=np.array([t]))
    full = np.full((cfg.h_kv, n, cfg.k_top), -1, dtype=np.int64)
    full[:, t] = top[:, 0]
    O, L = sparse_attention(Q, Kn, Vn, full, cfg, rows=np.array([t]))
    return O[0], L[0], top[:, 0]


# --------------------------------------------------------------------------- counts

def sparse_visible_tokens(i: int, cfg: Profile) -> int:
    """bench.py:96-100."""
    b = i // cfg.B
    picked = min(b + 1, cfg.N_init + cfg.N_local + cfg.k_top)
    return (picked - 1) * cfg.B + (i - b * cfg.B) + 1
