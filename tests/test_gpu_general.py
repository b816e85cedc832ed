"""GPU: the general drop-in surface added in round 2 --

* sparse_forward over ANY BlockSelection (the reference constructor,
  selection.py:51-66): every-causal-block selections (the reference's
  _all_blocks_selection, bench.py:207-210) against dense attention, random
  hand-made selections against a float64 restatement of sparse.py:43-98, a
  reference-written fixture through load_selection, and the empty-row error
  (sparse.py:75-76);
* batch x KV-group sharding through the C ABI (swattn_attend_groups /
  swattn_attend_rows_groups): the per-group calls reassemble the full attend
  bit for bit;
* decode with an empty batch slot, scratch workspaces per stream.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import swattn_oracle as O
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.dense import tiled_gqa_forward
from paper_2509_24663_b200.selection import BlockSelection, load_selection, select_blocks
from paper_2509_24663_b200.sparse import sparse_forward
from paper_2509_24663_b200.switch import SwitchPolicy, attend

pytestmark = pytest.mark.gpu

O_MAX_ABS, O_MEAN_ABS, LSE_ABS = 2e-2, 2e-3, 1e-3


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


def _f32(t):
    return t.float().cpu().numpy()


def _ref_rows(Q, K, V, sel, rows, B=64):
    """float64 softmax over each row's visible keys of an arbitrary selection
    (sparse.py:70-91 with visible_spans, selection.py:73-87)."""
    n, h_q, d = Q.shape
    G = h_q // K.shape[1]
    out = np.empty((len(rows), h_q, d))
    lse = np.empty((len(rows), h_q))
    for r, i in enumerate(rows):
        for g in range(K.shape[1]):
            keys = np.concatenate([np.arange(s, e) for s, e in sel.visible_spans(g, i)])
            q = Q[i, g * G:(g + 1) * G].astype(np.float64)
            S = q @ K[keys, g].astype(np.float64).T / np.sqrt(d)
            mx = S.max(1)
            z = np.exp(S - mx[:, None])
            out[r, g * G:(g + 1) * G] = (z / z.sum(1)[:, None]) @ V[keys, g].astype(np.float64)
            lse[r, g * G:(g + 1) * G] = mx + np.log(z.sum(1))
    return out, lse


def _check(o_dev, l_dev, rows, ref_o, ref_l):
    o = _f32(o_dev)[rows]
    err = np.abs(o - ref_o)
    assert err.max() <= O_MAX_ABS and err.mean() <= O_MEAN_ABS, (err.max(), err.mean())
    assert np.abs(_f32(l_dev)[rows] - ref_l).max() <= LSE_ABS


@pytest.mark.parametrize("n", [4096, 8192])
def test_all_blocks_selection_equals_dense(n):
    """bench.py:207-210: selecting every causal block is dense causal attention.
    At 4K every row is still init U local U (<= 63 top) -> part A + part B; at
    8K rows carry up to 95 middle blocks -> the general list kernel."""
    cfg = AttentionConfig()
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 11)
    nb = -(-n // 64)
    rows = tuple(np.arange(min(i // 64, nb - 1) + 1, dtype=np.int64) for i in range(n))
    sel = BlockSelection(64, n, (rows, rows))
    assert (sel.topk_form(cfg) is None) == (n > 4096)
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    res = sparse_forward(Qd, Kd, Vd, sel, cfg)
    dense = tiled_gqa_forward(Qd, Kd, Vd, cfg)
    torch.cuda.synchronize()
    d = np.abs(_f32(res.output) - _f32(dense.output))
    assert d.max() <= 2e-2 and d.mean() <= 1e-3
    assert np.abs(_f32(res.lse) - _f32(dense.lse)).max() <= 1e-3
    pick = np.array([0, 1, 63, 64, 1000, n // 2 + 5, n - 1])
    ro, rl = O.dense_attention(Q, K, V, O.PAPER, rows=pick)
    _check(res.output, res.lse, pick, ro, rl)


def test_random_general_selection_vs_float64():
    """Arbitrary sorted block sets (gaps, far blocks, blocks past the diagonal
    that clip to nothing, a ragged last block), n not a multiple of B."""
    cfg = AttentionConfig()
    n = 1500
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 12)
    rng = np.random.default_rng(3)
    nb = -(-n // 64)
    groups = []
    for g in range(2):
        rows = []
        for i in range(n):
            b = i // 64
            k = rng.integers(1, 8)
            cand = rng.choice(nb, size=min(k, nb), replace=False)
            cand = np.union1d(cand, [b]).astype(np.int64)   # keep the row non-empty
            rows.append(cand)
        groups.append(tuple(rows))
    sel = BlockSelection(64, n, tuple(groups))
    res = sparse_forward(_dev(Q), _dev(K), _dev(V), sel, cfg)
    torch.cuda.synchronize()
    pick = np.sort(rng.choice(n, 40, replace=False))
    ro, rl = _ref_rows(Q, K, V, sel, pick)
    _check(res.output, res.lse, pick, ro, rl)
    # host (numpy) inputs go through the same path and return host arrays
    res_h = sparse_forward(Q, K, V, sel, cfg)
    assert np.array_equal(np.asarray(res_h.output).view(np.uint16),
                          res.output.view(torch.int16).cpu().numpy().view(np.uint16))


def test_reference_fixture_through_load_selection(tmp_path):
    """A selection file written by the reference (golden paper_n300_s5) loads
    with the reference signature and runs sparse_forward to the golden output."""
    rec = load_golden("paper_n300_s5")
    cfg = AttentionConfig()
    Q, K, V = O.draw_qkv(int(rec["n"]), 32, 2, 128, int(rec["seed"]))
    p = tmp_path / "sel.bin"
    p.write_bytes(rec["selection_file"].tobytes())
    sel = load_selection(p)
    res = sparse_forward(_dev(Q), _dev(K), _dev(V), sel, cfg)
    torch.cuda.synchronize()
    rows = rec["sparse_rows"]
    want = rec["sparse_out_bits"].view(np.uint16).astype(np.uint32) << 16
    want = want.view(np.float32)
    _check(res.output, res.lse, rows, want, rec["sparse_lse"])
    # the same rows through the general kernel (a selection forced off the top-k form)
    groups = tuple(tuple(np.asarray(r) for r in grp) for grp in sel.blocks)
    sel_g = BlockSelection(64, int(rec["n"]), groups)
    blocks, ld, cnt = sel_g.list_form()
    O_ = torch.empty((int(rec["n"]), 32, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((int(rec["n"]), 32), dtype=torch.float32, device="cuda")
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    L = _lib.lib()
    _lib.check(L.swattn_sparse_fwd_lists(_lib.c_config(cfg), Qd.data_ptr(), Kd.data_ptr(),
                                         Vd.data_ptr(), int(rec["n"]), blocks.data_ptr(), ld,
                                         cnt.data_ptr(), O_.data_ptr(), lse.data_ptr(),
                                         _lib.stream_handle()), "lists")
    torch.cuda.synchronize()
    _check(O_, lse, rows, want, rec["sparse_lse"])


def test_empty_visible_set_raises():
    cfg = AttentionConfig()
    n = 200
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 13)
    rows = [np.array([0], dtype=np.int64)] * n
    rows[70] = np.array([2], dtype=np.int64)          # block 2 starts at 128 > 70
    sel = BlockSelection(64, n, (tuple(rows), tuple(rows)))
    with pytest.raises(RuntimeError, match="query 70 in group 0 has an empty visible set"):
        sparse_forward(_dev(Q), _dev(K), _dev(V), sel, cfg)


@pytest.mark.parametrize("n", [5000, 20000])
def test_group_sharded_attend_equals_full(n):
    """KV-group sharding: attend of group 0 and of group 1 (separate C-ABI
    calls, as two ranks would make them) fill O / lse bit-identically to one
    full attend; the same with row ranges split across ranks (group x CP)."""
    from paper_2509_24663_b200.parallel import group_cp_attend
    from paper_2509_24663_b200.selection import Workspace
    cfg = AttentionConfig()
    Qd, Kd, Vd = (_dev(x) for x in O.draw_qkv(n, 32, 2, 128, 14))
    full, _ = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    L = _lib.lib()
    c = _lib.c_config(cfg)
    O_ = torch.full((n, 32, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    lse = torch.full((n, 32), float("nan"), dtype=torch.float32, device="cuda")
    ws = Workspace.get(L.swattn_workspace_bytes(c, n), Qd.device)
    taken = _lib.ctypes.c_int32(0)
    for g in range(2):
        _lib.check(L.swattn_attend_groups(c, Qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n, g,
                                          g + 1, -1, 2, 2, O_.data_ptr(), lse.data_ptr(),
                                          _lib.ctypes.byref(taken), ws.data_ptr(), ws.numel(),
                                          _lib.stream_handle()), "attend_groups")
        if g == 0:   # group 1's heads untouched so far
            torch.cuda.synchronize()
            assert torch.isnan(lse[:, 16:]).all() and not torch.isnan(lse[:, :16]).any()
    torch.cuda.synchronize()
    assert torch.equal(O_, full.output) and torch.equal(lse, full.lse)
    for world in (2, 4, 8):
        O2 = torch.full_like(O_, float("nan"))
        l2 = torch.full_like(lse, float("nan"))
        for rank in range(world):
            group_cp_attend(Qd, Kd, Vd, cfg, world, rank, O=O2, lse=l2)
        torch.cuda.synchronize()
        assert torch.equal(O2, full.output) and torch.equal(l2, full.lse), world


def test_group_range_validation():
    cfg = AttentionConfig()
    L = _lib.lib()
    rc = L.swattn_attend_groups(_lib.c_config(cfg), 1, 1, 1, 100, 1, 1, -1, 0, 2, 1, 1, None,
                                None, 0, None)
    assert rc == _lib.SWATTN_EINVAL and "group range" in _lib.last_error()


def test_decode_empty_slot():
    """A batch slot with no cached token yields O = 0, lse = -inf and reads no
    page; the other slots are unaffected."""
    from paper_2509_24663_b200.decode import PagedKVCache, decode_step
    cfg = AttentionConfig()
    lens = [3000, 0, 5000]
    cache = PagedKVCache(cfg, batch=3, max_pages=-(-max(lens) // 64) + 1, seed=9)
    data = {}
    for b, Ln in enumerate(lens):
        if Ln:
            Q, K, V = O.draw_qkv(Ln, 32, 2, 128, 50 + b)
            data[b] = (Q, K, V)
            cache.append(b, _dev(K), _dev(V))
    q = torch.stack([_dev(data[b][0][lens[b] - 1]) if lens[b] else
                     torch.zeros((32, 128), dtype=torch.bfloat16, device="cuda") for b in range(3)])
    res = decode_step(cache, q)
    torch.cuda.synchronize()
    assert torch.all(res.output[1] == 0) and torch.all(torch.isneginf(res.lse[1]))
    for b in (0, 2):
        Q, K, V = data[b]
        o, l, _ = O.decode_row(Q[lens[b] - 1], K, V, lens[b] - 1, O.PAPER)
        err = np.abs(_f32(res.output[b]) - o)
        assert err.max() <= O_MAX_ABS and err.mean() <= O_MEAN_ABS


def test_workspace_per_stream():
    """Two attends in flight on two streams use separate scratch."""
    cfg = AttentionConfig()
    n = 9000
    a = [_dev(x) for x in O.draw_qkv(n, 32, 2, 128, 21)]
    b = [_dev(x) for x in O.draw_qkv(n, 32, 2, 128, 22)]
    ra, _ = attend(*a, cfg)
    rb, _ = attend(*b, cfg)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            x, _ = attend(*a, cfg)
        with torch.cuda.stream(s2):
            y, _ = attend(*b, cfg)
        outs.append((x, y))
    torch.cuda.synchronize()
    for x, y in outs:
        assert torch.equal(x.output, ra.output) and torch.equal(y.output, rb.output)


def test_select_blocks_returns_topk_form():
    cfg = AttentionConfig()
    n = 9000
    Qd, Kd, _ = (_dev(x) for x in O.draw_qkv(n, 32, 2, 128, 23))
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    assert sel.is_topk_form and sel.topk.shape == (2, n, 63)
    top, cnt = sel.topk_form(cfg, Qd.device)
    assert top.data_ptr() == sel.topk.data_ptr() or torch.equal(top, sel.topk)
