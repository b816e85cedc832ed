"""File formats (CPU): .swt tensors (core.py:258-311) and selection fixtures
(selection.py:386-430) -- byte-identical to the reference's own writers
(golden paper_n300_s5 carries the files the reference wrote) and the same
TensorFormatError cases."""

import os

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2509_24663_b200.core import TensorFormatError, load_tensor, save_tensor
from paper_2509_24663_b200.selection import BlockSelection, load_selection, save_selection


def test_tensor_bytes_match_reference(tmp_path):
    rec = load_golden("paper_n300_s5")
    p = tmp_path / "t.swt"
    save_tensor(np.asarray(rec["sparse_lse"], dtype=np.float64), p)
    assert p.read_bytes() == rec["tensor_file"].tobytes()
    back = load_tensor(p)
    assert np.array_equal(back, rec["sparse_lse"]) and back.dtype == np.float64


@pytest.mark.parametrize("arr", [np.float32(3.5), np.arange(6, dtype=np.float32).reshape(2, 3),
                                 np.zeros((0, 4)), np.random.default_rng(0).random((3, 1, 5))])
def test_tensor_round_trip(tmp_path, arr):
    p = tmp_path / "x.swt"
    save_tensor(np.asarray(arr), p)
    back = load_tensor(p)
    # like the reference (np.ascontiguousarray, core.py:311) a rank-0 tensor loads as shape (1,)
    want_shape = np.asarray(arr).shape or (1,)
    assert back.shape == want_shape and np.array_equal(back.reshape(np.shape(arr)), arr)
    save_tensor(torch.as_tensor(np.asarray(arr)), p)
    assert np.array_equal(load_tensor(p).reshape(np.shape(arr)), arr)


def test_tensor_errors(tmp_path):
    p = tmp_path / "x.swt"
    with pytest.raises(TensorFormatError):
        save_tensor(np.zeros(3, dtype=np.int32), p)
    save_tensor(np.zeros(4, dtype=np.float32), p)
    blob = p.read_bytes()
    for bad, msg in ((b"XXXXXXXX" + blob[8:], "bad magic"), (blob[:-1], "truncated"),
                     (blob + b"\0", "oversized"), (blob[:20] + b"\x07" + blob[21:], "tag")):
        p.write_bytes(bad)
        with pytest.raises(TensorFormatError, match=msg):
            load_tensor(p)


def _golden_selection():
    rec = load_golden("paper_n300_s5")
    top = rec["topk"].astype(np.int32)
    k = 63
    full = np.full(top.shape[:2] + (k,), -1, dtype=np.int32)
    full[:, :, :top.shape[2]] = top
    cnt = (full >= 0).sum(axis=2).astype(np.int32)
    return rec, BlockSelection.from_topk(64, int(rec["n"]), torch.from_numpy(full),
                                         torch.from_numpy(cnt), 1, 32)


def test_selection_bytes_match_reference(tmp_path):
    rec, sel = _golden_selection()
    p = tmp_path / "s.bin"
    save_selection(sel, p)
    assert p.read_bytes() == rec["selection_file"].tobytes()


def test_selection_load_reference_file(tmp_path):
    rec, sel = _golden_selection()
    p = tmp_path / "s.bin"
    p.write_bytes(rec["selection_file"].tobytes())
    got = load_selection(p)   # the reference signature: stored lists exactly, counts=None
    assert got.n == sel.n and got.num_groups == 2 and got.block_size == 64
    assert got.counts is None and not got.is_topk_form
    for g in range(2):
        for i in range(sel.n):
            assert np.array_equal(got.blocks[g][i], sel.blocks[g][i])
    # the paper-config split recovers the device top-k lists bit for bit
    from paper_2509_24663_b200.core import AttentionConfig
    top, cnt = got.topk_form(AttentionConfig(), "cpu")
    assert torch.equal(top, sel.topk) and torch.equal(cnt, sel.topk_cnt)
    blob = p.read_bytes()
    for bad in (blob[:-4], blob + b"\0\0\0\0", b"SWATTNS1" + b"\x00" + blob[9:]):
        p.write_bytes(bad)
        with pytest.raises(TensorFormatError):
            load_selection(p)


def test_selection_load_keeps_stored_blocks(tmp_path):
    """A fixture written under another N_local loads row for row as stored
    (no rewrite to the default init / local structure)."""
    from paper_2509_24663_b200.core import AttentionConfig
    n, B = 300, 64
    rows = []
    for i in range(n):
        b = i // B
        lo = max(0, b - 2 + 1)
        rows.append(np.union1d(np.arange(min(1, b + 1)), np.arange(lo, b + 1)).astype(np.int64))
    sel = BlockSelection(B, n, (tuple(rows), tuple(rows)))
    p = tmp_path / "s.bin"
    save_selection(sel, p)
    got = load_selection(p)
    assert np.array_equal(got.blocks[0][299], [0, 3, 4])
    # under the paper config (N_local = 32) those rows are not init U local: general form
    assert got.topk_form(AttentionConfig(), "cpu") is None
    # under the writer's config they are, with empty top-k lists
    top, cnt = got.topk_form(AttentionConfig(N_local=2, w=64), "cpu")
    assert int(cnt.sum()) == 0 and top.shape == (2, n, 63)


def test_save_selection_k_top_zero(tmp_path):
    """a k_top = 0 top-k-form selection writes init U local rows."""
    n = 200
    top = torch.zeros((2, n, 0), dtype=torch.int32)
    cnt = torch.zeros((2, n), dtype=torch.int32)
    sel = BlockSelection.from_topk(64, n, top, cnt, 1, 32)
    p = tmp_path / "s.bin"
    save_selection(sel, p)
    got = load_selection(p)
    assert np.array_equal(got.blocks[1][199], [0, 1, 2, 3])


def test_all_blocks_selection_is_general():
    """bench.py:207-210's every-causal-block selection: once a row has more
    than k_top blocks between the init block and its local window it is not
    the init U local U top-k shape, so it takes the general list form."""
    from paper_2509_24663_b200.core import AttentionConfig
    n, B = 8192, 64
    nb = -(-n // B)
    rows = tuple(np.arange(min(i // B, nb - 1) + 1, dtype=np.int64) for i in range(n))
    sel = BlockSelection(B, n, (rows, rows))
    cfg = AttentionConfig()
    # 128 blocks in the last rows: 95 non-local blocks > k_top = 63 -> general list form
    assert sel.topk_form(cfg, "cpu") is None
    blocks, ld, cnt = sel.list_form("cpu")
    assert ld == 128 and int(cnt[0, n - 1]) == 128 and int(blocks[0, n - 1, 127]) == 127
    assert sel.first_empty_row() is None
    v = sel.key_visits()
    assert v[0, 0] == 1 and v[1, n - 1] == n


def test_first_empty_row_order():
    n = 100
    rows0 = tuple(np.array([1], dtype=np.int64) if i in (10, 70) else np.array([0], dtype=np.int64)
                  for i in range(n))
    sel = BlockSelection(64, n, (rows0, rows0))
    # block 1 starts at token 64: row 10 sees nothing, row 70 sees 64..70
    assert sel.first_empty_row() == (0, 10)
