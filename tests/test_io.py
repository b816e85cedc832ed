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
    return rec, BlockSelection(64, int(rec["n"]), torch.from_numpy(full), torch.from_numpy(cnt), 1, 32)


def test_selection_bytes_match_reference(tmp_path):
    rec, sel = _golden_selection()
    p = tmp_path / "s.bin"
    save_selection(sel, p)
    assert p.read_bytes() == rec["selection_file"].tobytes()


def test_selection_load_reference_file(tmp_path):
    rec, sel = _golden_selection()
    p = tmp_path / "s.bin"
    p.write_bytes(rec["selection_file"].tobytes())
    got = load_selection(p, device="cpu")
    assert got.n == sel.n and got.num_groups == 2 and got.block_size == 64
    k = got.topk.shape[2]
    assert torch.equal(got.topk, sel.topk[:, :, :k]) and torch.equal(got.topk_cnt, sel.topk_cnt)
    blob = p.read_bytes()
    for bad in (blob[:-4], blob + b"\0\0\0\0", b"SWATTNS1" + b"\x00" + blob[9:]):
        p.write_bytes(bad)
        with pytest.raises(TensorFormatError):
            load_selection(p, device="cpu")
