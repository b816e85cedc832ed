"""Sparse backward (sparse.py:130-185) on the GPU vs the reference's own
gradients (golden, bwd_paper_n7000_s8) and the float64 oracle.

Bars (bf16 storage, bf16 MMA inputs for P / dS, fp32 accumulation), relative
to the largest |gradient| of the reference tensor: max-abs <= 2e-2, mean-abs
<= 2e-3."""

import ml_dtypes
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import swattn_oracle as O
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.selection import select_blocks
from paper_2509_24663_b200.sparse import sparse_backward

pytestmark = pytest.mark.gpu
REL_MAX, REL_MEAN = 2e-2, 2e-3


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _close(got, want, what):
    scale = max(np.abs(want).max(), 1e-30)
    err = np.abs(got - want)
    print(f"{what}: max {err.max() / scale:.2e} mean {err.mean() / scale:.2e} (x |ref|max {scale:.3g})")
    assert err.max() <= REL_MAX * scale, (what, err.max() / scale)
    assert err.mean() <= REL_MEAN * scale, (what, err.mean() / scale)


def _inputs(n, seed):
    Q, K, V = O.draw_qkv(n, 32, 2, 128, seed)
    dO, _, _ = O.draw_qkv(n, 32, 2, 128, seed + 1000)
    return Q, K, V, dO


def test_backward_matches_reference_golden():
    rec = load_golden("bwd_paper_n7000_s8")
    n = int(rec["n"])
    Q, K, V, dO = _inputs(n, int(rec["seed"]))
    assert O.digest(Q, K, V) == str(rec["digest"])
    cfg = AttentionConfig()
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    assert np.array_equal(sel.topk.cpu().numpy(), rec["topk"].astype(np.int32))
    dQ, dK, dV = sparse_backward(Qd, Kd, Vd, sel, _dev(dO), cfg)
    torch.cuda.synchronize()
    bf = lambda b: b.view(ml_dtypes.bfloat16).astype(np.float64)
    rows, krows = rec["bwd_rows"], rec["bwd_key_rows"]
    _close(_f64(dQ)[rows], bf(rec["bwd_dQ_bits"]), "dQ")
    _close(_f64(dK)[krows], bf(rec["bwd_dK_bits"]), "dK")
    _close(_f64(dV)[krows], bf(rec["bwd_dV_bits"]), "dV")


def test_backward_matches_oracle_and_is_deterministic():
    n = 1000
    Q, K, V, dO = _inputs(n, 21)
    cfg = AttentionConfig()
    Qd, Kd, Vd, dOd = _dev(Q), _dev(K), _dev(V), _dev(dO)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    top = sel.topk.cpu().numpy().astype(np.int64)
    dQ, dK, dV = sparse_backward(Qd, Kd, Vd, sel, dOd, cfg)
    wq, wk, wv = O.sparse_backward(Q, K, V, top, dO, O.PAPER)
    _close(_f64(dQ), wq, "dQ")
    _close(_f64(dK), wk, "dK")
    _close(_f64(dV), wv, "dV")
    again = sparse_backward(Qd, Kd, Vd, sel, dOd, cfg)
    for a, b in zip((dQ, dK, dV), again):
        assert torch.equal(a, b)


def test_backward_errors():
    cfg = AttentionConfig()
    Q, K, V, dO = _inputs(128, 3)
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    with pytest.raises(ValueError):
        sparse_backward(Qd, Kd, Vd, sel, _dev(dO)[:64], cfg)


@pytest.mark.parametrize("causal", [True, False])
def test_dense_backward(causal):
    """naive_gqa_backward (dense.py:173-221) vs the reference's own gradients
    (golden, causal) and the float64 oracle (non-causal), deterministic."""
    from paper_2509_24663_b200.dense import naive_gqa_backward
    rec = load_golden("bwd_dense_paper_n200_s4")
    n = int(rec["n"])
    Q, K, V, dO = _inputs(n, int(rec["seed"]))
    assert O.digest(Q, K, V) == str(rec["digest"])
    cfg = AttentionConfig()
    Qd, Kd, Vd, dOd = _dev(Q), _dev(K), _dev(V), _dev(dO)
    dQ, dK, dV = naive_gqa_backward(Qd, Kd, Vd, dOd, cfg, causal=causal)
    if causal:
        bf = lambda b: b.view(ml_dtypes.bfloat16).astype(np.float64)
        want = (bf(rec["dbwd_dQ_bits"]), bf(rec["dbwd_dK_bits"]), bf(rec["dbwd_dV_bits"]))
    else:
        want = O.dense_backward(Q, K, V, dO, O.PAPER, causal=False)
    for got, w, nm in zip((dQ, dK, dV), want, ("dQ", "dK", "dV")):
        _close(_f64(got), w, nm)
    again = naive_gqa_backward(Qd, Kd, Vd, dOd, cfg, causal=causal)
    for a, b in zip((dQ, dK, dV), again):
        assert torch.equal(a, b)
