"""Pin the CPU oracle (oracle/swattn_oracle.py) against golden vectors minted
from the unmodified reference (oracle/make_golden.py)."""

import glob
import os

import ml_dtypes
import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from oracle import swattn_oracle as O

NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
FAST = [n for n in NAMES if not n.startswith("paper_n16384") and not n.startswith("paper_n10000")]


def _cfg(rec):
    c = [int(x) for x in rec["cfg"]]
    return O.Profile(h_q=c[0], h_kv=c[1], d_h=c[2], B=c[3], l_C1=c[4], s_C1=c[5], l_C2=c[6],
                     s_C2=c[7], l=c[8], s=c[9], N_init=c[10], N_local=c[11], k_top=c[12], w=c[13])


def _inputs(rec):
    cfg = _cfg(rec)
    Q, K, V = O.draw_qkv(int(rec["n"]), cfg.h_q, cfg.h_kv, cfg.d_h, int(rec["seed"]))
    assert O.digest(Q, K, V) == str(rec["digest"]), "input generator drifted from make_qkv"
    return cfg, Q, K, V


@pytest.mark.parametrize("name", NAMES)
def test_inputs_and_pooled_keys(name):
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    c1 = O.pool(K, cfg.l_C1, cfg.s_C1)
    c2 = O.pool(K, cfg.l_C2, cfg.s_C2)
    assert O.digest(c1) == str(rec["c1_digest"])
    assert O.digest(c2) == str(rec["c2_digest"])
    if "c1_bits" in rec:
        assert np.array_equal(c1.view(np.uint16), rec["c1_bits"])
        assert np.array_equal(O.pool_exact_windows(K, cfg.l_C1, cfg.s_C1).view(np.uint16),
                              rec["c1_bits"])


@pytest.mark.parametrize("name", FAST)
def test_selection_matches_reference(name):
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    top, counts, _ = O.select(Q, K, cfg, "approx")
    k = rec["topk"].shape[2]
    assert np.array_equal(top[:, :, :k], rec["topk"].astype(np.int64))
    assert np.array_equal(counts, rec["counts"].astype(np.int64))
    if "topk_exact" in rec:
        tope, _, _ = O.select(Q, K, cfg, "exact")
        assert np.array_equal(tope[:, :, :k], rec["topk_exact"].astype(np.int64))


@pytest.mark.parametrize("name", [n for n in FAST if "score" in "".join(load_golden(n).keys())])
def test_scores_match_reference(name):
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    rows = rec["score_rows"]
    S, _ = O.shared_scores(Q, K, cfg, "approx", rows=rows)
    np.testing.assert_allclose(S, rec["shared_approx"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(O.block_scores(S, cfg.l, cfg.s), rec["cmp_approx"], rtol=1e-12,
                               atol=1e-15)
    if "shared_exact" in rec:
        Se, _ = O.shared_scores(Q, K, cfg, "exact")
        np.testing.assert_allclose(Se, rec["shared_exact"], rtol=1e-12, atol=1e-15)


def _bf16_close(got_f64, want_bits):
    want = want_bits.view(ml_dtypes.bfloat16).astype(np.float64)
    got = got_f64.astype(ml_dtypes.bfloat16).astype(np.float64)
    # identical up to float64 summation-order ties at a bf16 rounding boundary
    ulp = np.abs(want) * 2.0 ** -7 + 1e-30
    assert np.all(np.abs(got - want) <= ulp), float(np.max(np.abs(got - want)))
    assert np.mean(got != want) < 1e-3


@pytest.mark.parametrize("name", FAST)
def test_attention_matches_reference(name):
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    if "sparse_rows" in rec:
        rows = rec["sparse_rows"]
        top, _, _ = O.select(Q, K, cfg, "approx")
        if str(rec["sparse_mode"]) == "sparse":
            Osp, L = O.sparse_attention(Q, K, V, top, cfg, rows=rows)
        else:
            Osp, L = O.dense_attention(Q, K, V, cfg, rows=rows)
        _bf16_close(Osp, rec["sparse_out_bits"])
        np.testing.assert_allclose(L, rec["sparse_lse"], rtol=0, atol=1e-9)
    if "dense_rows" in rec:
        rows = rec["dense_rows"]
        Od, L = O.dense_attention(Q, K, V, cfg, rows=rows)
        _bf16_close(Od, rec["dense_out_bits"])
        np.testing.assert_allclose(L, rec["dense_lse"], rtol=0, atol=1e-9)


def test_spec_known_answers():
    # n=80, pool 32/16 -> m = 4
    assert O.n_pooled(80, 32, 16) == 4
    # max-pool [0,0,1,0,0,0,0,0], l=5, s=4 -> [1, 0]
    S = np.array([[[0, 0, 1, 0, 0, 0, 0, 0]]], dtype=np.float64)
    assert O.block_scores(S, 5, 4).ravel().tolist() == [1.0, 0.0]
    # SPEC.md:312-314 / :272-274: |I(i)| = 96 blocks at 32K, 6144 visible tokens
    cfg = O.PAPER
    assert (cfg.N_init + cfg.N_local + cfg.k_top) * cfg.B == 6144
    assert O.sparse_visible_tokens(32767, cfg) == 6144


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith("bwd_") and "dense" not in n])
def test_backward_matches_reference(name):
    """sparse_backward (sparse.py:130-185) with dO = make_qkv(seed + 1000).Q:
    dQ on the stored rows; dK / dV on the stored key rows when the oracle can
    afford every query row (small n)."""
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    n = int(rec["n"])
    dO, _, _ = O.draw_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, int(rec["seed"]) + 1000)
    top = rec["topk"].astype(np.int64)
    top = np.concatenate([top, np.full(top.shape[:2] + (cfg.k_top - top.shape[2],), -1)], 2) \
        if top.shape[2] < cfg.k_top else top
    rows = rec["bwd_rows"]
    full = n <= 512
    dQ, dK, dV = O.sparse_backward(Q, K, V, top, dO, cfg, rows=None if full else rows)
    _bf16_close(dQ[rows] if full else dQ, rec["bwd_dQ_bits"])
    if full:
        kr = rec["bwd_key_rows"]
        _bf16_close(dK[kr], rec["bwd_dK_bits"])
        _bf16_close(dV[kr], rec["bwd_dV_bits"])


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith("bwd_dense")])
def test_dense_backward_matches_reference(name):
    """naive_gqa_backward (dense.py:173-221), dO = make_qkv(seed + 1000).Q."""
    rec = load_golden(name)
    cfg, Q, K, V = _inputs(rec)
    n = int(rec["n"])
    dO, _, _ = O.draw_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, int(rec["seed"]) + 1000)
    dQ, dK, dV = O.dense_backward(Q, K, V, dO, cfg)
    _bf16_close(dQ, rec["dbwd_dQ_bits"])
    _bf16_close(dK, rec["dbwd_dK_bits"])
    _bf16_close(dV, rec["dbwd_dV_bits"])


@pytest.mark.parametrize("name", ["paper_n8192_s0", "paper_n10000_s1"])
def test_torch_f64_restatement_pinned(name):
    """oracle/torch_f64.py (the full-size parity checker of the GPU tests)
    reproduces the reference's own selection on every row of the goldens."""
    import torch
    from oracle import torch_f64
    rec = load_golden(name)
    c = [int(x) for x in rec["cfg"]]
    prof = O.Profile(h_q=c[0], h_kv=c[1], d_h=c[2], B=c[3], l_C1=c[4], s_C1=c[5], l_C2=c[6],
                     s_C2=c[7], l=c[8], s=c[9], N_init=c[10], N_local=c[11], k_top=c[12], w=c[13])
    Q, K, V = O.draw_qkv(int(rec["n"]), prof.h_q, prof.h_kv, prof.d_h, int(rec["seed"]))

    def t(x):
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16)
    top = torch_f64.select_f64(t(Q), t(K), prof, rows_per_chunk=512).numpy()
    assert np.array_equal(top, rec["topk"].astype(np.int64))
    c1 = torch_f64.pool_bf16(t(K), prof.l_C1, prof.s_C1)
    assert np.array_equal(c1.view(torch.int16).numpy().view(np.uint16),
                          O.pool(K, prof.l_C1, prof.s_C1).view(np.uint16))
