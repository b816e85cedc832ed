"""GPU parity: every hot-path kernel vs the reference-pinned golden vectors and
the CPU oracle, through the C ABI (via the drop-in Python API).

Bars (north star / SURVEY §8c):
  * pooled keys, block indices: bit-exact (ties broken as the reference);
  * S^cmp: relative error <= kScoreRelErr (1e-6) vs float64;
  * attention O: max-abs <= 2e-2 and mean-abs <= 2e-3 vs the float64
    reference values, lse abs <= 1e-3 (bf16 storage, fp32 softmax).
"""

import ml_dtypes
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import swattn_oracle as O
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.compression import mean_pool_keys
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.dense import tiled_gqa_forward
from paper_2509_24663_b200.selection import select_blocks
from paper_2509_24663_b200.sparse import sparse_forward
from paper_2509_24663_b200.switch import SwitchPolicy, attend

pytestmark = pytest.mark.gpu

O_MAX_ABS, O_MEAN_ABS, LSE_ABS = 2e-2, 2e-3, 1e-3
SCORE_REL = 1e-6  # = kScoreRelErr (csrc/common.cuh)

PAPER_GOLDEN = ["paper_n300_s5", "paper_n4096_s0", "paper_n8192_s0", "paper_n10000_s1",
                "paper_n16384_s2"]
SMALL_GOLDEN = ["small_n64_s0", "small_n257_s0", "small_n1000_s3"]


def _cfgs(rec):
    c = [int(x) for x in rec["cfg"]]
    prof = O.Profile(h_q=c[0], h_kv=c[1], d_h=c[2], B=c[3], l_C1=c[4], s_C1=c[5], l_C2=c[6],
                     s_C2=c[7], l=c[8], s=c[9], N_init=c[10], N_local=c[11], k_top=c[12],
                     w=c[13])
    cfg = AttentionConfig(h_q=c[0], h_kv=c[1], d_h=c[2], B=c[3], l_C1=c[4], s_C1=c[5],
                          l_C2=c[6], s_C2=c[7], l=c[8], s=c[9], N_init=c[10], N_local=c[11],
                          k_top=c[12], w=c[13])
    return prof, cfg


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


def _load(name):
    rec = load_golden(name)
    prof, cfg = _cfgs(rec)
    Q, K, V = O.draw_qkv(int(rec["n"]), prof.h_q, prof.h_kv, prof.d_h, int(rec["seed"]))
    assert O.digest(Q, K, V) == str(rec["digest"])
    return rec, prof, cfg, (Q, K, V), (_dev(Q), _dev(K), _dev(V))


def _host_bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("name", PAPER_GOLDEN + SMALL_GOLDEN)
def test_k1_pooled_keys_bit_exact(name):
    rec, prof, cfg, host, (Qd, Kd, Vd) = _load(name)
    c1 = mean_pool_keys(Kd, cfg.l_C1, cfg.s_C1)
    c2 = mean_pool_keys(Kd, cfg.l_C2, cfg.s_C2)
    torch.cuda.synchronize()
    assert O.digest(_host_bits(c1.keys)) == str(rec["c1_digest"])
    assert O.digest(_host_bits(c2.keys)) == str(rec["c2_digest"])
    # fused one-pass kernel (both profiles at once) through the raw C ABI
    L = _lib.lib()
    n = Kd.shape[0]
    m1, m2 = L.swattn_num_pooled(n, cfg.l_C1, cfg.s_C1), L.swattn_num_pooled(n, cfg.l_C2, cfg.s_C2)
    k1 = torch.empty((m1, cfg.h_kv, cfg.d_h), dtype=torch.bfloat16, device="cuda")
    k2 = torch.empty((max(m2, 1), cfg.h_kv, cfg.d_h), dtype=torch.bfloat16, device="cuda")
    _lib.check(L.swattn_compress_keys(_lib.c_config(cfg), Kd.data_ptr(), n, k1.data_ptr(),
                                      k2.data_ptr() if m2 else None, _lib.stream_handle()), "k1")
    torch.cuda.synchronize()
    assert O.digest(_host_bits(k1)) == str(rec["c1_digest"])
    if m2:
        assert O.digest(_host_bits(k2[:m2])) == str(rec["c2_digest"])


@pytest.mark.parametrize("name", PAPER_GOLDEN)
def test_selection_topk_fused_in_k2(name, monkeypatch):
    """Row f1 (opt-in SWATTN_K2_TOPK=1): the top-k selected in K2's pass-2
    epilogue from a per-token candidate set gives the reference's selection,
    including the float64 re-rank of the rows it flags."""
    rec, prof, cfg, host, (Qd, Kd, Vd) = _load(name)
    monkeypatch.setenv("SWATTN_K2_TOPK", "1")
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    torch.cuda.synchronize()
    got = sel.topk.cpu().numpy().astype(np.int64)
    want = rec["topk"].astype(np.int64)[:, :, :cfg.k_top]
    bad = np.argwhere((got != want).any(axis=2))
    assert bad.size == 0, f"{len(bad)} rows differ, first {bad[:5].tolist()}"
    assert np.array_equal(sel.counts, rec["counts"].astype(np.int64))


@pytest.mark.parametrize("name", PAPER_GOLDEN + SMALL_GOLDEN)
def test_selection_bit_exact(name):
    rec, prof, cfg, host, (Qd, Kd, Vd) = _load(name)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    torch.cuda.synchronize()
    k = cfg.k_top
    got = sel.topk.cpu().numpy().astype(np.int64)
    want = rec["topk"].astype(np.int64)[:, :, :k]
    bad = np.argwhere((got != want).any(axis=2))
    assert bad.size == 0, f"{len(bad)} rows differ, first {bad[:5].tolist()}; reranked={int(sel.n_reranked)}"
    assert np.array_equal(sel.counts, rec["counts"].astype(np.int64))
    if "topk_exact" in rec:
        for mode in ("fused-exact", "exact"):
            sel_e = select_blocks(Qd, Kd, cfg, mode=mode)
            got_e = sel_e.topk.cpu().numpy().astype(np.int64)
            assert np.array_equal(got_e, rec["topk_exact"].astype(np.int64)[:, :, :k]), mode


@pytest.mark.parametrize("name", ["paper_n8192_s0", "paper_n16384_s2", "paper_n10000_s1"])
def test_k2_score_error_bound(name):
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load(name)
    L = _lib.lib()
    c = _lib.c_config(cfg)
    n = Qd.shape[0]
    c1 = mean_pool_keys(Kd, cfg.l_C1, cfg.s_C1).keys
    c2 = mean_pool_keys(Kd, cfg.l_C2, cfg.s_C2).keys
    m1 = c1.shape[0]
    n_cols = -(-m1 // cfg.s)
    ld = (n_cols + 3) // 4 * 4
    scmp = torch.full((cfg.h_kv, n, ld), float("nan"), dtype=torch.float32, device="cuda")
    _lib.check(L.swattn_block_scores(c, Qd.data_ptr(), c1.data_ptr(), c2.data_ptr(), n, 2,
                                     scmp.data_ptr(), ld, None, _lib.stream_handle()), "k2")
    torch.cuda.synchronize()
    rows = rec["score_rows"]
    want = rec["cmp_approx"]  # [R, h_kv, n_cols] float64 from the reference
    got = scmp.cpu().numpy()[:, rows, :n_cols].transpose(1, 0, 2)
    worst = 0.0
    for ri, i in enumerate(rows):
        b = int(i) // cfg.B
        hi = min(max(0, b - cfg.N_local + 1), n_cols)
        if hi <= cfg.N_init:
            continue
        w = want[ri, :, cfg.N_init:hi]
        g = got[ri, :, cfg.N_init:hi]
        worst = max(worst, float(np.max(np.abs(g - w) / np.abs(w))))
    print(f"{name}: max rel err of S^cmp = {worst:.3e}")
    assert worst <= SCORE_REL


def _tol(got_bf16_dev, want_f64, lse_dev, want_lse):
    got = got_bf16_dev.float().cpu().numpy().astype(np.float64)
    err = np.abs(got - want_f64)
    assert err.max() <= O_MAX_ABS, err.max()
    assert err.mean() <= O_MEAN_ABS, err.mean()
    lerr = np.abs(lse_dev.cpu().numpy().astype(np.float64) - want_lse)
    assert lerr.max() <= LSE_ABS, lerr.max()
    return float(err.max()), float(err.mean()), float(lerr.max())


@pytest.mark.parametrize("name", PAPER_GOLDEN)
def test_sparse_attention_tolerance(name):
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load(name)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    res = sparse_forward(Qd, Kd, Vd, sel, cfg)
    torch.cuda.synchronize()
    rows = rec["sparse_rows"]
    top = rec["topk"].astype(np.int64)
    if str(rec["sparse_mode"]) == "sparse":
        want_o, want_l = O.sparse_attention(Q, K, V, top, prof, rows=rows)
    else:
        want_o, want_l = O.dense_attention(Q, K, V, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    stats = _tol(res.output[r], want_o, res.lse[r], want_l)
    # and against the reference's own bf16 output
    ref_bf16 = rec["sparse_out_bits"].view(ml_dtypes.bfloat16).astype(np.float64)
    got = res.output[r].float().cpu().numpy()
    assert np.abs(got - ref_bf16).max() <= O_MAX_ABS
    print(name, "sparse max/mean/lse err", stats)


@pytest.mark.parametrize("name", ["paper_n300_s5", "paper_n4096_s0", "paper_n8192_s0"])
def test_dense_attention_tolerance(name):
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load(name)
    res = tiled_gqa_forward(Qd, Kd, Vd, cfg)
    torch.cuda.synchronize()
    rows = rec["dense_rows"]
    want_o, want_l = O.dense_attention(Q, K, V, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    print(name, "dense max/mean/lse err", _tol(res.output[r], want_o, res.lse[r], want_l))


def test_attend_switch_dispatch():
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load("paper_n4096_s0")
    res, mode = attend(Qd, Kd, Vd, cfg)
    assert mode == "dense"  # 4096 <= 6144 (switch.py:69)
    res_s, mode_s = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    assert mode_s == "sparse"
    res_t, mode_t = attend(Qd, Kd, Vd, cfg, SwitchPolicy(threshold_tokens=4095))
    assert mode_t == "sparse"
    torch.cuda.synchronize()
    # at 4K every causal block is selected (budget 96 >= 64 blocks): sparse == dense
    d = (res.output.float() - res_s.output.float()).abs().max().item()
    assert d <= 2e-2
    assert torch.equal(res_s.output, res_t.output)
    with pytest.raises(ValueError):
        attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="bogus"))


def test_attend_host_arrays_roundtrip():
    rec, prof, cfg, (Q, K, V), _ = _load("paper_n8192_s0")
    res, mode = attend(Q, K, V, cfg)  # numpy bf16 in -> numpy out (H2D/D2H inside)
    assert mode == "sparse"
    assert isinstance(res.output, np.ndarray) and res.output.dtype == ml_dtypes.bfloat16
    rows = rec["sparse_rows"]
    ref = rec["sparse_out_bits"].view(ml_dtypes.bfloat16).astype(np.float64)
    assert np.abs(res.output[rows].astype(np.float64) - ref).max() <= O_MAX_ABS
    assert np.abs(res.lse[rows] - rec["sparse_lse"]).max() <= LSE_ABS


def test_determinism_bitwise():
    rec, prof, cfg, _, (Qd, Kd, Vd) = _load("paper_n10000_s1")
    outs = [attend(Qd, Kd, Vd, cfg)[0] for _ in range(2)]
    torch.cuda.synchronize()
    assert torch.equal(outs[0].output, outs[1].output)
    assert torch.equal(outs[0].lse, outs[1].lse)


def test_errors_match_reference_behaviour():
    cfg = AttentionConfig()
    Qd = torch.zeros((64, 32, 128), dtype=torch.bfloat16, device="cuda")
    Kd = torch.zeros((64, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="K shape"):
        tiled_gqa_forward(Qd, Kd[:32], Kd[:32], cfg)
    with pytest.raises(ValueError, match="unknown selection mode"):
        select_blocks(Qd, Kd, cfg, mode="fast")
    with pytest.raises(ValueError, match="tile sizes"):
        select_blocks(Qd, Kd, cfg, B_q=0)


def _random_rows(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.choice(n, size=k, replace=False), [n - 1, n // 2]]))


@pytest.mark.parametrize("n,seed,route", [(32768, 11, None), (131072, 12, None), (65536, 13, "60")])
def test_full_size_properties_and_sampled_rows(n, seed, route, monkeypatch):
    """BASELINE sizes: the oracle checks sampled rows exactly (selection) and
    within tolerance (attention); size-independent properties cover the rest.
    (32K routes tiles to the FA tile by default; 64K forces it, route.cuh.)"""
    if route is not None:
        monkeypatch.setenv("SWATTN_ROUTE_PCT", route)
    prof, cfg = O.PAPER, AttentionConfig()
    Q, K, V = O.draw_qkv(n, 32, 2, 128, seed)
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    res = sparse_forward(Qd, Kd, Vd, sel, cfg)
    torch.cuda.synchronize()
    top = sel.topk.cpu().numpy()
    cnt = sel.topk_cnt.cpu().numpy()
    i = np.arange(n)
    b = i // 64
    lo = np.maximum(0, b - 31)
    ncand = np.maximum(0, np.minimum(lo, -(-O.n_pooled(n, 32, 16) // 4)) - 1)
    assert np.array_equal(cnt, np.broadcast_to(np.minimum(63, ncand), cnt.shape))
    valid = top >= 0
    assert np.array_equal(valid.sum(axis=2), cnt)
    # ascending, inside the candidate pool
    t = np.where(valid, top, np.iinfo(np.int32).max)
    assert np.all(np.diff(t, axis=2)[valid[:, :, 1:]] > 0)
    assert np.all((top >= 1)[valid]) and np.all((top < lo[None, :, None])[valid])
    # 96 random rows plus the first rows with a competitive top-k (query block
    # 96: candidates just above k) and the last query block
    rows = np.unique(np.concatenate([_random_rows(n, 96, seed), np.arange(96 * 64, 96 * 64 + 4),
                                     np.arange(n - 4, n)]))
    want_top, _, _ = O.select(Q, K, prof, "approx", rows=rows)
    assert np.array_equal(top[:, rows, :], want_top)
    full = np.full((2, n, 63), -1, dtype=np.int64)
    full[:, rows] = want_top
    want_o, want_l = O.sparse_attention(Q, K, V, full, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    print(n, "sampled-row sparse err", _tol(res.output[r], want_o, res.lse[r], want_l),
          "reranked rows", int(sel.n_reranked))


@pytest.mark.parametrize("name", ["paper_n8192_s0", "paper_n16384_s2", "paper_n10000_s1"])
def test_routed_tiles_match_part_b(name, monkeypatch):
    """Tiles routed to the tensor-core FA tile (union of the tile's top-k
    blocks, per-row block mask, merged with part A -- route.cuh) give the same
    attention as part B's per-token gathers: both within the oracle bars and
    within 4e-3 of each other, on every sampled row."""
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load(name)
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    out = {}
    for pct in ("0", "100"):
        monkeypatch.setenv("SWATTN_ROUTE_PCT", pct)
        res = sparse_forward(Qd, Kd, Vd, sel, cfg)
        torch.cuda.synchronize()
        out[pct] = (res.output.float(), res.lse)
    d = (out["0"][0] - out["100"][0]).abs()
    assert float(d.max()) <= 4e-3 and float(d.mean()) <= 1e-4, (float(d.max()), float(d.mean()))
    assert float((out["0"][1] - out["100"][1]).abs().max()) <= 1e-4
    rows = rec["sparse_rows"]
    top = rec["topk"].astype(np.int64)
    want_o, want_l = O.sparse_attention(Q, K, V, top, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    res_o, res_l = out["100"]
    print(name, "routed max/mean/lse err", _tol(res_o[r].to(torch.bfloat16), want_o, res_l[r], want_l))


def test_all_rows_dense_and_forced_sparse_n4096():
    """Every row (not a sample): at 4K all causal blocks are selected, so the
    dense kernel and the two-part sparse kernels must both equal dense attention."""
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load("paper_n4096_s0")
    dense, _ = attend(Qd, Kd, Vd, cfg)
    sparse, _ = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    torch.cuda.synchronize()
    want_o, want_l = O.dense_attention(Q, K, V, prof)
    for res in (dense, sparse):
        got = res.output.float().cpu().numpy().astype(np.float64)
        err = np.abs(got - want_o)
        bad = np.argwhere(err.max(axis=(1, 2)) > O_MAX_ABS).ravel()
        assert bad.size == 0, f"rows {bad[:10].tolist()} exceed tolerance (max {err.max():.3e})"
        assert err.mean() <= O_MEAN_ABS
        assert np.abs(res.lse.cpu().numpy() - want_l).max() <= LSE_ABS


def test_decode_paged_matches_oracle_last_row():
    """K6 decode over a shuffled paged cache == row L-1 of the reference's
    sparse path (selection bit-exact, output within tolerance)."""
    from paper_2509_24663_b200.decode import PagedKVCache, decode_step
    prof, cfg = O.PAPER, AttentionConfig()
    lens = [9000, 12345, 20000]
    data = [O.draw_qkv(L, 32, 2, 128, 40 + b) for b, L in enumerate(lens)]
    cache = PagedKVCache(cfg, batch=len(lens), max_pages=-(-max(lens) // 64) + 2, seed=5)
    for b, (Q, K, V) in enumerate(data):
        cache.append(b, _dev(K), _dev(V))
    q = torch.stack([_dev(Q[L - 1]) for (Q, K, V), L in zip(data, lens)])
    res, topk = decode_step(cache, q, return_topk=True)
    torch.cuda.synchronize()
    for b, ((Q, K, V), L) in enumerate(zip(data, lens)):
        o, l, top = O.decode_row(Q[L - 1], K, V, L - 1, prof)
        assert np.array_equal(topk[b].cpu().numpy(), top), b
        err = np.abs(res.output[b].float().cpu().numpy() - o)
        assert err.max() <= O_MAX_ABS and err.mean() <= O_MEAN_ABS, (b, err.max())
        assert np.abs(res.lse[b].cpu().numpy() - l).max() <= LSE_ABS
    # pooled-key slabs equal the one-shot K1 pooling of the whole context
    for b, ((Q, K, V), L) in enumerate(zip(data, lens)):
        c1 = O.pool(K, 32, 16)
        got = cache.kc1[b, :c1.shape[0]].contiguous().view(torch.int16).cpu().numpy()
        assert np.array_equal(got, c1.view(np.int16))


def test_decode_incremental_append_equals_bulk():
    """Appending token by token keeps the compressed keys identical to a
    bulk append (windows completing at 16/64-token boundaries)."""
    from paper_2509_24663_b200.decode import PagedKVCache
    cfg = AttentionConfig()
    Q, K, V = O.draw_qkv(700, 32, 2, 128, 77)
    a = PagedKVCache(cfg, batch=1, max_pages=12, seed=1)
    b = PagedKVCache(cfg, batch=1, max_pages=12, seed=2)
    a.append(0, _dev(K), _dev(V))
    b.append(0, _dev(K[:500]), _dev(V[:500]))
    for t in range(500, 700):
        b.append(0, _dev(K[t:t + 1]), _dev(V[t:t + 1]))
    torch.cuda.synchronize()
    assert torch.equal(a.kc1, b.kc1) and torch.equal(a.kc2, b.kc2)


@pytest.mark.gpu
def test_decode_append_tokens_equals_bulk():
    """The serving-loop append (one token per sequence per launch, seq_lens
    advanced on the device, masked sequences left alone) builds the same
    cache as bulk appends, and decode over it matches the oracle."""
    from paper_2509_24663_b200.decode import PagedKVCache, decode_step
    cfg, prof = AttentionConfig(), O.PAPER
    start, steps = [0, 60, 127, 6000], 70
    skip = {1: range(10, 20)}                      # sequence 1 idles for ten steps
    total = [s + steps - len(skip.get(b, ())) for b, s in enumerate(start)]
    data = [O.draw_qkv(L, 32, 2, 128, 90 + b) for b, L in enumerate(total)]
    mp = -(-max(total) // 64) + 1
    a = PagedKVCache(cfg, batch=4, max_pages=mp, seed=3)
    ref = PagedKVCache(cfg, batch=4, max_pages=mp, seed=4)
    for b, (Q, K, V) in enumerate(data):
        ref.append(b, _dev(K), _dev(V))
        if start[b]:
            a.append(b, _dev(K[:start[b]]), _dev(V[:start[b]]))
    pos = list(start)
    for t in range(steps):
        act = np.array([t not in skip.get(b, ()) for b in range(4)])
        Kt = torch.zeros((4, 2, 128), dtype=torch.bfloat16, device="cuda")
        Vt = torch.zeros_like(Kt)
        for b in range(4):
            if act[b]:
                Kt[b], Vt[b] = _dev(data[b][1][pos[b]]), _dev(data[b][2][pos[b]])
                pos[b] += 1
        a.append_tokens(Kt, Vt, active=None if act.all() else act)
    torch.cuda.synchronize()
    assert pos == total and a.lens_h.tolist() == total
    assert a.seq_lens.cpu().tolist() == total
    assert torch.equal(a.kc1, ref.kc1) and torch.equal(a.kc2, ref.kc2)
    q = torch.stack([_dev(Q[L - 1]) for (Q, K, V), L in zip(data, total)])
    ra, ta = decode_step(a, q, return_topk=True)
    rr, tr = decode_step(ref, q, return_topk=True)
    torch.cuda.synchronize()
    assert torch.equal(ta, tr)
    assert torch.equal(ra.output, rr.output) and torch.equal(ra.lse, rr.lse)
    for b, ((Q, K, V), L) in enumerate(zip(data, total)):
        o, l, top = O.decode_row(Q[L - 1], K, V, L - 1, prof)
        assert np.array_equal(ta[b].cpu().numpy(), top), b
        err = np.abs(ra.output[b].float().cpu().numpy() - o)
        assert err.max() <= O_MAX_ABS and err.mean() <= O_MEAN_ABS, (b, err.max())


@pytest.mark.gpu
@pytest.mark.parametrize("name,rows", [("paper_n16384_s2", 4096), ("paper_n10000_s1", 2048)])
def test_chunked_host_pipeline_equals_whole(name, rows):
    """attend_host_chunked (Q streamed in row chunks, copies overlapped with
    swattn_attend_rows) reproduces the whole-sequence call bit for bit."""
    from paper_2509_24663_b200.switch import attend_host_chunked
    rec, prof, cfg, (Q, K, V), (Qd, Kd, Vd) = _load(name)
    whole, mode = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    torch.cuda.synchronize()
    Qh, Kh, Vh = (x.cpu().pin_memory() for x in (Qd, Kd, Vd))
    O_h, lse_h = attend_host_chunked(Qh, Kh, Vh, cfg, "approx", chunk_rows=rows)
    assert torch.equal(O_h, whole.output.cpu())
    assert torch.equal(lse_h, whole.lse.cpu())
    # and the public attend() on host arrays takes the same path
    res, _ = attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
    ref = whole.output.cpu().view(torch.int16).numpy().view(ml_dtypes.bfloat16)
    assert np.array_equal(res.output.view(np.int16), ref.view(np.int16))


@pytest.mark.gpu
def test_context_parallel_ranks_reassemble_whole():
    """Context parallelism: every rank's cost-balanced row range computed
    with swattn_attend_prepare + swattn_attend_rows (ranks run one after the
    other on this GPU) reassembles the whole-sequence attend bit for bit."""
    from paper_2509_24663_b200.parallel import context_parallel_attend
    rec, prof, cfg, _, (Qd, Kd, Vd) = _load("paper_n16384_s2")
    whole, _ = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    for world in (2, 4):
        O = torch.full_like(whole.output, float("nan"))
        lse = torch.full_like(whole.lse, float("nan"))
        covered = []
        for rank in range(world):
            _, _, rr = context_parallel_attend(Qd, Kd, Vd, cfg, world, rank, O=O, lse=lse)
            covered.append(rr)
        torch.cuda.synchronize()
        assert covered[0][0] == 0 and covered[-1][1] == Qd.shape[0]
        assert torch.equal(O, whole.output) and torch.equal(lse, whole.lse), world


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("paper_n16384_s2", 4), ("paper_n10000_s1", 3)])
def test_context_parallel_sharded_inputs(name, world):
    """Sequence-sharded context parallelism (parallel.context_parallel_attend_
    sharded) with its collectives replaced by in-process gathers: per-rank K1
    on the shard + halo reassembles the global compressed keys bit for bit,
    and each rank's rows computed from separately allocated Q / O shards
    (virtual row-0 base pointers) equal the whole-sequence attend."""
    from paper_2509_24663_b200.parallel import (cp_attend_rows, cp_halo_rows, cp_install_ckeys,
                                                cp_local_ckeys, shard_rows)
    from paper_2509_24663_b200.selection import Workspace
    rec, prof, cfg, _, (Qd, Kd, Vd) = _load(name)
    n = Qd.shape[0]
    whole, _ = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    k1, k2 = mean_pool_keys(Kd, cfg.l_C1, cfg.s_C1), mean_pool_keys(Kd, cfg.l_C2, cfg.s_C2)
    bounds = shard_rows(n, world)
    H = cp_halo_rows(cfg)
    parts = [cp_local_ckeys(Kd[a: min(n, b + H)].clone(), cfg, n, a, b) for a, b in bounds]
    kc1 = torch.cat([p[0] for p in parts])
    kc2 = torch.cat([p[1] for p in parts])
    assert torch.equal(kc1, k1.keys) and torch.equal(kc2, k2.keys)
    L = _lib.lib()
    ws = Workspace.get(L.swattn_workspace_bytes(_lib.c_config(cfg), n), Qd.device)
    cp_install_ckeys(ws, cfg, n, kc1, kc2)
    for a, b in bounds:
        Q_sh = Qd[a:b].clone()
        O_sh = torch.full((b - a, 32, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
        l_sh = torch.full((b - a, 32), float("nan"), dtype=torch.float32, device="cuda")
        cp_attend_rows(Q_sh, Kd, Vd, cfg, n, a, b, ws, O_sh, l_sh)
        torch.cuda.synchronize()
        assert torch.equal(O_sh, whole.output[a:b]) and torch.equal(l_sh, whole.lse[a:b]), (a, b)


@pytest.mark.gpu
def test_selection_all_tied_scores():
    """Q = 0 makes every candidate block of a row score exactly the same
    (shared = G / visible in float64 and float32 alike), so the stable
    argsort (selection.py:125) keeps the k lowest block ids.  Exercises K3's
    massive-tie path (the register path's survivor overflow) and the float64
    re-rank of every flagged row; checked in closed form for all rows and
    against the oracle on sampled rows."""
    n = 8192
    cfg = AttentionConfig()
    prof = O.Profile()
    _, K, _ = O.draw_qkv(n, 32, 2, 128, 11)
    Q = np.zeros((n, 32, 128), dtype=K.dtype)
    sel = select_blocks(_dev(Q), _dev(K), cfg, mode="approx")
    got = sel.topk.cpu().numpy().astype(np.int64)
    cnt = sel.topk_cnt.cpu().numpy()
    for i in range(0, n, 7):
        k = int(cnt[0, i])
        for g in range(2):
            assert np.array_equal(got[g, i, :k], np.arange(cfg.N_init, cfg.N_init + k)), (g, i)
    rows = np.array([4100, 5000, 8191])
    want, _, _ = O.select(Q, K, prof, mode="approx", rows=rows)
    assert np.array_equal(got[:, rows, :cfg.k_top], want.astype(np.int64)[:, :, :cfg.k_top])


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("scale", [3.0, 8.0])
def test_large_logits_dense_and_part_a(scale):
    """Logits spread wide enough that the running row max of the FA tile
    (K5 and part A) grows by more than its lazy-rescale threshold at
    different blocks for different rows of one warp: the O rescale must
    stay warp-collective (regression: a divergent tcgen05.ld hung the GPU on
    projected MiniCPM activations) and match the float64 oracle."""
    n = 8192
    cfg = AttentionConfig()
    prof = O.Profile()
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 5)
    Qs = (Q.astype(np.float32) * scale).astype(Q.dtype)
    Qd, Kd, Vd = _dev(Qs), _dev(K), _dev(V)
    rows = np.array([0, 1, 63, 64, 700, 4095, 4096, 6000, 8191])
    dense = tiled_gqa_forward(Qd, Kd, Vd, cfg)
    torch.cuda.synchronize()
    want_o, want_l = O.dense_attention(Qs, K, V, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    _tol(dense.output[r], want_o, dense.lse[r], want_l)
    res, mode = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    torch.cuda.synchronize()
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    topk = sel.topk.cpu().numpy().astype(np.int64)
    want_o, want_l = O.sparse_attention(Qs, K, V, topk, prof, rows=rows)
    _tol(res.output[r], want_o, res.lse[r], want_l)


@pytest.mark.gpu
def test_attend_cuda_graph_capture():
    """The sparse attend (K1..K4, part A forked onto the library's side stream
    and joined back) can be captured in a CUDA graph and replayed -- the
    serving path -- with results bit-identical to the eager call."""
    from paper_2509_24663_b200.core import make_qkv
    cfg = AttentionConfig()
    n = 16384
    Q, K, V = make_qkv(n, 32, 2, 128, seed=4)
    eager, _ = attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))   # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        res, _ = attend(Q, K, V, cfg, SwitchPolicy(forced_mode="sparse"))
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(res.output, eager.output) and torch.equal(res.lse, eager.lse)


@pytest.mark.gpu
def test_part_b_overflow_slow_path():
    """A top-k key whose logit exceeds the part-A offset m_A by far more than
    2^64 (log2) overflows part B's fixed-offset softmax; the token must go
    through the exact CUDA-core path and still match the float64 oracle."""
    n = 8192
    cfg = AttentionConfig()
    prof = O.Profile()
    Q, K, V = O.draw_qkv(n, 32, 2, 128, 13)
    i, j = 8000, 40                                   # query block 125, candidate block 40
    K = K.copy()
    K[j * 64 + 5, 0] = (Q[i, 0].astype(np.float32) * 8.0).astype(K.dtype)   # huge logit, head 0
    Qd, Kd, Vd = _dev(Q), _dev(K), _dev(V)
    res, mode = attend(Qd, Kd, Vd, cfg, SwitchPolicy(forced_mode="sparse"))
    sel = select_blocks(Qd, Kd, cfg, mode="approx")
    torch.cuda.synchronize()
    top = sel.topk.cpu().numpy().astype(np.int64)
    assert j in top[0, i]
    rows = np.array([i, i - 1, i + 1])
    want_o, want_l = O.sparse_attention(Q, K, V, top, prof, rows=rows)
    r = torch.as_tensor(rows, device="cuda")
    _tol(res.output[r], want_o, res.lse[r], want_l)


@pytest.mark.gpu
def test_decode_serving_loop_cuda_graph():
    """One serving step -- swattn_kcache_append_tokens (device-side seq_lens
    advance) + swattn_decode_step -- captured once in a CUDA graph and
    replayed step after step gives the eager loop's outputs bit for bit
    (pages mapped ahead by the host, as PagedKVCache.append_tokens does)."""
    from paper_2509_24663_b200.decode import PagedKVCache
    cfg, steps, B = AttentionConfig(), 6, 3
    gen = torch.Generator(device="cuda").manual_seed(7)
    prompt = [3000, 640, 1]
    ctx = [torch.randn((L, 2, 128), generator=gen, device="cuda").to(torch.bfloat16) for L in prompt]
    new_k = torch.randn((steps, B, 2, 128), generator=gen, device="cuda").to(torch.bfloat16)
    new_v = torch.randn_like(new_k)
    qs = torch.randn((steps, B, 32, 128), generator=gen, device="cuda").to(torch.bfloat16)
    L = _lib.lib()
    c = _lib.c_config(cfg)

    def make():
        cache = PagedKVCache(cfg, batch=B, max_pages=60, seed=2)
        for b, K in enumerate(ctx):
            cache.append(b, K, K.flip(0))
        for b in range(B):
            cache._ensure_pages(b, prompt[b] + steps)
        cache.block_table.copy_(torch.from_numpy(cache.block_table_h))
        nbytes = L.swattn_decode_workspace_bytes(c, B, cache.max_pages)
        return cache, torch.empty(nbytes, dtype=torch.uint8, device="cuda"), nbytes

    def step(cache, ws, nbytes, k, v, q, o, lse, topk, stream):
        kv = cache._descriptor()
        _lib.check(L.swattn_kcache_append_tokens(c, kv, k.data_ptr(), v.data_ptr(), None, B, stream),
                   "append_tokens")
        _lib.check(L.swattn_decode_step(c, kv, q.data_ptr(), B, o.data_ptr(), lse.data_ptr(),
                                        topk.data_ptr(), ws.data_ptr(), nbytes, stream), "decode")

    # eager loop
    cache, ws, nbytes = make()
    st = torch.cuda.current_stream().cuda_stream
    eager = []
    for t in range(steps):
        o = torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda")
        lse = torch.empty((B, 32), dtype=torch.float32, device="cuda")
        topk = torch.empty((B, 2, cfg.k_top), dtype=torch.int32, device="cuda")
        step(cache, ws, nbytes, new_k[t], new_v[t], qs[t], o, lse, topk, st)
        eager.append((o, lse, topk))
    torch.cuda.synchronize()
    assert cache.seq_lens.cpu().tolist() == [L0 + steps for L0 in prompt]
    # graph: static inputs / outputs, one warm-up step eagerly on the capture stream
    cache, ws, nbytes = make()
    k_in, v_in, q_in = new_k[0].clone(), new_v[0].clone(), qs[0].clone()
    o = torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((B, 32), dtype=torch.float32, device="cuda")
    topk = torch.empty((B, 2, cfg.k_top), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(cache, ws, nbytes, k_in, v_in, q_in, o, lse, topk, s.cuda_stream)   # = eager step 0
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step(cache, ws, nbytes, k_in, v_in, q_in, o, lse, topk, s.cuda_stream)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    assert torch.equal(o, eager[0][0]) and torch.equal(topk, eager[0][2])
    for t in range(1, steps):
        k_in.copy_(new_k[t]); v_in.copy_(new_v[t]); q_in.copy_(qs[t])
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(topk, eager[t][2]), t
        assert torch.equal(o, eager[t][0]) and torch.equal(lse, eager[t][1]), t
    assert cache.seq_lens.cpu().tolist() == [L0 + steps for L0 in prompt]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [300, 1000, 4100, 6144])
def test_dense_two_tile_matches_one_tile(n, monkeypatch):
    """The dense causal default (two query tiles per CTA, attention_tc2.cu)
    equals the one-tile FA kernel bit for bit, including a partial last tile
    pair (n % 16 != 0) -- both are checked against the oracle elsewhere."""
    from paper_2509_24663_b200.core import make_qkv
    cfg = AttentionConfig()
    Q, K, V = make_qkv(n, 32, 2, 128, seed=9)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("SWATTN_FA2", v)
        res = tiled_gqa_forward(Q, K, V, cfg)
        torch.cuda.synchronize()
        out[v] = (res.output.clone(), res.lse.clone())
    assert torch.equal(out["0"][0], out["1"][0]) and torch.equal(out["0"][1], out["1"][1])
