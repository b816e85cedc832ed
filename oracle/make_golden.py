"""Mint golden vectors from the UNMODIFIED reference (test infrastructure).

Runs ``swattn`` from ``/root/reference/pkg/src`` (read-only; never copied)
on bf16 storage arrays (ml_dtypes) -- the reference is dtype-generic, so this
is its own code path with storage = bf16 -- and writes small fixtures to
``tests/golden/``.  Inputs are NOT stored: they are regenerated with
``make_qkv`` (Philox) and pinned by a sha256 digest stored in each fixture.

Usage (build container only; /root/reference does not exist on the GPU box):
    python oracle/make_golden.py [--quick]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def _topk_array(sel, cfg, n):
    """BlockSelection -> (topk [h_kv, n, k_top] int16 -1 padded, counts)."""
    top = np.full((cfg.h_kv, n, max(cfg.k_top, 1)), -1, dtype=np.int16)
    for g in range(cfg.h_kv):
        for i in range(n):
            b = i // cfg.B
            lo = max(0, b - cfg.N_local + 1)
            base = set(range(min(cfg.N_init, b + 1))) | set(range(lo, b + 1))
            t = [int(j) for j in sel.blocks[g][i] if int(j) not in base]
            top[g, i, :len(t)] = t
    return top, np.asarray(sel.counts, dtype=np.int16)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the 16K case")
    ap.add_argument("--only", default=None, help="regenerate only fixtures whose name contains this")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.dirname(HERE))
    import ml_dtypes
    from swattn.core import AttentionConfig, make_qkv
    from swattn.compression import mean_pool_keys, max_pool_scores
    from swattn.selection import (select_blocks, fused_shared_scores_approx,
                                  fused_shared_scores_exact)
    from swattn.sparse import sparse_forward
    from swattn.dense import tiled_gqa_forward
    from swattn.switch import attend, SwitchPolicy
    from oracle.swattn_oracle import digest

    bf = ml_dtypes.bfloat16
    os.makedirs(OUT, exist_ok=True)
    small = AttentionConfig(h_q=4, h_kv=2, d_h=16, B=16, l_C1=8, s_C1=4, l_C2=32,
                            s_C2=16, l=5, s=4, N_init=1, N_local=2, k_top=3, w=16)
    paper = AttentionConfig()

    def case(name, cfg, n, seed, *, scores=False, exact=False, sparse_rows=None,
             dense_rows=None, forced=None, backward_rows=None, dense_backward=False):
        if args.only and args.only not in name:
            return
        t0 = time.time()
        Q, K, V = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed, dtype=bf)
        rec = {"n": n, "seed": seed, "digest": digest(Q, K, V),
               "cfg": np.array([cfg.h_q, cfg.h_kv, cfg.d_h, cfg.B, cfg.l_C1, cfg.s_C1,
                                cfg.l_C2, cfg.s_C2, cfg.l, cfg.s, cfg.N_init, cfg.N_local,
                                cfg.k_top, cfg.w])}
        ck1 = mean_pool_keys(K, cfg.l_C1, cfg.s_C1)
        ck2 = mean_pool_keys(K, cfg.l_C2, cfg.s_C2)
        rec["c1_digest"] = digest(ck1.keys)
        rec["c2_digest"] = digest(ck2.keys)
        if n <= 2048:
            rec["c1_bits"] = _bits(ck1.keys)
            rec["c2_bits"] = _bits(ck2.keys)
        sel = select_blocks(Q, K, cfg, mode="approx")
        rec["topk"], rec["counts"] = _topk_array(sel, cfg, n)
        if exact:
            sel_e = select_blocks(Q, K, cfg, mode="fused-exact")
            rec["topk_exact"], _ = _topk_array(sel_e, cfg, n)
        if scores:
            sh = fused_shared_scores_approx(Q, ck1, ck2, cfg)
            cmp_ = max_pool_scores(sh, cfg.l, cfg.s)
            rows = np.arange(n) if n <= 1024 else np.unique(
                np.linspace(0, n - 1, 48).astype(np.int64))
            rec["score_rows"] = rows
            rec["shared_approx"] = sh.scores[rows]
            rec["cmp_approx"] = cmp_.scores[rows]
            if n <= 1024:
                rec["shared_exact"] = fused_shared_scores_exact(Q, ck1, cfg).scores
        if sparse_rows is not None:
            res, mode = attend(Q, K, V, cfg, SwitchPolicy(forced_mode=forced or "sparse"))
            rows = np.asarray(sparse_rows)
            rec["sparse_rows"] = rows
            rec["sparse_out_bits"] = _bits(res.output[rows])
            rec["sparse_lse"] = res.lse[rows]
            rec["sparse_mode"] = mode
        if dense_rows is not None:
            res = tiled_gqa_forward(Q, K, V, cfg)
            rows = np.asarray(dense_rows)
            rec["dense_rows"] = rows
            rec["dense_out_bits"] = _bits(res.output[rows])
            rec["dense_lse"] = res.lse[rows]
        if backward_rows is not None:
            # sparse_backward (sparse.py:130-185) with dO = the Q of seed + 1000
            from swattn.sparse import sparse_backward
            dO, _, _ = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed + 1000, dtype=bf)
            dQ, dK, dV = sparse_backward(Q, K, V, sel, dO, cfg)
            rows = np.asarray(backward_rows)
            rec["bwd_rows"] = rows
            rec["bwd_dQ_bits"] = _bits(dQ[rows])
            krows = rows if n <= 512 else np.unique(np.concatenate([
                rows, np.arange(0, 64), np.arange(n - 64, n)]))   # block 0 gets every query
            rec["bwd_key_rows"] = krows
            rec["bwd_dK_bits"] = _bits(dK[krows])
            rec["bwd_dV_bits"] = _bits(dV[krows])
            rec["bwd_digest"] = digest(dQ, dK, dV)
        if dense_backward:
            # naive_gqa_backward (dense.py:173-221), dO = the Q of seed + 1000
            from swattn.dense import naive_gqa_backward
            dO, _, _ = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed + 1000, dtype=bf)
            dQ, dK, dV = naive_gqa_backward(Q, K, V, dO, cfg)
            rec["dbwd_dQ_bits"] = _bits(dQ)
            rec["dbwd_dK_bits"] = _bits(dK)
            rec["dbwd_dV_bits"] = _bits(dV)
        if name == "paper_n300_s5":
            # the reference's own file writers (core.py:258-275, selection.py:386-400)
            import tempfile
            from swattn.core import save_tensor
            from swattn.selection import save_selection
            with tempfile.TemporaryDirectory() as d:
                save_selection(sel, os.path.join(d, "s.bin"))
                save_tensor(np.asarray(rec["sparse_lse"], dtype=np.float64), os.path.join(d, "t.swt"))
                rec["selection_file"] = np.frombuffer(open(os.path.join(d, "s.bin"), "rb").read(), np.uint8)
                rec["tensor_file"] = np.frombuffer(open(os.path.join(d, "t.swt"), "rb").read(), np.uint8)
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **rec)
        print(f"{name}: {time.time() - t0:.1f}s -> {os.path.getsize(path) / 1e6:.2f} MB",
              flush=True)

    def sample(n, k, seed):
        r = np.random.Generator(np.random.Philox(key=np.uint64(seed + 77))).choice(
            n, size=min(k, n), replace=False)
        return np.unique(np.concatenate([r, [0, n - 1]]))

    # small profile of the reference's own harness (bench.py:199-204)
    case("small_n64_s0", small, 64, 0, scores=True, exact=True,
         sparse_rows=np.arange(64), dense_rows=np.arange(64))
    case("small_n257_s0", small, 257, 0, scores=True, exact=True,
         sparse_rows=np.arange(257), dense_rows=np.arange(257))
    case("small_n1000_s3", small, 1000, 3, exact=True,
         sparse_rows=np.arange(1000), dense_rows=np.arange(1000))
    # paper profile (core.py:78-91)
    case("paper_n300_s5", paper, 300, 5, scores=True, sparse_rows=sample(300, 40, 6),
         dense_rows=sample(300, 40, 7))
    # backward (sparse.py:130-185): small profile, and the paper profile at
    # a length where top-k is competitive (n > 96 blocks * 64)
    case("bwd_small_n257_s0", small, 257, 0, backward_rows=np.arange(257))
    case("bwd_dense_paper_n200_s4", paper, 200, 4, dense_backward=True)
    case("bwd_paper_n7000_s8", paper, 7000, 8, backward_rows=sample(7000, 24, 9))
    case("paper_n4096_s0", paper, 4096, 0, sparse_rows=sample(4096, 96, 0),
         dense_rows=sample(4096, 96, 1))
    case("paper_n8192_s0", paper, 8192, 0, scores=True, exact=True,
         sparse_rows=sample(8192, 128, 2), dense_rows=sample(8192, 48, 3))
    case("paper_n10000_s1", paper, 10000, 1, scores=True, sparse_rows=sample(10000, 96, 4))
    if not args.quick:
        case("paper_n16384_s2", paper, 16384, 2, scores=True,
             sparse_rows=sample(16384, 64, 5))


if __name__ == "__main__":
    main()
