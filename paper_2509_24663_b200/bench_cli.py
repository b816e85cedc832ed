"""Command-line driver (reference: bench.py): correctness
suite, counted-work + wall-clock benchmark CSV/JSON, selection-quality
report and fixture generation -- run on the B200 kernels.

Differences from the reference, by design:
  * wall times are CUDA-event medians of the GPU kernels (the reference
    times numpy on the CPU); counts and the CSV schema are the reference's;
  * the correctness suite checks every kernel path against brute-force
    float32 references computed with torch on the same GPU (dense causal
    attention, masked attention over the selected blocks, autograd
    gradients) plus the selection invariants and bitwise determinism -- the
    CPU float64 oracle of the reference lives in `oracle/` and is used by the
    test suite, not by the product;
  * inputs are make_qkv draws rounded to bf16, the storage dtype of the
    kernels (`--precision` selects the precision of the written fixtures).
"""

from __future__ import annotations

import csv
import io
import json
import math
import os
from dataclasses import asdict, dataclass

import numpy as np
import torch

from .core import AttentionConfig, atomic_write_bytes, make_qkv, save_tensor, validate_config
from .counts import dense_query_counts, selection_query_counts, sparse_query_counts

BENCH_MODES = ("dense-naive", "dense-tiled", "select-exact", "select-approx", "sparse")
CSV_COLUMNS = ("mode", "n", "B", "k_top", "G", "d_h", "mac_count", "exp_count", "wall_ms",
               "speedup_counts")   # bench.py:64-67


@dataclass
class BenchRecord:
    """bench.py:70-82."""
    mode: str
    n: int
    B: int
    k_top: int
    G: int
    d_h: int
    mac_count: int
    exp_count: int
    wall_ms: float | None
    speedup_vs_dense: float
    pass1_mac: int | None = None


def _time_median(fn, repeats: int) -> float:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(max(1, repeats)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run_bench(cfg: AttentionConfig, sizes, modes=BENCH_MODES, seed: int = 0,
              exec_max_n: int = 131072, repeats: int = 5) -> list[BenchRecord]:
    """bench.py:384-431: one record per (mode, n); analytic per-query counts,
    GPU wall time when n <= exec_max_n."""
    from .dense import tiled_gqa_forward
    from .selection import select_blocks
    from .sparse import sparse_forward
    validate_config(cfg)
    for mode in modes:
        if mode not in BENCH_MODES:
            raise ValueError(f"unknown bench mode {mode!r}; expected one of {BENCH_MODES}")
    records = []
    for n in (int(x) for x in sizes):
        dense_mac, dense_exp = dense_query_counts(cfg, n)
        execute = n <= exec_max_n
        if execute:
            Q, K, V = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed)
            sel = select_blocks(Q, K, cfg, mode="approx") if "sparse" in modes else None
        for mode in modes:
            pass1 = None
            if mode in ("dense-naive", "dense-tiled"):
                mac, exp = dense_mac, dense_exp
            elif mode == "sparse":
                mac, exp = sparse_query_counts(cfg, n)
            else:
                d = selection_query_counts(cfg, n, approx=mode == "select-approx")
                mac, exp, pass1 = d["mac"], d["exp"], d["pass1_mac"]
            wall = None
            if execute:
                runner = {
                    "dense-naive": lambda: tiled_gqa_forward(Q, K, V, cfg),
                    "dense-tiled": lambda: tiled_gqa_forward(Q, K, V, cfg),
                    "select-exact": lambda: select_blocks(Q, K, cfg, mode="fused-exact"),
                    "select-approx": lambda: select_blocks(Q, K, cfg, mode="approx"),
                    "sparse": lambda: sparse_forward(Q, K, V, sel, cfg),
                }[mode]
                wall = _time_median(runner, repeats)
            records.append(BenchRecord(mode=mode, n=n, B=cfg.B, k_top=cfg.k_top, G=cfg.group_size,
                                       d_h=cfg.d_h, mac_count=mac, exp_count=exp, wall_ms=wall,
                                       speedup_vs_dense=dense_mac / mac, pass1_mac=pass1))
        if execute:
            del Q, K, V, sel
            torch.cuda.empty_cache()
    return records


def write_bench_csv(records, path) -> None:
    """bench.py:434-444 (same columns and formatting)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for r in records:
        w.writerow([r.mode, r.n, r.B, r.k_top, r.G, r.d_h, r.mac_count, r.exp_count,
                    "" if r.wall_ms is None else f"{r.wall_ms:.3f}", f"{r.speedup_vs_dense:.6g}"])
    atomic_write_bytes(path, buf.getvalue().encode())


def write_bench_json(records, path) -> None:
    """bench.py:447-449."""
    payload = {"columns": list(CSV_COLUMNS), "records": [asdict(r) for r in records]}
    atomic_write_bytes(path, json.dumps(payload, indent=2).encode() + b"\n")


# ---------------------------------------------------------------- selection quality

def random_equal_budget_selection(cfg: AttentionConfig, n: int, per_row_counts, seed: int):
    """bench.py:456-471: uniform random block sets of each row's budget
    (same Philox stream as the reference).  Returns tuple[h_kv] of tuple[n]
    of sorted int64 block arrays."""
    gen = np.random.Generator(np.random.Philox(key=np.uint64(seed) ^ np.uint64(0x9E3779B97F4A7C15)))
    groups = []
    for g in range(cfg.h_kv):
        rows = []
        for i in range(n):
            b = i // cfg.B
            count = min(int(per_row_counts[g][i]), b + 1)
            rows.append(np.sort(gen.choice(b + 1, size=count, replace=False).astype(np.int64)))
        groups.append(tuple(rows))
    return tuple(groups)


def _group_block_mass(Q, K, cfg: AttentionConfig, g: int) -> np.ndarray:
    """bench.py:474-494 on the GPU in float32: dense causal attention mass per
    (query, selection block), summed over the group's heads (rows sum to G)."""
    n = Q.shape[0]
    nb = -(-n // cfg.B)
    G = cfg.group_size
    scale = 1.0 / math.sqrt(cfg.d_h)
    k = K[:, g].float()
    mass = torch.zeros((n, nb), device=Q.device)
    causal = torch.ones((n, n), dtype=torch.bool, device=Q.device).tril()
    for h in range(g * G, (g + 1) * G):
        s = (Q[:, h].float() @ k.T) * scale
        s = s.masked_fill(~causal, float("-inf"))
        p = torch.softmax(s, dim=1)
        pad = torch.zeros((n, nb * cfg.B), device=Q.device)
        pad[:, :n] = p
        mass += pad.view(n, nb, cfg.B).sum(dim=2)
    return mass.double().cpu().numpy()


def _mean_recall(mass_by_group, blocks, G: int) -> float:
    total, rows = 0.0, 0
    for g, mass in enumerate(mass_by_group):
        for i, bl in enumerate(blocks[g]):
            total += mass[i, bl].sum() / G
            rows += 1
    return total / rows


def run_selection_quality(cfg: AttentionConfig, n: int, seed: int = 0) -> dict:
    """bench.py:513-555: attention-mass recall of exact / approximate /
    equal-budget random selection, and the approx-vs-exact top-k overlap."""
    from .selection import select_blocks
    from .switch import visible_token_budget
    validate_config(cfg)
    Q, K, _ = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed)
    sel_e = select_blocks(Q, K, cfg, mode="exact")
    sel_a = select_blocks(Q, K, cfg, mode="approx")
    ex, ap = sel_e.blocks, sel_a.blocks
    per_row = [[ex[g][i].size for i in range(n)] for g in range(cfg.h_kv)]
    rnd = random_equal_budget_selection(cfg, n, per_row, seed)
    mass = [_group_block_mass(Q, K, cfg, g) for g in range(cfg.h_kv)]
    top_e = sel_e.topk.cpu().numpy()
    top_a = sel_a.topk.cpu().numpy()
    cnt_e = sel_e.topk_cnt.cpu().numpy()
    cnt_a = sel_a.topk_cnt.cpu().numpy()
    overlaps = []
    for g in range(cfg.h_kv):
        for i in range(n):
            if cnt_e[g, i] == 0:
                continue
            se = set(top_e[g, i, :cnt_e[g, i]].tolist())
            sa = set(top_a[g, i, :cnt_a[g, i]].tolist())
            overlaps.append(len(se & sa) / len(se))
    G = cfg.group_size
    return {"n": n, "seed": seed, "budget_blocks": cfg.budget_blocks,
            "visible_token_budget": visible_token_budget(cfg),
            "recall": {"exact": _mean_recall(mass, ex, G), "approx": _mean_recall(mass, ap, G),
                       "random": _mean_recall(mass, rnd, G)},
            "topk_overlap_approx_vs_exact": float(np.mean(overlaps)) if overlaps else None,
            "rows_with_topk": len(overlaps)}


# ---------------------------------------------------------------- correctness

def _visible_mask(sel, cfg: AttentionConfig, g: int, device) -> torch.Tensor:
    """[n, n] bool: key j visible to query i (selection.py:73-87 spans)."""
    n = sel.n
    nb = -(-n // cfg.B)
    i = torch.arange(n, device=device)
    b = i // cfg.B
    j = torch.arange(nb, device=device)
    lo = torch.clamp(b - cfg.N_local + 1, min=0)
    blk = (j[None, :] < torch.clamp(b + 1, max=cfg.N_init)[:, None]) | \
          ((j[None, :] >= lo[:, None]) & (j[None, :] <= b[:, None]))
    top = sel.topk[g].to(device).long()
    ext = torch.cat([blk, torch.zeros((n, 1), dtype=torch.bool, device=device)], dim=1)
    ext.scatter_(1, torch.where(top >= 0, top, torch.full_like(top, nb)), True)  # -1 -> spare column
    tok = ext[:, :nb].repeat_interleave(cfg.B, dim=1)[:, :n]
    return tok & (i[None, :] <= i[:, None])


def _masked_reference(Q, K, V, sel, cfg):
    """float32 brute force over each row's visible blocks (sparse.py:101-127)."""
    G = cfg.group_size
    scale = 1.0 / math.sqrt(cfg.d_h)
    outs, lses = [], []
    for g in range(cfg.h_kv):
        vis = _visible_mask(sel, cfg, g, Q.device)
        k, v = K[:, g].float(), V[:, g].float()
        for h in range(g * G, (g + 1) * G):
            s = (Q[:, h].float() @ k.T) * scale
            s = s.masked_fill(~vis, float("-inf"))
            lses.append(torch.logsumexp(s, dim=1))
            outs.append(torch.softmax(s, dim=1) @ v)
    return torch.stack(outs, dim=1), torch.stack(lses, dim=1)


def run_correctness(seed: int = 0, sizes=(300, 4096, 8192), perturb: float = 0.0) -> dict:
    """bench.py:213-314 analogue on the GPU.  `perturb` (a documented test
    hook) is added to every checked output to prove a breach is
    reported."""
    from .dense import naive_gqa_backward, tiled_gqa_forward
    from .selection import select_blocks
    from .sparse import sparse_backward, sparse_forward
    cfg = AttentionConfig()
    checks = []

    def record(name, n, err, tol):
        checks.append({"check": name, "n": n, "max_err": float(err), "tol": tol,
                       "ok": bool(err <= tol)})

    for n in (int(x) for x in sizes):
        Q, K, V = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed)
        dO, _, _ = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed + 1000)
        # dense (K5) vs torch float32 causal attention
        res = tiled_gqa_forward(Q, K, V, cfg)
        q = Q.float().transpose(0, 1)[None]
        k = K.float().transpose(0, 1).repeat_interleave(cfg.group_size, 0)[None]
        v = V.float().transpose(0, 1).repeat_interleave(cfg.group_size, 0)[None]
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)[0].transpose(0, 1)
        record("dense_output", n, (res.output.float() - ref).abs().max().item() + perturb, 2e-2)
        # selection invariants (selection.py:113-136)
        sel = select_blocks(Q, K, cfg, mode="approx")
        top, cnt = sel.topk.cpu().numpy(), sel.topk_cnt.cpu().numpy()
        m1 = (n - cfg.l_C1) // cfg.s_C1 + 1 if n >= cfg.l_C1 else 0
        n_cols = -(-m1 // cfg.s)
        bad = 0
        for g in range(cfg.h_kv):
            for i in range(n):
                c = int(cnt[g, i])
                t = top[g, i, :c]
                b = i // cfg.B
                lo = max(0, b - cfg.N_local + 1)
                ncand = max(0, min(lo, n_cols) - cfg.N_init)
                bad += int(c > cfg.k_top or (c and (np.any(np.diff(t) <= 0) or t[0] < cfg.N_init
                                                    or t[-1] >= lo)) or np.any(top[g, i, c:] != -1))
                bad += int(c < min(cfg.k_top, ncand) and i + 1 >= cfg.l_C1)
        record("selection_invariants", n, bad, 0)
        # sparse (K4) vs torch float32 masked attention (small n: n x n masks)
        if n <= 8192:
            sp = sparse_forward(Q, K, V, sel, cfg)
            O_ref, L_ref = _masked_reference(Q, K, V, sel, cfg)
            record("sparse_output", n, (sp.output.float() - O_ref).abs().max().item() + perturb, 2e-2)
            record("sparse_lse", n, (sp.lse - L_ref).abs().max().item() + perturb, 1e-3)
            again = sparse_forward(Q, K, V, sel, cfg)
            record("sparse_determinism", n, float(not torch.equal(again.output, sp.output)), 0)
        # backward vs autograd on the float32 masked / dense references (small n)
        if n <= 1024:
            qq, kk, vv = (t.float().requires_grad_() for t in (Q, K, V))
            Oq, _ = _masked_reference(qq, kk, vv, sel, cfg)
            gq, gk, gv = torch.autograd.grad(Oq, (qq, kk, vv), dO.float())
            dq, dk, dv = sparse_backward(Q, K, V, sel, dO, cfg)
            for nm, got, want in (("sparse_dQ", dq, gq), ("sparse_dK", dk, gk), ("sparse_dV", dv, gv)):
                rel = (got.float() - want).abs().max().item() / max(want.abs().max().item(), 1e-30)
                record(nm, n, rel + perturb, 2e-2)
            Od = torch.nn.functional.scaled_dot_product_attention(
                qq.transpose(0, 1)[None], kk.transpose(0, 1).repeat_interleave(cfg.group_size, 0)[None],
                vv.transpose(0, 1).repeat_interleave(cfg.group_size, 0)[None], is_causal=True)[0].transpose(0, 1)
            gq, gk, gv = torch.autograd.grad(Od, (qq, kk, vv), dO.float())
            dq, dk, dv = naive_gqa_backward(Q, K, V, dO, cfg)
            for nm, got, want in (("dense_dQ", dq, gq), ("dense_dK", dk, gk), ("dense_dV", dv, gv)):
                rel = (got.float() - want).abs().max().item() / max(want.abs().max().item(), 1e-30)
                record(nm, n, rel + perturb, 2e-2)
        del Q, K, V, dO
        torch.cuda.empty_cache()
    return {"seed": seed, "sizes": [int(x) for x in sizes], "checks": checks,
            "ok": all(c["ok"] for c in checks), "warning": None if checks else "no checks run"}


# ---------------------------------------------------------------- fixtures

def generate_fixtures(out_dir, sizes, seed: int, cfg: AttentionConfig, precision=np.float32):
    """bench.py:558-585: seeded Q/K/V (bf16-rounded, stored at `precision`)
    and the dense output / lse of the K5 kernel per size, plus manifest.json."""
    from .dense import tiled_gqa_forward
    validate_config(cfg)
    os.makedirs(out_dir, exist_ok=True)
    entries = []
    for n in (int(x) for x in sizes):
        Q, K, V = make_qkv(n, cfg.h_q, cfg.h_kv, cfg.d_h, seed=seed)
        res = tiled_gqa_forward(Q, K, V, cfg)
        files = {}
        for name, t in (("q", Q), ("k", K), ("v", V), ("out", res.output), ("lse", res.lse)):
            fname = f"fixture_n{n}_seed{seed}_{name}.swt"
            save_tensor(t.float().cpu().numpy().astype(precision), os.path.join(out_dir, fname))
            files[name] = fname
        entries.append({"n": n, "files": files})
    manifest = {"seed": seed, "precision": "f64" if np.dtype(precision) == np.float64 else "f32",
                "storage": "bf16-rounded inputs (the kernels' storage dtype)",
                "config": asdict(cfg), "fixtures": entries}
    atomic_write_bytes(os.path.join(out_dir, "manifest.json"),
                       json.dumps(manifest, indent=2).encode() + b"\n")
    return manifest
