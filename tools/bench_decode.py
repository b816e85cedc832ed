"""BASELINE config 4: decode, batch 16 with a 128K paged KV cache, per-step
block selection + sparse attention (K6).  Prints one JSON line.

  python tools/bench_decode.py [--batch 16] [--ctx 131072] [--steps 20]

Synthetic K/V (torch.randn, bf16, seeded) written straight into a shuffled
page pool; the timed step is swattn_decode_step for all sequences (pass 1 /
pass 2 scoring over the compressed keys, top-k + fp64 re-rank, split-KV
attention over <= 96 pages), CUDA events on the launching stream, L2 flushed
between steps (a 256 MB write) because one step's working set (~190 MB) is
close to the L2 size.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.decode import PagedKVCache


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--graph", action="store_true",
                    help="capture the step in a CUDA graph and time graph replays")
    ap.add_argument("--serve", action="store_true",
                    help="serving-loop step: swattn_kcache_append_tokens (one new token per "
                         "sequence, seq_lens advanced on the device) + swattn_decode_step")
    args = ap.parse_args()
    cfg = AttentionConfig()
    B, L = args.batch, args.ctx
    g = torch.Generator(device="cuda").manual_seed(args.seed)
    cache = PagedKVCache(cfg, batch=B, max_pages=-(-L // cfg.B) + 1, seed=3)
    for b in range(B):
        K = torch.randn((L, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
        V = torch.randn((L, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
        cache.append(b, K, V)
        del K, V
    q = torch.randn((B, cfg.h_q, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty((B, cfg.h_q), dtype=torch.float32, device="cuda")
    topk = torch.empty((B, cfg.h_kv, cfg.k_top), dtype=torch.int32, device="cuda")
    Lb = _lib.lib()
    c = _lib.c_config(cfg)
    nbytes = Lb.swattn_decode_workspace_bytes(c, B, cache.max_pages)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    kv = cache._descriptor()
    stream = torch.cuda.current_stream()
    if args.serve:
        # map the pages the timed appends will write (the host-side part of
        # PagedKVCache.append_tokens), so the device step needs no host work
        extra = args.warmup + args.steps + 2
        if (L + extra) > cache.max_pages * cfg.B:
            raise SystemExit("--serve needs ctx + steps below max_pages * 64")
        for b in range(B):
            cache._ensure_pages(b, L + extra)
        cache.block_table.copy_(torch.from_numpy(cache.block_table_h))
        knew = torch.randn((B, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
        vnew = torch.randn((B, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(sp=None):
        sp = sp or stream.cuda_stream
        if args.serve:
            _lib.check(Lb.swattn_kcache_append_tokens(c, kv, knew.data_ptr(), vnew.data_ptr(), None, B,
                                                      sp), "append_tokens")
        _lib.check(Lb.swattn_decode_step(c, kv, q.data_ptr(), B, o.data_ptr(), lse.data_ptr(),
                                         topk.data_ptr(), ws.data_ptr(), nbytes, sp),
                   "decode")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    run = step
    if args.graph:
        # the step's seven launches (+ one memset) replayed as one graph:
        # no per-launch host overhead or inter-kernel launch gaps
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                step(torch.cuda.current_stream().cuda_stream)
        stream.wait_stream(gs)
        torch.cuda.synchronize()
        run = graph.replay
        run()
        torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    off = Lb.swattn_decode_reranked_offset(c, B, cache.max_pages)
    reranked = int(ws[off:off + 4].view(torch.int32).item())
    # dense decode comparator: flash-attn 2.8 decode over the same 16 x 128K
    # contexts held contiguously (its paged path needs 256-token pages)
    dense = {}
    try:
        from flash_attn import flash_attn_with_kvcache
        kc = torch.randn((B, L, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
        vc = torch.randn((B, L, cfg.h_kv, cfg.d_h), generator=g, device="cuda").to(torch.bfloat16)
        lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
        qd = q[:, None]

        def dstep():
            flash_attn_with_kvcache(qd, kc, vc, cache_seqlens=lens, causal=True)
        dstep()
        torch.cuda.synchronize()
        dts = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dstep()
            b.record(stream)
            torch.cuda.synchronize()
            dts.append(a.elapsed_time(b))
        dense = {"impl": "flash_attn 2.8.3 flash_attn_with_kvcache (dense, contiguous cache)",
                 "ms": float(np.median(dts))}
        del kc, vc
    except Exception as e:  # pragma: no cover - comparator unavailable
        dense = {"error": str(e)[:160]}
    # algorithmic HBM bytes per step: per (sequence, group) the compressed keys
    # read by both scoring passes + K/V of the selected <= 96 blocks
    m1 = Lb.swattn_num_pooled(L, cfg.l_C1, cfg.s_C1)
    m2 = Lb.swattn_num_pooled(L, cfg.l_C2, cfg.s_C2)
    kv_blocks = min(cfg.N_init + cfg.N_local + cfg.k_top, -(-L // cfg.B))
    per = (m1 + m2) * cfg.d_h * 2 + kv_blocks * cfg.B * cfg.d_h * 2 * 2
    bytes_step = B * cfg.h_kv * per
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json"))) if os.path.exists("MEASURED_PEAKS.json") else {}
    hbm = peaks.get("hbm_gbs", 6552.0)
    line = {"metric": "decode tokens/s (batch x 128K paged cache, per-step selection + sparse attention)",
            "value": B / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms, "steps": args.steps,
            "higher_is_better": True, "dtype": "bf16", "data": "synthetic (torch.randn K/V/q, seeded)",
            "config": {"workload": f"decode batch {B}, context {L}, paged (64-token pages, shuffled pool)",
                       "launch": "CUDA graph replay" if args.graph else "eager launches",
                       "step": ("swattn_kcache_append_tokens + swattn_decode_step" if args.serve
                                else "swattn_decode_step"),
                       "l2": "flushed between steps (256 MB write)"},
            "roofline": {"bound": "hbm", "achieved": bytes_step / (ms / 1e3) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": bytes_step / (ms / 1e3) / 1e9 / hbm,
                         "algorithmic_bytes_per_step": bytes_step},
            "rows_reranked_per_step": reranked,
            "dense_decode_comparator": dense}
    if "ms" in dense:
        line["speedup_vs_dense_decode"] = dense["ms"] / ms
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
