"""BASELINE configs 2 and 5: the dense/sparse switch sweep 1K-128K through
`switch.attend` with the default policy (dense K5 at n <= 6144, SPEC.md:442;
sparse K1-K4 above), each n beside dense causal attention of the same shape
(own K5, FA2, cuDNN; bench.dense_comparator).  One JSON line per n on
stdout; inputs make_qkv(seed=0) resident in HBM, CUDA-event timing, median
of `reps` after warm-up.
  python tools/switch_sweep.py [n ...] > profiles/<round>_switch_sweep.jsonl
"""
import json
import os
import sys

import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2509_24663_b200.core import AttentionConfig, make_qkv  # noqa: E402
from paper_2509_24663_b200.switch import attend  # noqa: E402

SIZES = [1024, 2048, 4096, 6144, 8192, 16384, 32768, 65536, 131072]


def median_ms(fn, stream, reps):
    fn()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    sizes = [int(x) for x in sys.argv[1:]] or SIZES
    cfg = AttentionConfig()
    stream = torch.cuda.current_stream()
    for n in sizes:
        Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
        mode = {}

        def step():
            _, mode["m"] = attend(Q, K, V, cfg)
        reps = 20 if n <= 16384 else 7
        ms = median_ms(step, stream, reps)
        dense = bench.dense_comparator(Q, K, V, cfg, n, stream, reps=3 if n > 32768 else 10)
        best = dense.get("best", {})
        line = {"n": n, "mode": mode["m"], "ms": ms, "tokens_per_s": n / (ms / 1e3),
                "dense": {k: v.get("ms") for k, v in dense.items() if k != "best"},
                "best_dense": best.get("impl"), "best_dense_ms": best.get("ms"),
                "speedup_vs_best_dense": (best["ms"] / ms) if best else None}
        print(json.dumps(line), flush=True)
        del Q, K, V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
