"""Block-sharing fraction of K4 part B: how many K/V block gathers remain when
T consecutive tokens of one query block (same KV group) load the union of
their top-k blocks once, relative to one gather per (token, block).

  python tools/sharing_probe.py [n ...]

Inputs: make_qkv (the bench workload) and MiniCPM-like projected q/k/v
(random weights + RoPE, tools/minicpm_prefill.py).  Prints one JSON line per
(input, n) with the ratio for T = 1, 4, 8, 16, 32, 64.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from paper_2509_24663_b200.core import AttentionConfig, make_qkv  # noqa: E402
from paper_2509_24663_b200.selection import select_blocks  # noqa: E402


def sharing(topk, cnt, B, T):
    """topk [G, n, k] int32 (-1 padded), cnt [G, n]: gathers with T-token unions."""
    G, n, k = topk.shape
    nb = 2048 * 4
    total = int(cnt.sum())
    un = 0
    r0 = (n // B) * B
    tk = topk[:, :r0].reshape(G, r0 // T, T * k).long()
    valid = tk >= 0
    # bitmap per (group, T-chunk) over block ids
    nbk = int(tk.max().item()) + 1 if total else 1
    for g in range(G):
        for c0 in range(0, tk.shape[1], 4096):
            t = tk[g, c0:c0 + 4096]
            v = valid[g, c0:c0 + 4096]
            bm = torch.zeros((t.shape[0], nbk), dtype=torch.bool, device=t.device)
            bm.scatter_(1, torch.where(v, t, torch.zeros_like(t)), v)
            # scatter with v=False at index 0 may clear a true bit: redo index 0
            has0 = ((t == 0) & v).any(1)
            bm[:, 0] = has0
            un += int(bm.sum())
    del nb
    return un / max(total, 1)


def main():
    ns = [int(x) for x in sys.argv[1:]] or [32768, 131072]
    cfg = AttentionConfig()
    dev = torch.device("cuda")
    for n in ns:
        inputs = {"make_qkv": lambda: make_qkv(n, 32, 2, 128, seed=0, device="cuda")}
        try:
            import minicpm_prefill as M

            def model():
                gen = torch.Generator(device=dev).manual_seed(0)
                L = M.Layer(dev, gen)
                h = torch.randn(n, M.D, device=dev, generator=gen).to(torch.bfloat16)
                cos, sin = M.rope_tables(n, dev)
                x = M.rms_norm(h, L.ln1)
                qkv = x @ L.wqkv.t()
                q = M.rope(qkv[:, :4096].view(n, 32, 128), cos, sin).contiguous()
                k = M.rope(qkv[:, 4096:4352].view(n, 2, 128), cos, sin).contiguous()
                return q, k, None
            inputs["minicpm_projected"] = model
        except Exception as e:  # pragma: no cover
            print("no model inputs:", e, file=sys.stderr)
        for name, fn in inputs.items():
            Q, K, _ = fn()
            sel = select_blocks(Q, K, cfg, mode="approx")
            res = {T: round(sharing(sel.topk, sel.topk_cnt, cfg.B, T), 4) for T in (1, 4, 8, 16, 32, 64)}
            print(json.dumps({"n": n, "inputs": name, "gather_ratio_vs_T": res}), flush=True)
            del Q, K, sel
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
