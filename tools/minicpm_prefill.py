"""BASELINE config 5 (second half): full 32-layer MiniCPM4.1-8B prefill with
random-init weights, attention through `switch.attend` (dense K5 at n <= 6144,
sparse K1-K4 above -- the reference's switch), everything else
plain PyTorch / cuBLAS bf16 (the reference has no projections or FFN,
SPEC.md:441, so parity is pinned only at the attention boundary).

Architecture (MiniCPM4-8B public config): d_model 4096, 32
layers, 32 query heads / 2 KV heads, head_dim 128, SwiGLU FFN 16384, RMSNorm,
rotary position embedding (plain RoPE, base 10000 -- the LongRoPE rescaling
changes the rotation angles, not the cost), MiniCPM depth-scaled residuals
(scale_depth / sqrt(n_layers)).  Embedding and LM head are omitted (the
prefill output is the final hidden state); weights N(0, 0.02).

Per n it times one prefill with our attention and one with torch SDPA
(cuDNN) dense causal attention in the same layers, and reports the
attention share of the step.
  python tools/minicpm_prefill.py [n ...] > profiles/<round>_minicpm_prefill.jsonl
"""
import json
import math
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2509_24663_b200.core import AttentionConfig  # noqa: E402
from paper_2509_24663_b200.switch import attend  # noqa: E402

D, HQ, HKV, DH, FF = 4096, 32, 2, 128, 16384
LAYERS = int(os.environ.get("MINICPM_LAYERS", 32))
SCALE_DEPTH = 1.4
ROWS = 16384  # row chunk of the FFN (bounds the 2 x 16384-wide intermediate)


class Layer:
    def __init__(self, dev, gen):
        def w(*shape):
            return (torch.randn(*shape, device=dev, dtype=torch.float32, generator=gen) * 0.02).to(
                torch.bfloat16)
        self.ln1 = torch.ones(D, device=dev, dtype=torch.bfloat16)
        self.ln2 = torch.ones(D, device=dev, dtype=torch.bfloat16)
        self.wqkv = w((HQ + 2 * HKV) * DH, D)
        self.wo = w(D, HQ * DH)
        self.wgu = w(2 * FF, D)
        self.wd = w(D, FF)


def rms_norm(x, w, eps=1e-6):
    return F.rms_norm(x, (x.shape[-1],), w, eps)


def rope_tables(n, dev):
    inv = 1.0 / (10000 ** (torch.arange(0, DH, 2, device=dev, dtype=torch.float32) / DH))
    ang = torch.arange(n, device=dev, dtype=torch.float32)[:, None] * inv[None]
    return torch.cos(ang).to(torch.bfloat16)[:, None], torch.sin(ang).to(torch.bfloat16)[:, None]


def rope(x, cos, sin):
    x1, x2 = x[..., : DH // 2], x[..., DH // 2:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def attn_ours(q, k, v, cfg):
    res, mode = attend(q, k, v, cfg)
    return res.output, mode


def attn_cudnn(q, k, v, cfg):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    qt = q.transpose(0, 1)[None]
    kt = k.transpose(0, 1)[None]
    vt = v.transpose(0, 1)[None]
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        o = F.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)
    return o[0].transpose(0, 1), "cudnn"


def prefill(h, layers, cfg, attn_fn, timers):
    n = h.shape[0]
    cos, sin = rope_tables(n, h.device)
    res_scale = SCALE_DEPTH / math.sqrt(LAYERS)
    mode = None
    for L in layers:
        x = rms_norm(h, L.ln1)
        qkv = x @ L.wqkv.t()
        q = qkv[:, : HQ * DH].view(n, HQ, DH)
        k = qkv[:, HQ * DH: (HQ + HKV) * DH].view(n, HKV, DH)
        v = qkv[:, (HQ + HKV) * DH:].view(n, HKV, DH).contiguous()
        q = rope(q, cos, sin).contiguous()
        k = rope(k, cos, sin).contiguous()
        timers[0].record()
        o, mode = attn_fn(q, k, v, cfg)
        timers[1].record()
        h = h + (o.reshape(n, HQ * DH) @ L.wo.t()) * res_scale
        for r0 in range(0, n, ROWS):
            xs = rms_norm(h[r0: r0 + ROWS], L.ln2)
            gu = xs @ L.wgu.t()
            y = F.silu(gu[:, :FF]) * gu[:, FF:]
            h[r0: r0 + ROWS] += (y @ L.wd.t()) * res_scale
        timers[2].append((timers[0], timers[1]))
        timers[0] = torch.cuda.Event(enable_timing=True)
        timers[1] = torch.cuda.Event(enable_timing=True)
    return h, mode


def run(n, layers, cfg, attn_fn, reps=2):
    dev = layers[0].wqkv.device
    gen = torch.Generator(device=dev).manual_seed(n)
    h0 = torch.randn(n, D, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    best = None
    for rep in range(reps + 1):
        # [start event, end event, [(start, end) per layer]] of the attention calls
        timers = [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), []]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        h, mode = prefill(h0.clone(), layers, cfg, attn_fn, timers)
        b.record()
        torch.cuda.synchronize()
        if rep == 0:
            continue  # warm-up
        total = a.elapsed_time(b)
        att = sum(s.elapsed_time(e) for s, e in timers[2])
        if best is None or total < best[0]:
            best = (total, att, mode, bool(torch.isfinite(h.float()).all()))
        del h
    return best


def main():
    if os.environ.get("MINICPM_WATCHDOG"):  # debugging: dump the stacks of a hung run
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ["MINICPM_WATCHDOG"]), exit=True)
    sizes = [int(x) for x in sys.argv[1:]] or [4096, 32768, 131072]
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(0)
    print("building weights", file=sys.stderr, flush=True)
    layers = [Layer(dev, gen) for _ in range(LAYERS)]
    cfg = AttentionConfig()
    lin_flops_per_tok = 2 * LAYERS * (D * (HQ + 2 * HKV) * DH + HQ * DH * D + D * 2 * FF + FF * D)
    print(f"weights ready ({LAYERS} layers)", file=sys.stderr, flush=True)
    for n in sizes:
        ours = run(n, layers, cfg, attn_ours)
        print(f"n={n} ours {ours[0]:.1f} ms", file=sys.stderr, flush=True)
        dense = run(n, layers, cfg, attn_cudnn)
        print(f"n={n} cudnn {dense[0]:.1f} ms", file=sys.stderr, flush=True)
        line = {"n": n, "layers": LAYERS, "weights": "random N(0,0.02) bf16", "attention_mode": ours[2],
                "ms": ours[0], "tokens_per_s": n / (ours[0] / 1e3), "attention_ms": ours[1],
                "attention_share": ours[1] / ours[0], "finite": ours[3],
                "cudnn_dense": {"ms": dense[0], "attention_ms": dense[1],
                                "attention_share": dense[1] / dense[0]},
                "speedup_vs_cudnn_model": dense[0] / ours[0],
                "linear_tflops": lin_flops_per_tok * n / (ours[0] - ours[1]) / 1e9}
        print(json.dumps(line), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
