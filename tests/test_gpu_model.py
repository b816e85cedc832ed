"""Parity beyond the attention boundary: a MiniCPM4.1-8B
style layer stack (tools/minicpm_prefill.py: RMSNorm, fused QKV projection,
RoPE, GQA 32/2 x 128, depth-scaled residuals, SwiGLU FFN; random weights) run
with `switch.attend` in every layer against the same stack run with a plain
PyTorch float32 attention over the same selected blocks (init U local U
top-k of the approx selection, causal -- sparse.py:70-91).  n = 8192 takes
the sparse branch (threshold 6144, switch.py:27-82).

Per layer the attention outputs must agree within the bf16 bars of the
attention tests, and the final hidden state within 2 % relative (the
residual stream is bf16 in both stacks)."""
import importlib
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
N_LAYERS = 2
N = 8192


def _model():
    os.environ["MINICPM_LAYERS"] = str(N_LAYERS)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import minicpm_prefill as M
    return importlib.reload(M)


def _masked_attention_f32(q, k, v, topk, cfg):
    """Float32 attention of every row over init U local U top-k blocks (causal)."""
    n, h_q, d = q.shape
    G = h_q // k.shape[1]
    B = cfg.B
    nb = -(-n // B)
    out = torch.empty((n, h_q, d), dtype=torch.float32, device=q.device)
    keys = torch.arange(n, device=q.device)
    blk_of_key = keys // B
    for g in range(k.shape[1]):
        kg, vg = k[:, g].float(), v[:, g].float()
        for r0 in range(0, n, 512):
            rows = torch.arange(r0, min(n, r0 + 512), device=q.device)
            b = rows // B
            allowed = torch.zeros((rows.numel(), nb), dtype=torch.bool, device=q.device)
            allowed[:, : cfg.N_init] = (torch.arange(cfg.N_init, device=q.device)[None] <= b[:, None])
            j = torch.arange(nb, device=q.device)
            allowed |= (j[None] >= (b[:, None] - cfg.N_local + 1)) & (j[None] <= b[:, None])
            t = topk[g, r0: r0 + rows.numel()].long()
            tv = t >= 0
            allowed.scatter_(1, t.clamp_min(0), tv | allowed.gather(1, t.clamp_min(0)))
            vis = allowed[:, blk_of_key] & (keys[None] <= rows[:, None])
            qg = q[r0: r0 + rows.numel(), g * G:(g + 1) * G].float()
            s = torch.einsum("rhd,kd->rhk", qg, kg) / d ** 0.5
            s = s.masked_fill(~vis[:, None, :], float("-inf"))
            out[r0: r0 + rows.numel(), g * G:(g + 1) * G] = torch.einsum(
                "rhk,kd->rhd", torch.softmax(s, dim=-1), vg)
    return out


def test_layer_stack_matches_float32_attention_stack():
    M = _model()
    from paper_2509_24663_b200.core import AttentionConfig
    from paper_2509_24663_b200.selection import select_blocks
    from paper_2509_24663_b200.switch import attend

    cfg = AttentionConfig()
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(0)
    layers = [M.Layer(dev, gen) for _ in range(N_LAYERS)]
    h0 = (torch.randn(N, M.D, device=dev, generator=gen) * 1.0).to(torch.bfloat16)

    per_layer = []

    def ours(q, k, v, c):
        res, mode = attend(q, k, v, c)
        assert mode == "sparse"
        sel = select_blocks(q, k, c, mode="approx")
        ref = _masked_attention_f32(q, k, v, sel.topk, c)
        err = (res.output.float() - ref).abs()
        per_layer.append((float(err.max()), float(err.mean())))
        return res.output, mode

    def reference(q, k, v, c):
        sel = select_blocks(q, k, c, mode="approx")
        return _masked_attention_f32(q, k, v, sel.topk, c).to(torch.bfloat16), "f32"

    ev = lambda: [torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), []]
    h_ours, _ = M.prefill(h0.clone(), layers, cfg, ours, ev())
    h_ref, _ = M.prefill(h0.clone(), layers, cfg, reference, ev())
    torch.cuda.synchronize()
    for li, (mx, mean) in enumerate(per_layer):
        assert mx <= 2e-2 and mean <= 2e-3, (li, mx, mean)
    rel = float((h_ours.float() - h_ref.float()).norm() / h_ref.float().norm())
    print(f"{N_LAYERS} layers, n={N}: attention max-abs {[round(m, 5) for m, _ in per_layer]}, "
          f"final hidden state relative error {rel:.3g}")
    assert torch.isfinite(h_ours.float()).all()
    assert rel <= 2e-2
