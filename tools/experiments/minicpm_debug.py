import os, sys, faulthandler, math
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import minicpm_prefill as M
from paper_2509_24663_b200.core import AttentionConfig
from paper_2509_24663_b200.switch import attend
dev = torch.device("cuda")
gen = torch.Generator(device=dev).manual_seed(0)
L = M.Layer(dev, gen)
n = 4096
h = torch.randn(n, M.D, device=dev, generator=gen).to(torch.bfloat16)
cos, sin = M.rope_tables(n, dev)
x = M.rms_norm(h, L.ln1); torch.cuda.synchronize(); print("norm", flush=True)
qkv = x @ L.wqkv.t(); torch.cuda.synchronize(); print("qkv", flush=True)
q = qkv[:, : 32 * 128].view(n, 32, 128)
k = qkv[:, 32 * 128: 34 * 128].view(n, 2, 128)
v = qkv[:, 34 * 128:].view(n, 2, 128).contiguous()
q = M.rope(q, cos, sin).contiguous(); k = M.rope(k, cos, sin).contiguous(); torch.cuda.synchronize(); print("rope", q.abs().max().item(), k.abs().max().item(), flush=True)
cfg = AttentionConfig()
for scale in (0.25, 0.5, 1.0):
    res, mode = attend(q * scale, k, v, cfg); torch.cuda.synchronize(); print("attend", scale, mode, res.output.float().abs().max().item(), flush=True)
