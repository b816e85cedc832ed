"""Hash of a sparse attend's O / lse (compare part-B variants bit for bit:
SWATTN_PARTB=warp vs the default union form)."""
import hashlib, sys
import torch
sys.path.insert(0, ".")
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend

for n in [int(a) for a in sys.argv[1:]] or [8192, 32768, 131072]:
    Q, K, V = make_qkv(n, 32, 2, 128, seed=1, device="cuda")
    res, m = attend(Q, K, V, AttentionConfig(), SwitchPolicy(forced_mode="sparse"))
    torch.cuda.synchronize()
    h = hashlib.sha256(res.output.view(torch.int16).cpu().numpy().tobytes() + res.lse.cpu().numpy().tobytes())
    print(n, h.hexdigest()[:16])
