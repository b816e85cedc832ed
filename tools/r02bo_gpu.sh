python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
cfg = AttentionConfig(); pol = SwitchPolicy(forced_mode="sparse")
for n in (8192, 20000, 65536):
    Q, K, V = make_qkv(n, 32, 2, 128, seed=2, device="cuda")
    os.environ["SWATTN_FA2_PARTA"] = "0"; a, _ = attend(Q, K, V, cfg, pol); a = (a.output.clone(), a.lse.clone())
    os.environ["SWATTN_FA2_PARTA"] = "1"; b, _ = attend(Q, K, V, cfg, pol)
    torch.cuda.synchronize()
    print(n, "bit-identical", torch.equal(a[0], b.output) and torch.equal(a[1], b.lse), float((a[0].float() - b.output.float()).abs().max()), flush=True)
PY
for n in 16384 32768 131072; do N=$n ROUNDS=4 VARIANTS='base:SWATTN_FA2_PARTA=0;parta2:SWATTN_FA2_PARTA=1' timeout 600 python tools/route_ab.py; done
