"""Kernel timeline of one sparse attend at n = $N (torch.profiler / CUPTI):
start offset, duration and stream of every kernel and memset, to see the
critical path and the gaps between stages."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.switch import SwitchPolicy, attend
n = int(os.environ.get("N", "131072"))
cfg = AttentionConfig(); pol = SwitchPolicy(forced_mode="sparse")
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
for _ in range(2): attend(Q, K, V, cfg, pol)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    attend(Q, K, V, cfg, pol)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
end = max(e.time_range.end for e in evs)
for e in evs:
    print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  +{(e.time_range.end - e.time_range.start) / 1e3:8.3f} ms  "
          f"stream {getattr(e, 'device_index', '?')}/{e.kernel_name if hasattr(e, 'kernel_name') else ''} {e.name[:70]}")
print(f"total {(end - t0) / 1e3:.3f} ms")
