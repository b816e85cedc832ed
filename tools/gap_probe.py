"""Is there GPU idle time between K1 (compress) and K2 (block scores)?  Times
K1 alone, K2 alone and K1 + K2 back to back with CUDA events at n = $N."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.compression import mean_pool_keys
n = int(os.environ.get("N", "131072")); cfg = AttentionConfig(); L = _lib.lib(); c = _lib.c_config(cfg)
Q, K, V = make_qkv(n, 32, 2, 128, seed=0, device="cuda")
c1 = mean_pool_keys(K, cfg.l_C1, cfg.s_C1).keys.clone(); c2 = mean_pool_keys(K, cfg.l_C2, cfg.s_C2).keys.clone()
n_cols = -(-c1.shape[0] // cfg.s); ld = (n_cols + 3) // 4 * 4
scmp = torch.empty((cfg.h_kv, n, ld), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def k1(): _lib.check(L.swattn_compress_keys(c, K.data_ptr(), n, c1.data_ptr(), c2.data_ptr(), st), "k1")
def k2(): _lib.check(L.swattn_block_scores(c, Q.data_ptr(), c1.data_ptr(), c2.data_ptr(), n, 2, scmp.data_ptr(), ld, None, st), "k2")
def both(): k1(); k2()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return round(sorted(ts)[reps // 2], 3)
print("K1", t(k1), "K2", t(k2), "K1+K2", t(both), "K2+K2", t(lambda: (k2(), k2())), flush=True)
from torch.profiler import profile, ProfilerActivity
def timeline(label, fn):
    fn(); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn(); torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(label, " | ".join(f"{e.name[:24]} @{(e.time_range.start - t0) / 1e3:.3f} +{(e.time_range.end - e.time_range.start) / 1e3:.3f}" for e in evs), flush=True)
small = torch.zeros(1024, device="cuda")
timeline("K1,K2", both)
timeline("K2,K2", lambda: (k2(), k2()))
timeline("fill,K2", lambda: (small.fill_(1.0), k2()))
timeline("K1,fill,K2", lambda: (k1(), small.fill_(1.0), k2()))
