"""K2 (swattn_block_scores, approx) A/B: dumps S^cmp of one build to compare
bitwise with another, and times the kernel at n = $N.  SWATTN_B200_LIB picks the build."""
import os, sys, torch, hashlib
sys.path.insert(0, os.getcwd())
from paper_2509_24663_b200 import _lib
from paper_2509_24663_b200.core import AttentionConfig, make_qkv
from paper_2509_24663_b200.compression import mean_pool_keys
n = int(os.environ.get("N", "131072"))
cfg = AttentionConfig(); L = _lib.lib(); c = _lib.c_config(cfg)
Q, K, V = make_qkv(n, 32, 2, 128, seed=3, device="cuda")
c1 = mean_pool_keys(K, cfg.l_C1, cfg.s_C1).keys; c2 = mean_pool_keys(K, cfg.l_C2, cfg.s_C2).keys
n_cols = -(-c1.shape[0] // cfg.s); ld = (n_cols + 3) // 4 * 4
scmp = torch.zeros((cfg.h_kv, n, ld), dtype=torch.float32, device="cuda")
def run():
    _lib.check(L.swattn_block_scores(c, Q.data_ptr(), c1.data_ptr(), c2.data_ptr(), n, 2, scmp.data_ptr(), ld, None,
                                     _lib.stream_handle()), "k2")
run(); torch.cuda.synchronize()
digest = hashlib.sha1(scmp.cpu().numpy().tobytes()).hexdigest()[:16]
ts = []
for _ in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(os.environ.get("SWATTN_B200_LIB", "cur").split("/")[-1], n, "scmp sha1", digest, "K2 ms", round(sorted(ts)[3], 3), flush=True)
