"""Phase timing (clock64) of the re-rank kernel's first CTA on a decode step
with a flagged row (variant build with -DSWATTN_RERANK_PROF)."""
import ctypes, os, subprocess, sys
sys.argv = [sys.argv[0], "--seed", "0", "--steps", "3", "--warmup", "1"]
import runpy
runpy.run_path(os.path.join(os.path.dirname(__file__), "bench_decode.py"), run_name="__main__")
from paper_2509_24663_b200 import _lib
L = _lib.lib()
buf = (ctypes.c_ulonglong * 16)()
L.swattn_debug_rerank_prof(buf)
st = list(buf[:7])
print("rerank phases (cycles from start):", [st[k] - st[0] for k in range(7)])
print("deltas: wait/count", st[1]-st[0], "load_q", st[2]-st[1], "pass1-combine", st[3]-st[2], "cluster scan", st[4]-st[3], "member scoring", st[5]-st[4], "settle/out", st[6]-st[5])
