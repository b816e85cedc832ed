timeout 300 python tools/timeline.py 2>&1 | grep -E "ms  \+|total"
for r in 1 2 3; do for v in prev prio; do SWATTN_B200_LIB=$PWD/variants/$v.so N=131072 ROUNDS=1 VARIANTS='x:' timeout 300 python tools/route_ab.py | sed "s/^/$v /"; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
