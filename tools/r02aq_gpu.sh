timeout 600 python tools/route_sweep.py 2>&1 | tail -8
SWATTN_ROUTE_PCT=45 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
