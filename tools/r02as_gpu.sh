PCTS=0,45,60,80 timeout 600 python tools/route_sweep.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
