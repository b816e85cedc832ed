set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_tc_probe.py -q 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -s -k "dense or sparse or attend or determinism or errors" 2>&1 | grep -v "^$" | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --n 32768 --no-cpu 2>&1 | tail -2
timeout 900 python bench.py --steps 2 --warmup 3 --n 131072 --no-cpu 2>&1 | tail -2
