set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -s --timeout 600 2>&1 | grep -E "err|passed|failed|Error|assert|FAIL|max rel|reranked" | head -60
timeout 600 python tools/diag_scores.py 16384 131072 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --n 131072 --no-cpu 2>&1 | tail -2
