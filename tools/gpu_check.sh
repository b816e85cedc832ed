set -x
export PYTHONUNBUFFERED=1
timeout 300 ./tools/gather_bench 2>&1 | tee gpurun_out/gather_bench3.txt
timeout 900 python bench.py --steps 5 --warmup 3 --n 131072 --no-cpu 2>&1 | tail -1
