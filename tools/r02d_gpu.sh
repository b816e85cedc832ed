#!/bin/bash
# r02d: GPU suite (general + fullsize + rest), bench N=1, reference arm
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_general.py -m gpu -q -x -s --timeout 900 > gpurun_out/r02d_pytest_general.log 2>&1; echo "general rc=$?"; tail -8 gpurun_out/r02d_pytest_general.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 --ignore=tests/test_gpu_general.py --ignore=tests/test_gpu_fullsize.py > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r02d_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02d_bench.json; tail -5 gpurun_out/r02d_bench.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r02d_bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02d_bench_ref.json
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 1800 > gpurun_out/r02d_pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "mismatch|decode|passed|failed|Error|rerank" gpurun_out/r02d_pytest_fullsize.log | tail -20
