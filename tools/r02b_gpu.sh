#!/bin/bash
# r02b: full GPU test suite + bench N=1 (new multi-GPU-aware bench) + reference arm sample
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "general" > gpurun_out/r02b_pytest_general.log 2>&1; echo "pytest general rc=$?"; tail -15 gpurun_out/r02b_pytest_general.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -k "not general" > gpurun_out/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02b_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02b_bench.json; tail -5 gpurun_out/r02b_bench.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r02b_bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02b_bench_ref.json
timeout 600 python bench.py --cp --no-cpu --no-dense --steps 5 > gpurun_out/r02b_bench_cp1.json 2>&1; echo "cp rc=$?"; tail -1 gpurun_out/r02b_bench_cp1.json
