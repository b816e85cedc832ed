#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/bench_decode.py > gpurun_out/r02u_bench_decode.json 2>&1; echo "eager rc=$?"; tail -1 gpurun_out/r02u_bench_decode.json | cut -c1-200
timeout 300 python tools/bench_decode.py --graph > gpurun_out/r02u_bench_decode_graph.json 2>&1; echo "graph rc=$?"; tail -1 gpurun_out/r02u_bench_decode_graph.json | cut -c1-200
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02u_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02u_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02u_bench.json | cut -c1-400
