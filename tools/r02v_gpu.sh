#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"rerank" -c 2 -f -o gpurun_out/r02v_rerank_full python tools/bench_decode.py --steps 1 --warmup 1 > gpurun_out/r02v.log 2>&1; echo "ncu rc=$?"
