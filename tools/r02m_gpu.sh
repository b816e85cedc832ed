#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/bench_decode.py --graph > gpurun_out/r02m_bench_decode_graph.json 2>&1; echo "graph rc=$?"; tail -1 gpurun_out/r02m_bench_decode_graph.json | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none -k regex:"decode_|rerank" --csv python tools/bench_decode.py --steps 2 --warmup 1 > gpurun_out/r02m_decode_launches_warm.csv 2>&1; echo "ncu rc=$?"
timeout 900 python tools/decode_gaps.py > gpurun_out/r02m_decode_gaps.txt 2>&1; echo "gaps rc=$?"; grep -c FLAG gpurun_out/r02m_decode_gaps.txt; grep FLAG gpurun_out/r02m_decode_gaps.txt; tail -2 gpurun_out/r02m_decode_gaps.txt
