#!/bin/bash
# r02l: decode v2 (tie flags, CTA top-k, 4-deep attention ring, batched pass-2 merge), K1 grid
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 > gpurun_out/r02l_pytest.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r02l_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s --timeout 600 -k decode > gpurun_out/r02l_fullsize_decode.log 2>&1; echo "decode16x128K rc=$?"; grep -E "decode|passed|failed" gpurun_out/r02l_fullsize_decode.log | tail -3
timeout 300 python tools/bench_decode.py > gpurun_out/r02l_bench_decode.json 2>&1; echo "decode bench rc=$?"; tail -1 gpurun_out/r02l_bench_decode.json | cut -c1-400
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"decode_|rerank" --csv python tools/bench_decode.py --steps 2 --warmup 1 > gpurun_out/r02l_decode_launches.csv 2>&1; echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:compress -c 2 --csv python tools/one_attend.py 131072 > gpurun_out/r02l_compress.csv 2>&1; echo "ncu compress rc=$?"; grep compress gpurun_out/r02l_compress.csv | tail -2 | cut -c1-300
