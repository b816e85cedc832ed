#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 -k "decode" > gpurun_out/r02aj_pytest.log 2>&1; echo "decode tests rc=$?"; tail -2 gpurun_out/r02aj_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s --timeout 600 -k decode > gpurun_out/r02aj_fullsize_decode.log 2>&1; echo "decode16x128K rc=$?"; grep -E "decode|passed|failed" gpurun_out/r02aj_fullsize_decode.log | tail -2
timeout 300 python tools/bench_decode.py > gpurun_out/r02aj_bench_decode.json 2>&1; echo "eager rc=$?"; tail -1 gpurun_out/r02aj_bench_decode.json | cut -c1-250
timeout 300 python tools/bench_decode.py --graph > gpurun_out/r02aj_bench_decode_graph.json 2>&1; echo "graph rc=$?"; tail -1 gpurun_out/r02aj_bench_decode_graph.json | cut -c1-250
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none -k regex:"decode_|rerank" --csv python tools/bench_decode.py --steps 2 --warmup 1 > gpurun_out/r02aj_decode_launches_warm.csv 2>&1; echo "ncu rc=$?"
for s in 0 1 3; do
timeout 300 python tools/bench_decode.py --seed $s > gpurun_out/r02aj_decode_seed$s.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/r02aj_decode_seed$s.json').read().strip().splitlines()[-1]);print('seed $s', round(d['ms_per_step']*1000,1),'us', 'reranked', d['rows_reranked_per_step'])"
done
