#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 > gpurun_out/r02al_pytest.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02al_pytest.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -x --timeout 1000 > gpurun_out/r02al_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "mismatch|decode|passed|failed|Error" gpurun_out/r02al_fullsize.log | tail -4
for s in 0 2 1; do
timeout 300 python tools/bench_decode.py --seed $s > gpurun_out/r02al_decode_seed$s.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/r02al_decode_seed$s.json').read().strip().splitlines()[-1]);print('seed $s', round(d['ms_per_step']*1000,1),'us', 'reranked', d['rows_reranked_per_step'])"
done
timeout 600 python bench.py --no-cpu --no-dense > gpurun_out/r02al_bench.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02al_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],{k:round(v,3) for k,v in d['stages_ms'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rerank" --csv python tools/bench_decode.py --steps 2 --warmup 1 --seed 0 > gpurun_out/r02al_rerank_dec.csv 2>&1; python3 -c "import csv;[print(r[4][:30], r[-1]) for r in csv.reader(open('gpurun_out/r02al_rerank_dec.csv')) if len(r)>14 and 'rerank' in r[4]]"
