#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for s in 0 1 2 3 4; do
timeout 300 python tools/bench_decode.py --seed $s > gpurun_out/r02ab_decode_seed$s.json 2>&1; python -c "import json;d=json.loads(open('gpurun_out/r02ab_decode_seed$s.json').read().strip().splitlines()[-1]);print('seed $s', round(d['ms_per_step']*1000,1),'us', 'reranked', d['rows_reranked_per_step'])"
done
