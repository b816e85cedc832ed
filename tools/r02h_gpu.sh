#!/bin/bash
# r02h: part B time vs persistent grid (is it chip-L2-bound?)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in 148 128 111 96 74; do
SWATTN_PB_CTAS=$c timeout 300 python bench.py --no-cpu --no-dense --steps 5 > gpurun_out/r02h_pb_$c.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02h_pb_$c.json').read().strip().splitlines()[-1]);s=d['stages_ms'];print('ctas=$c', round(d['ms_per_step'],2), 'partB', round(s['K4_part_B_est'],2), 'K2', round(s['K2_block_scores'],2))"
done
