#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for v in base sleep1 sleep2 base; do
if [ $v = base ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/varlibs/$v.so; fi
timeout 600 python bench.py --no-cpu --no-dense --steps 8 > gpurun_out/r02y_bench_$v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02y_bench_$v.json').read().strip().splitlines()[-1]);s=d['stages_ms'];print('$v', round(d['ms_per_step'],2), 'K2', round(s['K2_block_scores'],3), 'A', round(s['K4_part_A_fa_tile'],3), 'B', round(s['K4_part_B_est'],3))"
done
