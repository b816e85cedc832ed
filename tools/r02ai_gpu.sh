#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/r02ai_pytest.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02ai_pytest.log
timeout 300 python tools/partb_hash.py 8192 32768 131072 > gpurun_out/r02ai_hash.txt 2>&1; cat gpurun_out/r02ai_hash.txt
for r in 1 2; do timeout 600 python bench.py --no-cpu --no-dense > gpurun_out/r02ai_bench_$r.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/r02ai_bench_$r.json').read().strip().splitlines()[-1]);s=d['stages_ms'];print(round(d['ms_per_step'],2), 'A', round(s['K4_part_A_fa_tile'],3), 'B', round(s['K4_part_B_est'],3))"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"sparse_pw" --csv python tools/one_attend.py 131072 > gpurun_out/r02ai_partb.csv 2>&1; python3 -c "import csv;[print(r[4][:30], r[-3], r[-1]) for r in csv.reader(open('gpurun_out/r02ai_partb.csv')) if len(r)>14 and 'sparse_pw' in r[4]]"
