#!/bin/bash
export PYTHONUNBUFFERED=1
for v in persist oneitem persist oneitem; do
if [ $v = oneitem ]; then export SWATTN_PA_ONEITEM=1; else unset SWATTN_PA_ONEITEM; fi
timeout 300 python bench.py --no-cpu --no-dense --steps 8 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);s=d['stages_ms'];print('$v', round(d['ms_per_step'],3), 'A', round(s['K4_part_A_fa_tile'],3), 'B', round(s['K4_part_B_est'],3))"
done
unset SWATTN_PA_ONEITEM
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > /tmp/p.log 2>&1; echo "parity rc=$?"; tail -1 /tmp/p.log
