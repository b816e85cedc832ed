#!/bin/bash
export PYTHONUNBUFFERED=1
for n in 16384 32768 65536; do
for v in warp union; do
if [ $v = union ]; then export SWATTN_PARTB_UNION=1; else unset SWATTN_PARTB_UNION; fi
timeout 300 python bench.py --no-cpu --no-dense --n $n --steps 8 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);s=d['stages_ms'];print('n=$n $v', round(d['ms_per_step'],3), 'B', round(s['K4_part_B_est'],3))"
done; done
