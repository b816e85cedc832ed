#!/bin/bash
# A/B the part-B variant libraries (tools/build_variants.sh) on the 128K bench stages
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in default "$@"; do
  if [ $v = default ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/tools/variants/$v/lib/libswattn_b200.so; fi
  timeout 300 python bench.py --no-cpu --no-dense --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})"
done
