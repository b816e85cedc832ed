cd $GRAFT_REPO_ROOT
for v in default noflags default noflags; do
  if [ $v = default ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/tools/variants/$v/lib/libswattn_b200.so; fi
  timeout 300 python bench.py --no-cpu --no-dense --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})"
done
