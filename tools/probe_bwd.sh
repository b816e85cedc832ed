cd $GRAFT_REPO_ROOT
for v in default q10 q12; do
  if [ $v = default ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/tools/variants/$v/lib/libswattn_b200.so; fi
  echo $v; timeout 300 python tools/bench_backward.py 131072 2>&1 | cut -c1-80
done
