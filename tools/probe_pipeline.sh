cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default w4 w8np w4np w8np64; do
  if [ $v = default ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/tools/variants/$v/lib/libswattn_b200.so; fi
  timeout 300 python tools/pipeline_probe.py 131072 4 8 16 >> gpurun_out/pipeline_probe.txt 2>&1
done
