#!/bin/bash
# A/B the FA-tile variant libraries (tools/build_variants.sh)
cd $GRAFT_REPO_ROOT
for v in default "$@"; do
  if [ $v = default ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/tools/variants/$v/lib/libswattn_b200.so; fi
  timeout 300 python tools/experiments/fa_probe.py 2>&1 | tail -1
done
