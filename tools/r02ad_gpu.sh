#!/bin/bash
export PYTHONUNBUFFERED=1
for v in base fapoly4 fapoly8 base; do
if [ $v = base ]; then unset SWATTN_B200_LIB; else export SWATTN_B200_LIB=$PWD/varlibs/$v.so; fi
timeout 300 python tools/fa_time.py
done
