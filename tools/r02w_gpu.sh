#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scores_tc" -c 1 -f -o gpurun_out/r02w_k2_full python tools/one_attend.py 131072 > gpurun_out/r02w.log 2>&1; echo "ncu rc=$?"
