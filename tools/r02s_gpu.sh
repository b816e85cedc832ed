#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in 148 128 116; do
SWATTN_PB_CTAS=$c timeout 300 python tools/pipeline_probe.py 131072 4 8 > gpurun_out/r02s_pipe_$c.txt 2>&1; echo "pb_ctas=$c"; cat gpurun_out/r02s_pipe_$c.txt | tail -3
done
