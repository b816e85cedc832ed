#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TAG=r02ay
timeout 900 python tools/switch_sweep.py > gpurun_out/${TAG}_switch_sweep.jsonl 2> gpurun_out/${TAG}_switch_sweep.err; echo "sweep rc=$?"; cut -c1-120 gpurun_out/${TAG}_switch_sweep.jsonl
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fa_tile --launch-skip 1 -c 1 -f -o gpurun_out/${TAG}_full_routed_fa python tools/one_attend.py 32768 > gpurun_out/${TAG}_full_routed.log 2>&1; echo "ncu routed rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_32k.csv python tools/one_attend.py 32768 > /dev/null 2>&1; echo "launches rc=$?"
