#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py --cp-sharded --no-cpu --no-dense --steps 5 > gpurun_out/r02z_cp_sharded.json 2> gpurun_out/r02z_cp_sharded.err; echo "cps rc=$?"; tail -1 gpurun_out/r02z_cp_sharded.json | cut -c1-300; tail -3 gpurun_out/r02z_cp_sharded.err
timeout 600 python bench.py --cp --no-cpu --no-dense --steps 5 > gpurun_out/r02z_cp.json 2> gpurun_out/r02z_cp.err; echo "cp rc=$?"; tail -1 gpurun_out/r02z_cp.json | cut -c1-300
timeout 300 python tools/experiments/cp_sharded_timing.py > gpurun_out/r02z_cps_timing.txt 2>&1; echo "timing rc=$?"; tail -15 gpurun_out/r02z_cps_timing.txt
