#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_general.py -m gpu -q -s --timeout 900 > gpurun_out/r02c_pytest_general.log 2>&1; echo "general rc=$?"; tail -15 gpurun_out/r02c_pytest_general.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s --timeout 1800 > gpurun_out/r02c_pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "mismatch|decode 16|passed|failed|Error" gpurun_out/r02c_pytest_fullsize.log | tail -15
