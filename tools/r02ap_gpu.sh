#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 > gpurun_out/r02ap_pytest.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02ap_pytest.log
timeout 1500 python tools/long_ctx_check.py 262144 393216 524288 557056 > gpurun_out/r02ap_long_ctx.txt 2>&1; echo "long rc=$?"; grep "^n=" gpurun_out/r02ap_long_ctx.txt; tail -3 gpurun_out/r02ap_long_ctx.txt
timeout 600 python tools/bench_decode.py --ctx 393216 --batch 4 > gpurun_out/r02ap_decode_384k.json 2>&1; echo "decode384k rc=$?"; tail -1 gpurun_out/r02ap_decode_384k.json | cut -c1-250
