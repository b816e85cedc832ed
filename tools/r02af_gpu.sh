#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/r02af_pytest.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02af_pytest.log
timeout 600 python bench.py --no-cpu --no-dense > gpurun_out/r02af_bench.json 2>/dev/null; echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02af_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],{k:round(v,3) for k,v in d['stages_ms'].items()})"
