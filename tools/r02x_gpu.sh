#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-dense > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo "bench rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02x_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e']['ms_per_step'],{k:round(v,3) for k,v in d['stages_ms'].items()})"
timeout 300 python tools/bench_decode.py > gpurun_out/r02x_bench_decode.json 2>&1; echo "decode rc=$?"; tail -1 gpurun_out/r02x_bench_decode.json | cut -c1-200
timeout 300 python tools/partb_hash.py 8192 32768 > gpurun_out/r02x_hash.txt 2>&1; cat gpurun_out/r02x_hash.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 > gpurun_out/r02x_pytest.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02x_pytest.log
