#!/bin/bash
# r02am: the N>1 bench paths on a one-GPU lease (both ranks on cuda:0 over gloo; timings meaningless)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
SWATTN_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-dense --n 32768 > gpurun_out/r02am_bench_g2.json 2> gpurun_out/r02am_bench_g2.err; echo "g2 rc=$?"; tail -1 gpurun_out/r02am_bench_g2.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print({k:d[k] for k in ['n_gpus','value','ms_per_step','scaling']}, d.get('strong_scaling',{}).get('ms_per_step'), d['config']['parallelism'][:80])"; tail -3 gpurun_out/r02am_bench_g2.err
SWATTN_BENCH_SHARE_GPU=1 timeout 600 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --n 32768 > gpurun_out/r02am_ref_g2.json 2>&1; echo "ref g2 rc=$?"; grep -c metric gpurun_out/r02am_ref_g2.json
SWATTN_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-dense --n 32768 --cp > gpurun_out/r02am_bench_g2_cp.json 2> gpurun_out/r02am_bench_g2_cp.err; echo "g2 cp rc=$?"; tail -1 gpurun_out/r02am_bench_g2_cp.json | cut -c1-200; tail -3 gpurun_out/r02am_bench_g2_cp.err
