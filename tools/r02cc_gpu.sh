timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_general.py -q -x -k "decode or serving" 2>&1 | tail -3
for s in 0 1; do timeout 120 python tools/bench_decode.py --graph --seed $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph seed $s', round(d['ms_per_step']*1000,1), 'us')"; done
timeout 120 python tools/bench_decode.py --seed 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager seed 1', round(d['ms_per_step']*1000,1), 'us')"
