timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_general.py -q -x -k "decode or tied or long" 2>&1 | tail -2
for s in 0 1; do python tools/bench_decode.py --graph --seed $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('seed $s', round(d['ms_per_step']*1000,1), 'us')"; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_topk --csv python tools/bench_decode.py --steps 2 --warmup 1 2>/dev/null | grep decode_topk | tail -1 | awk -F'","' '{print "decode_topk ns", $NF}'
timeout 900 python tools/long_ctx_check.py 2>&1 | grep "^n=" | head -3
