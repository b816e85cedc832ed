timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_general.py -q -x -k "decode" 2>&1 | tail -3
for s in 0 1 3; do python tools/bench_decode.py --graph --seed $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph seed', $s, d['ms_per_step'], d['rows_reranked_per_step'])"; done
python tools/bench_decode.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager', d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode --csv python tools/bench_decode.py --steps 3 --warmup 1 2>/dev/null | grep -E "decode_(scan|scores)" | tail -4 | cut -c1-40,200-
