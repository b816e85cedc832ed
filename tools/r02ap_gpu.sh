set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "decode" 2>&1 | tail -3
python tools/bench_decode.py --graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph', d['ms_per_step'])"
python tools/bench_decode.py --graph --serve 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph+serve', d['ms_per_step'])"
python tools/bench_decode.py --serve 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager+serve', d['ms_per_step'])"
