for r in 1 2; do for v in p2s2c13 p2s3c9 p2s3c13 p2s4c6; do
  for s in 0 1; do SWATTN_B200_LIB=$PWD/variants/$v.so python tools/bench_decode.py --graph --seed $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v seed $s', round(d['ms_per_step']*1000,1), 'us')"; done
done; done
SWATTN_B200_LIB=$PWD/variants/p2s3c9.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_general.py -q -x -k "decode" 2>&1 | tail -2
for v in p2s2c13 p2s3c9; do SWATTN_B200_LIB=$PWD/variants/$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:decode_pass --csv python tools/bench_decode.py --steps 2 --warmup 1 2>/dev/null | grep -E "decode_pass2" | tail -1 | awk -F'","' '{print "'$v' pass2 ns", $NF}'; done
