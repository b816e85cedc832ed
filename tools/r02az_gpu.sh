for n in 8192 16384 32768; do N=$n ROUNDS=4 VARIANTS='base:SWATTN_ROUTE_PCT=0;default:;r60:SWATTN_ROUTE_PCT=60' timeout 600 python tools/route_ab.py; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "routed or sparse_attention or full_size" 2>&1 | tail -2
