timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
N=32768 ROUNDS=4 VARIANTS='base:SWATTN_ROUTE_PCT=0;default:' timeout 600 python tools/route_ab.py
N=131072 ROUNDS=3 VARIANTS='base:SWATTN_ROUTE_PCT=0;default:' timeout 600 python tools/route_ab.py
