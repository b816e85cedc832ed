for c in 8 16; do SWATTN_HOST_CHUNKS=$c python tools/e2e_time.py | sed "s/^/chunks=$c /"; done
for c in 8 16; do SWATTN_HOST_CHUNKS=$c timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench chunks=$c', d['ms_per_step'], d['e2e']['ms_per_step'])"; done
