nvidia-smi topo -m 2>&1 | head -5
for r in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e'].get('host_cpus'))"; done
