#!/bin/bash
# r02f: union-staged part B -- parity, A/B timing vs the per-token ring, full-size selection
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 600 > gpurun_out/r02f_pytest.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/r02f_pytest.log
for n in 131072 32768; do
timeout 600 python bench.py --no-cpu --no-dense --n $n > gpurun_out/r02f_bench_union_$n.json 2> gpurun_out/r02f_bench_union_$n.err; echo "union $n rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02f_bench_union_$n.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
SWATTN_PARTB=warp timeout 600 python bench.py --no-cpu --no-dense --n $n > gpurun_out/r02f_bench_warp_$n.json 2> gpurun_out/r02f_bench_warp_$n.err; echo "warp $n rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02f_bench_warp_$n.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
done
timeout 300 python tools/partb_hash.py > gpurun_out/r02f_hash_union.txt; SWATTN_PARTB=warp timeout 300 python tools/partb_hash.py > gpurun_out/r02f_hash_warp.txt; echo "hash diff:"; diff gpurun_out/r02f_hash_union.txt gpurun_out/r02f_hash_warp.txt && echo identical; cat gpurun_out/r02f_hash_union.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:sparse_ --csv python tools/one_attend.py 131072 > gpurun_out/r02f_ncu_partb.csv 2>&1; echo "ncu rc=$?"; grep -E "sparse_" gpurun_out/r02f_ncu_partb.csv | head -12
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -x --timeout 1000 > gpurun_out/r02f_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "mismatch|decode|passed|failed|Error" gpurun_out/r02f_fullsize.log | tail -8
