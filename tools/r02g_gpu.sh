#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 120 python tools/partb_hash.py 8192 > gpurun_out/r02g_hash_union.txt 2>&1; echo "union8k rc=$?"
SWATTN_PARTB=warp timeout 120 python tools/partb_hash.py 8192 > gpurun_out/r02g_hash_warp.txt 2>&1; echo "warp8k rc=$?"
diff gpurun_out/r02g_hash_union.txt gpurun_out/r02g_hash_warp.txt && echo identical8k
tail -3 gpurun_out/r02g_hash_union.txt
timeout 300 python tools/partb_hash.py 32768 131072 > gpurun_out/r02g_hash_union2.txt 2>&1; echo "union rc=$?"
SWATTN_PARTB=warp timeout 300 python tools/partb_hash.py 32768 131072 > gpurun_out/r02g_hash_warp2.txt 2>&1; echo "warp rc=$?"
diff gpurun_out/r02g_hash_union2.txt gpurun_out/r02g_hash_warp2.txt && echo identical
for n in 131072 32768; do
timeout 300 python bench.py --no-cpu --no-dense --n $n > gpurun_out/r02g_bench_union_$n.json 2> gpurun_out/r02g_bench_union_$n.err; echo "union $n rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r02g_bench_union_$n.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general.py -m gpu -q -x --timeout 300 > gpurun_out/r02g_pytest.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/r02g_pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:sparse_ --csv python tools/one_attend.py 131072 > gpurun_out/r02g_ncu_partb.csv 2>&1; echo "ncu rc=$?"; grep -E "sparse_" gpurun_out/r02g_ncu_partb.csv | cut -d, -f5,13,15 | head -12
