#!/bin/bash
# r02cf: round-2 final validation of the last build -- full GPU suite, smoke, bench (ours + reference), decode bench,
# launch list @128K, ncu full of the dominant kernels
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TAG=r02cf
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.json | cut -c1-300
timeout 300 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${TAG}_bench_ref.json | cut -c1-200
for s in 0 1; do timeout 300 python tools/bench_decode.py --graph --seed $s > gpurun_out/${TAG}_bench_decode_seed$s.json 2>&1; echo "decode rc=$?"; tail -1 gpurun_out/${TAG}_bench_decode_seed$s.json | cut -c1-160; done
K='regex:compress|scores|topk|rerank|fa_tile|sparse_pw|attention_list|route'
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k "$K" --csv --log-file gpurun_out/${TAG}_launches_128k.csv python tools/one_attend.py 131072 > /dev/null 2>&1; echo "launches rc=$?"
for k in sparse_pw fa_tile scores_tc topk_kernel; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/${TAG}_full_$k python tools/one_attend.py 131072 > gpurun_out/${TAG}_full_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout 900 python tools/switch_sweep.py > gpurun_out/${TAG}_switch_sweep.jsonl 2> gpurun_out/${TAG}_switch_sweep.err; echo "sweep rc=$?"
