#!/bin/bash
# One gpurun call: parity tests, smoke, bench (ours + reference arm), launch list,
# one ncu --set full capture per hot kernel. Outputs under gpurun_out/.
set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${TAG}_bench_ref.json
if [ -z "$NO_NCU" ]; then
K='regex:compress|scores|topk|rerank|fa_tile|sparse_pw|attention_list|maxpool'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/${TAG}_launches_128k.csv python tools/one_attend.py 131072 > /dev/null 2>&1
grep -v "^==" gpurun_out/${TAG}_launches_128k.csv | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | tail -12
for k in ${NCU_KERNELS:-sparse_pw scores_tc fa_tile topk rerank}; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/${TAG}_full_$k python tools/one_attend.py 131072 > gpurun_out/${TAG}_full_$k.log 2>&1; echo "ncu $k rc=$?"
done
fi
ls -la gpurun_out
