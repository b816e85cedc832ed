set -x
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "selection_bit or k2_score" 2>&1 | grep -E "passed|failed|Error|assert|FAIL" | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_pb -s 1 -c 1 -o gpurun_out/prof_pb4 python tools/one_attend.py 131072 > gpurun_out/ncu_pb4.log 2>&1; tail -1 gpurun_out/ncu_pb4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rerank -s 1 -c 1 -o gpurun_out/prof_rr python tools/one_attend.py 131072 > gpurun_out/ncu_rr.log 2>&1; tail -1 gpurun_out/ncu_rr.log
K='regex:compress|scores|topk|rerank|fa_tile|sparse_pb|attention_list'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_128k.csv python tools/one_attend.py 131072 > /dev/null 2>&1
grep -v "^==" gpurun_out/launches_128k.csv | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | tail -8
