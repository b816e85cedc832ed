set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "sparse or attend or full_size" 2>&1 | grep -E "passed|failed|Error|assert|FAIL" | head -20
K='regex:compress|scores|topk|rerank|fa_tile|sparse_pb|attention_list'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_128k.csv python tools/one_attend.py 131072 > /dev/null 2>&1
grep -v "^==" gpurun_out/launches_128k.csv | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | tail -8
