set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
timeout 600 python tools/diag_scores.py 16384 131072 2>&1 | tail -3
K='regex:compress|scores|topk|rerank|fa_tile|sparse_pb|attention_list'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/launches_128k.csv python tools/one_attend.py 131072 > /dev/null 2>&1
grep -v "^==" gpurun_out/launches_128k.csv | awk -F'","' '{print $5, $NF}' | sed 's/"//g' | tail -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/prof_scores python tools/one_attend.py 131072 > gpurun_out/ncu_scores.log 2>&1; tail -2 gpurun_out/ncu_scores.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_pb -s 1 -c 1 -o gpurun_out/prof_pb python tools/one_attend.py 131072 > gpurun_out/ncu_pb.log 2>&1; tail -2 gpurun_out/ncu_pb.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_tile -s 1 -c 1 -o gpurun_out/prof_fa python tools/one_attend.py 131072 > gpurun_out/ncu_fa.log 2>&1; tail -2 gpurun_out/ncu_fa.log
timeout 900 python bench.py --steps 5 --warmup 3 --n 131072 --no-cpu 2>&1 | tail -1
