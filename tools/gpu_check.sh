set -x
export PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_pb -s 1 -c 1 -o gpurun_out/prof_pb2 python tools/one_attend.py 131072 > gpurun_out/ncu_pb2.log 2>&1; tail -2 gpurun_out/ncu_pb2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/prof_sc2 python tools/one_attend.py 131072 > gpurun_out/ncu_sc2.log 2>&1; tail -2 gpurun_out/ncu_sc2.log
