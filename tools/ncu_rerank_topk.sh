cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in rerank_kernel topk_kernel; do
timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/r01c_full_$k python tools/one_attend.py 131072 > gpurun_out/r01c_full_$k.log 2>&1; echo "ncu $k rc=$?"
done
