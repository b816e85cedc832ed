mkdir -p gpurun_out
for k in decode_pass1 decode_pass2 decode_topk_cta decode_attn_cluster; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/r02ch_full_$k python tools/bench_decode.py --steps 1 --warmup 1 > /dev/null 2>&1; echo "$k rc=$?"
done
timeout 300 ncu --set full --clock-control none -k regex:compress -c 1 -f -o gpurun_out/r02ch_full_compress python tools/one_attend.py 131072 > /dev/null 2>&1; echo "compress rc=$?"
