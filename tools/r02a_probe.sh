#!/bin/bash
# r02a: sharing probe, K1 + decode ncu captures, compute-sanitizer on small shapes
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python tools/sharing_probe.py 32768 131072 > gpurun_out/r02a_sharing.jsonl 2> gpurun_out/r02a_sharing.err; echo "sharing rc=$?"; cat gpurun_out/r02a_sharing.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:compress -c 1 -f -o gpurun_out/r02a_full_compress python tools/one_attend.py 131072 > gpurun_out/r02a_full_compress.log 2>&1; echo "ncu compress rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02a_decode_launches.csv python tools/bench_decode.py --steps 3 --warmup 1 > gpurun_out/r02a_decode_ncu.log 2>&1; echo "ncu decode rc=$?"
timeout 400 python tools/bench_decode.py > gpurun_out/r02a_bench_decode.json 2>&1; echo "decode rc=$?"; tail -1 gpurun_out/r02a_bench_decode.json
for tool in racecheck synccheck; do
timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/one_attend.py 8192 > gpurun_out/r02a_sanitizer_$tool.log 2>&1; echo "sanitizer $tool rc=$?"; tail -5 gpurun_out/r02a_sanitizer_$tool.log
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/one_attend.py 8192 > gpurun_out/r02a_sanitizer_memcheck.log 2>&1; echo "sanitizer memcheck rc=$?"; tail -5 gpurun_out/r02a_sanitizer_memcheck.log
