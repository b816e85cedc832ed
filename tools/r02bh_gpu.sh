mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/one_attend.py 8192 > gpurun_out/r02bh_sanitizer_${tool}_attend8192.log 2>&1; echo "attend $tool rc=$?"; tail -2 gpurun_out/r02bh_sanitizer_${tool}_attend8192.log
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/decode_once.py > gpurun_out/r02bh_sanitizer_${tool}_decode.log 2>&1; echo "decode $tool rc=$?"; tail -2 gpurun_out/r02bh_sanitizer_${tool}_decode.log
done
