mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/one_attend.py 8192 > gpurun_out/r02bj_sanitizer_synccheck_attend8192.log 2>&1; echo "attend synccheck rc=$?"; tail -2 gpurun_out/r02bj_sanitizer_synccheck_attend8192.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/one_attend.py 4096 dense > gpurun_out/r02bj_sanitizer_synccheck_dense4096.log 2>&1; echo "dense synccheck rc=$?"; tail -2 gpurun_out/r02bj_sanitizer_synccheck_dense4096.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/one_attend.py 8192 > gpurun_out/r02bj_sanitizer_racecheck_attend8192.log 2>&1; echo "attend racecheck rc=$?"; tail -1 gpurun_out/r02bj_sanitizer_racecheck_attend8192.log
timeout 300 python tools/fa_time.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_model.py tests/test_gpu_general.py -q -x 2>&1 | tail -2
