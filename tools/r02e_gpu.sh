export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 120 ./tools/mcast_bench > gpurun_out/r02e_mcast.txt 2>&1; echo "mcast rc=$?"; cat gpurun_out/r02e_mcast.txt
timeout 900 python tools/diag_mismatch.py > gpurun_out/r02e_diag.txt 2>&1; echo "diag rc=$?"; cat gpurun_out/r02e_diag.txt | tail -40
