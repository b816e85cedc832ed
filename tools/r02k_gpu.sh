#!/bin/bash
# r02i: full ncu captures of the decode kernels (pass 2, top-k, attention, rerank)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_pass2|decode_topk_cta|decode_attn|rerank|decode_pass1|decode_combine" -c 8 -f -o gpurun_out/r02k_decode_full python tools/bench_decode.py --steps 1 --warmup 1 > gpurun_out/r02k_decode_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r02k_decode_full.log
