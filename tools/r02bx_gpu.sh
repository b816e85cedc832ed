for n in 16384 131072; do for r in 1 2; do for v in prev k3one; do N=$n SWATTN_B200_LIB=$PWD/variants/$v.so timeout 300 python tools/k3_ab.py; done; done; done
SWATTN_B200_LIB=$PWD/variants/k3one.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk_kernel --csv python tools/one_attend.py 131072 2>/dev/null | grep topk | tail -1 | awk -F'","' '{print "k3one topk ns", $NF}'
SWATTN_B200_LIB=$PWD/variants/k3one.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "selection or full_size or tied" 2>&1 | tail -2
