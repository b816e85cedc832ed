for n in 16384 131072; do for r in 1 2; do for v in prev k3nch; do N=$n SWATTN_B200_LIB=$PWD/variants/$v.so timeout 300 python tools/k3_ab.py; done; done; done
SWATTN_B200_LIB=$PWD/variants/k3nch.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk_kernel --csv python tools/one_attend.py 131072 2>/dev/null | grep topk | tail -1 | awk -F'","' '{print "k3nch topk ns", $NF}'
