SWATTN_B200_LIB=$PWD/variants/split.so NS=1000,4096,32768 timeout 300 python tools/fa2_check.py 2>&1 | cut -c1-200
for r in 1 2; do for v in base split; do SWATTN_B200_LIB=$PWD/variants/$v.so NS=4096,32768,131072 timeout 300 python tools/fa2_ab.py | sed "s/^/$v /"; done; done
