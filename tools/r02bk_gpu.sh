for r in 1 2 3; do for v in prev cur; do SWATTN_B200_LIB=$PWD/variants/$v.so timeout 300 python tools/fa_time.py; done; done
