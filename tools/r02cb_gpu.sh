for n in 16384 131072; do for r in 1 2 3; do for v in prev k2db; do N=$n SWATTN_B200_LIB=$PWD/variants/$v.so timeout 300 python tools/k2_ab.py; done; done; done
