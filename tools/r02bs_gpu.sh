for r in 1 2; do for v in fa2base fa2poly16 fa2poly8 fa2poly4; do SWATTN_B200_LIB=$PWD/variants/$v.so NS=4096,32768,131072 timeout 300 python tools/fa2_ab.py | sed "s/^/$v /"; done; done
