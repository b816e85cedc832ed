for r in 1 2 3; do
  SWATTN_B200_LIB=$PWD/variants/base.so timeout 300 python tools/fa_time.py
  timeout 300 python tools/fa_time.py
done
