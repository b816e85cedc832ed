for r in 1 2 3; do
  SWATTN_B200_LIB=$PWD/variants/pre_route.so python tools/e2e_time.py
  python tools/e2e_time.py
done
