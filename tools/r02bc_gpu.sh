for r in 1 2; do
  for v in nopoly poly8 poly4 poly3; do SWATTN_B200_LIB=$PWD/variants/$v.so timeout 300 python tools/fa_time.py; done
done
SWATTN_B200_LIB=$PWD/variants/poly4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or large_logits or sparse_attention or all_rows" 2>&1 | tail -2
