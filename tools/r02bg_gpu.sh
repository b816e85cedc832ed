for r in 1 2; do for c in 16 8 6 12 24; do SWATTN_HOST_CHUNKS=$c python tools/e2e_time.py | sed "s/^/chunks=$c /"; done; done
