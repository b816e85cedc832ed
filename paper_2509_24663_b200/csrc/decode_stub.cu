#include "common.cuh"
extern "C" {
int32_t swattn_kcache_append(const swattn_config *, const swattn_paged_kv *, const int32_t *,
                             int32_t, void *) {
  swattn::set_error("decode path not built yet");
  return SWATTN_EUNSUPPORTED;
}
int32_t swattn_decode_step(const swattn_config *, const swattn_paged_kv *, const void *, int32_t,
                           void *, float *, int32_t *, void *, size_t, void *) {
  swattn::set_error("decode path not built yet");
  return SWATTN_EUNSUPPORTED;
}
size_t swattn_decode_workspace_bytes(const swattn_config *, int32_t, int32_t) { return 0; }
}
