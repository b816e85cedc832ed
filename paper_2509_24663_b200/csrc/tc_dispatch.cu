// Tensor-core kernel availability switches.  The tcgen05 kernels register
// themselves here; until a kernel is compiled in, the C ABI routes to the
// CUDA-core forms.
#include "common.cuh"

namespace swattn {

bool scores_tc_available() { return false; }
bool attention_tc_available() { return false; }

int32_t launch_scores_tc(const swattn_config *, const void *, const void *, const void *, int64_t,
                         int32_t, float *, int64_t, uint64_t *, int64_t, cudaStream_t) {
  set_error("tcgen05 scoring kernel not built");
  return SWATTN_EUNSUPPORTED;
}
int32_t launch_sparse_tc(const swattn_config *, const void *, const void *, const void *, int64_t,
                         const int32_t *, const int32_t *, void *, float *, cudaStream_t) {
  set_error("tcgen05 sparse attention kernel not built");
  return SWATTN_EUNSUPPORTED;
}
int32_t launch_dense_tc(const swattn_config *, const void *, const void *, const void *, int64_t,
                        int, void *, float *, cudaStream_t) {
  set_error("tcgen05 dense attention kernel not built");
  return SWATTN_EUNSUPPORTED;
}

}  // namespace swattn
