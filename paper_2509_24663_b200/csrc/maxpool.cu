// Generic max-pool of S^shared columns (compression.py:160-173) for the
// any-profile selection path: block j = max over columns [j*s, min(j*s+l, m)).
#include "common.cuh"

namespace swattn {

namespace {

__global__ void maxpool_kernel(const float *__restrict__ shared, int64_t n, int h_kv, int64_t m1,
                               int l, int s, int64_t n_cols, float *__restrict__ s_cmp,
                               int64_t ld) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)h_kv * n * n_cols) return;
  const int64_t j = t % n_cols;
  const int64_t i = (t / n_cols) % n;
  const int g = (int)(t / (n_cols * n));
  const float *row = shared + (i * h_kv + g) * m1;
  float mx = -INFINITY;
  for (int e = 0; e < l; ++e) {
    const int64_t c = j * s + e;
    if (c >= m1) break;
    mx = fmaxf(mx, row[c]);
  }
  s_cmp[((int64_t)g * n + i) * ld + j] = mx;
}

}  // namespace

int32_t launch_maxpool(const swattn_config *cfg, const float *shared, int64_t n, float *s_cmp,
                       int64_t ld, cudaStream_t stream) {
  const int64_t m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  const int64_t n_cols = m1 ? cdiv(m1, cfg->s) : 0;
  const int64_t total = (int64_t)cfg->h_kv * n * n_cols;
  if (total == 0) return SWATTN_OK;
  maxpool_kernel<<<(unsigned)cdiv(total, 256), 256, 0, stream>>>(shared, n, cfg->h_kv, m1, cfg->l,
                                                                 cfg->s, n_cols, s_cmp, ld);
  SWATTN_LAUNCH_CHECK("maxpool_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
