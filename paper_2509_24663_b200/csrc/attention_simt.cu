// K4/K5 (portable CUDA-core form): block-sparse and dense GQA attention
// forward with the online max/sum recurrence of dense.py:140-165 /
// sparse.py:70-91.  One warp per (query token, head), one CTA per
// (token, KV group) so the 16 heads of a group share the visible-key list.
// Baseline / fallback for the tensor-core kernels in attention_tc.cu.
#include "common.cuh"

namespace swattn {

namespace {

constexpr int kMaxBlocks = 512;  // visible-block list bound (dense path walks ranges)

struct AttnArgs {
  const __nv_bfloat16 *Q, *K, *V;
  int64_t n;
  int h_q, h_kv, G;
  int B, N_init, N_local, k_top;
  const int32_t *topk, *topk_cnt;  // sparse only
  int sparse, causal;
  float scale_log2;
  __nv_bfloat16 *O;
  float *lse;
  int *err;
};

// one warp: fold keys [k0, k1) into (m, l, acc) -- log2 domain
__device__ __forceinline__ void fold_range(const AttnArgs &a, const float *q_s, int g, int64_t k0,
                                           int64_t k1, float &m, float &l, float (&acc)[4]) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = k0; base < k1; base += 32) {
    const int64_t key = base + lane;
    float s = -INFINITY;
    if (key < k1) {
      const uint4 *kr = reinterpret_cast<const uint4 *>(a.K + (key * a.h_kv + g) * kD);
      float d0 = 0.f, d1 = 0.f;
#pragma unroll 4
      for (int t = 0; t < kD / 8; ++t) {
        const uint4 raw = __ldg(kr + t);
        const __nv_bfloat162 *p2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(p2[e]);
          d0 = fmaf(q_s[t * 8 + 2 * e], f.x, d0);
          d1 = fmaf(q_s[t * 8 + 2 * e + 1], f.y, d1);
        }
      }
      s = (d0 + d1) * a.scale_log2;
    }
    float cmax = s;
    for (int o = 16; o; o >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    const float m_new = fmaxf(m, cmax);
    const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - m_new);
    const float p = (key < k1) ? fast_exp2(s - m_new) : 0.f;
    float psum = p;
    for (int o = 16; o; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
    l = l * alpha + psum;
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e] *= alpha;
    const int cnt = (int)min((int64_t)32, k1 - base);
    for (int kk = 0; kk < cnt; ++kk) {
      const float pk = __shfl_sync(0xffffffffu, p, kk);
      const uint2 raw = __ldg(reinterpret_cast<const uint2 *>(a.V + ((base + kk) * a.h_kv + g) * kD + lane * 4));
      const __nv_bfloat162 *v2 = reinterpret_cast<const __nv_bfloat162 *>(&raw);
      const float2 f0 = __bfloat1622float2(v2[0]), f1 = __bfloat1622float2(v2[1]);
      acc[0] = fmaf(pk, f0.x, acc[0]);
      acc[1] = fmaf(pk, f0.y, acc[1]);
      acc[2] = fmaf(pk, f1.x, acc[2]);
      acc[3] = fmaf(pk, f1.y, acc[3]);
    }
    m = m_new;
  }
}

__device__ void attend_row(const AttnArgs &a, int64_t i, int g) {
  __shared__ float q_all[kG][kD];
  __shared__ int blocks_s[kMaxBlocks];
  __shared__ int nblocks_s;
  __syncthreads();  // smem reuse across rows of a persistent loop
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hq = g * a.G + warp;
  for (int t = threadIdx.x; t < kG * kD; t += blockDim.x)
    q_all[t / kD][t % kD] = bf2f(a.Q[(i * a.h_q + g * a.G) * kD + t]);
  if (a.sparse && threadIdx.x == 0) {
    const int b = (int)(i / a.B);
    const int n_init = min(a.N_init, b + 1);
    const int lo = max(0, b - a.N_local + 1);
    int c = 0;
    for (int j = 0; j < n_init; ++j) blocks_s[c++] = j;
    const int tc = a.topk_cnt[(int64_t)g * a.n + i];
    const int32_t *tr = a.topk + ((int64_t)g * a.n + i) * a.k_top;
    for (int t = 0; t < tc; ++t) blocks_s[c++] = tr[t];
    for (int j = max(lo, n_init); j <= b; ++j) blocks_s[c++] = j;
    nblocks_s = c;
  }
  __syncthreads();
  float m = -INFINITY, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  const float *q_s = q_all[warp];
  if (a.sparse) {
    const int nb = nblocks_s;
    for (int t = 0; t < nb; ++t) {
      const int64_t k0 = (int64_t)blocks_s[t] * a.B;
      const int64_t k1 = min(min(k0 + a.B, a.n), i + 1);
      if (k1 > k0) fold_range(a, q_s, g, k0, k1, m, l, acc);
    }
  } else {
    fold_range(a, q_s, g, 0, a.causal ? i + 1 : a.n, m, l, acc);
  }
  if (l == 0.f) {
    if (lane == 0 && a.err != nullptr) atomicExch(a.err, 1);
    l = 1.f;  // empty visible set: flagged; keep the warp in lock-step
  }
  const float inv = 1.f / l;
  __nv_bfloat16 *o = a.O + (i * a.h_q + hq) * kD + lane * 4;
  __align__(8) __nv_bfloat16 ov[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) ov[e] = __float2bfloat16_rn(acc[e] * inv);
  *reinterpret_cast<uint2 *>(o) = *reinterpret_cast<const uint2 *>(ov);
  if (lane == 0) a.lse[i * a.h_q + hq] = (m + __log2f(l)) * 0.6931471805599453f;
}

__global__ void __launch_bounds__(kG * 32) attention_rows_kernel(AttnArgs a) {
  attend_row(a, blockIdx.x, blockIdx.y);
}

// exact recomputation of listed (group, token) rows (g * n + i)
__global__ void __launch_bounds__(kG * 32) attention_list_kernel(AttnArgs a, const int32_t *count,
                                                                 const int32_t *list) {
  const int total = *count;
  for (int e = blockIdx.x; e < total; e += gridDim.x) {
    const int32_t row = list[e];
    attend_row(a, row % a.n, (int)(row / a.n));
  }
}

}  // namespace

int32_t launch_attention_list(const swattn_config *cfg, const void *Q, const void *K,
                              const void *V, int64_t n, const int32_t *topk,
                              const int32_t *topk_cnt, const int32_t *count, const int32_t *list,
                              void *O, float *lse, int grid, cudaStream_t stream) {
  AttnArgs a;
  a.Q = static_cast<const __nv_bfloat16 *>(Q);
  a.K = static_cast<const __nv_bfloat16 *>(K);
  a.V = static_cast<const __nv_bfloat16 *>(V);
  a.n = n;
  a.h_q = cfg->h_q;
  a.h_kv = cfg->h_kv;
  a.G = cfg->h_q / cfg->h_kv;
  a.B = cfg->B;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.k_top = cfg->k_top;
  a.topk = topk;
  a.topk_cnt = topk_cnt;
  a.sparse = 1;
  a.causal = 1;
  a.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  a.O = static_cast<__nv_bfloat16 *>(O);
  a.lse = lse;
  a.err = nullptr;
  attention_list_kernel<<<grid, kG * 32, 0, stream>>>(a, count, list);
  SWATTN_LAUNCH_CHECK("attention_list_kernel");
  return SWATTN_OK;
}

int32_t launch_attention_simt(const swattn_config *cfg, const void *Q, const void *K,
                              const void *V, int64_t n, const int32_t *topk,
                              const int32_t *topk_cnt, int sparse, int causal, void *O, float *lse,
                              int *err_flag, cudaStream_t stream) {
  AttnArgs a;
  a.Q = static_cast<const __nv_bfloat16 *>(Q);
  a.K = static_cast<const __nv_bfloat16 *>(K);
  a.V = static_cast<const __nv_bfloat16 *>(V);
  a.n = n;
  a.h_q = cfg->h_q;
  a.h_kv = cfg->h_kv;
  a.G = cfg->h_q / cfg->h_kv;
  a.B = cfg->B;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.k_top = cfg->k_top;
  a.topk = topk;
  a.topk_cnt = topk_cnt;
  a.sparse = sparse;
  a.causal = causal;
  a.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  a.O = static_cast<__nv_bfloat16 *>(O);
  a.lse = lse;
  a.err = err_flag;
  if (sparse && cfg->N_init + cfg->N_local + cfg->k_top > kMaxBlocks) {
    set_error("unsupported: block budget exceeds %d", kMaxBlocks);
    return SWATTN_EUNSUPPORTED;
  }
  dim3 grid((unsigned)n, (unsigned)cfg->h_kv);
  attention_rows_kernel<<<grid, kG * 32, 0, stream>>>(a);
  SWATTN_LAUNCH_CHECK("attention_rows_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
