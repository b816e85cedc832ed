// K2 (portable CUDA-core form) -- fused two-pass block scoring.
//
//  * scores_rows_kernel: the compiled paper profile (G=16, d=128, l=5, s=4),
//    CTA = 16 query tokens x 16 heads of one KV group, one thread per
//    (token, head) row.  Pass 1 streams the online log-sum-exp over the
//    visible normaliser columns (C2 for approx, C1 for exact;
//    selection.py:165-196), pass 2 recomputes the C1 logits of the top-k
//    candidate tiles, normalises with that lse, sums the 16 heads of a token
//    with warp shuffles (selection.py:199-222) and max-pools 5/4 into
//    S^cmp (compression.py:160-173).  This is the CUDA-core baseline the
//    tcgen05 kernel (scores_tc.cu) replaces; it also serves shapes the
//    tensor-core kernel does not tile.
//  * shared_* kernels: any profile, full S^shared for the parity/debug API
//    (fused_shared_scores_{exact,approx}), including the fallback rows
//    (selection.py:303-324).
#include "common.cuh"

namespace swattn {

namespace {

constexpr int kTok = 16;               // tokens per CTA
constexpr int kThreads = kTok * kG;    // 256
constexpr int kChunk = 64;             // normaliser columns staged per step
constexpr int kTileCols = 128;         // C1 columns per pass-2 tile
constexpr int kTileBlocks = 31;        // blocks per tile (tile stride 124 cols)

struct ScoreArgs {
  const __nv_bfloat16 *Q, *kc1, *kc2;
  int64_t n, m1, m2;
  int h_q, h_kv;
  int l_C1, s_C1, l_C2, s_C2;
  int N_init, N_local, B, n_cols;
  int approx;
  float scale_log2;   // logit scale * log2(e)
  float *s_cmp;
  int64_t ld;
  uint64_t *flags;
  int64_t ld_f;
  int64_t tok0;       // first token handled
};

__device__ __forceinline__ float dot_q_k(const uint32_t (&q)[kD / 2], const __nv_bfloat16 *k_s) {
  const __nv_bfloat162 *k2 = reinterpret_cast<const __nv_bfloat162 *>(k_s);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int t = 0; t < kD / 2; ++t) {
    const float2 kf = __bfloat1622float2(k2[t]);
    a0 = fmaf(__uint_as_float(q[t] << 16), kf.x, a0);
    a1 = fmaf(__uint_as_float(q[t] & 0xffff0000u), kf.y, a1);
  }
  return a0 + a1;
}

__global__ void __launch_bounds__(kThreads) scores_rows_kernel(ScoreArgs a) {
  __shared__ __align__(16) __nv_bfloat16 k_s[kTileCols][kD];   // 32 KB
  __shared__ float sc[kTok][kTileCols + 4];
  __shared__ unsigned long long fl[kTok];

  const int g = blockIdx.y;
  const int tok = threadIdx.x / kG, h = threadIdx.x % kG;
  const int64_t i0 = a.tok0 + (int64_t)blockIdx.x * kTok;
  const int64_t i = i0 + tok;
  const bool valid = i < a.n;
  const int64_t ii = valid ? i : a.n - 1;

  uint32_t q[kD / 2];
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(a.Q + (ii * a.h_q + g * kG + h) * kD);
#pragma unroll
    for (int t = 0; t < kD / 8; ++t) {
      const uint4 v = __ldg(src + t);
      q[4 * t] = v.x; q[4 * t + 1] = v.y; q[4 * t + 2] = v.z; q[4 * t + 3] = v.w;
    }
  }

  // ---------------- pass 1: online lse (log2 domain) over normaliser columns
  const int64_t vis1 = vis_count(ii, a.l_C1, a.s_C1);
  const int64_t vis2 = a.approx ? vis_count(ii, a.l_C2, a.s_C2) : 0;
  const bool use_c2 = a.approx && vis2 > 0;
  const int64_t vis = valid ? (use_c2 ? vis2 : vis1) : 0;
  // all rows of the CTA share the normaliser key set choice in the compiled
  // profile (tokens >= tok0 always see C2); fall back per row otherwise.
  const __nv_bfloat16 *kc = use_c2 ? a.kc2 : a.kc1;
  // vis is monotone in the row index: the CTA's last valid token bounds it
  const int64_t i_last = min(i0 + kTok - 1, a.n - 1);
  const int64_t vmax = use_c2 ? vis_count(i_last, a.l_C2, a.s_C2) : vis_count(i_last, a.l_C1, a.s_C1);
  float m = -INFINITY, l = 0.f;
  for (int64_t c0 = 0; c0 < vmax; c0 += kChunk) {
    __syncthreads();
    for (int t = threadIdx.x; t < kChunk * (kD / 8); t += kThreads) {
      const int c = t / (kD / 8), v = t % (kD / 8);
      uint4 val = make_uint4(0, 0, 0, 0);
      if (c0 + c < vmax) val = __ldg(reinterpret_cast<const uint4 *>(kc + ((c0 + c) * a.h_kv + g) * kD) + v);
      reinterpret_cast<uint4 *>(&k_s[c][0])[v] = val;
    }
    __syncthreads();
    const int cend = (int)min((int64_t)kChunk, vis - c0);
    for (int c = 0; c < cend; ++c) {
      const float s = dot_q_k(q, k_s[c]) * a.scale_log2;
      if (s > m) { l = l * fast_exp2(m - s) + 1.f; m = s; }
      else l += fast_exp2(s - m);
    }
  }
  // p = exp2(s - m) / l  ==  exp(logit - lse)
  const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
  const float m_safe = (m == -INFINITY) ? 0.f : m;

  // ---------------- pass 2: candidate tiles of C1 columns
  const int b = (int)(i0 / a.B);  // all 16 tokens share the query block
  const int hi = cand_hi(b, a.N_local, a.n_cols);
  const int n_tiles = hi > a.N_init ? (hi + kTileBlocks - 1) / kTileBlocks : 0;
  for (int t = 0; t < n_tiles; ++t) {
    const int64_t c0 = (int64_t)t * kTileBlocks * kPoolS;
    __syncthreads();
    for (int x = threadIdx.x; x < kTileCols * (kD / 8); x += kThreads) {
      const int c = x / (kD / 8), v = x % (kD / 8);
      uint4 val = make_uint4(0, 0, 0, 0);
      if (c0 + c < a.m1) val = __ldg(reinterpret_cast<const uint4 *>(a.kc1 + ((c0 + c) * a.h_kv + g) * kD) + v);
      reinterpret_cast<uint4 *>(&k_s[c][0])[v] = val;
    }
    if (threadIdx.x < kTok) fl[threadIdx.x] = 0ull;
    __syncthreads();
    for (int c = 0; c < kTileCols; ++c) {
      const int64_t col = c0 + c;
      float p = 0.f;
      if (col < vis1 && valid) p = fast_exp2(dot_q_k(q, k_s[c]) * a.scale_log2 - m_safe) * inv_l;
      p += __shfl_xor_sync(0xffffffffu, p, 8);
      p += __shfl_xor_sync(0xffffffffu, p, 4);
      p += __shfl_xor_sync(0xffffffffu, p, 2);
      p += __shfl_xor_sync(0xffffffffu, p, 1);
      if (h == 0) sc[tok][c] = (col < a.m1) ? p : -INFINITY;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < kTok * kTileBlocks; o += kThreads) {
      const int tk = o / kTileBlocks, qb = o % kTileBlocks;
      const int j = t * kTileBlocks + qb;
      const int64_t row_i = i0 + tk;
      if (row_i >= a.n || j < a.N_init || j >= hi) continue;
      float v[kPoolL];
#pragma unroll
      for (int e = 0; e < kPoolL; ++e) v[e] = sc[tk][qb * kPoolS + e];
      float mx = v[0];
#pragma unroll
      for (int e = 1; e < kPoolL; ++e) mx = fmaxf(mx, v[e]);
      a.s_cmp[((int64_t)g * a.n + row_i) * a.ld + j] = mx;
      if (a.flags != nullptr) {
        const float thr0 = v[0] / (1.f + 4.f * kScoreRelErr);
        const float thr4 = v[4] / (1.f + 4.f * kScoreRelErr);
        bool L = true, R = true;
#pragma unroll
        for (int e = 1; e < kPoolL; ++e) L = L && v[e] < thr0;
#pragma unroll
        for (int e = 0; e < kPoolL - 1; ++e) R = R && v[e] < thr4;
        const unsigned long long bits = ((unsigned long long)L << (2 * qb)) |
                                        ((unsigned long long)R << (2 * qb + 1));
        if (bits) atomicOr(&fl[tk], bits);
      }
    }
    __syncthreads();
    if (a.flags != nullptr && threadIdx.x < kTok && i0 + threadIdx.x < a.n)
      a.flags[((int64_t)g * a.n + i0 + threadIdx.x) * a.ld_f + t] = fl[threadIdx.x];
  }
}

// ---------------- any-profile debug path: full S^shared
// lse over the normaliser columns, one thread per (row, head); natural log.
__global__ void shared_lse_kernel(const __nv_bfloat16 *Q, const __nv_bfloat16 *kc1,
                                  const __nv_bfloat16 *kc2, int64_t n, int h_q, int h_kv,
                                  int d, int l1, int s1, int l2, int s2, int approx, int64_t m2,
                                  float scale, float *lse) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * h_q) return;
  const int64_t i = t / h_q;
  const int hq = (int)(t % h_q);
  const int g = hq / (h_q / h_kv);
  const int64_t v1 = vis_count(i, l1, s1);
  const int64_t v2 = (approx && m2 > 0) ? vis_count(i, l2, s2) : 0;
  const bool use2 = approx && v2 > 0;
  const int64_t vis = use2 ? v2 : (approx && !(v2 == 0 && v1 > 0) ? 0 : v1);
  const __nv_bfloat16 *kc = use2 ? kc2 : kc1;
  const __nv_bfloat16 *qr = Q + (i * h_q + hq) * d;
  float m = -INFINITY, l = 0.f;
  for (int64_t c = 0; c < vis; ++c) {
    const __nv_bfloat16 *kr = kc + (c * h_kv + g) * d;
    float s = 0.f;
    for (int e = 0; e < d; ++e) s = fmaf(bf2f(qr[e]), bf2f(kr[e]), s);
    s *= scale;
    if (s > m) { l = l * expf(m - s) + 1.f; m = s; } else l += expf(s - m);
  }
  lse[t] = (m == -INFINITY) ? 0.f : m + logf(l);  // lse_safe (selection.py:204)
}

__global__ void shared_pass2_kernel(const __nv_bfloat16 *Q, const __nv_bfloat16 *kc1, int64_t n,
                                    int h_q, int h_kv, int d, int l1, int s1, int64_t m1,
                                    float scale, const float *lse, float *shared,
                                    uint8_t *no_visible) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * h_kv * m1) return;
  const int64_t c = t % m1;
  const int g = (int)((t / m1) % h_kv);
  const int64_t i = t / (m1 * h_kv);
  const int64_t v1 = vis_count(i, l1, s1);
  if (no_visible != nullptr && c == 0 && g == 0) no_visible[i] = v1 == 0;
  float acc = 0.f;
  if (c < v1) {
    const int G = h_q / h_kv;
    const __nv_bfloat16 *kr = kc1 + (c * h_kv + g) * d;
    for (int hh = 0; hh < G; ++hh) {
      const int hq = g * G + hh;
      const __nv_bfloat16 *qr = Q + (i * h_q + hq) * d;
      float s = 0.f;
      for (int e = 0; e < d; ++e) s = fmaf(bf2f(qr[e]), bf2f(kr[e]), s);
      acc += expf(s * scale - lse[i * h_q + hq]);
    }
  }
  shared[t] = acc;
}

}  // namespace

int32_t launch_scores_simt(const swattn_config *cfg, const void *Q, const void *kc1,
                           const void *kc2, int64_t n, int32_t mode, float *s_cmp, int64_t ld,
                           uint64_t *flags, int64_t ld_f, cudaStream_t stream) {
  ScoreArgs a;
  a.Q = static_cast<const __nv_bfloat16 *>(Q);
  a.kc1 = static_cast<const __nv_bfloat16 *>(kc1);
  a.kc2 = static_cast<const __nv_bfloat16 *>(kc2);
  a.n = n;
  a.m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  a.m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  a.h_q = cfg->h_q;
  a.h_kv = cfg->h_kv;
  a.l_C1 = cfg->l_C1; a.s_C1 = cfg->s_C1; a.l_C2 = cfg->l_C2; a.s_C2 = cfg->s_C2;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.B = cfg->B;
  a.n_cols = (int)(a.m1 ? cdiv(a.m1, cfg->s) : 0);
  a.approx = mode == SWATTN_SELECT_APPROX;
  const float scale = cfg->scale_compressed_logits ? 1.f / sqrtf((float)cfg->d_h) : 1.f;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.s_cmp = s_cmp;
  a.ld = ld;
  a.flags = flags;
  a.ld_f = ld_f;
  // rows below the first candidate-bearing query block select no top-k
  a.tok0 = (int64_t)(cfg->N_init + cfg->N_local) * cfg->B;
  if (a.tok0 >= n || a.n_cols <= cfg->N_init) return SWATTN_OK;
  const int64_t tiles = cdiv(n - a.tok0, kTok);
  dim3 grid((unsigned)tiles, (unsigned)cfg->h_kv);
  scores_rows_kernel<<<grid, kThreads, 0, stream>>>(a);
  SWATTN_LAUNCH_CHECK("scores_rows_kernel");
  return SWATTN_OK;
}

int32_t launch_shared_scores(const swattn_config *cfg, const void *Q, const void *kc1,
                             const void *kc2, int64_t n, int32_t mode, float *shared,
                             uint8_t *no_visible, float *lse_ws, cudaStream_t stream) {
  const int64_t m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  const int64_t m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  const float scale = cfg->scale_compressed_logits ? 1.f / sqrtf((float)cfg->d_h) : 1.f;
  const int approx = mode == SWATTN_SELECT_APPROX;
  auto Qp = static_cast<const __nv_bfloat16 *>(Q);
  auto k1 = static_cast<const __nv_bfloat16 *>(kc1);
  auto k2 = static_cast<const __nv_bfloat16 *>(kc2);
  const int64_t t1 = n * cfg->h_q;
  shared_lse_kernel<<<(unsigned)cdiv(t1, 128), 128, 0, stream>>>(
      Qp, k1, k2, n, cfg->h_q, cfg->h_kv, cfg->d_h, cfg->l_C1, cfg->s_C1, cfg->l_C2, cfg->s_C2,
      approx, m2, scale, lse_ws);
  SWATTN_LAUNCH_CHECK("shared_lse_kernel");
  const int64_t t2 = n * cfg->h_kv * m1;
  if (t2 > 0) {
    shared_pass2_kernel<<<(unsigned)cdiv(t2, 128), 128, 0, stream>>>(
        Qp, k1, n, cfg->h_q, cfg->h_kv, cfg->d_h, cfg->l_C1, cfg->s_C1, m1, scale, lse_ws, shared,
        no_visible);
    SWATTN_LAUNCH_CHECK("shared_pass2_kernel");
  } else if (no_visible != nullptr) {
    cudaMemsetAsync(no_visible, 1, (size_t)n, stream);
  }
  return SWATTN_OK;
}

}  // namespace swattn
