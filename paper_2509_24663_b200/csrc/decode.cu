// K6 -- decode over a paged KV cache.  No reference symbol: the semantics are
// row t = L-1 of select_blocks(approx) + sparse_forward on the first L tokens
// (selection.py:93-136,165-222,279-348; sparse.py:43-98).
//
// Cache layout: pages of B = 64 tokens, k_pages / v_pages [num_pages][64][h_kv][d]
// bf16 (token-major inside a page, like the prefill tensors), block_table
// [batch][max_pages]; compressed keys per sequence kc1 [batch][max_m1][h_kv][d],
// kc2 [batch][max_m2][h_kv][d], appended incrementally as windows complete.
//
// One step, per (sequence, KV group) row -- all split across CTAs so that a
// batch of 16 fills the GPU, HBM-bound:
//   D1 kcache_append    new C1 / C2 entries (exact float64 window sums);
//   D2 pass 1           split over C2 columns: partial (max, sum) per head;
//   D3 pass 2           combine the partials -> lse, then per 124-column
//                       tile: 16-head sum of exp(logit - lse), 5/4 max-pool
//                       -> S^cmp row segment;
//   D4 top-k            decode_topk_kernel (topk.cu) + float64 re-rank of
//                       ambiguous rows (rerank.cu);
//   D5 attention        split-KV over <= 96 visible blocks, then combine.
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace swattn {

int32_t launch_decode_topk(const swattn_config *, const float *, int64_t, const int32_t *, int, int,
                           int32_t *, int32_t *, int32_t *, int32_t *, int32_t, cudaStream_t);
int32_t launch_rerank_decode(const swattn_config *, const void *, const void *, const void *,
                             int max_m1, int max_m2, const int32_t *seq_lens, int batch,
                             const float *, int64_t, const int32_t *, const int32_t *, int32_t,
                             int32_t *, int, cudaStream_t);

namespace {

constexpr int kP1Cols = 256;     // C2 columns per pass-1 CTA
constexpr int kTileBlocks = 31;  // pass-2 tile: 31 blocks, 124 (+4) columns
constexpr int kTileCols = 128;
constexpr int kAttnBlocks = 8;   // visible blocks per split-KV CTA
constexpr int kMaxSplits = 16;

struct DecodeArgs {
  const __nv_bfloat16 *q;            // [batch][h_q][d]
  const __nv_bfloat16 *k_pages, *v_pages;
  const int32_t *block_table, *seq_lens;
  int max_pages;
  const __nv_bfloat16 *kc1, *kc2;
  int max_m1, max_m2;
  int batch, h_q, h_kv;
  int l_C1, s_C1, l_C2, s_C2, B, N_init, N_local, k_top;
  float scale_log2;   // compressed-logit scale * log2(e)
  float attn_scale_log2;
};

__device__ __forceinline__ const __nv_bfloat16 *page_row(const __nv_bfloat16 *pages,
                                                         const int32_t *bt, int max_pages, int seq,
                                                         int64_t token, int h_kv, int g) {
  const int page = bt[(int64_t)seq * max_pages + token / kB];
  return pages + (((int64_t)page * kB + token % kB) * h_kv + g) * kD;
}

// dot of a q row held in smem (fp32) with a bf16 row in global memory
__device__ __forceinline__ float dot_row(const float *q, const __nv_bfloat16 *k) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
  for (int d = 0; d < kD; d += 8) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4 *>(k + d));
    const __nv_bfloat162 *v = reinterpret_cast<const __nv_bfloat162 *>(&raw);
    const float2 f0 = __bfloat1622float2(v[0]), f1 = __bfloat1622float2(v[1]);
    const float2 f2 = __bfloat1622float2(v[2]), f3 = __bfloat1622float2(v[3]);
    a0 = fmaf(q[d], f0.x, a0);
    a1 = fmaf(q[d + 1], f0.y, a1);
    a2 = fmaf(q[d + 2], f1.x, a2);
    a3 = fmaf(q[d + 3], f1.y, a3);
    a0 = fmaf(q[d + 4], f2.x, a0);
    a1 = fmaf(q[d + 5], f2.y, a1);
    a2 = fmaf(q[d + 6], f3.x, a2);
    a3 = fmaf(q[d + 7], f3.y, a3);
  }
  return (a0 + a1) + (a2 + a3);
}

// ------------------------------------------------------------ D1 append
// grid (batch, h_kv), 128 threads = d; new windows are few per step.
__global__ void kcache_append_kernel(DecodeArgs a, const int32_t *prev_lens) {
  const int seq = blockIdx.x, g = blockIdx.y, d = threadIdx.x;
  const int64_t L = a.seq_lens[seq], L0 = prev_lens ? prev_lens[seq] : 0;
  for (int which = 0; which < 2; ++which) {
    const int len = which ? a.l_C2 : a.l_C1, str = which ? a.s_C2 : a.s_C1;
    const int max_m = which ? a.max_m2 : a.max_m1;
    __nv_bfloat16 *dst = const_cast<__nv_bfloat16 *>(which ? a.kc2 : a.kc1) +
                         (int64_t)seq * max_m * a.h_kv * kD;
    const int64_t j0 = num_pooled(L0, len, str), j1 = min(num_pooled(L, len, str), (int64_t)max_m);
    for (int64_t j = j0; j < j1; ++j) {
      double s = 0.0;
      for (int r = 0; r < len; ++r)
        s += (double)bf2f(page_row(a.k_pages, a.block_table, a.max_pages, seq, j * str + r, a.h_kv,
                                   g)[d]);
      dst[(j * a.h_kv + g) * kD + d] = __float2bfloat16_rn(__double2float_rn(s / (double)len));
    }
  }
}

// ------------------------------------------------------------ D2 pass 1
// grid (batch*h_kv, splits), 256 threads: thread = C2 column, 16 heads each.
__global__ void __launch_bounds__(256) decode_pass1_kernel(DecodeArgs a, float2 *part, int splits) {
  __shared__ float q_s[kG][kD];
  __shared__ float2 red[8][kG];
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t vis2 = vis_count(L - 1, a.l_C2, a.s_C2);
  const int64_t vis1 = vis_count(L - 1, a.l_C1, a.s_C1);
  const bool use2 = vis2 > 0;
  const int64_t vis = use2 ? vis2 : vis1;  // fallback rows use the exact C1 lse
  const __nv_bfloat16 *kc = (use2 ? a.kc2 : a.kc1) + (int64_t)seq * (use2 ? a.max_m2 : a.max_m1) * a.h_kv * kD;
  for (int t = threadIdx.x; t < kG * kD; t += blockDim.x)
    q_s[t / kD][t % kD] = bf2f(a.q[((int64_t)seq * a.h_q + g * kG) * kD + t]);
  __syncthreads();
  float m[kG], l[kG];
#pragma unroll
  for (int h = 0; h < kG; ++h) { m[h] = -INFINITY; l[h] = 0.f; }
  const int64_t c = (int64_t)blockIdx.y * kP1Cols + threadIdx.x;
  if (c < vis) {
    const __nv_bfloat16 *kr = kc + (c * a.h_kv + g) * kD;
#pragma unroll
    for (int h = 0; h < kG; ++h) {
      m[h] = dot_row(q_s[h], kr) * a.scale_log2;
      l[h] = 1.f;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < kG; ++h) {
    float M = m[h];
    for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float S = (m[h] == -INFINITY) ? 0.f : l[h] * fast_exp2(m[h] - M);
    for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    if (lane == 0) red[warp][h] = make_float2(M, S);
  }
  __syncthreads();
  if (threadIdx.x < kG) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 8; ++w) M = fmaxf(M, red[w][h].x);
    float S = 0.f;
    for (int w = 0; w < 8; ++w)
      if (red[w][h].x != -INFINITY) S += red[w][h].y * fast_exp2(red[w][h].x - M);
    part[((int64_t)row * splits + blockIdx.y) * kG + h] = make_float2(M, S);
  }
}

// ------------------------------------------------------------ D3 pass 2
// grid (batch*h_kv, tiles), 128 threads: thread = C1 column of the tile.
__global__ void __launch_bounds__(128) decode_pass2_kernel(DecodeArgs a, const float2 *part,
                                                           int splits, float *s_cmp, int64_t ld) {
  __shared__ float q_s[kG][kD];
  __shared__ float2 stat[kG];  // (m, 1/l), log2 domain
  __shared__ float sc[kTileCols + 4];
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t i = L - 1;
  const int64_t m1 = num_pooled(L, a.l_C1, a.s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, kPoolS) : 0);
  const int hi = cand_hi((int)(i / a.B), a.N_local, n_cols);
  const int t = blockIdx.y;
  if (t * kTileBlocks >= hi) return;
  const int64_t vis1 = vis_count(i, a.l_C1, a.s_C1);
  for (int e = threadIdx.x; e < kG * kD; e += blockDim.x)
    q_s[e / kD][e % kD] = bf2f(a.q[((int64_t)seq * a.h_q + g * kG) * kD + e]);
  if (threadIdx.x < kG) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, part[((int64_t)row * splits + sp) * kG + h].x);
    float S = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      const float2 pv = part[((int64_t)row * splits + sp) * kG + h];
      if (pv.x != -INFINITY) S += pv.y * fast_exp2(pv.x - M);
    }
    stat[h] = make_float2(M == -INFINITY ? 0.f : M, S > 0.f ? 1.f / S : 0.f);
  }
  __syncthreads();
  const int64_t col = (int64_t)t * kTileBlocks * kPoolS + threadIdx.x;
  float v = -INFINITY;
  if (col < m1) {
    v = 0.f;
    if (col < vis1) {
      const __nv_bfloat16 *kr = a.kc1 + (((int64_t)seq * a.max_m1 + col) * a.h_kv + g) * kD;
      float acc = 0.f;
#pragma unroll
      for (int h = 0; h < kG; ++h)
        acc = fmaf(fast_exp2(dot_row(q_s[h], kr) * a.scale_log2 - stat[h].x), stat[h].y, acc);
      v = acc;
    }
  }
  sc[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x < kTileBlocks) {
    const int j = t * kTileBlocks + threadIdx.x;
    if (j >= a.N_init && j < hi) {
      float mx = sc[threadIdx.x * kPoolS];
#pragma unroll
      for (int e = 1; e < kPoolL; ++e) mx = fmaxf(mx, sc[threadIdx.x * kPoolS + e]);
      s_cmp[(int64_t)row * ld + j] = mx;
    }
  }
}

// ------------------------------------------------------------ D5 attention
__device__ __forceinline__ int visible_block(int idx, int n_init, int ntop, const int32_t *top,
                                             int lo2) {
  if (idx < n_init) return idx;
  idx -= n_init;
  if (idx < ntop) return top[idx];
  return lo2 + (idx - ntop);
}

// grid (batch*h_kv, splits), 256 threads (8 warps, 2 heads each)
__global__ void __launch_bounds__(256) decode_attn_kernel(DecodeArgs a, const int32_t *topk,
                                                          const int32_t *topk_cnt, float *part_o,
                                                          float2 *part_ml, int splits) {
  __shared__ float q_s[kG][kD];
  // rows padded by 16 B: lanes reading different key rows with 16-byte
  // vectors hit distinct banks
  __shared__ __align__(16) __nv_bfloat16 k_s[kB][kD + 8];
  __shared__ __align__(16) __nv_bfloat16 v_s[kB][kD + 8];
  __shared__ float p_s[kG][kB];
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t i = L - 1;
  const int b = (int)(i / kB);
  const int n_init = min(a.N_init, b + 1);
  const int lo = max(0, b - a.N_local + 1);
  const int lo2 = max(lo, n_init);
  const int ntop = topk_cnt[row];
  const int nvis = n_init + ntop + (b + 1 - lo2);
  const int32_t *top = topk + (int64_t)row * a.k_top;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < kG * kD; e += blockDim.x)
    q_s[e / kD][e % kD] = bf2f(a.q[((int64_t)seq * a.h_q + g * kG) * kD + e]);
  // per warp: heads 2w, 2w+1; lane owns d = 4*lane..4*lane+3
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f}, acc[2][4] = {};
  const int b0 = blockIdx.y * kAttnBlocks, b1 = min(nvis, b0 + kAttnBlocks);
  for (int vi = b0; vi < b1; ++vi) {
    const int j = visible_block(vi, n_init, ntop, top, lo2);
    const int64_t key0 = (int64_t)j * kB;
    const int nk = (int)min((int64_t)kB, i + 1 - key0);  // causal clip of the diagonal block
    __syncthreads();
    for (int e = threadIdx.x; e < kB * (kD / 8); e += blockDim.x) {
      const int r = e / (kD / 8), c = e % (kD / 8);
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (r < nk) {
        kv = __ldg(reinterpret_cast<const uint4 *>(page_row(a.k_pages, a.block_table, a.max_pages, seq, key0 + r, a.h_kv, g)) + c);
        vv = __ldg(reinterpret_cast<const uint4 *>(page_row(a.v_pages, a.block_table, a.max_pages, seq, key0 + r, a.h_kv, g)) + c);
      }
      reinterpret_cast<uint4 *>(&k_s[r][0])[c] = kv;
      reinterpret_cast<uint4 *>(&v_s[r][0])[c] = vv;
    }
    __syncthreads();
    // logits: warp w computes heads 2w, 2w+1 for keys lane, lane+32
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * warp + hh;
      float s0 = -INFINITY, s1 = -INFINITY;
      float d0 = 0.f, d1 = 0.f;
#pragma unroll 4
      for (int d = 0; d < kD; d += 8) {
        const uint4 ka = *reinterpret_cast<const uint4 *>(&k_s[lane][d]);
        const uint4 kb = *reinterpret_cast<const uint4 *>(&k_s[lane + 32][d]);
        const __nv_bfloat162 *pa = reinterpret_cast<const __nv_bfloat162 *>(&ka);
        const __nv_bfloat162 *pb = reinterpret_cast<const __nv_bfloat162 *>(&kb);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 fa = __bfloat1622float2(pa[e]), fb = __bfloat1622float2(pb[e]);
          d0 = fmaf(q_s[h][d + 2 * e], fa.x, d0);
          d0 = fmaf(q_s[h][d + 2 * e + 1], fa.y, d0);
          d1 = fmaf(q_s[h][d + 2 * e], fb.x, d1);
          d1 = fmaf(q_s[h][d + 2 * e + 1], fb.y, d1);
        }
      }
      if (lane < nk) s0 = d0 * a.attn_scale_log2;
      if (lane + 32 < nk) s1 = d1 * a.attn_scale_log2;
      float mx = fmaxf(s0, s1);
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float m_new = fmaxf(m[hh], mx);
      const float alpha = (m[hh] == -INFINITY) ? 0.f : fast_exp2(m[hh] - m_new);
      const float p0 = (lane < nk) ? fast_exp2(s0 - m_new) : 0.f;
      const float p1 = (lane + 32 < nk) ? fast_exp2(s1 - m_new) : 0.f;
      float ps = p0 + p1;
      for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l[hh] = l[hh] * alpha + ps;
      m[hh] = m_new;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[hh][e] *= alpha;
      p_s[h][lane] = p0;
      p_s[h][lane + 32] = p1;
    }
    __syncwarp();
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 2 * warp + hh;
      for (int r = 0; r < nk; ++r) {
        const float pr = p_s[h][r];
        const __nv_bfloat162 *vr = reinterpret_cast<const __nv_bfloat162 *>(&v_s[r][4 * lane]);
        const float2 f0 = __bfloat1622float2(vr[0]), f1 = __bfloat1622float2(vr[1]);
        acc[hh][0] = fmaf(pr, f0.x, acc[hh][0]);
        acc[hh][1] = fmaf(pr, f0.y, acc[hh][1]);
        acc[hh][2] = fmaf(pr, f1.x, acc[hh][2]);
        acc[hh][3] = fmaf(pr, f1.y, acc[hh][3]);
      }
    }
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int h = 2 * warp + hh;
    const int64_t pi = ((int64_t)row * splits + blockIdx.y) * kG + h;
    *reinterpret_cast<float4 *>(&part_o[pi * kD + 4 * lane]) =
        make_float4(acc[hh][0], acc[hh][1], acc[hh][2], acc[hh][3]);
    if (lane == 0) part_ml[pi] = make_float2(m[hh], l[hh]);
  }
}

// grid (batch*h_kv), 512 threads = 16 heads x 32 lanes (4 d each)
__global__ void __launch_bounds__(512) decode_combine_kernel(DecodeArgs a, const int32_t *topk_cnt,
                                                             const float *part_o,
                                                             const float2 *part_ml, int splits,
                                                             __nv_bfloat16 *o, float *lse) {
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t L = a.seq_lens[seq];
  const int b = (int)((L - 1) / kB);
  const int n_init = min(a.N_init, b + 1);
  const int lo2 = max(max(0, b - a.N_local + 1), n_init);
  const int nvis = n_init + topk_cnt[row] + (b + 1 - lo2);
  const int used = (int)cdiv(nvis, kAttnBlocks);
  float M = -INFINITY;
  for (int sp = 0; sp < used; ++sp) M = fmaxf(M, part_ml[((int64_t)row * splits + sp) * kG + h].x);
  float Ls = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int sp = 0; sp < used; ++sp) {
    const int64_t pi = ((int64_t)row * splits + sp) * kG + h;
    const float2 ml = part_ml[pi];
    if (ml.x == -INFINITY) continue;
    const float w = fast_exp2(ml.x - M);
    Ls += ml.y * w;
    const float4 po = *reinterpret_cast<const float4 *>(&part_o[pi * kD + 4 * lane]);
    acc[0] += po.x * w;
    acc[1] += po.y * w;
    acc[2] += po.z * w;
    acc[3] += po.w * w;
  }
  const float inv = 1.f / Ls;
  __nv_bfloat16 *dst = o + ((int64_t)seq * a.h_q + g * kG + h) * kD + 4 * lane;
  __align__(8) __nv_bfloat16 ov[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) ov[e] = __float2bfloat16_rn(acc[e] * inv);
  *reinterpret_cast<uint2 *>(dst) = *reinterpret_cast<const uint2 *>(ov);
  if (lane == 0) lse[(int64_t)seq * a.h_q + g * kG + h] = (M + __log2f(Ls)) * 0.6931471805599453f;
}

static DecodeArgs make_args(const swattn_config *cfg, const swattn_paged_kv *kv, const void *q,
                            int batch) {
  DecodeArgs a;
  memset(&a, 0, sizeof(a));
  a.q = static_cast<const __nv_bfloat16 *>(q);
  a.k_pages = static_cast<const __nv_bfloat16 *>(kv->k_pages);
  a.v_pages = static_cast<const __nv_bfloat16 *>(kv->v_pages);
  a.block_table = kv->block_table;
  a.seq_lens = kv->seq_lens;
  a.max_pages = kv->max_pages;
  a.kc1 = static_cast<const __nv_bfloat16 *>(kv->kc1);
  a.kc2 = static_cast<const __nv_bfloat16 *>(kv->kc2);
  a.max_m1 = kv->max_m1;
  a.max_m2 = kv->max_m2;
  a.batch = batch;
  a.h_q = cfg->h_q;
  a.h_kv = cfg->h_kv;
  a.l_C1 = cfg->l_C1; a.s_C1 = cfg->s_C1; a.l_C2 = cfg->l_C2; a.s_C2 = cfg->s_C2;
  a.B = cfg->B;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.k_top = cfg->k_top;
  const float scale = cfg->scale_compressed_logits ? 1.f / sqrtf((float)cfg->d_h) : 1.f;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.attn_scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  return a;
}

struct DecodeLayout {
  int p1_splits, tiles, attn_splits, max_ctx;
  int64_t ld;
  size_t off_p1, off_scmp, off_topk, off_cnt, off_count, off_rows, off_po, off_pml, total;
};

static inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static DecodeLayout decode_layout(const swattn_config *cfg, int batch, int max_pages) {
  DecodeLayout D{};
  D.max_ctx = max_pages * cfg->B;
  const int64_t m1 = num_pooled(D.max_ctx, cfg->l_C1, cfg->s_C1);
  const int64_t m2 = num_pooled(D.max_ctx, cfg->l_C2, cfg->s_C2);
  const int64_t n_cols = m1 ? cdiv(m1, cfg->s) : 0;
  D.p1_splits = (int)std::max<int64_t>(1, cdiv(std::max(m2, m1), kP1Cols));
  D.tiles = (int)std::max<int64_t>(1, cdiv(n_cols, kTileBlocks));
  D.attn_splits = (int)cdiv(cfg->N_init + cfg->N_local + cfg->k_top, kAttnBlocks);
  D.ld = ((n_cols + 3) / 4) * 4 + 4;
  const int64_t rows = (int64_t)batch * cfg->h_kv;
  size_t o = 0;
  D.off_p1 = o; o = al(o + rows * D.p1_splits * kG * sizeof(float2));
  D.off_scmp = o; o = al(o + rows * D.ld * sizeof(float));
  D.off_topk = o; o = al(o + rows * std::max(cfg->k_top, 1) * sizeof(int32_t));
  D.off_cnt = o; o = al(o + rows * sizeof(int32_t));
  D.off_count = o; o = al(o + 16);
  D.off_rows = o; o = al(o + rows * sizeof(int32_t));
  D.off_po = o; o = al(o + rows * D.attn_splits * kG * kD * sizeof(float));
  D.off_pml = o; o = al(o + rows * D.attn_splits * kG * sizeof(float2));
  D.total = o;
  return D;
}

static int num_sms_dec() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace
}  // namespace swattn

using namespace swattn;

extern "C" {

size_t swattn_decode_workspace_bytes(const swattn_config *cfg, int32_t batch, int32_t max_pages) {
  if (cfg == nullptr || batch < 1 || max_pages < 1) return 0;
  return decode_layout(cfg, batch, max_pages).total;
}

static int32_t check_decode(const swattn_config *cfg, const swattn_paged_kv *kv, int32_t batch) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (!swattn_profile_supported(cfg)) {
    set_error("unsupported profile for the decode kernels (need G=16, d_h=128, B=64, l=5, s=4)");
    return SWATTN_EUNSUPPORTED;
  }
  if (kv == nullptr || kv->k_pages == nullptr || kv->v_pages == nullptr ||
      kv->block_table == nullptr || kv->seq_lens == nullptr || kv->kc1 == nullptr ||
      kv->kc2 == nullptr) {
    set_error("paged KV descriptor has NULL members");
    return SWATTN_EINVAL;
  }
  if (batch < 1 || kv->max_pages < 1) {
    set_error("batch and max_pages must be >= 1");
    return SWATTN_EINVAL;
  }
  const int64_t ctx = (int64_t)kv->max_pages * cfg->B;
  if (kv->max_m1 < num_pooled(ctx, cfg->l_C1, cfg->s_C1) ||
      kv->max_m2 < num_pooled(ctx, cfg->l_C2, cfg->s_C2)) {
    set_error("compressed-key slabs too small for max_pages*B tokens");
    return SWATTN_EINVAL;
  }
  return SWATTN_OK;
}

int32_t swattn_kcache_append(const swattn_config *cfg, const swattn_paged_kv *kv,
                             const int32_t *prev_lens, int32_t batch, void *stream) {
  int32_t rc = check_decode(cfg, kv, batch);
  if (rc) return rc;
  DecodeArgs a = make_args(cfg, kv, nullptr, batch);
  kcache_append_kernel<<<dim3(batch, cfg->h_kv), kD, 0, static_cast<cudaStream_t>(stream)>>>(
      a, prev_lens);
  SWATTN_LAUNCH_CHECK("kcache_append_kernel");
  return SWATTN_OK;
}

int32_t swattn_decode_step(const swattn_config *cfg, const swattn_paged_kv *kv, const void *q,
                           int32_t batch, void *o, float *lse, int32_t *topk_out, void *workspace,
                           size_t workspace_bytes, void *stream) {
  int32_t rc = check_decode(cfg, kv, batch);
  if (rc) return rc;
  const DecodeLayout D = decode_layout(cfg, batch, kv->max_pages);
  if (workspace == nullptr || workspace_bytes < D.total) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, D.total);
    return SWATTN_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *ws = static_cast<char *>(workspace);
  float2 *p1 = reinterpret_cast<float2 *>(ws + D.off_p1);
  float *scmp = reinterpret_cast<float *>(ws + D.off_scmp);
  int32_t *topk = topk_out ? topk_out : reinterpret_cast<int32_t *>(ws + D.off_topk);
  int32_t *cnt = reinterpret_cast<int32_t *>(ws + D.off_cnt);
  int32_t *count = reinterpret_cast<int32_t *>(ws + D.off_count);
  int32_t *rows = reinterpret_cast<int32_t *>(ws + D.off_rows);
  float *po = reinterpret_cast<float *>(ws + D.off_po);
  float2 *pml = reinterpret_cast<float2 *>(ws + D.off_pml);
  DecodeArgs a = make_args(cfg, kv, q, batch);
  const int nrows = batch * cfg->h_kv;
  decode_pass1_kernel<<<dim3(nrows, D.p1_splits), 256, 0, st>>>(a, p1, D.p1_splits);
  SWATTN_LAUNCH_CHECK("decode_pass1_kernel");
  decode_pass2_kernel<<<dim3(nrows, D.tiles), 128, 0, st>>>(a, p1, D.p1_splits, scmp, D.ld);
  SWATTN_LAUNCH_CHECK("decode_pass2_kernel");
  if ((rc = cuda_check(cudaMemsetAsync(count, 0, 4, st), "memset"))) return rc;
  if ((rc = launch_decode_topk(cfg, scmp, D.ld, kv->seq_lens, batch, D.max_ctx, topk, cnt, count,
                               rows, nrows, st)))
    return rc;
  if ((rc = launch_rerank_decode(cfg, q, kv->kc1, kv->kc2, kv->max_m1, kv->max_m2, kv->seq_lens,
                                 batch, scmp, D.ld, count, rows, nrows, topk, num_sms_dec(), st)))
    return rc;
  decode_attn_kernel<<<dim3(nrows, D.attn_splits), 256, 0, st>>>(a, topk, cnt, po, pml,
                                                                 D.attn_splits);
  SWATTN_LAUNCH_CHECK("decode_attn_kernel");
  decode_combine_kernel<<<nrows, 512, 0, st>>>(a, cnt, po, pml, D.attn_splits,
                                               static_cast<__nv_bfloat16 *>(o), lse);
  SWATTN_LAUNCH_CHECK("decode_combine_kernel");
  return SWATTN_OK;
}

}  // extern "C"
