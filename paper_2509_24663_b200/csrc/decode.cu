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
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

int32_t launch_decode_topk(const swattn_config *, const float *, int64_t, const int32_t *, int, int,
                           int32_t *, int32_t *, int32_t *, int32_t *, int32_t, const uint64_t *,
                           int64_t, cudaStream_t);
int32_t launch_rerank_decode(const swattn_config *, const void *, const void *, const void *,
                             int max_m1, int max_m2, const int32_t *seq_lens, int batch,
                             const float *, int64_t, const int32_t *, const int32_t *, int32_t,
                             int32_t *, void *, int, cudaStream_t);
size_t rerank_partials_bytes();

namespace {

constexpr int kP1Cols = 128;     // normaliser columns per pass-1 CTA (4 warps x 32)
constexpr int kTileBlocks = 31;  // pass-2 tile: 31 blocks, 124 (+4) columns
constexpr int kTileCols = 128;
constexpr int kP2Smem = 2 * kTileCols * 256 + 1024;  // passes 1 and 2: two 128-row key tiles

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

// ------------------------------------------------------------ D1 append
// New C1 / C2 entries of one (sequence, group) when it grew from L0 to L
// tokens: thread d sums element d of each completed window in float64.
__device__ __forceinline__ void append_windows(const DecodeArgs &a, int seq, int g, int d, int64_t L0,
                                               int64_t L) {
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

// grid (batch, h_kv), 128 threads = d; new windows are few per step.
__global__ void kcache_append_kernel(DecodeArgs a, const int32_t *prev_lens) {
  const int seq = blockIdx.x, g = blockIdx.y, d = threadIdx.x;
  append_windows(a, seq, g, d, prev_lens ? prev_lens[seq] : 0, a.seq_lens[seq]);
}

// One decode token per sequence: grid (batch), h_kv * 128 threads (thread =
// group x element).  Writes the token's K/V row into its page (the block
// table already maps page L0 / B), extends the pooled keys, then advances
// seq_lens[seq] -- after every thread of the CTA has read the old length.
__global__ void kcache_append_tokens_kernel(DecodeArgs a, const __nv_bfloat16 *K,
                                            const __nv_bfloat16 *V, const int32_t *active,
                                            int32_t *seq_lens) {
  const int seq = blockIdx.x;
  if (active && !active[seq]) return;
  const int g = threadIdx.x / kD, d = threadIdx.x % kD;
  const int64_t L0 = seq_lens[seq];
  const int64_t src = ((int64_t)seq * a.h_kv + g) * kD + d;
  const int64_t dst = (page_row(a.k_pages, a.block_table, a.max_pages, seq, L0, a.h_kv, g) - a.k_pages) + d;
  const_cast<__nv_bfloat16 *>(a.k_pages)[dst] = K[src];
  const_cast<__nv_bfloat16 *>(a.v_pages)[dst] = V[src];
  append_windows(a, seq, g, d, L0, L0 + 1);  // reads only rows this thread wrote or older ones
  __syncthreads();
  if (threadIdx.x == 0) seq_lens[seq] = (int32_t)(L0 + 1);
}

// ------------------------------------------------------------ D2 pass 1
// grid (batch*h_kv, splits), 4 warps: warp w scores normaliser columns
// [128 split + 32 w, +32) on mma.sync (q as A fragments, key rows as B
// fragments from global memory) and keeps per-head online (max, sum); the
// four lanes sharing a head row, then the four warps, are merged.
__device__ __forceinline__ void merge_ml(float &m, float &l, float m2, float l2) {
  const float M = fmaxf(m, m2);
  if (M == -INFINITY) return;
  l = (m == -INFINITY ? 0.f : l * fast_exp2(m - M)) + (m2 == -INFINITY ? 0.f : l2 * fast_exp2(m2 - M));
  m = M;
}

__device__ __forceinline__ void mma16816_p1(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                            uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Persistent over 128-column slices like pass 2: grid (rows, kP1Ctas), CTA y
// takes slices y, y + kP1Ctas, ..., the next slice's key rows in flight
// (cp.async, double buffer) while the current one is scored from shared
// memory (ldmatrix); one (max, sum) partial per slice and head, merged in
// the same order as before (n-tiles of a lane, the lane quad, the 4 warps).
constexpr int kP1Ctas = 13;  // 416 CTAs at batch 16: one wave at 3 CTAs per SM

__device__ __forceinline__ void p1_issue_slice(uint32_t kt, const __nv_bfloat16 *kbase, int64_t col0,
                                               int64_t vis, int h_kv) {
  for (int c = threadIdx.x; c < kP1Cols * 16; c += blockDim.x) {
    const int rr = c >> 4, ch = c & 15;
    const uint32_t dst = kt + rr * 256 + (uint32_t)(((ch & 8) | ((ch & 7) ^ (rr & 7))) << 4);
    const int64_t col = col0 + rr;
    if (col < vis)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(kbase + col * h_kv * kD + ch * 8));
    else
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u));
  }
  asm volatile("cp.async.commit_group;");
}

__global__ void __launch_bounds__(128) decode_pass1_kernel(DecodeArgs a, float2 *part, int splits,
                                                           int32_t *amb_count) {
  extern __shared__ uint8_t p1_raw[];
  uint8_t *ktiles = p1_raw + ((128u - (tc::smem_u32(p1_raw) & 127u)) & 127u);  // [2][128 rows][256 B]
  __shared__ float2 red[4][kG];
  pdl_launch_dependents();
  // the step's flagged-row counter (read by top-k / re-rank after pass 2)
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *amb_count = 0;
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t vis2 = vis_count(L - 1, a.l_C2, a.s_C2);
  const int64_t vis1 = vis_count(L - 1, a.l_C1, a.s_C1);
  const bool use2 = vis2 > 0;
  const int64_t vis = use2 ? vis2 : vis1;  // fallback rows use the exact C1 lse
  const int n_sl = (int)min((int64_t)splits, cdiv(vis, (int64_t)kP1Cols));
  if ((int)blockIdx.y >= n_sl) return;
  const __nv_bfloat16 *kc = (use2 ? a.kc2 : a.kc1) + ((int64_t)seq * (use2 ? a.max_m2 : a.max_m1) * a.h_kv + g) * kD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, dw = lane & 3;
  const uint32_t kt0 = tc::smem_u32(ktiles);
  p1_issue_slice(kt0, kc, (int64_t)blockIdx.y * kP1Cols, vis, a.h_kv);
  uint32_t qa[8][4];
  {
    const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.q + (((int64_t)seq * a.h_q + g * kG + r) * kD));
    const uint32_t *q1 = q0 + 8 * (kD / 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = __ldg(q0 + ks * 8 + dw);
      qa[ks][1] = __ldg(q1 + ks * 8 + dw);
      qa[ks][2] = __ldg(q0 + ks * 8 + 4 + dw);
      qa[ks][3] = __ldg(q1 + ks * 8 + 4 + dw);
    }
  }
  const int lm = lane >> 3, lr = lane & 7;
  int buf = 0;
  for (int sl = blockIdx.y; sl < n_sl; sl += gridDim.y, buf ^= 1) {
    const uint32_t kt = kt0 + buf * (kP1Cols * 256);
    if (sl + (int)gridDim.y < n_sl) {
      p1_issue_slice(kt0 + (buf ^ 1) * (kP1Cols * 256), kc, (int64_t)(sl + gridDim.y) * kP1Cols, vis, a.h_kv);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();
    const int64_t col0 = (int64_t)sl * kP1Cols + warp * 32;
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int rr = warp * 32 + hf * 16 + (lm >> 1) * 8 + lr, ch = ks * 2 + (lm & 1);
        uint32_t b00, b01, b10, b11;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b00), "=r"(b01), "=r"(b10), "=r"(b11)
                     : "r"(kt + rr * 256 + (uint32_t)(((ch & 8) | ((ch & 7) ^ (rr & 7))) << 4)));
        mma16816_p1(acc[2 * hf], qa[ks], b00, b01);
        mma16816_p1(acc[2 * hf + 1], qa[ks], b10, b11);
      }
    }
    float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;  // heads r, r + 8
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      // columns 2 dw, 2 dw + 1 of this n-tile
      const int64_t c = col0 + nt * 8 + 2 * dw;
      const bool v0 = c < vis, v1 = c + 1 < vis;
      const float x0 = v0 ? acc[nt][0] * a.scale_log2 : -INFINITY, x1 = v1 ? acc[nt][1] * a.scale_log2 : -INFINITY;
      const float x2 = v0 ? acc[nt][2] * a.scale_log2 : -INFINITY, x3 = v1 ? acc[nt][3] * a.scale_log2 : -INFINITY;
      const float mm0 = fmaxf(x0, x1), mm1 = fmaxf(x2, x3);
      if (mm0 != -INFINITY) merge_ml(m0, l0, mm0, fast_exp2(x0 - mm0) + fast_exp2(x1 - mm0));
      if (mm1 != -INFINITY) merge_ml(m1, l1, mm1, fast_exp2(x2 - mm1) + fast_exp2(x3 - mm1));
    }
    // lanes 4 r .. 4 r + 3 share head rows r and r + 8
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const float om0 = __shfl_xor_sync(0xffffffffu, m0, o), ol0 = __shfl_xor_sync(0xffffffffu, l0, o);
      const float om1 = __shfl_xor_sync(0xffffffffu, m1, o), ol1 = __shfl_xor_sync(0xffffffffu, l1, o);
      merge_ml(m0, l0, om0, ol0);
      merge_ml(m1, l1, om1, ol1);
    }
    if (dw == 0) {
      red[warp][r] = make_float2(m0, l0);
      red[warp][r + 8] = make_float2(m1, l1);
    }
    __syncthreads();  // red complete; every warp is done with tile buffer `buf`
    if (threadIdx.x < kG) {
      const int h = threadIdx.x;
      float M = -INFINITY, S = 0.f;
      for (int w = 0; w < 4; ++w) merge_ml(M, S, red[w][h].x, red[w][h].y);
      part[((int64_t)row * splits + sl) * kG + h] = make_float2(M, S);
    }
    __syncthreads();  // red reuse
  }
}

// ------------------------------------------------------------ D3 pass 2
// grid (batch*h_kv, tiles), 4 warps: warp w scores columns [32 w, 32 w + 32)
// of the 128-column tile on the tensor cores -- S [16 heads x 32 columns] =
// q (A fragments, registers) . K_C1 rows (B fragments straight from global
// memory) with mma.sync.m16n8k16 -- then p = exp2(s c - m_h) / l_h summed over
// the 16 heads (two rows per thread + three shuffles), 5/4 max-pool from
// shared memory (compression.py:160-173).
__device__ __forceinline__ void mma16816_dec(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                             uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ unsigned long long spread_bits2(uint32_t x) {  // bit q -> bit 2q
  unsigned long long v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// Persistent over tiles: grid (rows, kP2Ctas); CTA y handles tiles y,
// y + kP2Ctas, ... of its row with the next tile's 32 KB of C1 rows in flight
// (cp.async, double buffer) while the current one is scored, and merges the
// row's pass-1 partials and loads q once (a CTA per tile repeated both 67
// times per row and ran 2.4 short waves: 26-31 us, profiles/r02k).
constexpr int kP2Ctas = 13;

__device__ __forceinline__ void p2_issue_tile(uint32_t kt, const __nv_bfloat16 *kbase, int64_t tile0,
                                              int64_t vis1, int h_kv) {
  // 128 C1 rows -> shared memory (256-byte rows, 16-byte chunk c of row rr at
  // c ^ (rr & 7): conflict-free ldmatrix), zeros past vis1
  for (int c = threadIdx.x; c < kTileCols * 16; c += blockDim.x) {
    const int rr = c >> 4, ch = c & 15;
    const uint32_t dst = kt + rr * 256 + (uint32_t)(((ch & 8) | ((ch & 7) ^ (rr & 7))) << 4);
    const int64_t col = tile0 + rr;
    if (col < vis1)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(kbase + col * h_kv * kD + ch * 8));
    else
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u));
  }
  asm volatile("cp.async.commit_group;");
}

__global__ void __launch_bounds__(128) decode_pass2_kernel(DecodeArgs a, const float2 *part,
                                                           int splits, float *s_cmp, int64_t ld,
                                                           uint64_t *flags, int ld_f) {
  extern __shared__ uint8_t p2_raw[];
  uint8_t *ktiles = p2_raw + ((128u - (tc::smem_u32(p2_raw) & 127u)) & 127u);  // [2][128 rows][256 B]
  __shared__ float2 stat[kG];  // (m, 1/l), log2 domain
  __shared__ float sc[kTileCols + 4];
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t i = L - 1;
  const int64_t m1 = num_pooled(L, a.l_C1, a.s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, kPoolS) : 0);
  const int hi = cand_hi((int)(i / a.B), a.N_local, n_cols);
  const int n_tiles = (int)cdiv(hi, kTileBlocks);
  if ((int)blockIdx.y >= n_tiles) return;
  const int64_t vis1 = vis_count(i, a.l_C1, a.s_C1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const __nv_bfloat16 *kbase = a.kc1 + ((int64_t)seq * a.max_m1 * a.h_kv + g) * kD;
  const uint32_t kt0 = tc::smem_u32(ktiles);
  p2_issue_tile(kt0, kbase, (int64_t)blockIdx.y * kTileBlocks * kPoolS, vis1, a.h_kv);
  pdl_launch_dependents();
  // q as A fragments (a step input): a0 = (head r, d k), a1 = (r + 8, k), a2 = (r, k + 8), a3 = (r + 8, k + 8)
  const int r = lane >> 2, dw = lane & 3;
  uint32_t qa[8][4];
  {
    const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.q + (((int64_t)seq * a.h_q + g * kG + r) * kD));
    const uint32_t *q1 = q0 + 8 * (kD / 2);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = __ldg(q0 + ks * 8 + dw);
      qa[ks][1] = __ldg(q1 + ks * 8 + dw);
      qa[ks][2] = __ldg(q0 + ks * 8 + 4 + dw);
      qa[ks][3] = __ldg(q1 + ks * 8 + 4 + dw);
    }
  }
  pdl_wait();  // pass-1 partials
  if (warp == 0) {
    // pass-1 partials of this row: only the slices pass 1 covered hold data
    // (C2 columns for approx rows, C1 for fallback rows); lane pairs (h, half)
    // merge half of the slices each (eight independent loads per round), then
    // one shuffle joins the halves
    const int64_t vis2 = vis_count(i, a.l_C2, a.s_C2);
    const int used = (int)min((int64_t)splits, cdiv(vis2 > 0 ? vis2 : vis1, (int64_t)kP1Cols));
    const int h = lane & 15, half = lane >> 4;
    float M = -INFINITY, S = 0.f;
    for (int sp0 = 0; sp0 < used; sp0 += 16) {
      float2 pv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int sp = sp0 + 2 * e + half;
        pv[e] = sp < used ? part[((int64_t)row * splits + sp) * kG + h] : make_float2(-INFINITY, 0.f);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (pv[e].x == -INFINITY) continue;
        const float Mn = fmaxf(M, pv[e].x);
        S = (M == -INFINITY ? 0.f : S * fast_exp2(M - Mn)) + pv[e].y * fast_exp2(pv[e].x - Mn);
        M = Mn;
      }
    }
    const float oM = __shfl_xor_sync(0xffffffffu, M, 16), oS = __shfl_xor_sync(0xffffffffu, S, 16);
    const float Mt = fmaxf(M, oM);
    float St = 0.f;
    if (Mt != -INFINITY)
      St = (M == -INFINITY ? 0.f : S * fast_exp2(M - Mt)) + (oM == -INFINITY ? 0.f : oS * fast_exp2(oM - Mt));
    if (half == 0) stat[h] = make_float2(Mt == -INFINITY ? 0.f : Mt, St > 0.f ? 1.f / St : 0.f);
  }
  const int lm = lane >> 3, lr = lane & 7;
  int buf = 0;
  for (int t = blockIdx.y; t < n_tiles; t += gridDim.y, buf ^= 1) {
    const int64_t tile0 = (int64_t)t * kTileBlocks * kPoolS;
    const uint32_t kt = kt0 + buf * (kTileCols * 256);
    if (t + (int)gridDim.y < n_tiles) {
      p2_issue_tile(kt0 + (buf ^ 1) * (kTileCols * 256), kbase,
                    (int64_t)(t + gridDim.y) * kTileBlocks * kPoolS, vis1, a.h_kv);
      asm volatile("cp.async.wait_group 1;");
    } else {
      asm volatile("cp.async.wait_group 0;");
    }
    __syncthreads();  // tile t (all threads' copies) and stat
    const int64_t col0 = tile0 + warp * 32;
    float acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        // rows (columns) 32 warp + 16 hf + 8 (lm >> 1) + lr; matrices (n-tile lo, k lo),
        // (n-tile lo, k hi), (n-tile hi, k lo), (n-tile hi, k hi)
        const int rr = warp * 32 + hf * 16 + (lm >> 1) * 8 + lr, ch = ks * 2 + (lm & 1);
        uint32_t b00, b01, b10, b11;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b00), "=r"(b01), "=r"(b10), "=r"(b11)
                     : "r"(kt + rr * 256 + (uint32_t)(((ch & 8) | ((ch & 7) ^ (rr & 7))) << 4)));
        mma16816_dec(acc[2 * hf], qa[ks], b00, b01);
        mma16816_dec(acc[2 * hf + 1], qa[ks], b10, b11);
      }
    }
    const float2 st0 = stat[r], st1 = stat[r + 8];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      // rows r (c0, c1) and r + 8 (c2, c3); columns 2 (lane % 4) + {0, 1}
      float c0 = fast_exp2(fmaf(acc[nt][0], a.scale_log2, -st0.x)) * st0.y +
                 fast_exp2(fmaf(acc[nt][2], a.scale_log2, -st1.x)) * st1.y;
      float c1 = fast_exp2(fmaf(acc[nt][1], a.scale_log2, -st0.x)) * st0.y +
                 fast_exp2(fmaf(acc[nt][3], a.scale_log2, -st1.x)) * st1.y;
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        c0 += __shfl_xor_sync(0xffffffffu, c0, o);
        c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      }
      if (r == 0) {
        const int cc = warp * 32 + nt * 8 + 2 * dw;
        const int64_t col = col0 + nt * 8 + 2 * dw;
        sc[cc] = col < m1 ? (col < vis1 ? c0 : 0.f) : -INFINITY;
        sc[cc + 1] = col + 1 < m1 ? (col + 1 < vis1 ? c1 : 0.f) : -INFINITY;
      }
    }
    __syncthreads();  // sc complete; every warp is done reading tile buffer `buf`
    if (warp == 0) {
      // 5/4 max-pool, one block per lane, plus the argmax-at-shared-column bits
      // (L: window column 0, R: column 4, with margin) that let top-k settle a
      // structural tie straddling the k-th boundary without the float64
      // re-rank -- the same flags K2 emits for prefill (scores_tc.cu)
      const int j = t * kTileBlocks + lane;
      const bool ok = lane < kTileBlocks && j >= a.N_init && j < hi;
      float v[kPoolL];
#pragma unroll
      for (int e = 0; e < kPoolL; ++e) v[e] = sc[min(lane * kPoolS + e, kTileCols + 3)];
      if (ok) s_cmp[(int64_t)row * ld + j] = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), v[4]);
      const float f = 1.f + 4.f * kScoreRelErr;
      const bool Lb = ok && v[1] * f < v[0] && v[2] * f < v[0] && v[3] * f < v[0] && v[4] * f < v[0];
      const bool Rb = ok && v[0] * f < v[4] && v[1] * f < v[4] && v[2] * f < v[4] && v[3] * f < v[4];
      const unsigned lmask = __ballot_sync(0xffffffffu, Lb);
      const unsigned rmask = __ballot_sync(0xffffffffu, Rb);
      if (lane == 0) flags[(int64_t)row * ld_f + t] = spread_bits2(lmask) | (spread_bits2(rmask) << 1);
    }
    __syncthreads();  // sc reuse by the next tile
  }
}

// ------------------------------------------------------------ D5 attention

// ---- D5 on the tensor cores: one warp = (row, split of kAttnBlocks blocks);
// the row's 16 query heads are the M = 16 of mma.sync.m16n8k16 (as in the
// prefill part B, csrc/sparse_warp.cu): Q in registers, S -> P in registers,
// O in registers, online softmax per 16-key stage.  K/V stages (16 rows of
// one page) come from the page pool by TMA -- one 4-D box {64 d, 16 rows,
// 2 d-halves, 1 group} per tensor into a per-warp 3-slot mbarrier ring
// stored [d half][row][64] with the 128-byte swizzle (conflict-free
// ldmatrix), lane 0 the warp's issuer -- the part-B scheme of
// csrc/sparse_warp.cu.  (16-byte cp.async copies needed ~60 instructions per
// stage per lane and reached 3.6 TB/s, profiles/r02o.)
constexpr int kDW = 4;                        // warps per CTA (2 CTAs per SM)
constexpr int kDCl = 8;                       // CTAs per cluster = per (sequence, group) row
constexpr int kDStages = 3;                   // ring depth: 2 stages in flight while one computes
constexpr int kDStageKeys = 16;
constexpr uint32_t kDTile = kDStageKeys * kD * 2;  // 4 KB

__device__ __forceinline__ uint32_t dswz(int row, int c) {  // c = 16-byte chunk 0..15
  const int line = (c >> 3) * kDStageKeys + row;
  return (uint32_t)(line * 128 + (((c & 7) ^ (line & 7)) << 4));
}
__device__ __forceinline__ void dldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                         uint32_t &r3, bool trans) {
  if (trans)
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
  else
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void dmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

struct AttnMaps {
  CUtensorMap k, v;  // page pools as (d lo/hi 64, pool row, half, group): box {64, 16, 2, 1}
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_cluster_f32x2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(kDCl, 1, 1) __launch_bounds__(kDW * 32)
    decode_attn_cluster_kernel(DecodeArgs a, const int32_t *topk, const int32_t * /* topk_cnt */,
                               __nv_bfloat16 *o_out, float *lse_out,
                               const __grid_constant__ AttnMaps maps) {
  extern __shared__ uint8_t dsm_raw[];
  uint8_t *dsm = dsm_raw + ((1024u - (tc::smem_u32(dsm_raw) & 1023u)) & 1023u);
  auto ring = reinterpret_cast<uint8_t(*)[kDStages][2][kDTile]>(dsm);  // [warp][stage][K|V]
  __shared__ uint64_t full_s[kDW][kDStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();   // = blockIdx.x (cluster spans x)
  const int wid = (int)crank * kDW + warp;    // warp of the row, 0 .. kDCl * kDW - 1
  const int row = blockIdx.y;
  uint64_t *full = full_s[warp];
  if (lane == 0) {
    for (int k = 0; k < kDStages; ++k) tc::mbar_init(&full[k], 1);
    tc::fence_barrier_init();
  }
  __syncwarp();
  pdl_launch_dependents();
  const int seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t i = L - 1;
  const int b = (int)(i / kB);
  const int n_init = min(a.N_init, b + 1);
  const int lo = max(0, b - a.N_local + 1);
  const int lo2 = max(lo, n_init);
  const int nloc = b + 1 - lo2;
  // the row's top-k count is a function of its length (topk_cta.cuh), so the
  // block -> warp map is known before the top-k kernels finish
  const int64_t m1_row = num_pooled(L, a.l_C1, a.s_C1);
  const int ncand = max(0, cand_hi(b, a.N_local, (int)(m1_row ? cdiv(m1_row, kPoolS) : 0)) - a.N_init);
  const int ntop = (L < 1 || i + 1 < a.l_C1) ? 0 : min(ncand, a.k_top);
  // an empty slot (no cached token) has no visible block: no page is read
  const int nvis = L < 1 ? 0 : n_init + nloc + ntop;
  const int32_t *top = topk + (int64_t)row * a.k_top;
  // visible blocks in the order init, local, top-k, spread evenly over the
  // row's kDCl x kDW warps: warps holding only init / local blocks (a third
  // of the row) need nothing from the top-k kernels and start streaming
  // before the programmatic-launch wait, the others wait for the selection
  const int per = (nvis + kDCl * kDW - 1) / (kDCl * kDW);
  const int vb0 = min(nvis, wid * per), vb1 = min(nvis, vb0 + per);
  if (vb1 > n_init + nloc) pdl_wait();  // top-k (and its re-rank)
  const int h0 = lane >> 2;
  // q of the group as A fragments straight from global memory:
  // a0 = (head h0, d k), a1 = (h0 + 8, k), a2 = (h0, k + 8), a3 = (h0 + 8, k + 8)
  const int lm = lane >> 3, lr = lane & 7;
  uint32_t qa[8][4];
  {
    const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.q + (((int64_t)seq * a.h_q + g * kG + h0) * kD));
    const uint32_t *q1 = q0 + 8 * (kD / 2);
    const int dw = lane & 3;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = __ldg(q0 + ks * 8 + dw);
      qa[ks][1] = __ldg(q1 + ks * 8 + dw);
      qa[ks][2] = __ldg(q0 + ks * 8 + 4 + dw);
      qa[ks][3] = __ldg(q1 + ks * 8 + 4 + dw);
    }
  }
  // the warp's <= 32 block ids and their pages, looked up once (lane l holds
  // block vb0 + l): a per-stage topk -> block_table -> page chain of
  // dependent loads was the kernel's top stall (profiles/r02n)
  int my_j = 0, my_page = 0;
  if (lane < vb1 - vb0) {
    const int idx = vb0 + lane;
    my_j = idx < n_init ? idx : idx < n_init + nloc ? lo2 + (idx - n_init) : top[idx - n_init - nloc];
    my_page = a.block_table[(int64_t)seq * a.max_pages + my_j];
  }
  // stage s of this warp's key stream: block vb0 + s / 4, rows (s % 4) * 16 ..
  const int nst = (vb1 - vb0) * (kB / kDStageKeys);
  auto issue = [&](int st_idx, int slot) {  // warp-collective (the shuffle); lane 0 issues
    const int page = __shfl_sync(0xffffffffu, my_page, st_idx / 4);
    if (lane == 0) {
      const int prow = page * kB + (st_idx % 4) * kDStageKeys;
      tc::mbar_arrive_expect_tx(&full[slot], 2 * kDTile);
      tc::tma_load_4d(&maps.k, &full[slot], ring[warp][slot][0], 0, prow, 0, g);
      tc::tma_load_4d(&maps.v, &full[slot], ring[warp][slot][1], 0, prow, 0, g);
    }
  };
  for (int s0 = 0; s0 < kDStages && s0 < nst; ++s0) issue(s0, s0);
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  for (int s2 = 0; s2 < nst; ++s2) {
    const int slot = s2 % kDStages;
    // refill the slot stage s2 - 1 used (every lane finished reading it at
    // the end of the previous iteration) with stage s2 + kDStages - 1
    if (s2 >= 1 && s2 + kDStages - 1 < nst) {
      if (lane == 0) tc::fence_proxy_async();
      issue(s2 + kDStages - 1, (s2 + kDStages - 1) % kDStages);
    }
    tc::mbar_wait(&full[slot], (uint32_t)((s2 / kDStages) & 1));
    const uint32_t kst = tc::smem_u32(ring[warp][slot][0]), vst = tc::smem_u32(ring[warp][slot][1]);
    float sc[2][4] = {};
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      uint32_t b00, b01, b10, b11;
      dldsm_x4(kst + dswz((lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), b00, b01, b10, b11, false);
      dmma(sc[0], qa[ks], b00, b01);
      dmma(sc[1], qa[ks], b10, b11);
    }
    // causal clip: keys after i (only in the diagonal block) are masked
    const int j = __shfl_sync(0xffffffffu, my_j, s2 / 4);
    const int64_t key0 = (int64_t)j * kB + (s2 % 4) * kDStageKeys;
    float x[2][4];
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int jt = 0; jt < 2; ++jt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t key = key0 + jt * 8 + (lane & 3) * 2 + (e & 1);
        const float v = key <= i ? sc[jt][e] * a.attn_scale_log2 : -INFINITY;
        x[jt][e] = v;
        if (e < 2) mx0 = fmaxf(mx0, v); else mx1 = fmaxf(mx1, v);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float al0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - mn0);
    const float al1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
    for (int jt = 0; jt < 2; ++jt) {
      x[jt][0] = (mn0 == -INFINITY) ? 0.f : fast_exp2(x[jt][0] - mn0);
      x[jt][1] = (mn0 == -INFINITY) ? 0.f : fast_exp2(x[jt][1] - mn0);
      x[jt][2] = (mn1 == -INFINITY) ? 0.f : fast_exp2(x[jt][2] - mn1);
      x[jt][3] = (mn1 == -INFINITY) ? 0.f : fast_exp2(x[jt][3] - mn1);
      ps0 += x[jt][0] + x[jt][1];
      ps1 += x[jt][2] + x[jt][3];
    }
    l0 = l0 * al0 + ps0;
    l1 = l1 * al1 + ps1;
#pragma unroll
    for (int jt = 0; jt < 16; ++jt) {
      o[jt][0] *= al0;
      o[jt][1] *= al0;
      o[jt][2] *= al1;
      o[jt][3] *= al1;
    }
    const uint32_t pa[4] = {pack2(x[0][0], x[0][1]), pack2(x[0][2], x[0][3]), pack2(x[1][0], x[1][1]),
                            pack2(x[1][2], x[1][3])};
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      uint32_t v00, v01, v10, v11;
      dldsm_x4(vst + dswz((lm & 1) * 8 + lr, dp * 2 + (lm >> 1)), v00, v01, v10, v11, true);
      dmma(o[2 * dp], pa, v00, v01);
      dmma(o[2 * dp + 1], pa, v10, v11);
    }
    __syncwarp();  // every lane's reads of this slot are done before it is refilled
  }
  // ---- the warp's state -> its (now idle) ring: stats [2][16] then O [16][128] fp32
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  float *st = reinterpret_cast<float *>(ring[warp][0][0]);  // [0,16) m, [16,32) l, [32, ...) O
  const int dc = (lane & 3) * 2;
#pragma unroll
  for (int jt = 0; jt < 16; ++jt) {
    *reinterpret_cast<float2 *>(&st[32 + h0 * kD + jt * 8 + dc]) = make_float2(o[jt][0], o[jt][1]);
    *reinterpret_cast<float2 *>(&st[32 + (h0 + 8) * kD + jt * 8 + dc]) = make_float2(o[jt][2], o[jt][3]);
  }
  if ((lane & 3) == 0) {
    st[h0] = m0;
    st[h0 + 8] = m1;
    st[16 + h0] = l0;
    st[16 + h0 + 8] = l1;
  }
  // ---- combine across the cluster through distributed shared memory: CTA
  // c finalises heads 2c, 2c + 1; thread = (head, 2 d); fixed warp order
  cluster_sync_all();
  {
    const int hh = 2 * (int)crank + (threadIdx.x >> 6), d = (threadIdx.x & 63) * 2;
    const uint32_t st_local = tc::smem_u32(ring[0][0][0]);
    constexpr uint32_t kWarpBytes = kDStages * 2 * kDTile;
    float mv[kDCl * kDW];
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDCl * kDW; ++w) {
      const uint32_t ra = mapa_u32(st_local + (w % kDW) * kWarpBytes + hh * 4, w / kDW);
      mv[w] = ld_cluster_f32(ra);
      M = fmaxf(M, mv[w]);
    }
    float Ls = 0.f, ox = 0.f, oy = 0.f;
#pragma unroll
    for (int w = 0; w < kDCl * kDW; ++w) {
      const uint32_t base = mapa_u32(st_local + (w % kDW) * kWarpBytes, w / kDW);
      const float wt = mv[w] == -INFINITY ? 0.f : fast_exp2(mv[w] - M);
      const float lw = ld_cluster_f32(base + (16 + hh) * 4);
      const float2 ow = ld_cluster_f32x2(base + (32 + hh * kD + d) * 4);
      Ls += lw * wt;
      ox += ow.x * wt;
      oy += ow.y * wt;
    }
    if (L >= 1) {
      const float inv = 1.f / Ls;
      __nv_bfloat16 *dst = o_out + ((int64_t)seq * a.h_q + g * kG + hh) * kD + d;
      *reinterpret_cast<__nv_bfloat162 *>(dst) = __floats2bfloat162_rn(ox * inv, oy * inv);
      if ((threadIdx.x & 63) == 0) lse_out[(int64_t)seq * a.h_q + g * kG + hh] = (M + __log2f(Ls)) * 0.6931471805599453f;
    } else {  // empty slot: defined outputs (O = 0, lse = -inf), nothing was read
      __nv_bfloat16 *dst = o_out + ((int64_t)seq * a.h_q + g * kG + hh) * kD + d;
      *reinterpret_cast<__nv_bfloat162 *>(dst) = __floats2bfloat162_rn(0.f, 0.f);
      if ((threadIdx.x & 63) == 0) lse_out[(int64_t)seq * a.h_q + g * kG + hh] = -INFINITY;
    }
  }
  cluster_sync_all();  // peers' shared memory stays valid until every read is done
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
  int p1_splits, tiles, max_ctx;
  int64_t ld;
  size_t off_p1, off_scmp, off_flags, off_topk, off_cnt, off_count, off_rows, off_part, total;
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
  D.ld = ((n_cols + 3) / 4) * 4 + 4;
  const int64_t rows = (int64_t)batch * cfg->h_kv;
  size_t o = 0;
  D.off_p1 = o; o = al(o + rows * D.p1_splits * kG * sizeof(float2));
  D.off_scmp = o; o = al(o + rows * D.ld * sizeof(float));
  D.off_flags = o; o = al(o + rows * D.tiles * sizeof(uint64_t));
  D.off_topk = o; o = al(o + rows * std::max(cfg->k_top, 1) * sizeof(int32_t));
  D.off_cnt = o; o = al(o + rows * sizeof(int32_t));
  D.off_count = o; o = al(o + 16);
  D.off_rows = o; o = al(o + 2 * rows * sizeof(int32_t));  // row ids + k-th keys
  D.off_part = o; o = al(o + rerank_partials_bytes());
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

int64_t swattn_decode_reranked_offset(const swattn_config *cfg, int32_t batch, int32_t max_pages) {
  if (cfg == nullptr || batch < 1 || max_pages < 1) return -1;
  return (int64_t)decode_layout(cfg, batch, max_pages).off_count;
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

int32_t swattn_kcache_append_tokens(const swattn_config *cfg, const swattn_paged_kv *kv,
                                    const void *K, const void *V, const int32_t *active,
                                    int32_t batch, void *stream) {
  int32_t rc = check_decode(cfg, kv, batch);
  if (rc) return rc;
  if (!K || !V) {
    set_error("K and V must be non-null");
    return SWATTN_EINVAL;
  }
  if (cfg->h_kv * kD > 1024) {
    set_error("h_kv * d_h > 1024 threads per sequence");
    return SWATTN_EUNSUPPORTED;
  }
  if (batch == 0) return SWATTN_OK;
  DecodeArgs a = make_args(cfg, kv, nullptr, batch);
  kcache_append_tokens_kernel<<<batch, cfg->h_kv * kD, 0, static_cast<cudaStream_t>(stream)>>>(
      a, static_cast<const __nv_bfloat16 *>(K), static_cast<const __nv_bfloat16 *>(V), active,
      const_cast<int32_t *>(kv->seq_lens));
  SWATTN_LAUNCH_CHECK("kcache_append_tokens_kernel");
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
  DecodeArgs a = make_args(cfg, kv, q, batch);
  const int nrows = batch * cfg->h_kv;
  {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(decode_pass1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2Smem);
      attr = true;
    }
    decode_pass1_kernel<<<dim3(nrows, kP1Ctas), 128, kP2Smem, st>>>(a, p1, D.p1_splits, count);
  }
  SWATTN_LAUNCH_CHECK("decode_pass1_kernel");
  uint64_t *flags = reinterpret_cast<uint64_t *>(ws + D.off_flags);
  {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(decode_pass2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kP2Smem);
      attr = true;
    }
    launch_pdl(decode_pass2_kernel, dim3(nrows, kP2Ctas), dim3(128), kP2Smem, st, a, p1, D.p1_splits,
               scmp, D.ld, flags, D.tiles);
  }
  SWATTN_LAUNCH_CHECK("decode_pass2_kernel");
  if ((rc = launch_decode_topk(cfg, scmp, D.ld, kv->seq_lens, batch, D.max_ctx, topk, cnt, count,
                               rows, nrows, flags, D.tiles, st)))
    return rc;
  if ((rc = launch_rerank_decode(cfg, q, kv->kc1, kv->kc2, kv->max_m1, kv->max_m2, kv->seq_lens,
                                 batch, scmp, D.ld, count, rows, nrows, topk, ws + D.off_part,
                                 num_sms_dec(), st)))
    return rc;
  {
    const int smem = kDW * kDStages * 2 * kDTile + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(decode_attn_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    AttnMaps maps;
    {
      // the pools as (d lo/hi 64, pool row, half, group), rows = num_pages * 64
      const int64_t pages = kv->num_pages > 0 ? kv->num_pages : (int64_t)batch * kv->max_pages;
      const uint64_t dims[4] = {64, (uint64_t)(pages * kB), 2, (uint64_t)cfg->h_kv};
      const uint64_t str[3] = {(uint64_t)cfg->h_kv * kD * 2, 128, (uint64_t)kD * 2};
      const uint32_t box[4] = {64, (uint32_t)kDStageKeys, 2, 1};
      if (!make_tmap_bf16(&maps.k, kv->k_pages, 4, dims, str, box) ||
          !make_tmap_bf16(&maps.v, kv->v_pages, 4, dims, str, box)) {
        set_error("cuTensorMapEncodeTiled(page pools) failed");
        return SWATTN_ECUDA;
      }
    }
    // one cluster of kDCl CTAs per (sequence, group) row; the split states
    // are combined in distributed shared memory (no partial-O round trip
    // through HBM, no combine kernel)
    launch_pdl(decode_attn_cluster_kernel, dim3(kDCl, nrows), dim3(kDW * 32), smem, st, a,
               (const int32_t *)topk, (const int32_t *)cnt, static_cast<__nv_bfloat16 *>(o), lse, maps);
    SWATTN_LAUNCH_CHECK("decode_attn_cluster_kernel");
  }
  return SWATTN_OK;
}

}  // extern "C"
