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

namespace swattn {

int32_t launch_decode_topk(const swattn_config *, const float *, int64_t, const int32_t *, int, int,
                           int32_t *, int32_t *, int32_t *, int32_t *, int32_t, cudaStream_t);
int32_t launch_rerank_decode(const swattn_config *, const void *, const void *, const void *,
                             int max_m1, int max_m2, const int32_t *seq_lens, int batch,
                             const float *, int64_t, const int32_t *, const int32_t *, int32_t,
                             int32_t *, void *, int, cudaStream_t);
size_t rerank_partials_bytes();

namespace {

constexpr int kP1Cols = 128;     // normaliser columns per pass-1 CTA (4 warps x 32)
constexpr int kTileBlocks = 31;  // pass-2 tile: 31 blocks, 124 (+4) columns
constexpr int kTileCols = 128;
constexpr int kAttnBlocks = 4;   // visible blocks per split-KV warp (24 splits at batch 16)

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

__global__ void __launch_bounds__(128) decode_pass1_kernel(DecodeArgs a, float2 *part, int splits) {
  __shared__ float2 red[4][kG];
  const int row = blockIdx.x, seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t vis2 = vis_count(L - 1, a.l_C2, a.s_C2);
  const int64_t vis1 = vis_count(L - 1, a.l_C1, a.s_C1);
  const bool use2 = vis2 > 0;
  const int64_t vis = use2 ? vis2 : vis1;  // fallback rows use the exact C1 lse
  const __nv_bfloat16 *kc = (use2 ? a.kc2 : a.kc1) + ((int64_t)seq * (use2 ? a.max_m2 : a.max_m1) * a.h_kv + g) * kD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = lane >> 2, dw = lane & 3;
  const int64_t col0 = (int64_t)blockIdx.y * 128 + warp * 32;
  float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;  // heads r, r + 8
  if (col0 < vis) {
    const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.q + (((int64_t)seq * a.h_q + g * kG + r) * kD));
    const uint32_t *q1 = q0 + 8 * (kD / 2);
    uint32_t qa[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = __ldg(q0 + ks * 8 + dw);
      qa[ks][1] = __ldg(q1 + ks * 8 + dw);
      qa[ks][2] = __ldg(q0 + ks * 8 + 4 + dw);
      qa[ks][3] = __ldg(q1 + ks * 8 + 4 + dw);
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const int64_t col = col0 + nt * 8 + r;
      const bool ok = col < vis;
      const uint32_t *kr = reinterpret_cast<const uint32_t *>(kc + (ok ? col : 0) * a.h_kv * kD);
      uint32_t kb[8][2];
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        kb[ks][0] = ok ? __ldg(kr + ks * 8 + dw) : 0u;
        kb[ks][1] = ok ? __ldg(kr + ks * 8 + 4 + dw) : 0u;
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) mma16816_p1(acc, qa[ks], kb[ks][0], kb[ks][1]);
      // columns 2 dw, 2 dw + 1 of this n-tile
      const int64_t c = col0 + nt * 8 + 2 * dw;
      const bool v0 = c < vis, v1 = c + 1 < vis;
      const float x0 = v0 ? acc[0] * a.scale_log2 : -INFINITY, x1 = v1 ? acc[1] * a.scale_log2 : -INFINITY;
      const float x2 = v0 ? acc[2] * a.scale_log2 : -INFINITY, x3 = v1 ? acc[3] * a.scale_log2 : -INFINITY;
      const float mm0 = fmaxf(x0, x1), mm1 = fmaxf(x2, x3);
      if (mm0 != -INFINITY) merge_ml(m0, l0, mm0, fast_exp2(x0 - mm0) + fast_exp2(x1 - mm0));
      if (mm1 != -INFINITY) merge_ml(m1, l1, mm1, fast_exp2(x2 - mm1) + fast_exp2(x3 - mm1));
    }
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
  __syncthreads();
  if (threadIdx.x < kG) {
    const int h = threadIdx.x;
    float M = -INFINITY, S = 0.f;
    for (int w = 0; w < 4; ++w) merge_ml(M, S, red[w][h].x, red[w][h].y);
    part[((int64_t)row * splits + blockIdx.y) * kG + h] = make_float2(M, S);
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

__global__ void __launch_bounds__(128) decode_pass2_kernel(DecodeArgs a, const float2 *part,
                                                           int splits, float *s_cmp, int64_t ld) {
  __shared__ __align__(128) uint8_t ktile[kTileCols * 256];  // 32 KB of C1 rows
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    // pass-1 partials of this row: only the slices pass 1 covered hold data
    // (C2 columns for approx rows, C1 for fallback rows); lane pairs (h, half)
    // merge half of the slices each, then one shuffle joins the halves
    const int64_t vis2 = vis_count(i, a.l_C2, a.s_C2);
    const int used = (int)min((int64_t)splits, cdiv(vis2 > 0 ? vis2 : vis1, (int64_t)kP1Cols));
    const int h = lane & 15, half = lane >> 4;
    float M = -INFINITY, S = 0.f;
    for (int sp = half; sp < used; sp += 2) {
      const float2 pv = part[((int64_t)row * splits + sp) * kG + h];
      if (pv.x == -INFINITY) continue;
      const float Mn = fmaxf(M, pv.x);
      S = (M == -INFINITY ? 0.f : S * fast_exp2(M - Mn)) + pv.y * fast_exp2(pv.x - Mn);
      M = Mn;
    }
    const float oM = __shfl_xor_sync(0xffffffffu, M, 16), oS = __shfl_xor_sync(0xffffffffu, S, 16);
    const float Mt = fmaxf(M, oM);
    float St = 0.f;
    if (Mt != -INFINITY)
      St = (M == -INFINITY ? 0.f : S * fast_exp2(M - Mt)) + (oM == -INFINITY ? 0.f : oS * fast_exp2(oM - Mt));
    if (half == 0) stat[h] = make_float2(Mt == -INFINITY ? 0.f : Mt, St > 0.f ? 1.f / St : 0.f);
  }
  // q as A fragments: a0 = (head r, d k), a1 = (r + 8, k), a2 = (r, k + 8), a3 = (r + 8, k + 8)
  const int r = lane >> 2, dw = lane & 3;
  const uint32_t *q0 = reinterpret_cast<const uint32_t *>(a.q + (((int64_t)seq * a.h_q + g * kG + r) * kD));
  const uint32_t *q1 = q0 + 8 * (kD / 2);
  uint32_t qa[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    qa[ks][0] = __ldg(q0 + ks * 8 + dw);
    qa[ks][1] = __ldg(q1 + ks * 8 + dw);
    qa[ks][2] = __ldg(q0 + ks * 8 + 4 + dw);
    qa[ks][3] = __ldg(q1 + ks * 8 + 4 + dw);
  }
  // the tile's 128 C1 rows -> shared memory by cp.async (256-byte rows, 16-byte
  // chunk c of row rr at c ^ (rr & 7): conflict-free ldmatrix), zeros past vis1
  const int64_t tile0 = (int64_t)t * kTileBlocks * kPoolS;
  const __nv_bfloat16 *kbase = a.kc1 + ((int64_t)seq * a.max_m1 * a.h_kv + g) * kD;
  const uint32_t kt = tc::smem_u32(ktile);
  for (int c = threadIdx.x; c < kTileCols * 16; c += blockDim.x) {
    const int rr = c >> 4, ch = c & 15;
    const uint32_t dst = kt + rr * 256 + (uint32_t)(((ch & 8) | ((ch & 7) ^ (rr & 7))) << 4);
    const int64_t col = tile0 + rr;
    if (col < vis1)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(kbase + col * a.h_kv * kD + ch * 8));
    else
      asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dst), "r"(0u));
  }
  asm volatile("cp.async.commit_group;");
  asm volatile("cp.async.wait_group 0;");
  const int64_t col0 = tile0 + warp * 32;
  float acc[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
  __syncthreads();  // tile and stat
  const int lm = lane >> 3, lr = lane & 7;
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

// ---- D5 on the tensor cores: one warp = (row, split of kAttnBlocks blocks);
// the row's 16 query heads are the M = 16 of mma.sync.m16n8k16 (as in the
// prefill part B, csrc/sparse_warp.cu): Q in registers, S -> P in registers,
// O in registers, online softmax per 16-key stage.  K/V rows are gathered
// from the page pool with cp.async into a per-warp 2-stage ring stored
// [d half][row][64] with the 16-byte chunk XOR-swizzled by row, so the
// ldmatrix reads are conflict-free.
constexpr int kDW = 4;                        // warps per CTA
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

__global__ void __launch_bounds__(kDW * 32) decode_attn_mma_kernel(DecodeArgs a, const int32_t *topk,
                                                                  const int32_t *topk_cnt,
                                                                  float *part_o, float2 *part_ml,
                                                                  int splits) {
  extern __shared__ uint8_t dsm_raw[];
  uint8_t *dsm = dsm_raw + ((1024u - (tc::smem_u32(dsm_raw) & 1023u)) & 1023u);
  auto ring = reinterpret_cast<uint8_t(*)[2][2][kDTile]>(dsm);  // [warp][stage][K|V]
  auto qs = reinterpret_cast<__nv_bfloat16(*)[kG * kD]>(dsm + kDW * 4 * kDTile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * kDW + warp;
  if (unit >= a.batch * a.h_kv * splits) return;
  const int row = unit / splits, split = unit % splits;
  const int seq = row / a.h_kv, g = row % a.h_kv;
  const int64_t L = a.seq_lens[seq];
  const int64_t i = L - 1;
  const int b = (int)(i / kB);
  const int n_init = min(a.N_init, b + 1);
  const int lo = max(0, b - a.N_local + 1);
  const int lo2 = max(lo, n_init);
  const int ntop = topk_cnt[row];
  // an empty slot (no cached token) has no visible block: no page is read
  const int nvis = L < 1 ? 0 : n_init + ntop + (b + 1 - lo2);
  const int32_t *top = topk + (int64_t)row * a.k_top;
  const int vb0 = split * kAttnBlocks, vb1 = min(nvis, vb0 + kAttnBlocks);
  const int64_t pi_base = ((int64_t)row * splits + split) * kG;
  const int h0 = lane >> 2;
  if (vb0 >= vb1) {
    if ((lane & 3) == 0) {
      part_ml[pi_base + h0] = make_float2(-INFINITY, 0.f);
      part_ml[pi_base + h0 + 8] = make_float2(-INFINITY, 0.f);
    }
    return;
  }
  // q rows of the group -> smem (row-major, 256 B) -> A fragments
  const __nv_bfloat16 *qg = a.q + ((int64_t)seq * a.h_q + g * kG) * kD;
  for (int e = lane; e < kG * kD / 8; e += 32)
    reinterpret_cast<uint4 *>(qs[warp])[e] = reinterpret_cast<const uint4 *>(qg)[e];
  __syncwarp();
  const int lm = lane >> 3, lr = lane & 7;
  uint32_t qa[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    // matrices: (heads 0-7, d lo), (heads 8-15, d lo), (heads 0-7, d hi), (heads 8-15, d hi)
    const int head = (lm & 1) * 8 + lr, d = ks * 16 + (lm >> 1) * 8;
    const uint32_t addr = tc::smem_u32(&qs[warp][head * kD + d]);
    dldsm_x4(addr, qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], false);
  }
  // stage s of this warp's key stream: block vb0 + s / 4, rows (s % 4) * 16 ..
  const int nst = (vb1 - vb0) * (kB / kDStageKeys);
  auto issue = [&](int st_idx, int slot) {
    const int j = visible_block(vb0 + st_idx / 4, n_init, ntop, top, lo2);
    const int page = a.block_table[(int64_t)seq * a.max_pages + j];
    const int r0 = (st_idx % 4) * kDStageKeys;
    // 16 rows x 16 chunks of 16 B per tensor: 8 per lane
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = e * 32 + lane, rr = idx >> 4, c = idx & 15;
      const int64_t off = (((int64_t)page * kB + r0 + rr) * a.h_kv + g) * kD + c * 8;
      const uint32_t dk = tc::smem_u32(ring[warp][slot][0]) + dswz(rr, c);
      const uint32_t dv = tc::smem_u32(ring[warp][slot][1]) + dswz(rr, c);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk), "l"(a.k_pages + off));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dv), "l"(a.v_pages + off));
    }
    asm volatile("cp.async.commit_group;");
  };
  issue(0, 0);
  if (nst > 1) issue(1, 1);
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  for (int s2 = 0; s2 < nst; ++s2) {
    const int slot = s2 & 1;
    if (s2 + 1 < nst) asm volatile("cp.async.wait_group 1;");
    else asm volatile("cp.async.wait_group 0;");
    __syncwarp();
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
    const int j = visible_block(vb0 + s2 / 4, n_init, ntop, top, lo2);
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
    __syncwarp();
    if (s2 + 2 < nst) issue(s2 + 2, slot);
  }
  // partial row sums over the quad, then the partial state of this split
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const int dc = (lane & 3) * 2;
#pragma unroll
  for (int jt = 0; jt < 16; ++jt) {
    *reinterpret_cast<float2 *>(&part_o[(pi_base + h0) * kD + jt * 8 + dc]) = make_float2(o[jt][0], o[jt][1]);
    *reinterpret_cast<float2 *>(&part_o[(pi_base + h0 + 8) * kD + jt * 8 + dc]) = make_float2(o[jt][2], o[jt][3]);
  }
  if ((lane & 3) == 0) {
    part_ml[pi_base + h0] = make_float2(m0, l0);
    part_ml[pi_base + h0 + 8] = make_float2(m1, l1);
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
  if (L < 1) {  // empty slot: defined outputs (O = 0, lse = -inf), nothing read
    o[((int64_t)seq * a.h_q + g * kG + h) * kD + 4 * lane + 0] = __float2bfloat16_rn(0.f);
    o[((int64_t)seq * a.h_q + g * kG + h) * kD + 4 * lane + 1] = __float2bfloat16_rn(0.f);
    o[((int64_t)seq * a.h_q + g * kG + h) * kD + 4 * lane + 2] = __float2bfloat16_rn(0.f);
    o[((int64_t)seq * a.h_q + g * kG + h) * kD + 4 * lane + 3] = __float2bfloat16_rn(0.f);
    if (lane == 0) lse[(int64_t)seq * a.h_q + g * kG + h] = -INFINITY;
    return;
  }
  const int b = (int)((L - 1) / kB);
  const int n_init = min(a.N_init, b + 1);
  const int lo2 = max(max(0, b - a.N_local + 1), n_init);
  const int nvis = n_init + topk_cnt[row] + (b + 1 - lo2);
  const int used = (int)cdiv(nvis, kAttnBlocks);  // <= 24 splits (96 blocks / 4)
  // lane s holds split s's (max, sum): one load, then warp reductions
  float2 ml = make_float2(-INFINITY, 0.f);
  if (lane < used) ml = part_ml[((int64_t)row * splits + lane) * kG + h];
  float M = ml.x;
#pragma unroll
  for (int off = 16; off; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const float wl = ml.x == -INFINITY ? 0.f : fast_exp2(ml.x - M);
  float Ls = ml.y * wl;
#pragma unroll
  for (int off = 16; off; off >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, off);
  // the splits' partial O rows are independent loads (4 in flight)
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int sp = 0; sp < used; ++sp) {
    const float w = __shfl_sync(0xffffffffu, wl, sp);
    const int64_t pi = ((int64_t)row * splits + sp) * kG + h;
    const float4 po = *reinterpret_cast<const float4 *>(&part_o[pi * kD + 4 * lane]);
    if (w != 0.f) {
      acc[0] += po.x * w;
      acc[1] += po.y * w;
      acc[2] += po.z * w;
      acc[3] += po.w * w;
    }
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
  size_t off_p1, off_scmp, off_topk, off_cnt, off_count, off_rows, off_part, off_po, off_pml, total;
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
  D.off_rows = o; o = al(o + 2 * rows * sizeof(int32_t));  // row ids + k-th keys
  D.off_part = o; o = al(o + rerank_partials_bytes());
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
  decode_pass1_kernel<<<dim3(nrows, D.p1_splits), 128, 0, st>>>(a, p1, D.p1_splits);
  SWATTN_LAUNCH_CHECK("decode_pass1_kernel");
  decode_pass2_kernel<<<dim3(nrows, D.tiles), 128, 0, st>>>(a, p1, D.p1_splits, scmp, D.ld);
  SWATTN_LAUNCH_CHECK("decode_pass2_kernel");
  if ((rc = cuda_check(cudaMemsetAsync(count, 0, 4, st), "memset"))) return rc;
  if ((rc = launch_decode_topk(cfg, scmp, D.ld, kv->seq_lens, batch, D.max_ctx, topk, cnt, count,
                               rows, nrows, st)))
    return rc;
  if ((rc = launch_rerank_decode(cfg, q, kv->kc1, kv->kc2, kv->max_m1, kv->max_m2, kv->seq_lens,
                                 batch, scmp, D.ld, count, rows, nrows, topk, ws + D.off_part,
                                 num_sms_dec(), st)))
    return rc;
  {
    const int units = nrows * D.attn_splits;
    const int smem = kDW * 4 * kDTile + kDW * kG * kD * 2 + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(decode_attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    decode_attn_mma_kernel<<<(units + kDW - 1) / kDW, kDW * 32, smem, st>>>(a, topk, cnt, po, pml,
                                                                           D.attn_splits);
    SWATTN_LAUNCH_CHECK("decode_attn_mma_kernel");
  }
  decode_combine_kernel<<<nrows, 512, 0, st>>>(a, cnt, po, pml, D.attn_splits,
                                               static_cast<__nv_bfloat16 *>(o), lse);
  SWATTN_LAUNCH_CHECK("decode_combine_kernel");
  return SWATTN_OK;
}

}  // extern "C"
