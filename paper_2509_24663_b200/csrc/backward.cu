// Sparse attention backward (sparse.py:130-185) on sm_100a: gradients of
// sum(O * dO) through the masked softmax over each row's visible blocks
// (init U local U top-k, selection.py:113-133), recomputing P from the
// forward lse.  No gradient flows into the selection.
//
//   B0  delta[i, h] = sum_d dO[i,h,d] O[i,h,d]                       (:169)
//   B1  dQ: one warp per (token, group), exactly the forward part-B warp
//       (Q and dO fragments in registers, a 2-stage TMA ring of 16-key K/V
//       stages per warp) over all visible blocks:
//         S = Q K^T, P = exp(S scale - lse), dP = dO V^T,
//         dS = P (dP - delta), dQ += dS K                       (:171-177)
//   B2  (group, key block, query) pairs of every visible (token, block),
//       radix-sorted by (group, block, token) -> per key block, the queries
//       that see it in ascending order;
//   B3  dK / dV: CTA = one segment of <= kSeg queries of one key block, warp
//       = 16 keys: S^T = K_w Q_i^T, P^T, dP^T = V_w dO_i^T,
//         dV_w += P^T dO_i, dK_w += dS^T Q_i                    (:178-179)
//       with Q_i / dO_i double-buffered in shared memory (cp.async); fp32
//       partials per segment;
//   B4  dK / dV = sum of a block's segment partials in segment order.
// Every reduction has a fixed order (no floating-point atomics), so repeated
// runs are bitwise identical (the reference's promise, sparse.py:139-143);
// the order differs from the reference's serial float64 loop, so results
// agree within bf16 tolerance, not bitwise.
#include <string.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

constexpr int kBlk = 64;
constexpr int kStageKeys = 16;
constexpr int kStagesPerBlock = kBlk / kStageKeys;
constexpr uint32_t kTileBytes = kStageKeys * kD * 2;  // 4 KB
#ifndef SWATTN_BWD_QWARPS
#define SWATTN_BWD_QWARPS 8
#endif
constexpr int kQWarps = SWATTN_BWD_QWARPS;             // B1 warps per CTA
constexpr int kQStages = 2;
constexpr int kSeg = 1024;                             // B3 queries per segment
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                        uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                          uint32_t &r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// TMA tile [d half][row][64] with the 128-byte swizzle (as sparse_warp.cu)
template <int kRows>
__device__ __forceinline__ uint32_t swz(int row, int c) {
  const int line = (c >> 3) * kRows + row;
  return (uint32_t)(line * 128 + (((c & 7) ^ (line & 7)) << 4));
}
// cp.async tile [row][128 d] (256-byte rows, 16-byte chunk c of row r at c ^ (r & 7))
__device__ __forceinline__ uint32_t swz256(int row, int c) {
  return (uint32_t)(row * 256 + (((c & 8) | ((c & 7) ^ (row & 7))) << 4));
}

// A fragments (16 rows x 128) of a row-major bf16 matrix in global memory
// (row stride `ld` elements): a0 = (r, k), a1 = (r + 8, k), a2 = (r, k + 8),
// a3 = (r + 8, k + 8) with r = lane / 4, k = 16 ks + 2 (lane % 4).
__device__ __forceinline__ void load_a_global(const __nv_bfloat16 *base, int64_t ld, int rows_ok,
                                              uint32_t (&a)[8][4]) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, dw = lane & 3;
  const uint32_t *r0 = reinterpret_cast<const uint32_t *>(base + (int64_t)r * ld);
  const uint32_t *r1 = reinterpret_cast<const uint32_t *>(base + (int64_t)(r + 8) * ld);
  const bool ok0 = r < rows_ok, ok1 = r + 8 < rows_ok;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    a[ks][0] = ok0 ? __ldg(r0 + ks * 8 + dw) : 0u;
    a[ks][1] = ok1 ? __ldg(r1 + ks * 8 + dw) : 0u;
    a[ks][2] = ok0 ? __ldg(r0 + ks * 8 + 4 + dw) : 0u;
    a[ks][3] = ok1 ? __ldg(r1 + ks * 8 + 4 + dw) : 0u;
  }
}

// Visible blocks of row i (selection.py:113-133): local [lo, b], then the
// init blocks below lo, then the top-k list (disjoint from both).
struct RowBlocks {
  int lo, nl, ni, nt;
  __device__ int count() const { return nl + ni + nt; }
};
// mode: 0 sparse (init U local U top-k), 1 dense causal ([0, b]), 2 dense
// non-causal (every block of the nb) -- dense.py:173-221
__device__ __forceinline__ RowBlocks row_blocks(int64_t i, int B, int N_init, int N_local, int cnt,
                                                int mode = 0, int nb = 0) {
  RowBlocks r;
  const int b = (int)(i / B);
  if (mode != 0) {
    r.lo = 0;
    r.nl = mode == 1 ? b + 1 : nb;
    r.ni = 0;
    r.nt = 0;
    return r;
  }
  r.lo = max(0, b - N_local + 1);
  r.nl = b - r.lo + 1;
  r.ni = min(N_init, r.lo);
  r.nt = cnt;
  return r;
}

// ------------------------------------------------------------------ B0
__global__ void bwd_delta_kernel(const __nv_bfloat16 *__restrict__ O, const __nv_bfloat16 *__restrict__ dO,
                                 int64_t rows, float *__restrict__ delta) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint2 o = *reinterpret_cast<const uint2 *>(O + row * kD + lane * 4);
  const uint2 g = *reinterpret_cast<const uint2 *>(dO + row * kD + lane * 4);
  const __nv_bfloat162 *o2 = reinterpret_cast<const __nv_bfloat162 *>(&o);
  const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&g);
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float2 a = __bfloat1622float2(o2[e]), c = __bfloat1622float2(g2[e]);
    s = fmaf(a.x, c.x, fmaf(a.y, c.y, s));
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) delta[row] = s;
}

// ------------------------------------------------------------------ B1
struct DqParams {
  CUtensorMap k_map, v_map;  // as sparse_warp.cu: box {64, 16 keys, 2, 1}
  const __nv_bfloat16 *Q, *dO;
  const float *lse, *delta;
  const int32_t *topk, *topk_cnt;
  __nv_bfloat16 *dQ;
  int64_t n;
  int h_q, h_kv, k_top, B, N_init, N_local, mode, nb;
  float scale, scale_log2;
};

struct __align__(1024) DqWarpSmem {
  uint8_t k[kQStages][kTileBytes];
  uint8_t v[kQStages][kTileBytes];
};
struct __align__(1024) DqSmem {
  DqWarpSmem w[kQWarps];
  uint64_t full[kQWarps][kQStages];
};

// per-warp stream of (item, stage): item = g * n + i, blocks of row_blocks()
struct DqStream {
  int64_t it, n_items;
  int g;
  int64_t t;
  RowBlocks rb;
  int s, id0, id1;  // topk ids: lane l holds entries l and l + 32
  __device__ void load(const DqParams &p, int lane) {
    for (; it < n_items; it += (int64_t)gridDim.x * kQWarps) {
      g = (int)(it / p.n);
      t = it % p.n;
      const int64_t row = (int64_t)g * p.n + t;
      rb = row_blocks(t, p.B, p.N_init, p.N_local, p.mode == 0 ? p.topk_cnt[row] : 0, p.mode, p.nb);
      const int32_t *tk = p.topk + (p.mode == 0 ? row * p.k_top : 0);
      id0 = lane < rb.nt ? tk[lane] : 0;
      id1 = lane + 32 < rb.nt ? tk[lane + 32] : 0;
      s = 0;
      return;
    }
  }
  __device__ bool valid() const { return it < n_items; }
  __device__ int block() const {  // warp-collective
    const int j = s / kStagesPerBlock;
    int blk;
    if (j < rb.nl) blk = rb.lo + j;
    else if (j < rb.nl + rb.ni) blk = j - rb.nl;
    else {
      const int q = j - rb.nl - rb.ni;
      blk = __shfl_sync(0xffffffffu, q < 32 ? id0 : id1, q & 31);
    }
    return blk;
  }
  __device__ void advance(const DqParams &p, int lane) {
    if (++s == rb.count() * kStagesPerBlock) {
      it += (int64_t)gridDim.x * kQWarps;
      load(p, lane);
    }
  }
};

__global__ void __launch_bounds__(kQWarps * 32, 1) bwd_dq_kernel(const __grid_constant__ DqParams p) {
  extern __shared__ uint8_t smem_raw[];
  DqSmem &sm = *reinterpret_cast<DqSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DqWarpSmem &ws = sm.w[warp];
  uint64_t *full = sm.full[warp];
  if (lane == 0) {
    for (int i = 0; i < kQStages; ++i) tc::mbar_init(&full[i], 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&p.k_map);
    tc::tma_prefetch(&p.v_map);
  }
  __syncwarp();
  const int64_t n_items = (int64_t)p.h_kv * p.n;
  DqStream prod;
  prod.n_items = n_items;
  prod.it = (int64_t)blockIdx.x * kQWarps + warp;
  prod.load(p, lane);
  if (!prod.valid()) return;
  int64_t issued = 0;
  auto issue = [&]() {
    const int blk = prod.block();
    if (lane == 0) {
      const int st = (int)(issued % kQStages);
      const int row0 = blk * kBlk + (prod.s % kStagesPerBlock) * kStageKeys;
      tc::mbar_arrive_expect_tx(&full[st], 2 * kTileBytes);
      tc::tma_load_4d(&p.k_map, &full[st], ws.k[st], 0, row0, 0, prod.g);
      tc::tma_load_4d(&p.v_map, &full[st], ws.v[st], 0, row0, 0, prod.g);
    }
    ++issued;
    prod.advance(p, lane);
  };
  for (int i = 0; i < kQStages && prod.valid(); ++i) issue();

  const uint32_t kbase = tc::smem_u32(ws.k[0]), vbase = tc::smem_u32(ws.v[0]);
  const int h0 = lane >> 2;
  const int lm = lane >> 3, lr = lane & 7;
  int64_t consumed = 0;
  DqStream cons;
  cons.n_items = n_items;
  cons.it = (int64_t)blockIdx.x * kQWarps + warp;
  cons.load(p, lane);
  while (cons.valid()) {
    const int64_t t = cons.t;
    const int64_t ridx = t * p.h_q + cons.g * kG;  // [n][h_q] row of head 0
    uint32_t qa[8][4], ga[8][4];
    load_a_global(p.Q + ridx * kD, kD, kG, qa);
    load_a_global(p.dO + ridx * kD, kD, kG, ga);
    const float l0 = p.lse[ridx + h0] * kLog2e, l1 = p.lse[ridx + h0 + 8] * kLog2e;
    const float d0 = p.delta[ridx + h0], d1 = p.delta[ridx + h0 + 8];
    float dq[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
    const int nst = cons.rb.count() * kStagesPerBlock;
    for (int s = 0; s < nst; ++s, ++consumed) {
      const int st = (int)(consumed % kQStages);
      // key index of this stage's column 0 (for the causal / length mask)
      const int64_t key0 = (int64_t)cons.block() * kBlk + (s % kStagesPerBlock) * kStageKeys;
      cons.s = s + 1;  // keep block() in step with the stage (advance() not used here)
      tc::mbar_wait(&full[st], (uint32_t)((consumed / kQStages) & 1));
      const uint32_t kst = kbase + st * kTileBytes, vst = vbase + st * kTileBytes;
      float sc[2][4], dp[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) sc[j][e] = dp[j][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b00, b01, b10, b11, c00, c01, c10, c11;
        ldsm_x4(kst + swz<kStageKeys>((lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), b00, b01, b10, b11);
        ldsm_x4(vst + swz<kStageKeys>((lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), c00, c01, c10, c11);
        mma16816(sc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b00, b01);
        mma16816(sc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b10, b11);
        mma16816(dp[0], ga[ks][0], ga[ks][1], ga[ks][2], ga[ks][3], c00, c01);
        mma16816(dp[1], ga[ks][0], ga[ks][1], ga[ks][2], ga[ks][3], c10, c11);
      }
      // dS = P (dP - delta), P = exp2(S scale log2e - lse log2e); invisible keys -> 0
      float ds[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t key = key0 + j * 8 + 2 * (lane & 3) + (e & 1);
          const bool vis = (p.mode == 2 || key <= t) && key < p.n;
          const float lse2 = e < 2 ? l0 : l1, dl = e < 2 ? d0 : d1;
          const float pr = vis ? fast_exp2(fmaf(sc[j][e], p.scale_log2, -lse2)) : 0.f;
          ds[j][e] = pr * (dp[j][e] - dl);
        }
      }
      const uint32_t pa0 = tc::pack_bf16(ds[0][0], ds[0][1]), pa1 = tc::pack_bf16(ds[0][2], ds[0][3]);
      const uint32_t pa2 = tc::pack_bf16(ds[1][0], ds[1][1]), pa3 = tc::pack_bf16(ds[1][2], ds[1][3]);
      // dQ += dS K over the 16 keys: K fragments by ldmatrix.trans ([key][d] = [k][n])
#pragma unroll
      for (int dpi = 0; dpi < 8; ++dpi) {
        uint32_t k00, k01, k10, k11;
        ldsm_x4_t(kst + swz<kStageKeys>((lm & 1) * 8 + lr, dpi * 2 + (lm >> 1)), k00, k01, k10, k11);
        mma16816(dq[2 * dpi], pa0, pa1, pa2, pa3, k00, k01);
        mma16816(dq[2 * dpi + 1], pa0, pa1, pa2, pa3, k10, k11);
      }
      __syncwarp();
      if (prod.valid()) {
        if (lane == 0) tc::fence_proxy_async();
        issue();
      }
    }
    // dQ = dS K * scale (sparse.py:176)
    __nv_bfloat16 *q0 = p.dQ + (ridx + h0) * kD, *q1 = p.dQ + (ridx + h0 + 8) * kD;
    const int dc = (lane & 3) * 2;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int d = j * 8 + dc;
      *reinterpret_cast<__nv_bfloat162 *>(q0 + d) = __floats2bfloat162_rn(dq[j][0] * p.scale, dq[j][1] * p.scale);
      *reinterpret_cast<__nv_bfloat162 *>(q1 + d) = __floats2bfloat162_rn(dq[j][2] * p.scale, dq[j][3] * p.scale);
    }
    cons.it += (int64_t)gridDim.x * kQWarps;
    cons.load(p, lane);
  }
}

// ------------------------------------------------------------------ B2
// key = (g * nb + block) << 32 | query
__global__ void bwd_pair_count_kernel(int64_t n, int h_kv, int B, int N_init, int N_local, int mode,
                                      int nb, const int32_t *__restrict__ topk_cnt,
                                      int64_t *__restrict__ cnt) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= (int64_t)h_kv * n) return;
  const int64_t i = it % n;
  cnt[it] = row_blocks(i, B, N_init, N_local, mode == 0 ? topk_cnt[it] : 0, mode, nb).count();
}

__global__ void bwd_pair_fill_kernel(int64_t n, int h_kv, int B, int N_init, int N_local, int k_top,
                                     int mode, int64_t nb, const int32_t *__restrict__ topk,
                                     const int32_t *__restrict__ topk_cnt,
                                     const int64_t *__restrict__ off, uint64_t *__restrict__ keys,
                                     int32_t *__restrict__ blk_count) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= (int64_t)h_kv * n) return;
  const int g = (int)(it / n);
  const int64_t i = it % n;
  const RowBlocks rb = row_blocks(i, B, N_init, N_local, mode == 0 ? topk_cnt[it] : 0, mode, (int)nb);
  uint64_t *out = keys + off[it];
  const int32_t *tk = topk + (mode == 0 ? it * k_top : 0);
  const int c = rb.count();
  for (int j = 0; j < c; ++j) {
    int blk;
    if (j < rb.nl) blk = rb.lo + j;
    else if (j < rb.nl + rb.ni) blk = j - rb.nl;
    else blk = tk[j - rb.nl - rb.ni];
    const int64_t gb = (int64_t)g * nb + blk;
    out[j] = ((uint64_t)gb << 32) | (uint64_t)i;
    atomicAdd(&blk_count[gb], 1);  // integer counts: order-independent
  }
}

// segment table: seg_off[gb] = first segment of key block gb (exclusive scan
// of ceil(count / kSeg)); one entry per segment = (gb, pair begin, pair end)
__global__ void bwd_seg_count_kernel(int64_t n_gb, const int32_t *__restrict__ blk_count,
                                     int32_t *__restrict__ nseg) {
  const int64_t gb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gb < n_gb) nseg[gb] = (blk_count[gb] + kSeg - 1) / kSeg;
}

struct Seg {
  int32_t gb;
  int32_t pos;  // segment index within its block
  int64_t begin, end;
};

__global__ void bwd_seg_fill_kernel(int64_t n_gb, const int32_t *__restrict__ blk_count,
                                    const int64_t *__restrict__ blk_off,
                                    const int32_t *__restrict__ seg_off, Seg *__restrict__ segs) {
  const int64_t gb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gb >= n_gb) return;
  const int c = blk_count[gb];
  const int ns = (c + kSeg - 1) / kSeg;
  for (int s = 0; s < ns; ++s) {
    Seg sg;
    sg.gb = (int32_t)gb;
    sg.pos = s;
    sg.begin = blk_off[gb] + (int64_t)s * kSeg;
    sg.end = blk_off[gb] + min((int64_t)c, (int64_t)(s + 1) * kSeg);
    segs[seg_off[gb] + s] = sg;
  }
}

// ------------------------------------------------------------------ B3
struct DkvParams {
  const __nv_bfloat16 *Q, *K, *V, *dO;
  const float *lse, *delta;
  const uint64_t *keys;  // sorted pairs
  const Seg *segs;
  const int32_t *n_segs;  // device total
  float *part;            // [segment][2][64][128] fp32 (dK, dV partials)
  int64_t n, nb;
  int h_q, h_kv, mode;
  float scale_log2;
};

constexpr int kKvWarps = 4;  // 16 keys each
constexpr int kKvBuf = 4;    // queries in flight (cp.async prefetch depth): the
                             // L2 -> smem latency exceeds one query's compute
struct __align__(128) DkvSmem {
  uint8_t q[kKvBuf][kG * kD * 2];   // 4 KB each, [head][d] swizzled (swz256)
  uint8_t go[kKvBuf][kG * kD * 2];
  __align__(16) float lse[kKvBuf][kG];  // natural log, as stored by the forward
  __align__(16) float delta[kKvBuf][kG];
  int32_t tok[kSeg];                    // the segment's queries, ascending
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}

__global__ void __launch_bounds__(kKvWarps * 32) bwd_dkdv_kernel(const __grid_constant__ DkvParams p) {
  extern __shared__ __align__(128) uint8_t dkv_smem[];
  DkvSmem &sm = *reinterpret_cast<DkvSmem *>(dkv_smem);
  const int seg_id = blockIdx.x;
  if (seg_id >= *p.n_segs) return;
  const Seg sg = p.segs[seg_id];
  const int g = (int)(sg.gb / p.nb);
  const int64_t blk = sg.gb % p.nb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t key_w = blk * kBlk + warp * 16;  // first key of this warp
  // K_w / V_w as A fragments (16 keys x 128 d), rows past n read as zero
  uint32_t ka[8][4], va[8][4];
  const int rows_ok = (int)max((int64_t)0, min((int64_t)16, p.n - key_w));
  load_a_global(p.K + (key_w * p.h_kv + g) * kD, (int64_t)p.h_kv * kD, rows_ok, ka);
  load_a_global(p.V + (key_w * p.h_kv + g) * kD, (int64_t)p.h_kv * kD, rows_ok, va);
  float dk[16][4], dv[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[j][e] = dv[j][e] = 0.f;

  const int64_t npairs = sg.end - sg.begin;
  // the segment's query ids once into shared memory (no dependent global
  // load on the per-query path)
  for (int t = threadIdx.x; t < npairs; t += blockDim.x)
    sm.tok[t] = (int32_t)(p.keys[sg.begin + t] & 0xffffffffull);
  __syncthreads();
  auto stage = [&](int64_t pi, int buf) {  // all 128 threads: Q_i, dO_i, lse_i, delta_i of group g
    const int64_t i = sm.tok[pi];
    const __nv_bfloat16 *qs = p.Q + (i * p.h_q + g * kG) * kD;
    const __nv_bfloat16 *gs = p.dO + (i * p.h_q + g * kG) * kD;
    for (int c = threadIdx.x; c < kG * 16; c += blockDim.x) {  // 16-byte chunks
      const int r = c >> 4, ch = c & 15;
      cp_async16(tc::smem_u32(sm.q[buf]) + swz256(r, ch), qs + r * kD + ch * 8);
      cp_async16(tc::smem_u32(sm.go[buf]) + swz256(r, ch), gs + r * kD + ch * 8);
    }
    if (threadIdx.x < 8) {  // 16 lse + 16 delta floats: 8 x 16 bytes
      const int part = threadIdx.x & 3;
      const float *src = (threadIdx.x < 4 ? p.lse : p.delta) + i * p.h_q + g * kG + part * 4;
      float *dst = (threadIdx.x < 4 ? sm.lse[buf] : sm.delta[buf]) + part * 4;
      cp_async16(tc::smem_u32(dst), src);
    }
    asm volatile("cp.async.commit_group;");
  };
  // prologue: queries 0 .. kKvBuf-2 in flight (one commit group each, empty
  // groups past the end keep the group count uniform)
  for (int q = 0; q < kKvBuf - 1; ++q) {
    if (q < npairs) stage(q, q);
    else asm volatile("cp.async.commit_group;");
  }
  const int lm = lane >> 3, lr = lane & 7;
  for (int64_t pi = 0; pi < npairs; ++pi) {
    const int buf = (int)(pi % kKvBuf);
    const int64_t ahead = pi + kKvBuf - 1;
    if (ahead < npairs) stage(ahead, (int)(ahead % kKvBuf));
    else asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group %0;" ::"n"(kKvBuf - 1));  // query pi has landed
    __syncthreads();
    const int64_t i = sm.tok[pi];
    const uint32_t qb = tc::smem_u32(sm.q[buf]), gb_ = tc::smem_u32(sm.go[buf]);
    // S^T (16 keys x 16 heads) = K_w Q_i^T, dP^T = V_w dO_i^T
    float st[2][4], dpt[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      // B fragments: rows = heads (n), 16 d (k): matrices (heads 0-7, d lo),
      // (heads 0-7, d hi), (heads 8-15, d lo), (heads 8-15, d hi)
      uint32_t b00, b01, b10, b11, c00, c01, c10, c11;
      const int hr = (lm >> 1) * 8 + lr, ch = ks * 2 + (lm & 1);
      ldsm_x4(qb + swz256(hr, ch), b00, b01, b10, b11);
      ldsm_x4(gb_ + swz256(hr, ch), c00, c01, c10, c11);
      mma16816(st[0], ka[ks][0], ka[ks][1], ka[ks][2], ka[ks][3], b00, b01);
      mma16816(st[1], ka[ks][0], ka[ks][1], ka[ks][2], ka[ks][3], b10, b11);
      mma16816(dpt[0], va[ks][0], va[ks][1], va[ks][2], va[ks][3], c00, c01);
      mma16816(dpt[1], va[ks][0], va[ks][1], va[ks][2], va[ks][3], c10, c11);
    }
    // element (key r, head c): r = lane/4 (+8 for e >= 2), c = 8 j + 2 (lane%4) + (e&1)
    float pt[2][4], dst[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = j * 8 + 2 * (lane & 3) + (e & 1);
        const int64_t key = key_w + (lane >> 2) + (e >= 2 ? 8 : 0);
        const bool vis = (p.mode == 2 || key <= i) && key < p.n;
        const float pr = vis ? fast_exp2(fmaf(st[j][e], p.scale_log2, -sm.lse[buf][h] * kLog2e)) : 0.f;
        pt[j][e] = pr;
        dst[j][e] = pr * (dpt[j][e] - sm.delta[buf][h]);
      }
    }
    const uint32_t pa0 = tc::pack_bf16(pt[0][0], pt[0][1]), pa1 = tc::pack_bf16(pt[0][2], pt[0][3]);
    const uint32_t pa2 = tc::pack_bf16(pt[1][0], pt[1][1]), pa3 = tc::pack_bf16(pt[1][2], pt[1][3]);
    const uint32_t sa0 = tc::pack_bf16(dst[0][0], dst[0][1]), sa1 = tc::pack_bf16(dst[0][2], dst[0][3]);
    const uint32_t sa2 = tc::pack_bf16(dst[1][0], dst[1][1]), sa3 = tc::pack_bf16(dst[1][2], dst[1][3]);
    // dV_w += P^T dO_i, dK_w += dS^T Q_i: B = [head][d] = [k][n] -> ldmatrix.trans
#pragma unroll
    for (int dpi = 0; dpi < 8; ++dpi) {
      uint32_t g00, g01, g10, g11, q00, q01, q10, q11;
      const int hr = (lm & 1) * 8 + lr, ch = dpi * 2 + (lm >> 1);
      ldsm_x4_t(gb_ + swz256(hr, ch), g00, g01, g10, g11);
      ldsm_x4_t(qb + swz256(hr, ch), q00, q01, q10, q11);
      mma16816(dv[2 * dpi], pa0, pa1, pa2, pa3, g00, g01);
      mma16816(dv[2 * dpi + 1], pa0, pa1, pa2, pa3, g10, g11);
      mma16816(dk[2 * dpi], sa0, sa1, sa2, sa3, q00, q01);
      mma16816(dk[2 * dpi + 1], sa0, sa1, sa2, sa3, q10, q11);
    }
    __syncthreads();  // this buffer is refilled by the next iteration's prefetch
  }
  // partials: [seg][0 = dK, 1 = dV][64 keys][128 d]
  float *pk = p.part + (int64_t)seg_id * 2 * kBlk * kD;
  float *pv = pk + kBlk * kD;
  const int r0 = warp * 16 + (lane >> 2);
  const int dc = (lane & 3) * 2;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int d = j * 8 + dc;
    *reinterpret_cast<float2 *>(pk + r0 * kD + d) = make_float2(dk[j][0], dk[j][1]);
    *reinterpret_cast<float2 *>(pk + (r0 + 8) * kD + d) = make_float2(dk[j][2], dk[j][3]);
    *reinterpret_cast<float2 *>(pv + r0 * kD + d) = make_float2(dv[j][0], dv[j][1]);
    *reinterpret_cast<float2 *>(pv + (r0 + 8) * kD + d) = make_float2(dv[j][2], dv[j][3]);
  }
}

// ------------------------------------------------------------------ B4
__global__ void bwd_reduce_kernel(int64_t n, int64_t nb, int h_kv, const int32_t *__restrict__ seg_off,
                                  const int32_t *__restrict__ nseg, const float *__restrict__ part,
                                  float scale, __nv_bfloat16 *__restrict__ dK,
                                  __nv_bfloat16 *__restrict__ dV) {
  const int64_t gb = blockIdx.x;  // g * nb + block
  const int g = (int)(gb / nb);
  const int64_t blk = gb % nb;
  const int s0 = seg_off[gb], ns = nseg[gb];
  for (int e = threadIdx.x; e < kBlk * kD; e += blockDim.x) {
    const int r = e / kD, d = e % kD;
    const int64_t key = blk * kBlk + r;
    if (key >= n) continue;
    float ak = 0.f, av = 0.f;
    for (int s = 0; s < ns; ++s) {
      const float *pk = part + (int64_t)(s0 + s) * 2 * kBlk * kD;
      ak += pk[e];
      av += pk[kBlk * kD + e];
    }
    dK[(key * h_kv + g) * kD + d] = __float2bfloat16_rn(ak * scale);
    dV[(key * h_kv + g) * kD + d] = __float2bfloat16_rn(av);
  }
}

// ------------------------------------------------------------------ workspace
struct BwdLayout {
  int64_t items, nb, n_gb, max_pairs, max_segs;
  size_t off_delta, off_cnt, off_off, off_keys, off_keys_alt, off_blk_count, off_blk_off,
      off_nseg, off_seg_off, off_nsegs_total, off_segs, off_part, off_temp, temp_bytes, total;
};

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

BwdLayout bwd_layout(const swattn_config *cfg, int64_t n, int mode) {
  BwdLayout L{};
  L.items = (int64_t)cfg->h_kv * n;
  L.nb = cdiv(n, cfg->B);
  L.n_gb = (int64_t)cfg->h_kv * L.nb;
  const int64_t per_row = mode == 0 ? std::min<int64_t>(cfg->N_init + cfg->N_local + cfg->k_top, L.nb)
                                    : L.nb;
  L.max_pairs = L.items * per_row;
  L.max_segs = L.max_pairs / kSeg + L.n_gb + 1;
  // CUB temp storage (queried with null buffers; no device work)
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (int64_t *)nullptr, (int64_t *)nullptr, (int)L.items);
  cub::DoubleBuffer<uint64_t> db(nullptr, nullptr);
  cub::DeviceRadixSort::SortKeys(nullptr, t2, db, (int)L.max_pairs, 0, 64);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, (int32_t *)nullptr, (int64_t *)nullptr, (int)L.n_gb);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, (int32_t *)nullptr, (int32_t *)nullptr, (int)L.n_gb + 1);
  L.temp_bytes = std::max(std::max(t1, t2), std::max(t3, t4));
  size_t o = 0;
  L.off_delta = o; o = al(o + (size_t)n * cfg->h_q * 4);
  L.off_cnt = o; o = al(o + (size_t)L.items * 8);
  L.off_off = o; o = al(o + (size_t)(L.items + 1) * 8);
  L.off_keys = o; o = al(o + (size_t)L.max_pairs * 8);
  L.off_keys_alt = o; o = al(o + (size_t)L.max_pairs * 8);
  L.off_blk_count = o; o = al(o + (size_t)(L.n_gb + 1) * 4);
  L.off_blk_off = o; o = al(o + (size_t)(L.n_gb + 1) * 8);
  L.off_nseg = o; o = al(o + (size_t)(L.n_gb + 1) * 4);
  L.off_seg_off = o; o = al(o + (size_t)(L.n_gb + 1) * 4);
  L.off_nsegs_total = o; o = al(o + 16);
  L.off_segs = o; o = al(o + (size_t)L.max_segs * sizeof(Seg));
  L.off_part = o; o = al(o + (size_t)L.max_segs * 2 * kBlk * kD * 4);
  L.off_temp = o; o = al(o + L.temp_bytes);
  L.total = o;
  return L;
}

__global__ void bwd_total_segs_kernel(const int32_t *seg_off, const int32_t *nseg, int64_t n_gb,
                                      int32_t *total) {
  *total = seg_off[n_gb - 1] + nseg[n_gb - 1];
}

}  // namespace

size_t sparse_bwd_workspace_bytes(const swattn_config *cfg, int64_t n, int mode) {
  return bwd_layout(cfg, n, mode).total;
}

// mode 0: sparse (topk / topk_cnt), 1: dense causal, 2: dense non-causal
int32_t launch_sparse_bwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, const int32_t *topk, const int32_t *topk_cnt, const void *O,
                          const float *lse, const void *dO, void *dQ, void *dK, void *dV,
                          void *workspace, size_t workspace_bytes, int num_sms, int mode,
                          cudaStream_t st) {
  const BwdLayout L = bwd_layout(cfg, n, mode);
  if (workspace == nullptr || workspace_bytes < L.total) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, L.total);
    return SWATTN_EINVAL;
  }
  char *ws = static_cast<char *>(workspace);
  float *delta = reinterpret_cast<float *>(ws + L.off_delta);
  int64_t *cnt = reinterpret_cast<int64_t *>(ws + L.off_cnt);
  int64_t *off = reinterpret_cast<int64_t *>(ws + L.off_off);
  uint64_t *keys = reinterpret_cast<uint64_t *>(ws + L.off_keys);
  uint64_t *keys_alt = reinterpret_cast<uint64_t *>(ws + L.off_keys_alt);
  int32_t *blk_count = reinterpret_cast<int32_t *>(ws + L.off_blk_count);
  int64_t *blk_off = reinterpret_cast<int64_t *>(ws + L.off_blk_off);
  int32_t *nseg = reinterpret_cast<int32_t *>(ws + L.off_nseg);
  int32_t *seg_off = reinterpret_cast<int32_t *>(ws + L.off_seg_off);
  int32_t *n_segs = reinterpret_cast<int32_t *>(ws + L.off_nsegs_total);
  Seg *segs = reinterpret_cast<Seg *>(ws + L.off_segs);
  float *part = reinterpret_cast<float *>(ws + L.off_part);
  void *temp = ws + L.off_temp;
  const float scale = 1.f / sqrtf((float)cfg->d_h);
  int32_t rc;

  // B0
  {
    const int64_t rows = n * cfg->h_q;
    bwd_delta_kernel<<<(unsigned)cdiv(rows, 8), 256, 0, st>>>(
        static_cast<const __nv_bfloat16 *>(O), static_cast<const __nv_bfloat16 *>(dO), rows, delta);
    SWATTN_LAUNCH_CHECK("bwd_delta_kernel");
  }
  // B1
  {
    DqParams p;
    memset(&p, 0, sizeof(p));
    const uint64_t dims[4] = {64, (uint64_t)n, 2, (uint64_t)cfg->h_kv};
    const uint64_t str[3] = {(uint64_t)cfg->h_kv * kD * 2, 128, (uint64_t)kD * 2};
    const uint32_t box[4] = {64, (uint32_t)kStageKeys, 2, 1};
    if (!make_tmap_bf16(&p.k_map, K, 4, dims, str, box) || !make_tmap_bf16(&p.v_map, V, 4, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(K/V) failed");
      return SWATTN_ECUDA;
    }
    p.Q = static_cast<const __nv_bfloat16 *>(Q);
    p.dO = static_cast<const __nv_bfloat16 *>(dO);
    p.lse = lse;
    p.delta = delta;
    p.topk = topk;
    p.topk_cnt = topk_cnt;
    p.dQ = static_cast<__nv_bfloat16 *>(dQ);
    p.n = n;
    p.h_q = cfg->h_q;
    p.h_kv = cfg->h_kv;
    p.k_top = cfg->k_top;
    p.B = cfg->B;
    p.N_init = cfg->N_init;
    p.N_local = cfg->N_local;
    p.mode = mode;
    p.nb = (int)L.nb;
    p.scale = scale;
    p.scale_log2 = scale * kLog2e;
    const size_t smem = sizeof(DqSmem) + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    int64_t grid = cdiv(L.items, kQWarps);
    if (grid > num_sms) grid = num_sms;
    bwd_dq_kernel<<<(unsigned)grid, kQWarps * 32, smem, st>>>(p);
    SWATTN_LAUNCH_CHECK("bwd_dq_kernel");
  }
  // B2: pairs, sorted by (group, block, query)
  {
    const unsigned g1 = (unsigned)cdiv(L.items, 256);
    bwd_pair_count_kernel<<<g1, 256, 0, st>>>(n, cfg->h_kv, cfg->B, cfg->N_init, cfg->N_local,
                                              mode, (int)L.nb, topk_cnt, cnt);
    SWATTN_LAUNCH_CHECK("bwd_pair_count_kernel");
    size_t tb = L.temp_bytes;
    if ((rc = cuda_check(cub::DeviceScan::ExclusiveSum(temp, tb, cnt, off, (int)L.items, st), "scan(pairs)")))
      return rc;
    if ((rc = cuda_check(cudaMemsetAsync(blk_count, 0, (size_t)(L.n_gb + 1) * 4, st), "memset")))
      return rc;
    bwd_pair_fill_kernel<<<g1, 256, 0, st>>>(n, cfg->h_kv, cfg->B, cfg->N_init, cfg->N_local,
                                             cfg->k_top, mode, L.nb, topk, topk_cnt, off, keys,
                                             blk_count);
    SWATTN_LAUNCH_CHECK("bwd_pair_fill_kernel");
    // the pair count is data-dependent (top-k counts): sort the max_pairs
    // buffer? no -- sort exactly the filled prefix, whose length is off[items-1]
    // + cnt[items-1]; read it back once (the only host sync of the backward)
    int64_t last_off = 0, last_cnt = 0;
    if ((rc = cuda_check(cudaMemcpyAsync(&last_off, off + L.items - 1, 8, cudaMemcpyDeviceToHost, st), "d2h")) ||
        (rc = cuda_check(cudaMemcpyAsync(&last_cnt, cnt + L.items - 1, 8, cudaMemcpyDeviceToHost, st), "d2h")) ||
        (rc = cuda_check(cudaStreamSynchronize(st), "sync")))
      return rc;
    const int64_t npairs = last_off + last_cnt;
    int end_bit = 32;
    while (end_bit < 64 && ((uint64_t)L.n_gb >> (end_bit - 32)) != 0) ++end_bit;
    cub::DoubleBuffer<uint64_t> db(keys, keys_alt);
    tb = L.temp_bytes;
    if ((rc = cuda_check(cub::DeviceRadixSort::SortKeys(temp, tb, db, (int)npairs, 0, end_bit, st), "sort(pairs)")))
      return rc;
    keys = db.Current();
    tb = L.temp_bytes;
    if ((rc = cuda_check(cub::DeviceScan::ExclusiveSum(temp, tb, blk_count, blk_off, (int)L.n_gb, st), "scan(blocks)")))
      return rc;
    const unsigned g2 = (unsigned)cdiv(L.n_gb, 256);
    bwd_seg_count_kernel<<<g2, 256, 0, st>>>(L.n_gb, blk_count, nseg);
    SWATTN_LAUNCH_CHECK("bwd_seg_count_kernel");
    tb = L.temp_bytes;
    if ((rc = cuda_check(cub::DeviceScan::ExclusiveSum(temp, tb, nseg, seg_off, (int)L.n_gb, st), "scan(segments)")))
      return rc;
    bwd_seg_fill_kernel<<<g2, 256, 0, st>>>(L.n_gb, blk_count, blk_off, seg_off, segs);
    SWATTN_LAUNCH_CHECK("bwd_seg_fill_kernel");
    bwd_total_segs_kernel<<<1, 1, 0, st>>>(seg_off, nseg, L.n_gb, n_segs);
    SWATTN_LAUNCH_CHECK("bwd_total_segs_kernel");
    // B3: one CTA per segment (upper bound grid; idle CTAs exit)
    DkvParams q;
    q.Q = static_cast<const __nv_bfloat16 *>(Q);
    q.K = static_cast<const __nv_bfloat16 *>(K);
    q.V = static_cast<const __nv_bfloat16 *>(V);
    q.dO = static_cast<const __nv_bfloat16 *>(dO);
    q.lse = lse;
    q.delta = delta;
    q.keys = keys;
    q.segs = segs;
    q.n_segs = n_segs;
    q.part = part;
    q.n = n;
    q.nb = L.nb;
    q.h_q = cfg->h_q;
    q.h_kv = cfg->h_kv;
    q.mode = mode;
    q.scale_log2 = scale * kLog2e;
    const int64_t max_segs = npairs / kSeg + L.n_gb + 1;
    static bool dkv_attr = false;
    if (!dkv_attr) {
      cudaFuncSetAttribute(bwd_dkdv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(DkvSmem));
      dkv_attr = true;
    }
    bwd_dkdv_kernel<<<(unsigned)max_segs, kKvWarps * 32, sizeof(DkvSmem), st>>>(q);
    SWATTN_LAUNCH_CHECK("bwd_dkdv_kernel");
    // B4
    bwd_reduce_kernel<<<(unsigned)L.n_gb, 256, 0, st>>>(n, L.nb, cfg->h_kv, seg_off, nseg, part, scale,
                                                        static_cast<__nv_bfloat16 *>(dK),
                                                        static_cast<__nv_bfloat16 *>(dV));
    SWATTN_LAUNCH_CHECK("bwd_reduce_kernel");
  }
  return SWATTN_OK;
}

}  // namespace swattn
