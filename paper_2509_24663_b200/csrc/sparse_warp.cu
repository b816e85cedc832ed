// K4 part B -- per-token top-k block attention, one warp per token (sm_100a).
//
// Part A (attention_tc.cu, mode 2) already folded every token's init + local
// blocks -- shared by the 64 tokens of a query block -- into (O_A, m_A, l_A).
// The top-k blocks are chosen per token (selection.py:123-126), so each warp
// owns one token at a time: its 16 query heads are exactly the M = 16 of a
// warp-level mma.sync.m16n8k16, so
//
//   S [16 heads x 16 keys] = Q_t [16 x 128] . K_stage^T     (8 k-steps x 2 n-tiles)
//   O [16 heads x 128 d]  += P [16 x 16 keys] . V_stage     (1 k-step x 16 n-tiles)
//
// with Q_t in registers for the whole token, P built in registers straight
// from the S accumulators (no shared-memory round trip), and O accumulated in
// registers.  Why not tcgen05 here: with N = 16 every tcgen05.mma costs
// ~80 cycles of issue/operand overhead regardless of N (tools/mma_bench.cu),
// i.e. ~400 MAC/clk/SM, while mma.sync sustains 1024 MAC/clk/SM
// (tools/mmasync_bench.cu) and needs no TMEM/mbarrier handoff between warps.
//
// The softmax offset is Part A's row max m_A (fixed for the token: no
// rescaling): p = exp2(s*c - m_A).  The merge O = (O_A l_A + O_B) / (l_A + l_B),
// lse = m_A + log2(l_A + l_B) completes sparse_forward (sparse.py:70-91).  A
// token whose logits exceed m_A by more than 2^64 is listed for the CUDA-core
// exact path (never on sane inputs).
//
// Data movement: each warp streams its token's selected blocks as 16-key
// stages (K and V, 4 KB each, one 4-D TMA box per tensor, 128-byte swizzle)
// through its own 2-stage mbarrier ring; lane 0 is the warp's TMA issuer, so
// a CTA has 12 independent issuers (a single issuing thread caps near
// 36 GB/s, tools/gather_bench.cu).  The ring runs across token boundaries.
// Q fragments are loaded straight from global memory (L2) into registers,
// which frees the Q smem slot: 12 warps x 2 stages (192 KB, 168 registers)
// measured best (tools/probe_partb.sh, profiles/r01c_partb_probe.txt:
// w12 34.3 ms, w10 37.4, w8 35.6, w8 + TMA'd Q 37.7, w8 x 3 stages 40.2,
// w6 x 4 stages 46.0 at 128K) -- deeper rings lose, more warps win.
// Roofline: the L2->SMEM gather of 2 x cnt x 16 KB per (token, group).
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

// geometry (overridable for tuning sweeps: tools/build_variants.sh EXTRA=-D...)
#ifndef SWATTN_PW_WARPS
#define SWATTN_PW_WARPS 12
#endif
#ifndef SWATTN_PW_STAGES
#define SWATTN_PW_STAGES 2
#endif
#ifndef SWATTN_PW_QGLOBAL
#define SWATTN_PW_QGLOBAL 1  // Q fragments straight from global memory (0: TMA into a Q smem slot)
#endif
#ifndef SWATTN_PW_IPW
#define SWATTN_PW_IPW 0  // items (tokens) per warp; 0 = persistent grid of num_sms CTAs
#endif
#ifndef SWATTN_PW_STAGE_KEYS
#define SWATTN_PW_STAGE_KEYS 16
#endif
constexpr int kWarps = SWATTN_PW_WARPS;
constexpr int kThreads = kWarps * 32;
constexpr int kStages = SWATTN_PW_STAGES;
constexpr int kStageKeys = SWATTN_PW_STAGE_KEYS;
constexpr int kBlk = 64;
constexpr int kStagesPerBlock = kBlk / kStageKeys;       // 4
constexpr uint32_t kTileBytes = kStageKeys * kD * 2;     // 4 KB (K or V of one stage)
constexpr uint32_t kQBytes = kG * kD * 2;                // 4 KB
constexpr float kOverflowSum = 1.8446744073709552e19f;  // 2^64

struct PwParams {
  CUtensorMap q_map;  // Q as (d lo/hi 64, head, half, token): box {64, 16, 2, 1}
  CUtensorMap k_map;  // K as (d lo/hi 64, token, half, group): box {64, 16, 2, 1}
  CUtensorMap v_map;
  int64_t n;
  int h_q, h_kv, k_top, g0;
  int64_t tok0, tok1;  // tokens [tok0, tok1) of this launch (all have top-k blocks)
  int64_t n_items;     // h_kv * (tok1 - tok0)
  const int32_t *topk, *topk_cnt;
  const float *m_a, *l_a;  // part A row statistics [n][h_q] (log2 max, sum)
  const __nv_bfloat16 *Q;  // [n][h_q][d] (QGLOBAL variant)
  __nv_bfloat16 *O;        // in: O_A (normalised), out: final
  float *lse;
  float scale_log2;
  int32_t *slow_count, *slow_list;
  const uint8_t *routed;  // [h_kv][ntiles] tiles finished by the FA tile (route.cuh), or null
  int64_t ntiles;
  const int32_t *plan;    // route plan: plan[1] = CTAs that work (the rest exit at once), or null
};

struct __align__(1024) WarpSmem {
  uint8_t k[kStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
#if !SWATTN_PW_QGLOBAL
  uint8_t q[kQBytes];
#endif
};
struct __align__(1024) PwSmem {
  WarpSmem w[kWarps];
  uint64_t full[kWarps][kStages];
  uint64_t qfull[kWarps];
};

__device__ __forceinline__ void item_of(const PwParams &p, int64_t it, int &g, int64_t &t) {
  const int64_t per = p.tok1 - p.tok0;
  g = p.g0 + (int)(it / per);
  t = p.tok0 + it % per;
}

// Tiles are stored [d half][row][64] (the tensor maps list the half after the
// row dimension), so the 8 rows of an ldmatrix 8x8 matrix fall on 8
// consecutive 128-byte lines and the 128-byte swizzle spreads them over all
// banks.  Byte offset of 16-byte chunk `c` (0..15, i.e. d / 8) of `row` in a
// tile of `rows` rows:
template <int kRows>
__device__ __forceinline__ uint32_t swz(int row, int c) {
  const int line = (c >> 3) * kRows + row;
  return (uint32_t)(line * 128 + (((c & 7) ^ (line & 7)) << 4));
}

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

// Per-warp stream of (token, stage) work: the producer side of the warp's
// ring.  Lane l holds block ids l and l+32 of the token.
struct Stream {
  int64_t it, step;  // step = working CTAs x warps
  int cnt, s, id0, id1, g;
  int64_t t;
  __device__ void load(const PwParams &p, int lane) {
    for (; it < p.n_items; it += step) {
      item_of(p, it, g, t);
      const int64_t row = (int64_t)g * p.n + t;
      cnt = p.topk_cnt[row];
      if (cnt > 0 && p.routed != nullptr && p.routed[(int64_t)g * p.ntiles + t / 8]) cnt = 0;
      if (cnt > 0) {
        const int32_t *b = p.topk + row * p.k_top;
        id0 = lane < p.k_top ? b[lane] : 0;
        id1 = lane + 32 < p.k_top ? b[lane + 32] : 0;
        s = 0;
        return;
      }
    }
  }
  __device__ bool valid(const PwParams &p) const { return it < p.n_items; }
  __device__ int block() const {  // warp-collective
    const int j = s / kStagesPerBlock;
    return __shfl_sync(0xffffffffu, j < 32 ? id0 : id1, j & 31);
  }
  __device__ void advance(const PwParams &p, int lane) {
    if (++s == cnt * kStagesPerBlock) {
      it += step;
      load(p, lane);
    }
  }
};

__global__ void __launch_bounds__(kThreads, 1) sparse_pw_kernel(const __grid_constant__ PwParams p) {
  extern __shared__ uint8_t smem_raw[];
  PwSmem &sm = *reinterpret_cast<PwSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Routed tiles run concurrently on the SMs this launch leaves free: every
  // CTA releases the dependent (programmatic) launch at once, and the CTAs
  // beyond the plan's count exit so their SMs take the FA tile's CTAs.
  pdl_launch_dependents();
  const int ctas = p.plan != nullptr ? p.plan[1] : (int)gridDim.x;
  if ((int)blockIdx.x >= ctas) return;
  const int64_t step = (int64_t)ctas * kWarps;
  WarpSmem &ws = sm.w[warp];
  uint64_t *full = sm.full[warp];
  uint64_t *qfull = &sm.qfull[warp];
  if (lane == 0) {
    for (int i = 0; i < kStages; ++i) tc::mbar_init(&full[i], 1);
    tc::mbar_init(qfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&p.q_map);
    tc::tma_prefetch(&p.k_map);
    tc::tma_prefetch(&p.v_map);
  }
  __syncwarp();

  // ---- producer cursor: prime the ring and the first Q
  Stream prod;
  prod.it = (int64_t)blockIdx.x * kWarps + warp;
  prod.step = step;
  prod.load(p, lane);
  if (!prod.valid(p)) return;
  uint32_t issued = 0;  // stages issued (ring position; only its low bits matter)
  auto issue = [&]() {
    const int blk = prod.block();
    if (lane == 0) {
      const int st = (int)(issued % kStages);
      const int row0 = blk * kBlk + (prod.s % kStagesPerBlock) * kStageKeys;
      tc::mbar_arrive_expect_tx(&full[st], 2 * kTileBytes);
      tc::tma_load_4d(&p.k_map, &full[st], ws.k[st], 0, row0, 0, prod.g);
      tc::tma_load_4d(&p.v_map, &full[st], ws.v[st], 0, row0, 0, prod.g);
    }
    ++issued;
    prod.advance(p, lane);
  };
#if !SWATTN_PW_QGLOBAL
  if (lane == 0) {
    tc::mbar_arrive_expect_tx(qfull, kQBytes);
    tc::tma_load_4d(&p.q_map, qfull, ws.q, 0, prod.g * kG, 0, (int)prod.t);
  }
#endif
  for (int i = 0; i < kStages && prod.valid(p); ++i) issue();

  const uint32_t kbase = tc::smem_u32(ws.k[0]), vbase = tc::smem_u32(ws.v[0]);
#if !SWATTN_PW_QGLOBAL
  const uint32_t qaddr = tc::smem_u32(ws.q);
#endif
  const int h0 = lane >> 2;  // rows (heads) h0 and h0 + 8 of every fragment
  // ldmatrix lane roles: matrix m = lane / 8, row-in-matrix = lane % 8
  const int lm = lane >> 3, lr = lane & 7;
  uint32_t consumed = 0;
  int64_t qphase = 0;
  Stream cons;
  cons.it = (int64_t)blockIdx.x * kWarps + warp;
  cons.step = step;
  cons.load(p, lane);
  while (cons.valid(p)) {
    const int64_t row = (int64_t)cons.g * p.n + cons.t;
    const int64_t ridx = cons.t * p.h_q + cons.g * kG;  // [n][h_q] row of head 0
    // ---- Q fragments (A operand, 16 heads x 128 d) for the whole token
    uint32_t qa[8][4];
#if SWATTN_PW_QGLOBAL
    {
      // a0 = (head h0, d 16 ks + 2 (lane & 3)), a1 = head h0 + 8, a2/a3 = d + 8
      const uint32_t *qg = reinterpret_cast<const uint32_t *>(p.Q + ridx * kD);
      const int dw = lane & 3;  // 32-bit word within the 8-column group
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qa[ks][0] = __ldg(qg + h0 * (kD / 2) + ks * 8 + dw);
        qa[ks][1] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + dw);
        qa[ks][2] = __ldg(qg + h0 * (kD / 2) + ks * 8 + 4 + dw);
        qa[ks][3] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + 4 + dw);
      }
    }
#else
    tc::mbar_wait(qfull, (uint32_t)(qphase & 1));
    ++qphase;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      // matrices: (heads 0-7, d lo), (heads 8-15, d lo), (heads 0-7, d hi), (heads 8-15, d hi)
      const int head = (lm & 1) * 8 + lr;
      ldsm_x4(qaddr + swz<kG>(head, ks * 2 + (lm >> 1)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    // next token's Q streams in while this token computes
    {
      Stream nx = cons;
      nx.it += nx.step;
      nx.load(p, lane);
      __syncwarp();
      if (lane == 0 && nx.valid(p)) {
        tc::fence_proxy_async();
        tc::mbar_arrive_expect_tx(qfull, kQBytes);
        tc::tma_load_4d(&p.q_map, qfull, ws.q, 0, nx.g * kG, 0, (int)nx.t);
      }
    }
#endif
    const float mA0 = p.m_a[ridx + h0], mA1 = p.m_a[ridx + h0 + 8];
    float lp0 = 0.f, lp1 = 0.f;
    float o[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

    const int nst = cons.cnt * kStagesPerBlock;
    for (int s = 0; s < nst; ++s, ++consumed) {
      const int st = (int)(consumed % kStages);
      tc::mbar_wait(&full[st], (consumed / kStages) & 1u);
      const uint32_t kst = kbase + st * kTileBytes, vst = vbase + st * kTileBytes;
#pragma unroll
      for (int sub = 0; sub < kStageKeys / 16; ++sub) {
      // ---- S = Q K^T over 16 keys: n-tiles (keys 0-7, 8-15)
      float sc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        // matrices: (keys 0-7, d lo), (keys 0-7, d hi), (keys 8-15, d lo), (keys 8-15, d hi)
        uint32_t b00, b01, b10, b11;
        ldsm_x4(kst + swz<kStageKeys>(sub * 16 + (lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), b00, b01, b10, b11);
        mma16816(sc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b00, b01);
        mma16816(sc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b10, b11);
      }
      // ---- fixed-offset softmax: rows h0 (c0, c1) and h0 + 8 (c2, c3)
      float x[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        x[j][0] = fmaf(sc[j][0], p.scale_log2, -mA0);
        x[j][1] = fmaf(sc[j][1], p.scale_log2, -mA0);
        x[j][2] = fmaf(sc[j][2], p.scale_log2, -mA1);
        x[j][3] = fmaf(sc[j][3], p.scale_log2, -mA1);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[j][e] = fast_exp2(x[j][e]);
        lp0 += x[j][0] + x[j][1];
        lp1 += x[j][2] + x[j][3];
      }
      const uint32_t pa0 = tc::pack_bf16(x[0][0], x[0][1]), pa1 = tc::pack_bf16(x[0][2], x[0][3]);
      const uint32_t pa2 = tc::pack_bf16(x[1][0], x[1][1]), pa3 = tc::pack_bf16(x[1][2], x[1][3]);
      // ---- O += P V over 16 keys: 16 d n-tiles, V fragments via ldmatrix.trans
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        // matrices: (keys 0-7, d tile 2dp), (keys 8-15, d tile 2dp),
        //           (keys 0-7, d tile 2dp+1), (keys 8-15, d tile 2dp+1)
        uint32_t v00, v01, v10, v11;
        ldsm_x4_t(vst + swz<kStageKeys>(sub * 16 + (lm & 1) * 8 + lr, dp * 2 + (lm >> 1)), v00, v01, v10, v11);
        mma16816(o[2 * dp], pa0, pa1, pa2, pa3, v00, v01);
        mma16816(o[2 * dp + 1], pa0, pa1, pa2, pa3, v10, v11);
      }
      }
      // ---- refill this slot with the stage kStages ahead (ring runs across tokens)
      __syncwarp();
      if (prod.valid(p)) {
        if (lane == 0) tc::fence_proxy_async();
        issue();
      }
    }

    // ---- per-token epilogue: merge with part A
    lp0 += __shfl_xor_sync(0xffffffffu, lp0, 1);
    lp0 += __shfl_xor_sync(0xffffffffu, lp0, 2);
    lp1 += __shfl_xor_sync(0xffffffffu, lp1, 1);
    lp1 += __shfl_xor_sync(0xffffffffu, lp1, 2);
    // overflow guard without a per-element max: any logit more than 64
    // (log2) above m_A makes its p > 2^64, so the row sum exceeds it too
    // (the test is conservative: huge sums of smaller p's are caught as well)
    const bool big = !(lp0 <= kOverflowSum) || !(lp1 <= kOverflowSum);  // also inf / NaN
    if (__any_sync(0xffffffffu, big) && lane == 0) {
      const int slot = atomicAdd(p.slow_count, 1);
      p.slow_list[slot] = (int32_t)row;
    }
    const float lA0 = p.l_a[ridx + h0], lA1 = p.l_a[ridx + h0 + 8];
    const float lt0 = lA0 + lp0, lt1 = lA1 + lp1;
    const float i0 = 1.f / lt0, i1 = 1.f / lt1;
    __nv_bfloat16 *o0 = p.O + (ridx + h0) * kD, *o1 = p.O + (ridx + h0 + 8) * kD;
    const int dc = (lane & 3) * 2;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int d = j * 8 + dc;
      const __nv_bfloat162 a0 = *reinterpret_cast<const __nv_bfloat162 *>(o0 + d);
      const __nv_bfloat162 a1 = *reinterpret_cast<const __nv_bfloat162 *>(o1 + d);
      const float2 f0 = __bfloat1622float2(a0), f1 = __bfloat1622float2(a1);
      *reinterpret_cast<__nv_bfloat162 *>(o0 + d) =
          __floats2bfloat162_rn((f0.x * lA0 + o[j][0]) * i0, (f0.y * lA0 + o[j][1]) * i0);
      *reinterpret_cast<__nv_bfloat162 *>(o1 + d) =
          __floats2bfloat162_rn((f1.x * lA1 + o[j][2]) * i1, (f1.y * lA1 + o[j][3]) * i1);
    }
    if ((lane & 3) == 0) {
      p.lse[ridx + h0] = (mA0 + __log2f(lt0)) * 0.6931471805599453f;
      p.lse[ridx + h0 + 8] = (mA1 + __log2f(lt1)) * 0.6931471805599453f;
    }
    cons.it += cons.step;
    cons.load(p, lane);
  }
}

}  // namespace

int32_t launch_sparse_part_b(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                             int64_t n, int64_t r0, int64_t r1, const int32_t *topk, const int32_t *topk_cnt,
                             const float *m_a, const float *l_a, void *O, float *lse,
                             int32_t *slow_count, int32_t *slow_list, int num_sms,
                             cudaStream_t stream, const uint8_t *routed, const int32_t *plan) {
  PwParams p;
  memset(&p, 0, sizeof(p));
  {
    const uint64_t dims[4] = {64, (uint64_t)cfg->h_q, 2, (uint64_t)n};
    const uint64_t str[3] = {(uint64_t)kD * 2, 128, (uint64_t)cfg->h_q * kD * 2};
    const uint32_t box[4] = {64, (uint32_t)kG, 2, 1};
    if (!make_tmap_bf16(&p.q_map, Q, 4, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(Q) failed");
      return SWATTN_ECUDA;
    }
  }
  {
    const uint64_t dims[4] = {64, (uint64_t)n, 2, (uint64_t)cfg->h_kv};
    const uint64_t str[3] = {(uint64_t)cfg->h_kv * kD * 2, 128, (uint64_t)kD * 2};
    const uint32_t box[4] = {64, (uint32_t)kStageKeys, 2, 1};
    if (!make_tmap_bf16(&p.k_map, K, 4, dims, str, box) ||
        !make_tmap_bf16(&p.v_map, V, 4, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(K/V) failed");
      return SWATTN_ECUDA;
    }
  }
  p.n = n;
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  p.k_top = cfg->k_top;
  p.tok0 = (int64_t)(cfg->N_init + cfg->N_local) * cfg->B;
  if (p.tok0 < r0) p.tok0 = r0;
  p.tok1 = r1;
  if (p.tok0 >= r1 || cfg->k_top == 0) return SWATTN_OK;
  const GroupRange gr = group_range(cfg);
  p.g0 = gr.g0;
  p.n_items = (int64_t)gr.gc * (r1 - p.tok0);
  p.topk = topk;
  p.topk_cnt = topk_cnt;
  p.m_a = m_a;
  p.l_a = l_a;
  p.Q = static_cast<const __nv_bfloat16 *>(Q);
  p.O = static_cast<__nv_bfloat16 *>(O);
  p.lse = lse;
  p.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  p.slow_count = slow_count;
  p.slow_list = slow_list;
  p.routed = routed;
  p.plan = plan;
  p.ntiles = cdiv(n, 8);
  const size_t smem = sizeof(PwSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sparse_pw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t per_cta = kWarps;
  int64_t grid = (p.n_items + per_cta - 1) / per_cta;
#if SWATTN_PW_IPW > 0
  // non-persistent: CTAs retire, so kernels on other streams can share SMs
  grid = (p.n_items + per_cta * SWATTN_PW_IPW - 1) / (per_cta * SWATTN_PW_IPW);
#else
  if (grid > num_sms) grid = num_sms;
#endif
  sparse_pw_kernel<<<(unsigned)grid, kThreads, smem, stream>>>(p);
  SWATTN_LAUNCH_CHECK("sparse_pw_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
