// K4 part B -- per-token top-k block attention on tcgen05 (sm_100a).
//
// Part A (attention_tc.cu, mode 2) already folded every token's init + local
// blocks -- shared by the 64 tokens of a query block -- into (O_A, m_A, l_A).
// The top-k blocks are per token (selection.py:123-126), so they are walked
// token by token in the swap-AB orientation, which keeps M = 128 on the
// tensor core although one token only has 16 query rows (its 16 heads):
//
//   S^T [128 keys x 16 heads] = K_pair [128 x 128] . Q_t^T        (SS, K-major)
//   O^T [128 d    x 16 heads] += V_pair^T [128 x 128] . P_t^T     (SS, A MN-major)
//
// with a "pair" = two selected 64-key blocks gathered by TMA into one
// 128-row tile.  The softmax offset is Part A's row max m_A (fixed for the
// token, so no rescaling and no cross-lane max): p = exp2(s*c - m_A);
// per-lane partial row sums are reduced once per token.  The merge
// O = (O_A l_A + O_B) / (l_A + l_B), lse = m_A + log2(l_A + l_B) completes
// sparse_forward (sparse.py:70-91).  A token whose logits exceed m_A by more
// than 2^64 is listed for the CUDA-core exact path (never on sane inputs).
//
// Warp roles (256 threads, 1 CTA / SM, persistent over (group, token)):
//   warps 0..2 TMA producers -- warp w owns ring stage w (pairs p = w mod 3):
//              a single issuing thread tops out near 36 GB/s of TMA traffic
//              (tools/gather_bench.cu), so the gather needs several issuers;
//   warp 3     MMA issuer; warps 4..7 softmax + per-token epilogue.
// Roofline: bound by the L2->SMEM gather of 2 x 63 x 16 KB per token
// (K and V of the selected blocks); FLOP = 4 * 16 * 64 * d per block.
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

constexpr int kThreads = 256;
constexpr int kMmaWarp = 3;  // warps [0, kStages) produce, then MMA, then 4 softmax warps
constexpr int kStages = 3;
constexpr int kBlk = 64;
constexpr uint32_t kPairBytes = 2 * kBlk * kD * 2;  // 32 KB (K or V of two blocks)
constexpr uint32_t kQTokBytes = kG * kD * 2;          // 4 KB
constexpr uint32_t kPBytes = kG * 128 * 2;            // 4 KB
constexpr uint32_t kTmemCols = 64;                    // S0 S1 O0 O1 (16 each)
constexpr float kOverflowExcess = 64.f;

struct PbParams {
  CUtensorMap q_map;  // Q [n][h_q][d]: box {64, 16, 1}
  CUtensorMap k_map;  // K [n][h_kv*d]: box {64, 64}
  CUtensorMap v_map;
  int64_t n;
  int h_q, h_kv, k_top;
  int64_t tok0;        // first token with top-k blocks
  int64_t n_items;     // h_kv * (n - tok0)
  const int32_t *topk, *topk_cnt;
  const float *m_a, *l_a;  // part A row statistics [n][h_q] (log2 max, sum)
  __nv_bfloat16 *O;        // in: O_A (normalised), out: final
  float *lse;
  float scale_log2;
  int32_t *slow_count, *slow_list;
};

struct __align__(1024) PbSmem {
  uint8_t k[kStages][kPairBytes];
  uint8_t v[kStages][kPairBytes];
  uint8_t q[2][kQTokBytes];
  uint8_t p[2][kPBytes];
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2];
  uint64_t o_full[2], o_empty[2];
  float lred[4][kG];
  uint32_t tmem_base;
};

__device__ __forceinline__ void item_of(const PbParams &p, int64_t it, int &g, int64_t &t) {
  const int64_t per = p.n - p.tok0;
  g = (int)(it / per);
  t = p.tok0 + it % per;
}

__device__ __forceinline__ int cnt_of(const PbParams &p, int64_t it) {
  int g;
  int64_t t;
  item_of(p, it, g, t);
  return p.topk_cnt[(int64_t)g * p.n + t];
}

__global__ void __launch_bounds__(kThreads, 1) sparse_pb_kernel(const __grid_constant__ PbParams p) {
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on smem_raw so accesses stay in the shared space
  PbSmem &s = *reinterpret_cast<PbSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.k_full[i], 1);
      tc::mbar_init(&s.k_empty[i], 1);
      tc::mbar_init(&s.v_full[i], 1);
      tc::mbar_init(&s.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.q_full[i], 1);
      tc::mbar_init(&s.q_empty[i], 1);
      tc::mbar_init(&s.s_full[i], 1);
      tc::mbar_init(&s.s_empty[i], 128);
      tc::mbar_init(&s.p_full[i], 128);
      tc::mbar_init(&s.p_empty[i], 1);
      tc::mbar_init(&s.o_full[i], 1);
      tc::mbar_init(&s.o_empty[i], 128);
    }
    tc::fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc<kTmemCols>(&s.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp < kStages) {
    // ------------------------------------------------------------ TMA producers
    // Whole warp walks the items; lane l holds block ids l and l+32 of the
    // current token, fetched one token ahead so no dependent global load sits
    // between two TMA issues (an L2 round trip per pair halves the gather rate).
    if (lane == 0) {
      tc::tma_prefetch(&p.q_map);
      tc::tma_prefetch(&p.k_map);
      tc::tma_prefetch(&p.v_map);
    }
    int64_t pair = 0;
    int tau = 0;
    auto fetch = [&](int64_t item, int &cnt, int &id0, int &id1) {
      int g;
      int64_t t;
      item_of(p, item, g, t);
      const int64_t row = (int64_t)g * p.n + t;
      cnt = p.topk_cnt[row];
      const int32_t *blocks = p.topk + row * p.k_top;
      id0 = lane < p.k_top ? blocks[lane] : 0;
      id1 = lane + 32 < p.k_top ? blocks[lane + 32] : 0;
    };
    int cnt = 0, id0 = 0, id1 = 0;
    int64_t it = blockIdx.x;
    if (it < p.n_items) fetch(it, cnt, id0, id1);
    while (it < p.n_items) {
      const int64_t nit = it + gridDim.x;
      int ncnt = 0, nid0 = 0, nid1 = 0;
      if (nit < p.n_items) fetch(nit, ncnt, nid0, nid1);
      if (cnt > 0) {
        int g;
        int64_t t;
        item_of(p, it, g, t);
        const int qs = tau & 1;
        if (lane == 0 && warp == 0) {
          tc::mbar_wait(&s.q_empty[qs], ((tau >> 1) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&s.q_full[qs], kQTokBytes);
          for (int h = 0; h < 2; ++h)
            tc::tma_load_3d(&p.q_map, &s.q_full[qs], s.q[qs] + h * (kQTokBytes / 2), h * 64,
                            g * kG, (int)t);
        }
        const int npairs = (cnt + 1) >> 1;
        for (int pi = 0; pi < npairs; ++pi, ++pair) {
          const int x0 = 2 * pi, x1 = (2 * pi + 1 < cnt) ? 2 * pi + 1 : 2 * pi;  // odd tail: duplicate, masked
          const int b0 = __shfl_sync(0xffffffffu, x0 < 32 ? id0 : id1, x0 & 31);
          const int b1 = __shfl_sync(0xffffffffu, x1 < 32 ? id0 : id1, x1 & 31);
          if (lane == 0 && (int)(pair % kStages) == warp) {
            const int st = warp;
            const uint32_t ph = ((pair / kStages) & 1) ^ 1;
            tc::mbar_wait(&s.k_empty[st], ph);
            tc::mbar_arrive_expect_tx(&s.k_full[st], kPairBytes);
            for (int h = 0; h < 2; ++h) {
              uint8_t *dst = s.k[st] + h * (kPairBytes / 2);
              tc::tma_load_2d(&p.k_map, &s.k_full[st], dst, g * kD + h * 64, b0 * kBlk);
              tc::tma_load_2d(&p.k_map, &s.k_full[st], dst + kBlk * 128, g * kD + h * 64, b1 * kBlk);
            }
            tc::mbar_wait(&s.v_empty[st], ph);
            tc::mbar_arrive_expect_tx(&s.v_full[st], kPairBytes);
            for (int h = 0; h < 2; ++h) {
              uint8_t *dst = s.v[st] + h * (kPairBytes / 2);
              tc::tma_load_2d(&p.v_map, &s.v_full[st], dst, g * kD + h * 64, b0 * kBlk);
              tc::tma_load_2d(&p.v_map, &s.v_full[st], dst + kBlk * 128, g * kD + h * 64, b1 * kBlk);
            }
          }
          __syncwarp();
        }
        ++tau;
      }
      it = nit;
      cnt = ncnt;
      id0 = nid0;
      id1 = nid1;
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id_s = tc::idesc_bf16(128, kG, false, false);
    const uint32_t id_o = tc::idesc_bf16(128, kG, true, false);
    int64_t pair = 0;      // global pair counter (S issued)
    int tau = 0;
    // deferred PV of the previous pair
    bool pend = false;
    int64_t pend_pair = 0;
    bool pend_first = false, pend_last = false;
    int pend_tau = 0;
    auto issue_pv = [&]() {
      const int st = (int)(pend_pair % kStages);
      const int pb = (int)(pend_pair & 1);
      tc::mbar_wait(&s.p_full[pb], (pend_pair >> 1) & 1);
      tc::mbar_wait(&s.v_full[st], (pend_pair / kStages) & 1);
      if (pend_first) tc::mbar_wait(&s.o_empty[pend_tau & 1], ((pend_tau >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t v_addr = tc::smem_u32(s.v[st]);
        const uint32_t p_addr = tc::smem_u32(s.p[pb]);
        const uint32_t d_o = tmem + 32 + (pend_tau & 1) * kG;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc::mma_ss(d_o, tc::desc_mnmajor(v_addr + kk * 16 * 128, kPairBytes / 2),
                     tc::desc_kmajor(p_addr + (kk >> 2) * (kPBytes / 2) + (kk & 3) * 32), id_o,
                     (!pend_first || kk > 0) ? 1u : 0u);
        tc::mma_commit(&s.v_empty[st]);
        tc::mma_commit(&s.p_empty[pb]);
        if (pend_last) tc::mma_commit(&s.o_full[pend_tau & 1]);
      }
      __syncwarp();
      pend = false;
    };
    int cnt_next = blockIdx.x < p.n_items ? cnt_of(p, blockIdx.x) : 0;
    for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      int g;
      int64_t t;
      item_of(p, it, g, t);
      const int cnt = cnt_next;  // fetched one item ahead
      cnt_next = it + gridDim.x < p.n_items ? cnt_of(p, it + gridDim.x) : 0;
      if (cnt == 0) continue;
      const int npairs = (cnt + 1) >> 1;
      const int qs = tau & 1;
      tc::mbar_wait(&s.q_full[qs], (tau >> 1) & 1);
      for (int pi = 0; pi < npairs; ++pi, ++pair) {
        const int st = (int)(pair % kStages);
        const int sb = (int)(pair & 1);
        tc::mbar_wait(&s.k_full[st], (pair / kStages) & 1);
        tc::mbar_wait(&s.s_empty[sb], ((pair >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t k_addr = tc::smem_u32(s.k[st]);
          const uint32_t q_addr = tc::smem_u32(s.q[qs]);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const int h = kk >> 2, j = kk & 3;
            tc::mma_ss(tmem + sb * kG, tc::desc_kmajor(k_addr + h * (kPairBytes / 2) + j * 32),
                       tc::desc_kmajor(q_addr + h * (kQTokBytes / 2) + j * 32), id_s, kk > 0);
          }
          tc::mma_commit(&s.s_full[sb]);
          tc::mma_commit(&s.k_empty[st]);
          if (pi == npairs - 1) tc::mma_commit(&s.q_empty[qs]);
        }
        __syncwarp();
        if (pend) issue_pv();
        pend = true;
        pend_pair = pair;
        pend_first = pi == 0;
        pend_last = pi == npairs - 1;
        pend_tau = tau;
      }
      ++tau;
    }
    if (pend) issue_pv();
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // key lane (S^T) / d lane (O^T)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int64_t pair = 0;
    int tau = 0;
    int cnt_next = blockIdx.x < p.n_items ? cnt_of(p, blockIdx.x) : 0;
    for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      int g;
      int64_t t;
      item_of(p, it, g, t);
      const int64_t row = (int64_t)g * p.n + t;
      const int cnt = cnt_next;  // fetched one item ahead
      cnt_next = it + gridDim.x < p.n_items ? cnt_of(p, it + gridDim.x) : 0;
      if (cnt == 0) continue;
      const int npairs = (cnt + 1) >> 1;
      const int64_t ridx = t * p.h_q + g * kG;  // [n][h_q] row of head 0 of the group
      float mA[kG], lp[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        mA[h] = p.m_a[ridx + h];
        lp[h] = 0.f;
      }
      float excess = -INFINITY;
      for (int pi = 0; pi < npairs; ++pi, ++pair) {
        const int sb = (int)(pair & 1);
        tc::mbar_wait(&s.s_full[sb], (pair >> 1) & 1);
        tc::tc_fence_after();
        uint32_t sv[kG];
        tc::tmem_ld16(tmem + lane_off + sb * kG, sv);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.s_empty[sb]);
        const bool valid = (2 * pi + (r >> 6)) < cnt;
        float pr[kG];
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          const float x = __uint_as_float(sv[h]) * p.scale_log2 - mA[h];
          excess = valid ? fmaxf(excess, x) : excess;
          pr[h] = valid ? fast_exp2(x) : 0.f;
          lp[h] += pr[h];
        }
        // P^T tile (K-major: row = head, 128 keys in two 64-key halves)
        tc::mbar_wait(&s.p_empty[sb], ((pair >> 1) & 1) ^ 1);
        uint8_t *pt = s.p[sb] + (r >> 6) * (kPBytes / 2);
        const int c = r & 63;
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          const uint32_t off = h * 128 + ((((c * 2) >> 4) ^ (h & 7)) << 4) + ((c * 2) & 15);
          *reinterpret_cast<__nv_bfloat16 *>(pt + off) = __float2bfloat16_rn(pr[h]);
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&s.p_full[sb]);
      }
      // ---- per-token epilogue
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        float v = lp[h];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        lp[h] = v;
      }
      excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, 16));
      excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, 8));
      excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, 4));
      excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, 2));
      excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, 1));
      if (lane == 0) {
#pragma unroll
        for (int h = 0; h < kG; ++h) s.lred[quad][h] = lp[h];
      }
      const int ob = tau & 1;
      tc::mbar_wait(&s.o_full[ob], (tau >> 1) & 1);
      tc::tc_fence_after();
      uint32_t ov[kG];
      tc::tmem_ld16(tmem + lane_off + 32 + ob * kG, ov);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&s.o_empty[ob]);
      // all 4 softmax warps: reduce the per-warp partial sums through smem
      asm volatile("bar.sync 1, 128;" ::: "memory");
      float lB[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h)
        lB[h] = s.lred[0][h] + s.lred[1][h] + s.lred[2][h] + s.lred[3][h];
      float exw = excess;
      if (exw > kOverflowExcess && lane == 0) {
        const int slot = atomicAdd(p.slow_count, 1);
        p.slow_list[slot] = (int32_t)row;
      }
      const int d = r;
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        const int64_t oi = (ridx + h) * kD + d;
        const float lA = p.l_a[ridx + h];
        const float oa = __bfloat162float(p.O[oi]);
        const float lt = lA + lB[h];
        p.O[oi] = __float2bfloat16_rn((oa * lA + __uint_as_float(ov[h])) / lt);
        if (d == 0) p.lse[ridx + h] = (mA[h] + __log2f(lt)) * 0.6931471805599453f;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // lred reuse
      ++tau;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

int32_t launch_sparse_part_b(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                             int64_t n, const int32_t *topk, const int32_t *topk_cnt,
                             const float *m_a, const float *l_a, void *O, float *lse,
                             int32_t *slow_count, int32_t *slow_list, int num_sms,
                             cudaStream_t stream) {
  PbParams p;
  memset(&p, 0, sizeof(p));
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cfg->h_q, (uint64_t)n};
    const uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)cfg->h_q * kD * 2};
    const uint32_t box[3] = {64, (uint32_t)kG, 1};
    if (!make_tmap_bf16(&p.q_map, Q, 3, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(Q) failed");
      return SWATTN_ECUDA;
    }
  }
  {
    const uint64_t dims[2] = {(uint64_t)cfg->h_kv * kD, (uint64_t)n};
    const uint64_t str[1] = {(uint64_t)cfg->h_kv * kD * 2};
    const uint32_t box[2] = {64, (uint32_t)kBlk};
    if (!make_tmap_bf16(&p.k_map, K, 2, dims, str, box) ||
        !make_tmap_bf16(&p.v_map, V, 2, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(K/V) failed");
      return SWATTN_ECUDA;
    }
  }
  p.n = n;
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  p.k_top = cfg->k_top;
  p.tok0 = (int64_t)(cfg->N_init + cfg->N_local) * cfg->B;
  if (p.tok0 >= n || cfg->k_top == 0) return SWATTN_OK;
  p.n_items = (int64_t)cfg->h_kv * (n - p.tok0);
  p.topk = topk;
  p.topk_cnt = topk_cnt;
  p.m_a = m_a;
  p.l_a = l_a;
  p.O = static_cast<__nv_bfloat16 *>(O);
  p.lse = lse;
  p.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  p.slow_count = slow_count;
  p.slow_list = slow_list;
  const size_t smem = sizeof(PbSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sparse_pb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const int64_t grid = p.n_items < num_sms ? p.n_items : num_sms;
  sparse_pb_kernel<<<(unsigned)grid, kThreads, smem, stream>>>(p);
  SWATTN_LAUNCH_CHECK("sparse_pb_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
