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
// Pipeline: the MMA issuer runs the S MMAs kLag pairs ahead of the PV MMAs,
// so the softmax warps always have S tiles queued and the chain
// S -> softmax -> PV never serialises the tensor pipe; K and V travel in
// separate TMA rings (K is released right after S, V is held until its PV,
// hence the deeper V ring).  Fixed-offset softmax makes the O accumulation
// order-free, which is what allows the lag across token boundaries.
//
// Warp roles (320 threads, 1 CTA / SM, persistent over (group, token)):
//   warps 0-1 K producers (ring stage q % 2), warps 2-3 V producers (stage
//   parity), warps 4-7 softmax + per-token epilogue (TMEM lane quadrant =
//   warp & 3), warp 8 MMA issuer.  Several issuing threads: one thread's TMA
//   issue rate caps near 36 GB/s (tools/gather_bench.cu).
// Roofline: bound by the L2->SMEM gather of 2 x 63 x 16 KB per token
// (K and V of the selected blocks); FLOP = 4 * 16 * 64 * d per block.
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

constexpr int kThreads = 288;
constexpr int kSoftmaxWarp0 = 4;
constexpr int kMmaWarp = 8;
constexpr int kKStages = 2;
constexpr int kVStages = 4;
constexpr int kLag = 2;                 // S issued kLag pairs ahead of PV
constexpr int kSBufs = kLag + 2;        // S tiles in TMEM
constexpr int kPBufs = kLag + 2;        // P tiles in smem
constexpr int kBlk = 64;
constexpr uint32_t kPairBytes = 2 * kBlk * kD * 2;  // 32 KB (K or V of two blocks)
constexpr uint32_t kQTokBytes = kG * kD * 2;          // 4 KB
constexpr uint32_t kPBytes = kG * 128 * 2;            // 4 KB
constexpr uint32_t kTmemCols = 128;                   // S x4 | O 2 tokens x 2 accumulators
constexpr uint32_t kTmemO = kSBufs * kG;
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
  uint8_t k[kKStages][kPairBytes];
  uint8_t v[kVStages][kPairBytes];
  uint8_t p[kPBufs][kPBytes];
  uint8_t q[2][kQTokBytes];
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full[kSBufs], s_empty[kSBufs], p_full[kPBufs], p_empty[kPBufs];
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

// ring position helpers: slot and phase parity of the q-th use
__device__ __forceinline__ uint32_t phase(int64_t q, int ring) { return (uint32_t)((q / ring) & 1); }

__global__ void __launch_bounds__(kThreads, 1) sparse_pb_kernel(const __grid_constant__ PbParams p) {
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on smem_raw so accesses stay in the shared space
  PbSmem &s = *reinterpret_cast<PbSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kKStages; ++i) {
      tc::mbar_init(&s.k_full[i], 1);
      tc::mbar_init(&s.k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      tc::mbar_init(&s.v_full[i], 1);
      tc::mbar_init(&s.v_empty[i], 1);
    }
    for (int i = 0; i < kSBufs; ++i) {
      tc::mbar_init(&s.s_full[i], 1);
      tc::mbar_init(&s.s_empty[i], 128);
    }
    for (int i = 0; i < kPBufs; ++i) {
      tc::mbar_init(&s.p_full[i], 128);
      tc::mbar_init(&s.p_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.q_full[i], 1);
      tc::mbar_init(&s.q_empty[i], 1);
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

  if (warp < kSoftmaxWarp0) {
    // ------------------------------------------------------------ TMA producers
    // warps 0/1: K of pairs with q % 2 == warp; warps 2/3: V of pairs whose V
    // stage (q % 4) has parity warp-2.  Each warp walks all items; lane l holds
    // block ids l and l+32 of the current token, fetched one token ahead.
    const bool is_v = warp >= 2;
    const int role = warp & 1;
    if (lane == 0) {
      tc::tma_prefetch(&p.q_map);
      tc::tma_prefetch(is_v ? &p.v_map : &p.k_map);
    }
    int64_t q = 0;
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
        if (lane == 0 && warp == 0) {
          const int qs = tau & 1;
          tc::mbar_wait(&s.q_empty[qs], phase(tau, 2) ^ 1);
          tc::mbar_arrive_expect_tx(&s.q_full[qs], kQTokBytes);
          for (int h = 0; h < 2; ++h)
            tc::tma_load_3d(&p.q_map, &s.q_full[qs], s.q[qs] + h * (kQTokBytes / 2), h * 64,
                            g * kG, (int)t);
        }
        const int npairs = (cnt + 1) >> 1;
        for (int pi = 0; pi < npairs; ++pi, ++q) {
          const int x0 = 2 * pi, x1 = (2 * pi + 1 < cnt) ? 2 * pi + 1 : 2 * pi;  // odd tail: duplicate, masked
          const int b0 = __shfl_sync(0xffffffffu, x0 < 32 ? id0 : id1, x0 & 31);
          const int b1 = __shfl_sync(0xffffffffu, x1 < 32 ? id0 : id1, x1 & 31);
          if (lane == 0 && !is_v && (int)(q % kKStages) == role) {
            const int st = role;
            tc::mbar_wait(&s.k_empty[st], phase(q, kKStages) ^ 1);
            tc::mbar_arrive_expect_tx(&s.k_full[st], kPairBytes);
            for (int h = 0; h < 2; ++h) {
              uint8_t *dst = s.k[st] + h * (kPairBytes / 2);
              tc::tma_load_2d(&p.k_map, &s.k_full[st], dst, g * kD + h * 64, b0 * kBlk);
              tc::tma_load_2d(&p.k_map, &s.k_full[st], dst + kBlk * 128, g * kD + h * 64, b1 * kBlk);
            }
          }
          if (lane == 0 && is_v && (int)(q % kVStages) % 2 == role) {
            const int st = (int)(q % kVStages);
            tc::mbar_wait(&s.v_empty[st], phase(q, kVStages) ^ 1);
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
    // An N = 16 MMA chain accumulating into one TMEM tile is latency-bound
    // (~130 cycles per dependent MMA while the tensor pipe is 95 % idle), so
    // pairs are issued two at a time with their k-steps interleaved: S of
    // pairs (q, q+1) and PV of the previous two pairs form four independent
    // accumulation chains.  PV of a token alternates between two O
    // accumulators (pair parity), summed in the epilogue.
    const uint32_t id_s = tc::idesc_bf16(128, kG, false, false);
    const uint32_t id_o = tc::idesc_bf16(128, kG, true, false);
    struct PairInfo {
      int64_t q;
      int tau, pi, npairs;
    };
    PairInfo cur[2], pv[2];
    int ncur = 0, npv = 0;
    auto issue_pv_group = [&]() {
      for (int e = 0; e < npv; ++e) {
        const int64_t qq = pv[e].q;
        tc::mbar_wait(&s.p_full[(int)(qq % kPBufs)], phase(qq, kPBufs));
        tc::mbar_wait(&s.v_full[(int)(qq % kVStages)], phase(qq, kVStages));
        if (pv[e].pi == 0) tc::mbar_wait(&s.o_empty[pv[e].tau & 1], phase(pv[e].tau, 2) ^ 1);
      }
      tc::tc_fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          for (int e = 0; e < npv; ++e) {
            const int64_t qq = pv[e].q;
            const uint32_t v_addr = tc::smem_u32(s.v[(int)(qq % kVStages)]);
            const uint32_t p_addr = tc::smem_u32(s.p[(int)(qq % kPBufs)]);
            const uint32_t d_o = tmem + kTmemO + ((pv[e].tau & 1) * 2 + (pv[e].pi & 1)) * kG;
            tc::mma_ss(d_o, tc::desc_mnmajor(v_addr + kk * 16 * 128, kPairBytes / 2),
                       tc::desc_kmajor(p_addr + (kk >> 2) * (kPBytes / 2) + (kk & 3) * 32), id_o,
                       (pv[e].pi >= 2 || kk > 0) ? 1u : 0u);
          }
        }
        for (int e = 0; e < npv; ++e) {
          const int64_t qq = pv[e].q;
          tc::mma_commit(&s.v_empty[(int)(qq % kVStages)]);
          tc::mma_commit(&s.p_empty[(int)(qq % kPBufs)]);
          if (pv[e].pi == pv[e].npairs - 1) tc::mma_commit(&s.o_full[pv[e].tau & 1]);
        }
      }
      __syncwarp();
      npv = 0;
    };
    auto flush = [&]() {
      for (int e = 0; e < ncur; ++e) {
        const int64_t qq = cur[e].q;
        if (cur[e].pi == 0) tc::mbar_wait(&s.q_full[cur[e].tau & 1], phase(cur[e].tau, 2));
        tc::mbar_wait(&s.k_full[(int)(qq % kKStages)], phase(qq, kKStages));
        tc::mbar_wait(&s.s_empty[(int)(qq % kSBufs)], phase(qq, kSBufs) ^ 1);
      }
      tc::tc_fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const int h = kk >> 2, j = kk & 3;
          for (int e = 0; e < ncur; ++e) {
            const int64_t qq = cur[e].q;
            const uint32_t k_addr = tc::smem_u32(s.k[(int)(qq % kKStages)]);
            const uint32_t q_addr = tc::smem_u32(s.q[cur[e].tau & 1]);
            tc::mma_ss(tmem + (int)(qq % kSBufs) * kG,
                       tc::desc_kmajor(k_addr + h * (kPairBytes / 2) + j * 32),
                       tc::desc_kmajor(q_addr + h * (kQTokBytes / 2) + j * 32), id_s, kk > 0);
          }
        }
        for (int e = 0; e < ncur; ++e) {
          const int64_t qq = cur[e].q;
          tc::mma_commit(&s.s_full[(int)(qq % kSBufs)]);
          tc::mma_commit(&s.k_empty[(int)(qq % kKStages)]);
          if (cur[e].pi == cur[e].npairs - 1) tc::mma_commit(&s.q_empty[cur[e].tau & 1]);
        }
      }
      __syncwarp();
      if (npv) issue_pv_group();
      for (int e = 0; e < ncur; ++e) pv[e] = cur[e];
      npv = ncur;
      ncur = 0;
    };
    int64_t q = 0;
    int tau = 0;
    int cnt_next = blockIdx.x < p.n_items ? cnt_of(p, blockIdx.x) : 0;
    for (int64_t it = blockIdx.x; it < p.n_items; it += gridDim.x) {
      const int cnt = cnt_next;  // fetched one item ahead
      cnt_next = it + gridDim.x < p.n_items ? cnt_of(p, it + gridDim.x) : 0;
      if (cnt == 0) continue;
      const int npairs = (cnt + 1) >> 1;
      for (int pi = 0; pi < npairs; ++pi, ++q) {
        cur[ncur++] = PairInfo{q, tau, pi, npairs};
        if (ncur == 2) flush();
      }
      ++tau;
    }
    if (ncur) flush();
    if (npv) issue_pv_group();
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // key lane (S^T) / d lane (O^T)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    int64_t q = 0;
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
      for (int pi = 0; pi < npairs; ++pi, ++q) {
        const int sb = (int)(q % kSBufs), pb = (int)(q % kPBufs);
        tc::mbar_wait(&s.s_full[sb], phase(q, kSBufs));
        tc::tc_fence_after();
        uint32_t sv[kG];
        tc::tmem_ld16(tmem + lane_off + sb * kG, sv);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.s_empty[sb]);
        const bool valid = (2 * pi + (r >> 6)) < cnt;
        uint32_t pk[kG / 2];
#pragma unroll
        for (int h = 0; h < kG; h += 2) {
          const float x0 = __uint_as_float(sv[h]) * p.scale_log2 - mA[h];
          const float x1 = __uint_as_float(sv[h + 1]) * p.scale_log2 - mA[h + 1];
          excess = valid ? fmaxf(excess, fmaxf(x0, x1)) : excess;
          const float p0 = valid ? fast_exp2(x0) : 0.f;
          const float p1 = valid ? fast_exp2(x1) : 0.f;
          lp[h] += p0;
          lp[h + 1] += p1;
          pk[h / 2] = tc::pack_bf16(p0, p1);
        }
        // P^T tile (K-major: row = head, 128 keys in two 64-key halves)
        tc::mbar_wait(&s.p_empty[pb], phase(q, kPBufs) ^ 1);
        uint8_t *pt = s.p[pb] + (r >> 6) * (kPBytes / 2);
        const int c = r & 63;
#pragma unroll
        for (int h = 0; h < kG; ++h) {
          const uint32_t off = h * 128 + ((((c * 2) >> 4) ^ (h & 7)) << 4) + ((c * 2) & 15);
          const uint32_t w = pk[h / 2];
          *reinterpret_cast<uint16_t *>(pt + off) = (h & 1) ? (uint16_t)(w >> 16) : (uint16_t)w;
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&s.p_full[pb]);
      }
      // ---- per-token epilogue
#pragma unroll
      for (int h = 0; h < kG; ++h) {
        float v = lp[h];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        lp[h] = v;
      }
      for (int o = 16; o; o >>= 1) excess = fmaxf(excess, __shfl_xor_sync(0xffffffffu, excess, o));
      if (lane == 0) {
#pragma unroll
        for (int h = 0; h < kG; ++h) s.lred[quad][h] = lp[h];
      }
      const int ob = tau & 1;
      tc::mbar_wait(&s.o_full[ob], phase(tau, 2));
      tc::tc_fence_after();
      uint32_t ov[kG], ov1[kG];
      tc::tmem_ld16(tmem + lane_off + kTmemO + (ob * 2) * kG, ov);
      tc::tmem_ld16(tmem + lane_off + kTmemO + (ob * 2 + 1) * kG, ov1);
      tc::tmem_ld_wait();
      if (npairs >= 2) {
#pragma unroll
        for (int h = 0; h < kG; ++h)
          ov[h] = __float_as_uint(__uint_as_float(ov[h]) + __uint_as_float(ov1[h]));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&s.o_empty[ob]);
      // all 4 softmax warps: reduce the per-warp partial sums through smem
      asm volatile("bar.sync 1, 128;" ::: "memory");
      float lB[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h)
        lB[h] = s.lred[0][h] + s.lred[1][h] + s.lred[2][h] + s.lred[3][h];
      if (excess > kOverflowExcess && r == 0) {
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
