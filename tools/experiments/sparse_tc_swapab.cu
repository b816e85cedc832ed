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

constexpr int kStages = 3;           // K ring and V ring depth (32 KB slots)
constexpr int kProducers = 2 * kStages;  // warp w < 3: K slot w; 3 <= w < 6: V slot w - 3
constexpr int kMmaWarp = kProducers;
constexpr int kSoftmaxWarp0 = kMmaWarp + 1;
constexpr int kThreads = (kSoftmaxWarp0 + 4) * 32;
constexpr int kSBufs = 4;            // S^T tiles in TMEM
constexpr int kPBufs = 4;            // P^T tiles in smem
constexpr int kBlk = 64;
constexpr uint32_t kPairBytes = 2 * kBlk * kD * 2;  // 32 KB (K or V of two blocks)
constexpr uint32_t kQTokBytes = kG * kD * 2;          // 4 KB
constexpr uint32_t kPBytes = kG * 128 * 2;            // 4 KB
// A dependent tcgen05.mma chain costs ~190 cycles per MMA at any N while
// independent accumulators interleave at ~50 cycles (tools/mma_bench.cu), so
// S^T is accumulated as 4 partial sums over d quarters and O^T as 4 partial
// sums over key quarters (4 chains of 2 k-steps each instead of 1 chain of 8).
constexpr int kChains = 4;
constexpr uint32_t kTmemS = 0;                             // kSBufs x 4 chains x 16 cols
constexpr uint32_t kTmemO = kSBufs * kChains * kG;         // 2 tokens x 4 chains x 16 cols
constexpr uint32_t kTmemCols = 512;
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
  uint8_t p[kPBufs][kPBytes];
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full[kSBufs], s_empty[kSBufs], p_full[kPBufs], p_empty[kPBufs];
  uint64_t o_full[2], o_empty[2];
  float lred[4][kG];
  float xred[4];
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
__device__ __forceinline__ uint32_t ph(int64_t q, int ring) { return (uint32_t)((q / ring) & 1); }

// Cycle accounting for the pipeline roles (variant builds with
// -DSWATTN_PB_PROFILE only; read back with swattn_debug_pb_profile).
#ifdef SWATTN_PB_PROFILE
__device__ unsigned long long g_pb_prof[4][8];
#define PB_T0(t) const long long t = clock64()
#define PB_ACC(t, acc, k) (acc)[k] += clock64() - t
#else
#define PB_T0(t)
#define PB_ACC(t, acc, k)
#endif

// Walks this CTA's pairs in order: (token ordinal tau, pair pi of npairs).
struct PairIter {
  int64_t it;
  int npairs, pi, tau;
  bool valid;
  __device__ void first(const PbParams &p) {
    it = blockIdx.x;
    tau = 0;
    skip(p);
  }
  __device__ void skip(const PbParams &p) {  // move to the first item >= it with pairs
    valid = false;
    for (; it < p.n_items; it += gridDim.x) {
      const int cnt = cnt_of(p, it);
      if (cnt > 0) {
        npairs = (cnt + 1) >> 1;
        pi = 0;
        valid = true;
        return;
      }
    }
  }
  __device__ void next(const PbParams &p) {
    if (++pi == npairs) {
      ++tau;
      it += gridDim.x;
      skip(p);
    }
  }
};

__device__ __forceinline__ bool warp_test(uint64_t *bar, uint32_t parity) {
  const int lane = threadIdx.x & 31;
  bool ok = lane == 0 ? tc::mbar_test_wait(bar, parity) : false;
  return __shfl_sync(0xffffffffu, ok, 0);
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

  if (warp < kProducers) {
    // ------------------------------------------------------------ TMA producers
    // One issuing warp per ring slot: a single thread's TMA issue rate caps
    // near 36 GB/s (tools/gather_bench.cu), so the gather needs several
    // issuers.  Each warp walks all items; lane l holds block ids l and l+32
    // of the current token, fetched one token ahead so no dependent global
    // load sits between two TMA issues.
    const bool is_v = warp >= kStages;
    const int slot = is_v ? warp - kStages : warp;
    const CUtensorMap *map = is_v ? &p.v_map : &p.k_map;
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    if (lane == 0) {
      tc::tma_prefetch(&p.q_map);
      tc::tma_prefetch(map);
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
        if (warp == 0 && lane == 0) {
          const int qs = tau & 1;
          PB_T0(_t1);
          tc::mbar_wait(&s.q_empty[qs], ph(tau, 2) ^ 1);
          PB_ACC(_t1, prof, 2);
          tc::mbar_arrive_expect_tx(&s.q_full[qs], kQTokBytes);
          for (int h = 0; h < 2; ++h)
            tc::tma_load_3d(&p.q_map, &s.q_full[qs], s.q[qs] + h * (kQTokBytes / 2), h * 64,
                            g * kG, (int)t);
        }
        const int npairs = (cnt + 1) >> 1;
        // first pair of this token that falls on my slot
        const int pi0 = (int)(((int64_t)slot - pair) % kStages + kStages) % kStages;
        for (int pi = pi0; pi < npairs; pi += kStages) {
          const int64_t q = pair + pi;
          const int x0 = 2 * pi, x1 = (2 * pi + 1 < cnt) ? 2 * pi + 1 : 2 * pi;  // odd tail: duplicate, masked
          const int b0 = __shfl_sync(0xffffffffu, x0 < 32 ? id0 : id1, x0 & 31);
          const int b1 = __shfl_sync(0xffffffffu, x1 < 32 ? id0 : id1, x1 & 31);
          if (lane == 0) {
            uint64_t *empty = is_v ? &s.v_empty[slot] : &s.k_empty[slot];
            uint64_t *full = is_v ? &s.v_full[slot] : &s.k_full[slot];
            uint8_t *buf = is_v ? s.v[slot] : s.k[slot];
            {
              PB_T0(_t2);
              tc::mbar_wait(empty, ph(q, kStages) ^ 1);
              PB_ACC(_t2, prof, 1);
            }
#if defined(SWATTN_PB_NO_GATHER)  // timing decomposition only (tools/build_variants.sh)
            tc::mbar_arrive(full);
#else
            tc::mbar_arrive_expect_tx(full, kPairBytes);
            for (int h = 0; h < 2; ++h) {
              uint8_t *dst = buf + h * (kPairBytes / 2);
              tc::tma_load_2d(map, full, dst, g * kD + h * 64, b0 * kBlk);
              tc::tma_load_2d(map, full, dst + kBlk * 128, g * kD + h * 64, b1 * kBlk);
            }
#endif
          }
          __syncwarp();
        }
        pair += npairs;
        ++tau;
      }
      it = nit;
      cnt = ncnt;
      id0 = nid0;
      id1 = nid1;
    }
    prof[0] = clock64() - tstart;
#ifdef SWATTN_PB_PROFILE
    if (lane == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&g_pb_prof[is_v ? 1 : 0][k], (unsigned long long)prof[k]);
#endif
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Two cursors over the same pair sequence: S (needs K and a free S tile)
    // and PV (needs the softmax's P tile and V).  The issuer polls both and
    // issues whichever is ready, PV first, keeping at most kSBufs pairs
    // between them -- no fixed lag, so neither the softmax nor the producers
    // wait on a rigid schedule.
    const uint32_t id_s = tc::idesc_bf16(128, kG, false, false);
    const uint32_t id_o = tc::idesc_bf16(128, kG, true, false);
    PairIter si, vi;
    si.first(p);
    vi = si;
    int64_t sq = 0, vq = 0;
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
    long long tidle = clock64();
    while (true) {
      if (vq < sq) {
        const int pb = (int)(vq % kPBufs), vs = (int)(vq % kStages);
        bool ready = warp_test(&s.p_full[pb], ph(vq, kPBufs)) && warp_test(&s.v_full[vs], ph(vq, kStages));
        if (ready && vi.pi == 0) ready = warp_test(&s.o_empty[vi.tau & 1], ph(vi.tau, 2) ^ 1);
        if (ready) {
          prof[1] += clock64() - tidle;
          ++prof[3];
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t v_addr = tc::smem_u32(s.v[vs]);
            const uint32_t p_addr = tc::smem_u32(s.p[pb]);
            const uint32_t d_o = tmem + kTmemO + (vi.tau & 1) * (kChains * kG);
            // key quarter c (k-steps 2c, 2c+1) accumulates into O chain c
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int c = i & 3, kk = 2 * c + (i >> 2);
#ifndef SWATTN_PB_NO_MMA
              tc::mma_ss(d_o + c * kG, tc::desc_mnmajor(v_addr + kk * 16 * 128, kPairBytes / 2),
                         tc::desc_kmajor(p_addr + (kk >> 2) * (kPBytes / 2) + (kk & 3) * 32), id_o,
                         (vi.pi > 0 || (i >> 2)) ? 1u : 0u);
#endif
            }
            tc::mma_commit(&s.v_empty[vs]);
            tc::mma_commit(&s.p_empty[pb]);
            if (vi.pi == vi.npairs - 1) tc::mma_commit(&s.o_full[vi.tau & 1]);
          }
          __syncwarp();
          vi.next(p);
          ++vq;
          tidle = clock64();
          continue;
        }
      } else if (!si.valid) {
        break;
      }
      if (si.valid && sq - vq < kSBufs) {
        const int ks = (int)(sq % kStages), sb = (int)(sq % kSBufs);
        bool ready = warp_test(&s.k_full[ks], ph(sq, kStages)) && warp_test(&s.s_empty[sb], ph(sq, kSBufs) ^ 1);
        if (ready && si.pi == 0) ready = warp_test(&s.q_full[si.tau & 1], ph(si.tau, 2));
        if (ready) {
          prof[2] += clock64() - tidle;
          ++prof[4];
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t k_addr = tc::smem_u32(s.k[ks]);
            const uint32_t q_addr = tc::smem_u32(s.q[si.tau & 1]);
            // d quarter c (k-steps 2c, 2c+1) accumulates into S chain c
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int c = i & 3, kk = 2 * c + (i >> 2);
              const int h = kk >> 2, j = kk & 3;
#ifndef SWATTN_PB_NO_MMA
              tc::mma_ss(tmem + kTmemS + (sb * kChains + c) * kG,
                         tc::desc_kmajor(k_addr + h * (kPairBytes / 2) + j * 32),
                         tc::desc_kmajor(q_addr + h * (kQTokBytes / 2) + j * 32), id_s, i >> 2);
#endif
            }
            tc::mma_commit(&s.s_full[sb]);
            tc::mma_commit(&s.k_empty[ks]);
            if (si.pi == si.npairs - 1) tc::mma_commit(&s.q_empty[si.tau & 1]);
          }
          __syncwarp();
          si.next(p);
          ++sq;
          tidle = clock64();
        }
      }
    }
    prof[0] = clock64() - tstart;
#ifdef SWATTN_PB_PROFILE
    if (lane == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&g_pb_prof[2][k], (unsigned long long)prof[k]);
#endif
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // key lane (S^T) / d lane (O^T)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    // P^T word offsets of this lane's 8 stores (see the store loop)
    const bool odd = lane & 1;
    uint32_t poff[8], wrd[8];
    {
      const int ce = (r & 63) & ~1;  // even key of the lane pair
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int h = odd ? 2 * (j ^ 2) + 1 : 2 * j;
        poff[j] = h * 128 + ((((ce * 2) >> 4) ^ (h & 7)) << 4) + ((ce * 2) & 15);
      }
    }
    int64_t pair = 0;
    int tau = 0;
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long tstart = clock64();
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
        const int sb = (int)(pair % kSBufs), pb = (int)(pair % kPBufs);
        {
          PB_T0(_t3);
          tc::mbar_wait(&s.s_full[sb], ph(pair, kSBufs));
          PB_ACC(_t3, prof, 1);
        }
        tc::tc_fence_after();
        PB_T0(_t4);
        uint32_t sa[2 * kG], sbv[2 * kG];
        tc::tmem_ld32(tmem + lane_off + kTmemS + sb * (kChains * kG), sa);
        tc::tmem_ld32(tmem + lane_off + kTmemS + sb * (kChains * kG) + 2 * kG, sbv);
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.s_empty[sb]);
        PB_ACC(_t4, prof, 4);
#if defined(SWATTN_PB_NO_MMA) || defined(SWATTN_PB_NO_GATHER)
        const bool valid = false;
#else
        const bool valid = (2 * pi + (r >> 6)) < cnt;
#endif
        // valid is warp-uniform (a warp's 32 keys lie in one 64-key block)
        float pr[kG];
        if (valid) {
          float xm = -INFINITY;
#pragma unroll
          for (int h = 0; h < kG; ++h) {
            const float sv = (__uint_as_float(sa[h]) + __uint_as_float(sa[kG + h])) +
                             (__uint_as_float(sbv[h]) + __uint_as_float(sbv[kG + h]));
            const float x = fmaf(sv, p.scale_log2, -mA[h]);
            xm = fmaxf(xm, x);
            pr[h] = fast_exp2(x);
            lp[h] += pr[h];
          }
          excess = fmaxf(excess, xm);
        } else {
#pragma unroll
          for (int h = 0; h < kG; ++h) pr[h] = 0.f;
        }
        // P^T tile (K-major: row = head, 128 keys in two 64-key halves)
        {
          PB_T0(_t5);
          tc::mbar_wait(&s.p_empty[pb], ph(pair, kPBufs) ^ 1);
          PB_ACC(_t5, prof, 2);
        }
        PB_T0(_t6);
        // Key pairs (c, c+1) of one head form a 32-bit word: lanes c and c^1
        // swap half their heads (4 shuffles of packed bf16x2), the even lane
        // then stores heads 0,2,..,14 and the odd lane heads 1,3,..,15; store
        // j pairs even head 2j with odd head 2(j^2)+1, which lies in the other
        // half of the 128-byte swizzle pattern, so the two rows never share a
        // bank.
        uint8_t *pt = s.p[pb] + (r >> 6) * (kPBytes / 2);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t A = tc::pack_bf16(pr[4 * k], pr[4 * k + 2]);
          const uint32_t B = tc::pack_bf16(pr[4 * k + 1], pr[4 * k + 3]);
          const uint32_t keep = odd ? B : A;
          const uint32_t recv = __shfl_xor_sync(0xffffffffu, odd ? A : B, 1);
          wrd[2 * k] = odd ? __byte_perm(recv, keep, 0x5410) : __byte_perm(keep, recv, 0x5410);
          wrd[2 * k + 1] = odd ? __byte_perm(recv, keep, 0x7632) : __byte_perm(keep, recv, 0x7632);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint32_t *>(pt + poff[j]) = odd ? wrd[j ^ 2] : wrd[j];
        tc::fence_proxy_async();
        tc::mbar_arrive(&s.p_full[pb]);
        PB_ACC(_t6, prof, 5);
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
        s.xred[quad] = excess;
      }
      const int ob = tau & 1;
      {
        PB_T0(_t7);
        tc::mbar_wait(&s.o_full[ob], ph(tau, 2));
        PB_ACC(_t7, prof, 3);
      }
      tc::tc_fence_after();
      uint32_t oa4[2 * kG], ob4[2 * kG];
      tc::tmem_ld32(tmem + lane_off + kTmemO + ob * (kChains * kG), oa4);
      tc::tmem_ld32(tmem + lane_off + kTmemO + ob * (kChains * kG) + 2 * kG, ob4);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&s.o_empty[ob]);
      float ov[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h)
        ov[h] = (__uint_as_float(oa4[h]) + __uint_as_float(oa4[kG + h])) +
                (__uint_as_float(ob4[h]) + __uint_as_float(ob4[kG + h]));
      // all 4 softmax warps: reduce the per-warp partial sums through smem
      asm volatile("bar.sync 1, 128;" ::: "memory");
      float lB[kG];
#pragma unroll
      for (int h = 0; h < kG; ++h)
        lB[h] = s.lred[0][h] + s.lred[1][h] + s.lred[2][h] + s.lred[3][h];
      excess = fmaxf(fmaxf(s.xred[0], s.xred[1]), fmaxf(s.xred[2], s.xred[3]));
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
        p.O[oi] = __float2bfloat16_rn((oa * lA + ov[h]) / lt);
        if (d == 0) p.lse[ridx + h] = (mA[h] + __log2f(lt)) * 0.6931471805599453f;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // lred reuse
      ++tau;
    }
    prof[0] = clock64() - tstart;
#ifdef SWATTN_PB_PROFILE
    if (lane == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&g_pb_prof[3][k], (unsigned long long)prof[k]);
#endif
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

#ifdef SWATTN_PB_PROFILE
extern "C" int swattn_debug_pb_profile(unsigned long long *out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_pb_prof, sizeof(g_pb_prof));
  if (reset) {
    static const unsigned long long zero[4][8] = {};
    cudaMemcpyToSymbol(g_pb_prof, zero, sizeof(zero));
  }
  return 0;
}
#endif

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
