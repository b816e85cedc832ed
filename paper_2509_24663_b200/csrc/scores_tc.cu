// K2 -- fused two-pass block scoring on tcgen05 (sm_100a).
//
// CTA = 8 query tokens x 16 heads of one KV group (128 rows), 2 CTAs / SM.
//   Pass 1 (normal orientation, selection.py:165-196): S = Q_tile . K_C2^T
//     over 128-column chunks of the normaliser keys (C2 for approx, C1 for
//     exact); one thread per (token, head) row keeps the online (max, sum)
//     in registers -> m, 1/l per row (log2 domain).
//   Pass 2 (swap-AB, selection.py:199-222): S^T = K_C1_tile . Q_tile^T with
//     M = 128 C1 columns, N = 128 (token, head) rows, so one thread owns one
//     compressed column and the 16-head group sum
//       shared(i, c) = sum_h exp2(s_h c' - m_h) / l_h
//     is thread-local.  The 5/4 max-pool (compression.py:160-173) runs on
//     warp shuffles; tiles advance by 124 columns so every 5-column window
//     of the tile's 31 blocks is inside the tile.  Only the top-k candidate
//     region [N_init, min(b - N_local + 1, n_cols)) is computed and written
//     (S^cmp fp32), plus the argmax-at-shared-column flag bits K3 uses to
//     classify exact ties.
// Warp roles (320 threads): warp 0 TMA (Q once; C2 chunks then C1 tiles
// through one 2-stage ring), warp 1 MMA issuer, warps 2..9 epilogues in two
// warpgroups that split every TMEM tile by columns (pass 1: key columns
// 0-63 / 64-127 of a chunk; pass 2: tokens 0-3 / 4-7), so each SM sub-
// partition runs 4 epilogue warps (2 per CTA) and keeps MUFU busy while the
// other warps wait on TMEM loads or the max-pool barrier.
// Roofline: tensor + MUFU; FLOP = 2 * h_q * d * (pass-1 cols + pass-2 cols)
// per row (bench.py:144-155).
#include <stddef.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"
#include "topk_cta.cuh"

namespace swattn {

namespace {

constexpr int kThreads = 320;
constexpr int kEpiThreads = 256;  // warps 2..9
constexpr int kTok = 8;
constexpr int kRows = kTok * kG;           // 128
constexpr int kCols = 128;                 // columns per chunk / tile
constexpr int kTileBlocks = 31;
constexpr int kTileStride = kTileBlocks * kPoolS;  // 124
constexpr int kStages = 2;
constexpr uint32_t kQBytes = kRows * kD * 2;      // 32 KB
constexpr uint32_t kKBytes = kCols * kD * 2;      // 32 KB
constexpr uint32_t kTmemCols = 256;

// heads 0, 4, .. 4 (SWATTN_K2_POLY_GROUPS - 1) of every 16 take their pass-2
// exp on the FMA pipe (0 = all on MUFU)
#ifndef SWATTN_K2_POLY_GROUPS
#define SWATTN_K2_POLY_GROUPS 2  // measured best: 8.09 -> 7.39 ms at 128K (tools/probe_partb.sh pf1-3)
#endif
// pass 1: every 8th column's exp on the FMA pipe as well
#ifndef SWATTN_K2_POLY_P1
#define SWATTN_K2_POLY_P1 0
#endif
// timing-decomposition switches for variant builds (tools/build_variants.sh)
#ifdef SWATTN_K2_NO_EXP
#define K2_EXP(x) (x)
#else
#define K2_EXP(x) fast_exp2(x)
#endif

struct ScParams {
  CUtensorMap q_map;    // Q [n][h_q][d]: box {64, 16, 8}
  CUtensorMap k1_map;   // K_C1 [m1][h_kv*d]: box {64, 128}
  CUtensorMap k2_map;   // K_C2 (or K_C1 again in exact mode)
  int64_t n, m1, m2;
  int h_q, h_kv, g0;
  int l_C1, s_C1, l_C2, s_C2;
  int N_init, N_local, B, n_cols;
  int approx;
  float scale_log2;
  int64_t tok0;         // first token of the launch (>= first token with candidates)
  int64_t r1;           // rows [tok0, r1) are computed
  int n_tiles_tok;      // CTAs along tokens
  float *s_cmp;
  int64_t ld;
  uint64_t *flags;
  int64_t ld_f;
  // top-k in the pass-2 epilogue (row f1; null topk = S^cmp only, K3 selects)
  int32_t *topk, *topk_cnt;
  int k_top;
  AmbList amb;
  int32_t *ovf_count, *ovf_rows;  // rows whose candidate set overflowed (massive ties)
};

// Per-token running candidate set of the fused top-k: every block score of
// a tile that reaches the token's threshold is appended (ballot) in block
// order; when the next tile might not fit, the set is compacted to the keys
// >= (k-th largest) x (1 - 4 eps), which keeps the final top-k, every key
// within the float32 error band below the final k-th, and every key above
// it (the threshold only rises, and stays below the final k-th by 4 eps).
constexpr int kCand = 128;

struct __align__(1024) ScSmem {
  uint8_t q[kQBytes];
  uint8_t k[kStages][kKBytes];
  uint64_t q_full, full[kStages], empty[kStages], tfull[2], tempty[2];
  __align__(16) float2 stat[kRows];  // (m, 1/l) per (token, head) row, log2 domain
  float2 stat_hi[kRows];             // warpgroup 1's pass-1 (m, l) before the merge
  float sc[kTok][kCols + 4];   // tile column scores for the max-pool
  uint32_t tmem_base;
  // fused top-k only (the default kernel is launched without these 6 KB):
  uint32_t ckey[kTok][kCand];  // candidate keys (f2key of S^cmp), block order
  uint16_t cid[kTok][kCand];   //   and their block ids
};

// k-th largest of the warp's candidate keys (lane holds entries lane + 32 e;
// invalid entries are 0): the largest X with #{key >= X} >= k, bit by bit
__device__ __forceinline__ uint32_t warp_kth_key(const uint32_t (&kv)[kCand / 32], int k) {
  uint32_t x = 0u;
#pragma unroll 1
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t c = x | (1u << bit);
    int n = 0;
#pragma unroll
    for (int e = 0; e < kCand / 32; ++e) n += kv[e] >= c;
    if (__reduce_add_sync(0xffffffffu, n) >= k) x = c;
  }
  return x;
}

// bit q of x -> bit 2q of the result (Morton spread)
__device__ __forceinline__ unsigned long long spread_bits(uint32_t x) {
  unsigned long long v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// kFuse: row f1 variant (top-k in the pass-2 epilogue); compiled separately
// so the default kernel carries none of its code
template <bool kFuse>
__global__ void __launch_bounds__(kThreads, 2) scores_tc_kernel(const __grid_constant__ ScParams p) {
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on smem_raw so accesses stay in the shared space
  ScSmem &s = *reinterpret_cast<ScSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heavy CTAs (late tokens) first
  const int tt = p.n_tiles_tok - 1 - (int)blockIdx.x;
  const int g = p.g0 + (int)blockIdx.y;
  const int64_t i0 = p.tok0 + (int64_t)tt * kTok;
  const int64_t i_last = min(i0 + kTok - 1, p.r1 - 1);
  const int b = (int)(i0 / p.B);
  const int hi = cand_hi(b, p.N_local, p.n_cols);
  const int n_t2 = (hi + kTileBlocks - 1) / kTileBlocks;  // pass-2 tiles
  const bool use_c2 = p.approx && vis_count(i0, p.l_C2, p.s_C2) > 0;
  const int64_t vmax = use_c2 ? vis_count(i_last, p.l_C2, p.s_C2) : vis_count(i_last, p.l_C1, p.s_C1);
  const int n_c1 = (int)cdiv(vmax, kCols);  // pass-1 chunks
  const int n_units = n_c1 + n_t2;

  if (threadIdx.x == 0) {
    tc::mbar_init(&s.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.full[i], 1);
      tc::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.tfull[i], 1);
      tc::mbar_init(&s.tempty[i], kEpiThreads);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&s.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 0) {
    // lanes 0 and 1 each own one ring stage (units u = lane mod 2): two issuing
    // threads, since one thread's TMA issue rate caps near 36 GB/s
    if (lane < kStages) {
      if (lane == 0) {
        tc::tma_prefetch(&p.q_map);
        tc::tma_prefetch(&p.k1_map);
        tc::tma_prefetch(&p.k2_map);
        tc::mbar_arrive_expect_tx(&s.q_full, kQBytes);
        for (int h = 0; h < 2; ++h)
          tc::tma_load_3d(&p.q_map, &s.q_full, s.q + h * (kQBytes / 2), h * 64, g * kG, (int)i0);
      }
      for (int u = lane; u < n_units; u += kStages) {
        const int st = u % kStages;
        tc::mbar_wait(&s.empty[st], ((u / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&s.full[st], kKBytes);
        const bool p1 = u < n_c1;
        const CUtensorMap *map = p1 ? (use_c2 ? &p.k2_map : &p.k1_map) : &p.k1_map;
        const int row0 = p1 ? u * kCols : (u - n_c1) * kTileStride;
        for (int h = 0; h < 2; ++h)
          tc::tma_load_2d(map, &s.full[st], s.k[st] + h * (kKBytes / 2), g * kD + h * 64, row0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = tc::idesc_bf16(128, 128, false, false);
    const uint32_t q_addr = tc::smem_u32(s.q);
    tc::mbar_wait(&s.q_full, 0);
    for (int u = 0; u < n_units; ++u) {
      const int st = u % kStages, tb = u & 1;
      tc::mbar_wait(&s.full[st], (u / kStages) & 1);
      tc::mbar_wait(&s.tempty[tb], ((u >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t k_addr = tc::smem_u32(s.k[st]);
        const bool p1 = u < n_c1;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const int h = kk >> 2, j = kk & 3;
          const uint64_t dq = tc::desc_kmajor(q_addr + h * (kQBytes / 2) + j * 32);
          const uint64_t dk = tc::desc_kmajor(k_addr + h * (kKBytes / 2) + j * 32);
          // pass 1: rows = (token, head), cols = keys; pass 2: rows = C1 columns
#ifndef SWATTN_K2_NO_MMA
          tc::mma_ss(tmem + tb * kCols, p1 ? dq : dk, p1 ? dk : dq, idesc, kk > 0);
#endif
        }
        tc::mma_commit(&s.tfull[tb]);
        tc::mma_commit(&s.empty[st]);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;           // TMEM lane quadrant of this warp
    const int half = (warp - 2) >> 2;    // epilogue warpgroup 0 / 1
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    // ---------------- pass 1: thread = row (token r/16, head r%16), key
    // columns [64 half, 64 half + 64) of every chunk
    const int64_t my_tok = min(i0 + r / kG, p.r1 - 1);
    const int64_t my_vis = use_c2 ? vis_count(my_tok, p.l_C2, p.s_C2) : vis_count(my_tok, p.l_C1, p.s_C1);
    float m = -INFINITY, l = 0.f;
    for (int u = 0; u < n_c1; ++u) {
      const int tb = u & 1;
      tc::mbar_wait(&s.tfull[tb], (u >> 1) & 1);
      tc::tc_fence_after();
      const int64_t c0 = (int64_t)u * kCols + half * 64;
      uint32_t va[32], vb[32];
      tc::tmem_ld32(tmem + lane_off + tb * kCols + half * 64, va);
      tc::tmem_ld32(tmem + lane_off + tb * kCols + half * 64 + 32, vb);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&s.tempty[tb]);
      // raw logits; the scale is folded into the exp FFMA and the visibility
      // mask only runs on the chunk that crosses my_vis
      float x[64];
#pragma unroll
      for (int e = 0; e < 64; ++e) x[e] = __uint_as_float(e < 32 ? va[e] : vb[e - 32]);
      if (c0 + 64 > my_vis) {
        const int64_t lim = my_vis - c0;  // columns e >= lim are not visible
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (e >= lim) x[e] = -INFINITY;
      }
      const float cm = max64(x) * p.scale_log2;
      if (cm > m) {
        l *= fast_exp2(m - cm);
        m = cm;
      }
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
      for (int e = 0; e < 64; e += 4) {
        const float y0 = fmaf(x[e], p.scale_log2, -m);
        a0 += (SWATTN_K2_POLY_P1 && e % 8 == 0) ? poly_exp2(y0) : fast_exp2(y0);
        a1 += fast_exp2(fmaf(x[e + 1], p.scale_log2, -m));
        a2 += fast_exp2(fmaf(x[e + 2], p.scale_log2, -m));
        a3 += fast_exp2(fmaf(x[e + 3], p.scale_log2, -m));
      }
      if (m != -INFINITY) l += (a0 + a1) + (a2 + a3);
    }
    // merge the two column halves of every row
    if (half == 1) s.stat_hi[r] = make_float2(m, l);
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    if (half == 0) {
      const float2 o = s.stat_hi[r];
      const float M = fmaxf(m, o.x);
      float L = 0.f;
      if (M != -INFINITY) L = l * fast_exp2(m - M) + o.y * fast_exp2(o.x - M);
      s.stat[r] = make_float2(M == -INFINITY ? 0.f : M, L > 0.f ? 1.f / L : 0.f);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");

    // ---------------- pass 2: thread = C1 column of the tile
    // No causal / edge masking is needed here: every column of a candidate
    // block's window (cols <= 4*hi) is visible to all 8 rows (vis1 >= 4b - 1)
    // and < m1; values of other columns are never written.
    constexpr bool fuse = kFuse;
    const int ksel = min(p.k_top, max(hi - p.N_init, 0));  // the same for the CTA's 8 tokens
    int ccnt = 0;          // fused top-k state of token warp - 2 (warp-uniform)
    uint32_t cthr = 0u;
    bool covf = false;
    uint32_t t1 = 0u, t2 = 0u, t3 = 0u;  // this lane's 3 largest keys so far
    for (int t = 0; t < n_t2; ++t) {
      const int u = n_c1 + t;
      const int tb = u & 1;
      tc::mbar_wait(&s.tfull[tb], (u >> 1) & 1);
      tc::tc_fence_after();
      // this warpgroup's 4 tokens x 16 heads = 64 TMEM columns, one wait
      float sc[4];
      {
        const int kb = half * 4;
        uint32_t va[32], vb[32];
        tc::tmem_ld32(tmem + lane_off + tb * kCols + kb * kG, va);
        tc::tmem_ld32(tmem + lane_off + tb * kCols + kb * kG + 32, vb);
        tc::tmem_ld_wait();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;  // independent chains
#pragma unroll
          for (int h = 0; h < kG; h += 4) {
            const int cidx = k * kG + h;
            const float4 st01 = *reinterpret_cast<const float4 *>(&s.stat[(kb + k) * kG + h]);
            const float4 st23 = *reinterpret_cast<const float4 *>(&s.stat[(kb + k) * kG + h + 2]);
            const uint32_t u0 = cidx < 32 ? va[cidx] : vb[cidx - 32];
            const uint32_t u1 = cidx + 1 < 32 ? va[cidx + 1] : vb[cidx + 1 - 32];
            const uint32_t u2 = cidx + 2 < 32 ? va[cidx + 2] : vb[cidx + 2 - 32];
            const uint32_t u3 = cidx + 3 < 32 ? va[cidx + 3] : vb[cidx + 3 - 32];
            // heads offloaded to the FMA pipe (poly_exp2) relieve MUFU, the
            // bound of this epilogue
            const float x0 = fmaf(__uint_as_float(u0), p.scale_log2, -st01.x);
            a0 = fmaf(((h / 4) < SWATTN_K2_POLY_GROUPS) ? poly_exp2(x0) : K2_EXP(x0), st01.y, a0);
            a1 = fmaf(K2_EXP(fmaf(__uint_as_float(u1), p.scale_log2, -st01.z)), st01.w, a1);
            a2 = fmaf(K2_EXP(fmaf(__uint_as_float(u2), p.scale_log2, -st23.x)), st23.y, a2);
            a3 = fmaf(K2_EXP(fmaf(__uint_as_float(u3), p.scale_log2, -st23.z)), st23.w, a3);
          }
          sc[k] = (a0 + a1) + (a2 + a3);
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&s.tempty[tb]);
      // stage the tile's column scores [token][column]; the 5/4 max-pool then
      // runs one block per lane (epilogue warp e pools token e), so the 31
      // block scores of a token are written coalesced and the tie flags come
      // straight out of two ballots
#pragma unroll
      for (int k = 0; k < 4; ++k) s.sc[half * 4 + k][r] = sc[k];
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      const int qb = lane;
      const int j = t * kTileBlocks + qb;
      const bool blk_ok = qb < kTileBlocks && j >= p.N_init && j < hi;
      {
        const int k = warp - 2;
        const int64_t tok = i0 + k;
        const bool ok = blk_ok && tok < p.r1;
        float v[kPoolL];
#pragma unroll
        for (int e = 0; e < kPoolL; ++e) v[e] = s.sc[k][min(qb * kPoolS + e, kCols - 1)];
        const float mx = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), v[4]);
        if (ok) p.s_cmp[((int64_t)g * p.n + tok) * p.ld + j] = mx;
        if (fuse && !covf) {
          // threshold: every lane holds >= 3 keys >= its 3rd largest, so >= 93
          // keys are >= tau = the lanes' minimum, and the final top-k is above
          // it; appending / keeping keys >= tau (1 - 4 eps) also keeps the
          // float32 error band below the final k-th.  Compaction is then one
          // ordered stream-compaction pass (no k-th search in the tile loop).
          const uint32_t key = ok ? f2key(mx) : 0u;
          if (key > t3) {
            if (key > t1) { t3 = t2; t2 = t1; t1 = key; }
            else if (key > t2) { t3 = t2; t2 = key; }
            else t3 = key;
          }
          const uint32_t tau = __reduce_min_sync(0xffffffffu, lane < kTileBlocks ? t3 : 0xffffffffu);
          if (tau != 0u) cthr = max(cthr, f2key(key2f(tau) * (1.f - 4.f * kScoreRelErr)));
          if (ccnt + kTileBlocks > kCand) {
            uint32_t kv[kCand / 32];
            uint16_t iv[kCand / 32];
#pragma unroll
            for (int e = 0; e < kCand / 32; ++e) {
              const int q = e * 32 + lane;
              kv[e] = q < ccnt ? s.ckey[k][q] : 0u;
              iv[e] = q < ccnt ? s.cid[k][q] : (uint16_t)0;
            }
            __syncwarp();
            int w = 0;
#pragma unroll
            for (int e = 0; e < kCand / 32; ++e) {
              const bool keep = kv[e] >= cthr && kv[e] != 0u;
              const unsigned km = __ballot_sync(0xffffffffu, keep);
              if (keep) {
                const int pos = w + __popc(km & ((1u << lane) - 1u));
                s.ckey[k][pos] = kv[e];
                s.cid[k][pos] = iv[e];
              }
              w += __popc(km);
            }
            ccnt = w;
            __syncwarp();
            if (ccnt + kTileBlocks > kCand) {
              // the lane bound was too loose: raise the threshold to the exact
              // k-th largest x (1 - 4 eps) and compact again (a few times per row)
#pragma unroll
              for (int e = 0; e < kCand / 32; ++e) {
                const int q = e * 32 + lane;
                kv[e] = q < ccnt ? s.ckey[k][q] : 0u;
                iv[e] = q < ccnt ? s.cid[k][q] : (uint16_t)0;
              }
              const uint32_t T = warp_kth_key(kv, ksel);
              cthr = max(cthr, f2key(key2f(T) * (1.f - 4.f * kScoreRelErr)));
              __syncwarp();
              w = 0;
#pragma unroll
              for (int e = 0; e < kCand / 32; ++e) {
                const bool keep = kv[e] >= cthr && kv[e] != 0u;
                const unsigned km = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                  const int pos = w + __popc(km & ((1u << lane) - 1u));
                  s.ckey[k][pos] = kv[e];
                  s.cid[k][pos] = iv[e];
                }
                w += __popc(km);
              }
              ccnt = w;
              __syncwarp();
            }
            covf = ccnt + kTileBlocks > kCand;  // massive ties: the fallback selects from S^cmp
          }
          const bool take = ok && !covf && key >= cthr;
          const unsigned tm = __ballot_sync(0xffffffffu, take);
          if (take) {
            const int pos = ccnt + __popc(tm & ((1u << lane) - 1u));
            s.ckey[k][pos] = key;
            s.cid[k][pos] = (uint16_t)j;
          }
          ccnt += __popc(tm);
          __syncwarp();
        }
        if (p.flags != nullptr) {
          // argmax-at-shared-column bits (L: window col 0, R: col 4) with margin
          const float f = 1.f + 4.f * kScoreRelErr;
          const bool L = ok && v[1] * f < v[0] && v[2] * f < v[0] && v[3] * f < v[0] && v[4] * f < v[0];
          const bool R = ok && v[0] * f < v[4] && v[1] * f < v[4] && v[2] * f < v[4] && v[3] * f < v[4];
          const unsigned lm = __ballot_sync(0xffffffffu, L);
          const unsigned rm = __ballot_sync(0xffffffffu, R);
          if (lane == 0 && tok < p.r1)
            p.flags[((int64_t)g * p.n + tok) * p.ld_f + t] = spread_bits(lm) | (spread_bits(rm) << 1);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");  // s.sc reuse by the next tile
    }
    if (fuse) {
      // ---- the token's selection from its candidate set (as K3 from S^cmp,
      // topk.cu / topk_cta.cuh: keys > T, then keys == T by ascending block
      // index, emitted ascending; the same float32 ambiguity test)
      const int k = warp - 2;
      const int64_t tok = i0 + k;
      if (tok < p.r1) {
        const int64_t row = (int64_t)g * p.n + tok;
        int32_t *out = p.topk + row * p.k_top;
        if (lane == 0) p.topk_cnt[row] = ksel;
        if (covf) {
          if (lane == 0) p.ovf_rows[atomicAdd(p.ovf_count, 1)] = (int32_t)row;
        } else {
          uint32_t kv[kCand / 32];
          uint16_t iv[kCand / 32];
#pragma unroll
          for (int e = 0; e < kCand / 32; ++e) {
            const int q = e * 32 + lane;
            kv[e] = q < ccnt ? s.ckey[k][q] : 0u;
            iv[e] = q < ccnt ? s.cid[k][q] : (uint16_t)0;
          }
          const bool all = ksel >= max(hi - p.N_init, 0);  // every candidate: no ranking
          const uint32_t T = all ? 0u : warp_kth_key(kv, ksel);
          int gt = 0, eq = 0;
          uint32_t below = 0u, above = 0xffffffffu;
#pragma unroll
          for (int e = 0; e < kCand / 32; ++e) {
            if (kv[e] == 0u) continue;
            if (kv[e] > T) { ++gt; above = min(above, kv[e]); }
            else if (kv[e] == T) ++eq;
            else below = max(below, kv[e]);
          }
          gt = __reduce_add_sync(0xffffffffu, gt);
          eq = __reduce_add_sync(0xffffffffu, eq);
          below = __reduce_max_sync(0xffffffffu, below);
          above = __reduce_min_sync(0xffffffffu, above);
          const int need_eq = ksel - gt;
          int written = 0, eq_seen = 0, first = -1, second = -1;
#pragma unroll
          for (int e = 0; e < kCand / 32; ++e) {
            const bool valid = kv[e] != 0u;
            const bool is_eq = valid && kv[e] == T && !all;
            const unsigned em = __ballot_sync(0xffffffffu, is_eq);
            const int eq_rank = eq_seen + __popc(em & ((1u << lane) - 1u));
            const bool tk = valid && (all || kv[e] > T || (is_eq && eq_rank < need_eq));
            const unsigned tkm = __ballot_sync(0xffffffffu, tk);
            if (tk) out[written + __popc(tkm & ((1u << lane) - 1u))] = iv[e];
            written += __popc(tkm);
            // the first two tied ids (ascending: buffer order)
            unsigned x = em;
            while (x && second < 0) {
              const int src = __ffs(x) - 1;
              x &= x - 1;
              const int id = __shfl_sync(0xffffffffu, (int)iv[e], src);
              if (first < 0) first = id; else second = id;
            }
            eq_seen += __popc(em);
          }
          for (int q = written + lane; q < p.k_top; q += 32) out[q] = -1;
          if (!all && p.amb.count != nullptr) {
            bool ambiguous;
            if (gt + eq > ksel) {
              ambiguous = true;
              if (eq == 2 && p.amb.flags != nullptr && second == first + 1) {
                const int jj = first;
                const uint64_t *fr = p.amb.flags + row * p.amb.ld_f;
                const int tj = jj / 31, qj = jj % 31, tj1 = (jj + 1) / 31, qj1 = (jj + 1) % 31;
                const bool R_j = (fr[tj] >> (2 * qj + 1)) & 1ull;
                const bool L_j1 = (fr[tj1] >> (2 * qj1)) & 1ull;
                ambiguous = !(R_j && L_j1) || tie_neighbours_close(T, below, above);
              }
            } else {
              const float vk = key2f(T);
              const float vb = below ? key2f(below) : -INFINITY;
              ambiguous = (vk - vb) <= 3.0f * kScoreRelErr * fabsf(vk);
            }
            if (ambiguous && lane == 0) {
              const int slot = atomicAdd(p.amb.count, 1);
              if (slot < p.amb.cap) {
                p.amb.rows[slot] = (int32_t)row;
                p.amb.rows[p.amb.cap + slot] = (int32_t)T;
              }
            }
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

bool scores_tc_available() { return true; }

int32_t launch_scores_tc(const swattn_config *cfg, const void *Q, const void *kc1, const void *kc2,
                         int64_t n, int64_t r0, int64_t r1, int32_t mode, float *s_cmp, int64_t ld,
                         uint64_t *flags, int64_t ld_f, cudaStream_t stream, const FusedTopk *fz) {
  ScParams p;
  memset(&p, 0, sizeof(p));
  if (fz != nullptr) {
    p.topk = fz->topk;
    p.topk_cnt = fz->topk_cnt;
    p.k_top = cfg->k_top;
    p.amb = AmbList{fz->amb_count, fz->amb_rows, fz->amb_cap, flags, ld_f};
    p.ovf_count = fz->ovf_count;
    p.ovf_rows = fz->ovf_rows;
  }
  p.n = n;
  p.m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  p.m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  p.l_C1 = cfg->l_C1; p.s_C1 = cfg->s_C1; p.l_C2 = cfg->l_C2; p.s_C2 = cfg->s_C2;
  p.N_init = cfg->N_init;
  p.N_local = cfg->N_local;
  p.B = cfg->B;
  p.n_cols = (int)(p.m1 ? cdiv(p.m1, cfg->s) : 0);
  p.approx = mode == SWATTN_SELECT_APPROX && p.m2 > 0;
  const float scale = cfg->scale_compressed_logits ? 1.f / sqrtf((float)cfg->d_h) : 1.f;
  p.scale_log2 = scale * 1.4426950408889634f;
  // rows before (N_init + N_local) * B have no candidates; tiles of 8 tokens
  // never straddle a query block (row ranges are multiples of 8)
  p.tok0 = std::max<int64_t>((int64_t)(cfg->N_init + cfg->N_local) * cfg->B, r0);
  p.r1 = r1;
  if (p.tok0 >= r1 || p.n_cols <= cfg->N_init) return SWATTN_OK;
  p.n_tiles_tok = (int)cdiv(r1 - p.tok0, kTok);
  p.s_cmp = s_cmp;
  p.ld = ld;
  p.flags = flags;
  p.ld_f = ld_f;
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cfg->h_q, (uint64_t)n};
    const uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)cfg->h_q * kD * 2};
    const uint32_t box[3] = {64, (uint32_t)kG, (uint32_t)kTok};
    if (!make_tmap_bf16(&p.q_map, Q, 3, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(Q) failed");
      return SWATTN_ECUDA;
    }
  }
  {
    const uint64_t dims[2] = {(uint64_t)cfg->h_kv * kD, (uint64_t)p.m1};
    const uint64_t str[1] = {(uint64_t)cfg->h_kv * kD * 2};
    const uint32_t box[2] = {64, (uint32_t)kCols};
    if (!make_tmap_bf16(&p.k1_map, kc1, 2, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(K_C1) failed");
      return SWATTN_ECUDA;
    }
    if (p.approx) {
      const uint64_t dims2[2] = {(uint64_t)cfg->h_kv * kD, (uint64_t)p.m2};
      if (!make_tmap_bf16(&p.k2_map, kc2, 2, dims2, str, box)) {
        set_error("cuTensorMapEncodeTiled(K_C2) failed");
        return SWATTN_ECUDA;
      }
    } else {
      p.k2_map = p.k1_map;
    }
  }
  const size_t smem_f = sizeof(ScSmem) + 1024, smem = offsetof(ScSmem, ckey) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(scores_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(scores_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_f);
    attr = true;
  }
  const GroupRange gr = group_range(cfg);
  p.g0 = gr.g0;
  dim3 grid((unsigned)p.n_tiles_tok, (unsigned)gr.gc);
  if (p.topk != nullptr)
    scores_tc_kernel<true><<<grid, kThreads, smem_f, stream>>>(p);
  else
    scores_tc_kernel<false><<<grid, kThreads, smem, stream>>>(p);
  SWATTN_LAUNCH_CHECK("scores_tc_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
