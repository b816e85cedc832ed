// K5 on tcgen05 with two query tiles per CTA (dense causal / non-causal,
// long sequences).  The same tile math as attention_tc.cu (128 GQA-packed
// rows = 8 tokens x 16 heads, 64-key blocks, S / P / O in TMEM, one thread
// per row, lazy rescaling), but a CTA owns 16 consecutive tokens as tiles A
// and B of one KV group: every K / V block is loaded once for both, and the
// two MMA issuers (one per tile) keep the tensor pipe fed from both tiles,
// so it works on one tile while the other tile's softmax warps run.  One CTA per SM (TMEM: S_A x2 | S_B x2 | O_A | O_B = 512 columns),
// 3-stage K / V rings (160 KB of shared memory).
//
// Warp roles (352 threads): warp 0 TMA (lane 0: Q_A, Q_B, K; lane 1: V),
// warps 1 / 10 the MMA issuers of tiles A / B, warps 2-5 softmax of tile A,
// warps 6-9 tile B.
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

constexpr int kRows = 128;
constexpr int kTokTile = kRows / kG;  // 8 tokens per tile
constexpr int kThreads = 352;
constexpr uint32_t kQBytes = kRows * kD * 2;  // 32 KB per tile
constexpr float kRescaleThresh = 8.0f;

// kStep keys per pipeline step: 64 (S double-buffered per tile, 3 K/V
// stages) or 128 (N = 128 S MMAs -- half the tcgen05.mma issues per key --
// single S buffer per tile, 2 K/V stages of 32 KB).
template <int kStep>
struct StepCfg {
  static constexpr int kStages = kStep == 64 ? 3 : 2;
  static constexpr int kSBuf = kStep == 64 ? 2 : 1;
  static constexpr uint32_t kKVBytes = kStep * kD * 2;
};

struct Fa2Params {
  CUtensorMap q_map;  // Q [n][h_q][d]: box {64, 16, 8}
  CUtensorMap k_map;  // K [n][h_kv*d]: box {64, 64}
  CUtensorMap v_map;
  int64_t n;
  int h_q, h_kv, g0, gc;
  int n_pairs;  // 16-token tile pairs of this launch
  int causal;
  int part_a;    // sparse part A (sparse.py:43-98): init U local blocks only
  int N_init, N_local;
  int64_t r0, r1;  // rows [r0, r1) of this launch (r0 a multiple of 16)
  float *m_out, *l_out;  // part A: per-row running max (log2) and sum
  float scale_log2;
  __nv_bfloat16 *O;
  float *lse;
};

#ifndef SWATTN_FA2_POLY
#define SWATTN_FA2_POLY 0  // every Nth column pair's exp2 on the FMA pipe (measurement)
#endif
// 2^x for a pair on the FMA pipe: degree-3 minimax on the rounded-off
// fraction (7.7e-5 relative, below the bf16 rounding of P)
__device__ __forceinline__ float2 poly_exp2x2_fa2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 r = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);
  float2 q = ffma2(make_float2(0.05508868f, 0.05508868f), f, make_float2(0.24260405f, 0.24260405f));
  q = ffma2(q, f, make_float2(0.6932762f, 0.6932762f));
  q = ffma2(q, f, make_float2(0.99992895f, 0.99992895f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

template <int kStep>
struct __align__(1024) Fa2Smem {
  static constexpr int kStages = StepCfg<kStep>::kStages;
  uint8_t q[2][kQBytes];
  uint8_t k[kStages][StepCfg<kStep>::kKVBytes];
  uint8_t v[kStages][StepCfg<kStep>::kKVBytes];
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2][2], p_full[2][2];  // [tile][buffer]
  uint64_t o_final[2];
  uint32_t tmem_base;
};

template <int kStep>
__global__ void __launch_bounds__(kThreads, 1) fa2_dense_kernel(const __grid_constant__ Fa2Params p) {
  constexpr int kBlk = kStep;
  constexpr int kStages = StepCfg<kStep>::kStages;
  constexpr int kSBuf = StepCfg<kStep>::kSBuf;
  constexpr uint32_t kKVBytes = StepCfg<kStep>::kKVBytes;
  extern __shared__ uint8_t smem_raw[];
  Fa2Smem<kStep> &s =
      *reinterpret_cast<Fa2Smem<kStep> *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heavy (late) pairs first, group-major within a wave
  const int w = blockIdx.x;
  const int g = p.g0 + w / p.n_pairs;
  const int pair = p.n_pairs - 1 - w % p.n_pairs;
  const int64_t t0 = p.r0 + (int64_t)pair * 2 * kTokTile;
  const int64_t nb_total = cdiv(p.n, kBlk);
  // block list: dense 0..b (causal) / all; part A [0, n_init) U [second, b]
  const int b = (int)(t0 / kBlk);
  int nblk, n_init = 0, second = 0;
  if (p.part_a) {
    n_init = min(p.N_init, b + 1);
    second = max(max(0, b - p.N_local + 1), n_init);
    nblk = n_init + (b + 1 - second);
  } else {
    nblk = p.causal ? b + 1 : (int)nb_total;  // steps of kStep keys
  }
  auto blk_at = [&](int i) { return p.part_a ? (i < n_init ? i : second + (i - n_init)) : i; };

  if (threadIdx.x == 0) {
    tc::mbar_init(&s.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.k_full[i], 1);
      tc::mbar_init(&s.k_empty[i], 2);  // one commit per tile's MMA issuer
      tc::mbar_init(&s.v_full[i], 1);
      tc::mbar_init(&s.v_empty[i], 2);
    }
    for (int t = 0; t < 2; ++t)
      for (int i = 0; i < kSBuf; ++i) {
        tc::mbar_init(&s.s_full[t][i], 1);
        tc::mbar_init(&s.p_full[t][i], 128);
      }
    tc::mbar_init(&s.o_final[0], 1);
    tc::mbar_init(&s.o_final[1], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&s.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  // columns: S of tile t, buffer j at 128 t + 64 j; O of tile t at 256 + 128 t

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    if (lane == 0) {
      tc::tma_prefetch(&p.q_map);
      tc::tma_prefetch(&p.k_map);
      tc::mbar_arrive_expect_tx(&s.q_full, 2 * kQBytes);
      for (int t = 0; t < 2; ++t)
        for (int h = 0; h < 2; ++h)
          tc::tma_load_3d(&p.q_map, &s.q_full, s.q[t] + h * (kQBytes / 2), h * 64, g * kG,
                          (int)(t0 + t * kTokTile));
      for (int i = 0; i < nblk; ++i) {
        const int st = i % kStages;
        tc::mbar_wait(&s.k_empty[st], ((i / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&s.k_full[st], kKVBytes);
        for (int h = 0; h < 2; ++h)
          tc::tma_load_2d(&p.k_map, &s.k_full[st], s.k[st] + h * (kKVBytes / 2), g * kD + h * 64,
                          blk_at(i) * kBlk);
      }
    } else if (lane == 1) {
      tc::tma_prefetch(&p.v_map);
      for (int i = 0; i < nblk; ++i) {
        const int st = i % kStages;
        tc::mbar_wait(&s.v_empty[st], ((i / kStages) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&s.v_full[st], kKVBytes);
        for (int h = 0; h < 2; ++h)
          tc::tma_load_2d(&p.v_map, &s.v_full[st], s.v[st] + h * (kKVBytes / 2), g * kD + h * 64,
                          blk_at(i) * kBlk);
      }
    }
    // drain: observe the last ring phases the MMA warp releases
    if (lane == 0 || lane == 1) {
      uint64_t *ring = lane == 0 ? s.k_empty : s.v_empty;
      for (int gd = nblk > kStages ? nblk - kStages : 0; gd < nblk; ++gd)
        tc::mbar_wait(&ring[gd % kStages], (gd / kStages) & 1);
    }
    __syncwarp();
  } else if (warp == 1 || warp == 10) {
    // ------------------------------------------------------------ MMA issuers
    // one issuing thread per tile (warp 1: A, warp 10: B): a tcgen05.mma has
    // a fixed issue cost that one thread would pay for both tiles; each
    // issuer commits its own ops, the K / V stages free after both
    const int t = warp == 1 ? 0 : 1;
    const uint32_t id_s = tc::idesc_bf16(kRows, kBlk, false, false);
    const uint32_t id_o = tc::idesc_bf16(kRows, kD, false, true);
    const uint32_t q_addr = tc::smem_u32(s.q[t]);
    tc::mbar_wait(&s.q_full, 0);
    tc::tc_fence_after();
    auto issue_s = [&](int i) {
      const int st = i % kStages;
      tc::mbar_wait(&s.k_full[st], (i / kStages) & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t k_addr = tc::smem_u32(s.k[st]);
        const uint32_t d_s = tmem + t * 128 + (i % kSBuf) * 64;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const int h = kk >> 2, j = kk & 3;
          tc::mma_ss(d_s, tc::desc_kmajor(q_addr + h * (kQBytes / 2) + j * 32),
                     tc::desc_kmajor(k_addr + h * (kKVBytes / 2) + j * 32), id_s, kk > 0);
        }
        tc::mma_commit(&s.s_full[t][i % kSBuf]);
        tc::mma_commit(&s.k_empty[st]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int j) {
      const int st = j % kStages;
      tc::mbar_wait(&s.v_full[st], (j / kStages) & 1);
      tc::mbar_wait(&s.p_full[t][j % kSBuf], (j / kSBuf) & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t v_addr = tc::smem_u32(s.v[st]);
        const uint32_t a_p = tmem + t * 128 + (j % kSBuf) * 64;
#pragma unroll
        for (int kk = 0; kk < kBlk / 16; ++kk)
          tc::mma_ts(tmem + 256 + t * 128, a_p + kk * 8,
                     tc::desc_mnmajor(v_addr + kk * 16 * 128, kKVBytes / 2), id_o,
                     (j > 0 || kk > 0) ? 1u : 0u);
        tc::mma_commit(&s.v_empty[st]);
        if (j == nblk - 1) tc::mma_commit(&s.o_final[t]);
      }
      __syncwarp();
    };
    // double-buffered S: S(i) goes out while the softmax still works on
    // S(i-1), then PV(i-1); single-buffered S (128-key steps): PV(i-1) must
    // consume P(i-1) before S(i) overwrites it -- the tile's own pipeline is
    // serial and the other tile's issuer fills the tensor pipe meanwhile
    for (int i = 0; i <= nblk; ++i) {
      if (kSBuf == 2) {
        if (i < nblk) issue_s(i);
        if (i >= 1) issue_pv(i - 1);
      } else {
        if (i >= 1) issue_pv(i - 1);
        if (i < nblk) issue_s(i);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int tile = (warp - 2) >> 2;  // 0: warps 2-5 (A), 1: warps 6-9 (B)
    const int quad = warp & 3;         // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tmem_s = tmem + tile * 128, tmem_o = tmem + 256 + tile * 128;
    const int64_t tok = t0 + tile * kTokTile + r / kG;
    float m = -INFINITY, l = 0.f;
    for (int i = 0; i < nblk; ++i) {
      tc::mbar_wait(&s.s_full[tile][i % kSBuf], (i / kSBuf) & 1);
      tc::tc_fence_after();
      const uint32_t sbuf = tmem_s + lane_off + (i % kSBuf) * 64;
      const int64_t key0 = (int64_t)blk_at(i) * kBlk;
      const bool diag = p.causal && (key0 + kBlk - 1 > tok);
      const bool pad = !p.causal && (key0 + kBlk > p.n);
      const int64_t lim = diag ? tok - key0 : p.n - 1 - key0;  // last visible column (diag / pad)
      // 64 columns of S (chunk c0) with the diagonal / padding mask
      auto load64 = [&](int c0, float (&x)[64]) {
        uint32_t ra[32], rb[32];
        tc::tmem_ld32(sbuf + c0, ra);
        tc::tmem_ld32(sbuf + c0 + 32, rb);
        tc::tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 64; ++c) x[c] = __uint_as_float(c < 32 ? ra[c] : rb[c - 32]);
        if (diag || pad) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c0 + c > lim) x[c] = -INFINITY;
        }
      };
      float x[64];
      load64(0, x);
      float mx = max64(x);
      if constexpr (kBlk == 128) {
        // pass 1 of 2 over TMEM: the second chunk's max only (x keeps chunk 0
        // for nothing -- it is reloaded in pass 2 to bound the registers)
        float y[64];
        load64(64, y);
        mx = fmaxf(mx, max64(y));
      }
      mx *= p.scale_log2;
      const bool want = mx > m + kRescaleThresh || m == -INFINITY;
      const float m_new = want ? fmaxf(mx, m) : m;
      const bool resc = want && m != -INFINITY && i > 0;
      if (__any_sync(0xffffffffu, resc)) {
        // PV(i-1) of both tiles is done once its V stage is released (one
        // commit per tile); that stage's next phase needs P(i+2) from this
        // warp: unambiguous parity
        const float alpha = resc ? fast_exp2(m - m_new) : 1.f;
        tc::mbar_wait(&s.v_empty[(i - 1) % kStages], ((i - 1) / kStages) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < kD; c0 += 32) {
          uint32_t o[32];
          tc::tmem_ld32(tmem_o + lane_off + c0, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tc::tmem_st32(tmem_o + lane_off + c0, o);
        }
        l *= alpha;
      }
      m = m_new;
      if constexpr (kBlk == 64) {
        // P first, released to the MMA warp, then the row sum off the critical path
        uint32_t pk[32];
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m, -m);
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float2 a2 = ffma2(make_float2(x[c], x[c + 1]), sc2, nm2);
#if SWATTN_FA2_POLY > 0
          if ((c / 2) % SWATTN_FA2_POLY == SWATTN_FA2_POLY - 1) {
            const float2 e2 = poly_exp2x2_fa2(a2);
            x[c] = e2.x;
            x[c + 1] = e2.y;
          } else
#endif
          {
            x[c] = fast_exp2(a2.x);
            x[c + 1] = fast_exp2(a2.y);
          }
          pk[c / 2] = tc::pack_bf16(x[c], x[c + 1]);
        }
        tc::tmem_st32(sbuf, pk);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.p_full[tile][i % kSBuf]);
        float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          s0 = fadd2(s0, make_float2(x[c], x[c + 1]));
          s1 = fadd2(s1, make_float2(x[c + 2], x[c + 3]));
        }
        l += (s0.x + s0.y) + (s1.x + s1.y);
      } else {
        // pass 2: both chunks reloaded, exps packed; P overwrites S columns
        // 0..63, so it is stored only after both chunks are read
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m, -m);
        float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
        uint32_t pw0[32], pw1[32];
        auto exps = [&](const float (&xx)[64], uint32_t (&pw)[32]) {
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const float2 a01 = ffma2(make_float2(xx[c], xx[c + 1]), sc2, nm2);
            const float2 a23 = ffma2(make_float2(xx[c + 2], xx[c + 3]), sc2, nm2);
            const float2 e01 = make_float2(fast_exp2(a01.x), fast_exp2(a01.y));
            const float2 e23 = make_float2(fast_exp2(a23.x), fast_exp2(a23.y));
            pw[c / 2] = tc::pack_bf16(e01.x, e01.y);
            pw[c / 2 + 1] = tc::pack_bf16(e23.x, e23.y);
            s0 = fadd2(s0, e01);
            s1 = fadd2(s1, e23);
          }
        };
        exps(x, pw0);  // chunk 0 is still in x
        load64(64, x);
        exps(x, pw1);
        tc::tmem_st32(sbuf, pw0);
        tc::tmem_st32(sbuf + 32, pw1);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.p_full[tile][i % kSBuf]);
        l += (s0.x + s0.y) + (s1.x + s1.y);
      }
    }
    tc::mbar_wait(&s.o_final[tile], 0);
    tc::tc_fence_after();
    const bool valid = tok < p.r1;
    const int hq = g * kG + (r % kG);
    const int64_t idx = tok * p.h_q + hq;
    const float inv_l = 1.f / l;
    __nv_bfloat16 *orow = p.O + idx * kD;
#pragma unroll
    for (int c0 = 0; c0 < kD; c0 += 32) {
      uint32_t o[32];
      tc::tmem_ld32(tmem_o + lane_off + c0, o);
      tc::tmem_ld_wait();
      if (valid) {
        uint4 *dst = reinterpret_cast<uint4 *>(orow + c0);
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 wv;
          wv.x = tc::pack_bf16(__uint_as_float(o[e]) * inv_l, __uint_as_float(o[e + 1]) * inv_l);
          wv.y = tc::pack_bf16(__uint_as_float(o[e + 2]) * inv_l, __uint_as_float(o[e + 3]) * inv_l);
          wv.z = tc::pack_bf16(__uint_as_float(o[e + 4]) * inv_l, __uint_as_float(o[e + 5]) * inv_l);
          wv.w = tc::pack_bf16(__uint_as_float(o[e + 6]) * inv_l, __uint_as_float(o[e + 7]) * inv_l);
          dst[e / 8] = wv;
        }
      }
    }
    if (valid) {
      p.lse[idx] = (m + __log2f(l)) * 0.6931471805599453f;
      if (p.m_out != nullptr) {
        p.m_out[idx] = m;
        p.l_out[idx] = l;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace

// Dense causal / non-causal attention of all n rows with two query tiles per
// CTA (requires n to be a multiple of 16 tokens; the caller falls back to the
// one-tile kernel otherwise).
template <int kStep>
static int32_t launch_fa2(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, int64_t r0, int64_t r1, int causal, int part_a, void *O,
                          float *lse, float *m_out, float *l_out, cudaStream_t stream) {
  if (r1 <= r0) return SWATTN_OK;
  Fa2Params p;
  memset(&p, 0, sizeof(p));
  {
    const uint64_t dims[3] = {(uint64_t)kD, (uint64_t)cfg->h_q, (uint64_t)n};
    const uint64_t str[2] = {(uint64_t)kD * 2, (uint64_t)cfg->h_q * kD * 2};
    const uint32_t box[3] = {64, (uint32_t)kG, (uint32_t)kTokTile};
    if (!make_tmap_bf16(&p.q_map, Q, 3, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(Q) failed");
      return SWATTN_ECUDA;
    }
  }
  {
    const uint64_t dims[2] = {(uint64_t)cfg->h_kv * kD, (uint64_t)n};
    const uint64_t str[1] = {(uint64_t)cfg->h_kv * kD * 2};
    const uint32_t box[2] = {64, (uint32_t)kStep};
    if (!make_tmap_bf16(&p.k_map, K, 2, dims, str, box) ||
        !make_tmap_bf16(&p.v_map, V, 2, dims, str, box)) {
      set_error("cuTensorMapEncodeTiled(K/V) failed");
      return SWATTN_ECUDA;
    }
  }
  p.n = n;
  p.h_q = cfg->h_q;
  p.h_kv = cfg->h_kv;
  const GroupRange gr = group_range(cfg);
  p.g0 = gr.g0;
  p.gc = gr.gc;
  p.n_pairs = (int)cdiv(r1 - r0, 2 * kTokTile);
  p.causal = causal;
  p.part_a = part_a;
  p.N_init = cfg->N_init;
  p.N_local = cfg->N_local;
  p.r0 = r0;
  p.r1 = r1;
  p.m_out = m_out;
  p.l_out = l_out;
  p.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  p.O = static_cast<__nv_bfloat16 *>(O);
  p.lse = lse;
  const size_t smem = sizeof(Fa2Smem<kStep>) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fa2_dense_kernel<kStep>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  fa2_dense_kernel<kStep><<<(unsigned)((int64_t)p.n_pairs * gr.gc), kThreads, smem, stream>>>(p);
  SWATTN_LAUNCH_CHECK("fa2_dense_kernel");
  return SWATTN_OK;
}

// Dense causal / non-causal attention of all n rows with two query tiles per
// CTA; step = 64 or 128 keys per pipeline step.
int32_t launch_dense_tc2(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int causal, void *O, float *lse, cudaStream_t stream, int step) {
  if (step == 128)
    return launch_fa2<128>(cfg, Q, K, V, n, 0, n, causal, 0, O, lse, nullptr, nullptr, stream);
  return launch_fa2<64>(cfg, Q, K, V, n, 0, n, causal, 0, O, lse, nullptr, nullptr, stream);
}

// Sparse part A of rows [r0, r1) (r0 a multiple of 16) on the two-tile kernel.
int32_t launch_part_a_tc2(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, int64_t r0, int64_t r1, void *O, float *lse, float *m_out,
                          float *l_out, cudaStream_t stream) {
  return launch_fa2<64>(cfg, Q, K, V, n, r0, r1, 1, 1, O, lse, m_out, l_out, stream);
}

}  // namespace swattn
