// K5 / K4-part-A -- block-list flash attention on tcgen05 (sm_100a).
//
// One work item = one GQA-packed query tile of 128 rows = 8 tokens x 16 heads
// of one KV group (row r <-> token t0 + r/16, head 16g + r%16), so every row
// of the tile reads the same K/V blocks.  Up to 8192 items the CTAs are
// persistent (two per SM walk the items); above that one CTA per item.  The tile walks a list of 64-key
// blocks:
//   dense (tiled_gqa_forward, dense.py:112-170): blocks 0..b, causal;
//   sparse part A (sparse.py:43-98, the init + local blocks every token of a
//   query block shares, selection.py:113-119): [0, n_init) U [lo, b].
//
// Warp roles (192 threads, 2 CTAs / SM):
//   warp 0      TMA producers: lane 0 issues Q once then K blocks, lane 1
//               V blocks, through two independent 2-stage rings (K freed
//               after QK^T, V after PV);
//   warp 1      MMA issuer (one elected lane): S_j = Q K_j^T into a
//               double-buffered TMEM S tile (128 x 64 fp32), then
//               O += P_{j-1} V_{j-1} with P read straight from TMEM (kind::f16
//               A-from-TMEM), O accumulated in TMEM (128 x 128 fp32);
//   warps 2..5  softmax: thread = row; online max (FMNMX3) with lazy
//               rescaling (O is rescaled in TMEM only when the row max grows
//               by > 2^8, warp-collectively), P = exp2(s*scale*log2e - m)
//               (one FFMA + ex2) packed to bf16 into the S buffer; epilogue
//               O / l -> bf16, lse.
// Roofline: tensor-bound; algorithmic FLOP = 4 * visible_pairs * d_h * h_q
// (dense.py:167-169 counts x 2).
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "route.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

constexpr int kRows = 128;         // query rows per tile
constexpr int kTokTile = kRows / kG;  // 8 tokens
constexpr int kBlk = 64;           // keys per block
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr uint32_t kQBytes = kRows * kD * 2;     // 32 KB
constexpr uint32_t kKVBytes = kBlk * kD * 2;     // 16 KB
constexpr uint32_t kTmemCols = 256;              // S0 | S1 | O
constexpr float kRescaleThresh = 8.0f;           // log2 units

struct FaParams {
  CUtensorMap q_map;   // Q [n][h_q][d]: box {64, 16, 8}
  CUtensorMap k_map;   // K [n][h_kv*d]: box {64, 64}
  CUtensorMap v_map;
  int64_t n;
  int h_q, h_kv, g0, gc;
  int n_tiles;         // token tiles of 8 in this launch
  int tile_end;        // tiles [tile_end - n_tiles, tile_end)
  int mode;            // 0 dense causal, 1 dense non-causal, 2 sparse part A,
                       // 3 routed tiles (union of the tiles' top-k blocks, route.cuh)
  int N_init, N_local;
  float scale_log2;
  __nv_bfloat16 *O;
  float *lse;          // [n][h_q]
  float *m_out, *l_out;  // part A: per-row running max (log2) and sum, [n][h_q] (mode 3: in)
  TileRoutes routes;     // mode 3
};

struct __align__(1024) FaSmem {
  uint8_t q[kQBytes];
  uint8_t k[kStages][kKVBytes];
  uint8_t v[kStages][kKVBytes];
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2];
  uint64_t o_final;
  uint64_t q_empty, o_empty;  // persistent CTAs: Q slot / O accumulator free for the next item
  uint32_t tmem_base;
};

// 2^x for a pair on the FMA pipe (degree-3 minimax on the rounded-off
// fraction, 7.7e-5 relative error -- far below the bf16 rounding of P):
// takes some exps off MUFU, which the softmax otherwise saturates
// (16 ex2 / clk / SM, profiles/r02ax_mufu_bench.txt).
__device__ __forceinline__ float2 poly_exp2x2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));  // 1.5 * 2^23: round to integer
  const float2 r = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);           // x - round(x), |f| <= 0.5
  float2 q = ffma2(make_float2(0.05508868f, 0.05508868f), f, make_float2(0.24260405f, 0.24260405f));
  q = ffma2(q, f, make_float2(0.6932762f, 0.6932762f));
  q = ffma2(q, f, make_float2(0.99992895f, 0.99992895f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

#ifndef SWATTN_FA_POLY
// every SWATTN_FA_POLY-th column pair's exps on the FMA pipe (0: none).  Off:
// 1/8, 1/4, 1/3 of the pairs measured 1 %, 10 %, 10 % slower at 128K dense
// (profiles/r02bc_fa_poly.txt) -- the softmax warp's issue / latency, not
// the MUFU rate, bounds it.
#define SWATTN_FA_POLY 0
#endif

// Block list of a tile (query block b): dense 0..b / 0..nb-1, part A init U local.
// Mode 3: the routed slot's ascending union list.
struct BlockList {
  int n_first, first_end;  // [0, first_end)
  int second_begin, second_end;  // [second_begin, second_end)
  const int16_t *ids;      // mode 3
  __device__ int size() const { return first_end + (second_end - second_begin); }
  __device__ int at(int i) const {
    if (ids != nullptr) return ids[i];
    return i < first_end ? i : second_begin + (i - first_end);
  }
};

template <bool kRouted>
__device__ __forceinline__ BlockList make_list(const FaParams &p, int b, int64_t nb_total,
                                               int64_t slot) {
  BlockList L;
  L.ids = nullptr;
  if (kRouted) {
    L.first_end = p.routes.ucount[slot];
    L.second_begin = L.second_end = 0;
    L.ids = p.routes.ulist + slot * kUCap;
  } else if (p.mode == 2) {
    const int n_init = min(p.N_init, b + 1);
    const int lo = max(0, b - p.N_local + 1);
    L.first_end = n_init;
    L.second_begin = max(lo, n_init);
    L.second_end = b + 1;
  } else {
    L.first_end = (p.mode == 0) ? b + 1 : (int)nb_total;
    L.second_begin = 0;
    L.second_end = 0;
  }
  L.n_first = 0;
  return L;
}

// Persistent: a CTA walks the (tile, group) items blockIdx.x, + gridDim.x, ...
// (heavy tiles first).  Every barrier phase is derived from running counters
// -- the global block index gi over all items of the CTA (K/V ring, S / P
// double buffers) and the item counter it (Q, o_final, q_empty,
// o_empty) -- which all four roles advance identically.  Q is reloaded once
// the previous item's last S MMA completed (q_empty); the first PV of an
// item waits until the softmax warps have read the previous O out of TMEM
// (o_empty).  TMEM is allocated once per CTA.
// Persistent CTAs take the items in zig-zag rounds (CTA c gets c, 2G-1-c,
// 2G+c, ...), so every CTA's heavy-first share sums to about the same work.
__device__ __forceinline__ int64_t fa_slot_item(int64_t w, int64_t n_items, int64_t G) {
  const int64_t r = w / G, c = w % G;
  return ((r & 1) && (r + 1) * G <= n_items) ? r * G + (G - 1 - c) : w;
}

template <bool kRouted>
__device__ __forceinline__ void fa_item(const FaParams &p, int64_t w, int &tile, int &g) {
  if (kRouted) {
    const int32_t it = p.routes.items[w];
    g = (int)(it / p.routes.ntiles);
    tile = (int)(it % p.routes.ntiles);
    return;
  }
  // group-major (one group's K/V, 67 MB at 128K, stays L2-resident while its
  // tiles run), heavy (late) tiles first within a group
  g = p.g0 + (int)(w / p.n_tiles);
  tile = p.tile_end - 1 - (int)(w % p.n_tiles);
}

// kPersist = false: one item per CTA (the grid covers the items); the item
// loops below then run once and the running counters fold to constants.
template <bool kPersist, bool kRouted = false>
__global__ void __launch_bounds__(kThreads, 2) fa_tile_kernel(const __grid_constant__ FaParams p) {
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on smem_raw so accesses stay in the shared space
  FaSmem &s = *reinterpret_cast<FaSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nb_total = cdiv(p.n, kBlk);
  const int64_t n_items = kRouted ? (int64_t)*p.routes.count : (int64_t)p.n_tiles * p.gc;
  // routed tiles run beside part B (programmatic launch): the plan's CTA count
  // works, the rest exit before touching TMEM; the working CTAs wait for part B
  // at the end so this grid's completion implies part B's.
  const int64_t ctas = kRouted ? (int64_t)p.routes.plan[0] : (int64_t)gridDim.x;
  if (kRouted && (int64_t)blockIdx.x >= (ctas > 0 ? ctas : 1)) return;
  if (kRouted && ctas == 0) {
    pdl_wait();
    return;
  }

  if (threadIdx.x == 0) {
    tc::mbar_init(&s.q_full, 1);
    tc::mbar_init(&s.q_empty, 1);
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&s.k_full[i], 1);
      tc::mbar_init(&s.k_empty[i], 1);
      tc::mbar_init(&s.v_full[i], 1);
      tc::mbar_init(&s.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s.s_full[i], 1);
      tc::mbar_init(&s.p_full[i], 128);
    }
    tc::mbar_init(&s.o_final, 1);
    tc::mbar_init(&s.o_empty, 128);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(&s.tmem_base);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t tmem_o = tmem + 128;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    // lane 0: Q + K blocks, lane 1: V blocks -- two issuing threads, since one
    // thread's TMA issue rate caps near 36 GB/s (tools/gather_bench.cu)
    if (lane == 0) {
      tc::tma_prefetch(&p.q_map);
      tc::tma_prefetch(&p.k_map);
    } else if (lane == 1) {
      tc::tma_prefetch(&p.v_map);
    }
    uint32_t gi0 = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += kPersist ? ctas : n_items, ++it) {
      int tile, g;
      const int64_t wi = kPersist ? fa_slot_item(w, n_items, ctas) : w;
      fa_item<kRouted>(p, wi, tile, g);
      const int64_t t0 = (int64_t)tile * kTokTile;
      const BlockList L = make_list<kRouted>(p, (int)(t0 / kBlk), nb_total, wi);
      const int nblk = L.size();
      if (lane == 0) {
        if (it > 0) tc::mbar_wait(&s.q_empty, (uint32_t)((it - 1) & 1));
        tc::mbar_arrive_expect_tx(&s.q_full, kQBytes);
        for (int h = 0; h < 2; ++h)
          tc::tma_load_3d(&p.q_map, &s.q_full, s.q + h * (kQBytes / 2), h * 64, g * kG, (int)t0);
        int nid = L.at(0);
        for (int i = 0; i < nblk; ++i) {
          const uint32_t gi = gi0 + (uint32_t)i;
          const int st = (int)(gi % kStages);
          const uint32_t ph = (((gi / kStages) & 1u) ^ 1u);
          const int key0 = nid * kBlk;
          if (i + 1 < nblk) nid = L.at(i + 1);
          tc::mbar_wait(&s.k_empty[st], ph);
          tc::mbar_arrive_expect_tx(&s.k_full[st], kKVBytes);
          for (int h = 0; h < 2; ++h)
            tc::tma_load_2d(&p.k_map, &s.k_full[st], s.k[st] + h * (kKVBytes / 2), g * kD + h * 64,
                            key0);
        }
      } else if (lane == 1) {
        int nid = L.at(0);
        for (int i = 0; i < nblk; ++i) {
          const uint32_t gi = gi0 + (uint32_t)i;
          const int st = (int)(gi % kStages);
          const uint32_t ph = (((gi / kStages) & 1u) ^ 1u);
          const int key0 = nid * kBlk;
          if (i + 1 < nblk) nid = L.at(i + 1);
          tc::mbar_wait(&s.v_empty[st], ph);
          tc::mbar_arrive_expect_tx(&s.v_full[st], kKVBytes);
          for (int h = 0; h < 2; ++h)
            tc::tma_load_2d(&p.v_map, &s.v_full[st], s.v[st] + h * (kKVBytes / 2), g * kD + h * 64,
                            key0);
        }
      }
      gi0 += (uint32_t)nblk;
    }
    // drain: observe the ring phases and the Q slot release the MMA warp
    // signals after the last issue, so no barrier phase completes unwaited
    // at exit (keeps compute-sanitizer synccheck clean; costs nothing)
    if (lane == 0 || lane == 1) {
      uint64_t *ring = lane == 0 ? s.k_empty : s.v_empty;
      for (uint32_t gd = gi0 > (uint32_t)kStages ? gi0 - kStages : 0u; gd < gi0; ++gd)
        tc::mbar_wait(&ring[gd % kStages], (gd / kStages) & 1u);
      if (lane == 0 && it > 0) tc::mbar_wait(&s.q_empty, (uint32_t)((it - 1) & 1));
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t id_s = tc::idesc_bf16(kRows, kBlk, false, false);
    const uint32_t id_o = tc::idesc_bf16(kRows, kD, false, true);
    const uint32_t q_addr = tc::smem_u32(s.q);
    uint32_t gi0 = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += kPersist ? ctas : n_items, ++it) {
      int tile, g;
      const int64_t wi = kPersist ? fa_slot_item(w, n_items, ctas) : w;
      fa_item<kRouted>(p, wi, tile, g);
      const int64_t t0 = (int64_t)tile * kTokTile;
      const BlockList L = make_list<kRouted>(p, (int)(t0 / kBlk), nb_total, wi);
      const int nblk = L.size();
      tc::mbar_wait(&s.q_full, (uint32_t)(it & 1));
      tc::tc_fence_after();
      for (int i = 0; i <= nblk; ++i) {
        if (i < nblk) {
          const uint32_t gi = gi0 + (uint32_t)i;
          const int st = (int)(gi % kStages);
          tc::mbar_wait(&s.k_full[st], ((gi / kStages) & 1u));
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t k_addr = tc::smem_u32(s.k[st]);
            const uint32_t d_s = tmem + (gi & 1u) * kBlk;
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
              const int h = kk >> 2, j = kk & 3;
              tc::mma_ss(d_s, tc::desc_kmajor(q_addr + h * (kQBytes / 2) + j * 32),
                         tc::desc_kmajor(k_addr + h * (kKVBytes / 2) + j * 32), id_s, kk > 0);
            }
            tc::mma_commit(&s.s_full[gi & 1u]);
            tc::mma_commit(&s.k_empty[st]);
            if (i == nblk - 1) tc::mma_commit(&s.q_empty);  // Q free once this S is done
          }
          __syncwarp();
        }
        if (i >= 1) {
          const int pi = i - 1;
          const uint32_t pg = gi0 + (uint32_t)pi;
          const int st = (int)(pg % kStages);
          if (pi == 0 && it > 0) {
            // the previous item's O has been read out of TMEM
            tc::mbar_wait(&s.o_empty, (uint32_t)((it - 1) & 1));
          }
          tc::mbar_wait(&s.p_full[pg & 1u], ((pg >> 1) & 1u));
          tc::mbar_wait(&s.v_full[st], ((pg / kStages) & 1u));
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t v_addr = tc::smem_u32(s.v[st]);
            const uint32_t a_p = tmem + (pg & 1u) * kBlk;
#pragma unroll
            for (int kk = 0; kk < kBlk / 16; ++kk)
              tc::mma_ts(tmem_o, a_p + kk * 8, tc::desc_mnmajor(v_addr + kk * 16 * 128, kKVBytes / 2),
                         id_o, (pi > 0 || kk > 0) ? 1u : 0u);
            tc::mma_commit(&s.v_empty[st]);  // also tells a rescaling softmax PV_pg is done
            if (pi == nblk - 1) tc::mma_commit(&s.o_final);
          }
          __syncwarp();
        }
      }
      gi0 += (uint32_t)nblk;
    }
    // drain: the last item's O release (no next item waits for it)
    if (it > 0) tc::mbar_wait(&s.o_empty, (uint32_t)((it - 1) & 1));
  } else {
    // ------------------------------------------------------------ softmax
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint32_t gi0 = 0;
    int it = 0;
    for (int64_t w = blockIdx.x; w < n_items; w += kPersist ? ctas : n_items, ++it) {
      int tile, g;
      const int64_t wi = kPersist ? fa_slot_item(w, n_items, ctas) : w;
      fa_item<kRouted>(p, wi, tile, g);
      const int64_t t0 = (int64_t)tile * kTokTile;
      const BlockList L = make_list<kRouted>(p, (int)(t0 / kBlk), nb_total, wi);
      const int nblk = L.size();
      const int64_t tok = t0 + r / kG;
      float m = -INFINITY, l = 0.f;
      // mode 3: this row's token takes block i of the union iff bit i is set
      const uint32_t *tbits =
          kRouted ? p.routes.tbits + (wi * kTokTile + r / kG) * kUWords : nullptr;
      uint32_t tword = 0;
      for (int i = 0; i < nblk; ++i) {
        const uint32_t gi = gi0 + (uint32_t)i;
        const int jb = kRouted ? 0 : L.at(i);
        if (kRouted && (i & 31) == 0) tword = tbits[i >> 5];
        const bool on = !kRouted || ((tword >> (i & 31)) & 1u);
        tc::mbar_wait(&s.s_full[gi & 1u], ((gi >> 1) & 1u));
        tc::tc_fence_after();
        uint32_t ra[32], rb[32];
        tc::tmem_ld32(tmem + lane_off + (gi & 1u) * kBlk, ra);
        tc::tmem_ld32(tmem + lane_off + (gi & 1u) * kBlk + 32, rb);
        tc::tmem_ld_wait();
        // raw logits; the scale is folded into the exp argument (one FFMA per
        // element) and masking runs only on the diagonal / padded block
        float x[kBlk];
        const int64_t key0 = (int64_t)jb * kBlk;
        const bool diag = !kRouted && (p.mode != 1) && (key0 + kBlk - 1 > tok);
        const bool pad = (p.mode == 1) && (key0 + kBlk > p.n);
#pragma unroll
        for (int c = 0; c < kBlk; ++c) x[c] = __uint_as_float(c < 32 ? ra[c] : rb[c - 32]);
        if (diag || pad) {
          const int64_t lim = diag ? tok - key0 : p.n - 1 - key0;  // last visible column
#pragma unroll
          for (int c = 0; c < kBlk; ++c)
            if (c > lim) x[c] = -INFINITY;
        }
        const float mx = on ? max64(x) * p.scale_log2 : -INFINITY;
        // Lazy rescale.  tcgen05.ld / st are warp-collective (.sync.aligned), so
        // the O read-modify-write runs for the whole warp whenever any of its
        // rows needs it; rows that do not scale by 1.
        const bool want = on && (mx > m + kRescaleThresh || m == -INFINITY);
        const float m_new = want ? fmaxf(mx, m) : m;
        const bool resc = want && m != -INFINITY && i > 0;
        if (__any_sync(0xffffffffu, resc)) {
          // PV_{gi-1} is complete when its V stage is released (v_empty is
          // committed right after it); that stage's next phase needs P_{gi+1}
          // from this warp, so the parity wait is unambiguous.
          const float alpha = resc ? fast_exp2(m - m_new) : 1.f;
          tc::mbar_wait(&s.v_empty[(gi - 1u) % kStages], ((gi - 1u) / kStages) & 1u);
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
        // P first (argument by packed FFMA2, ex2, pack), released to the MMA
        // warp, and only then the row sum over the kept exps -- off the
        // S -> P -> PV critical path
        uint32_t pk[kBlk / 2];
        if constexpr (kRouted) {
          // (routed tiles keep the inline sum: the deferred one spills at 168 registers)
          float rs = 0.f;
          if (on) {
#pragma unroll
            for (int c = 0; c < kBlk; c += 2) {
              const float p0 = fast_exp2(fmaf(x[c], p.scale_log2, -m));
              const float p1 = fast_exp2(fmaf(x[c + 1], p.scale_log2, -m));
              rs += p0 + p1;
              pk[c / 2] = tc::pack_bf16(p0, p1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < kBlk / 2; ++c) pk[c] = 0u;
          }
          l += rs;
          tc::tmem_st32(tmem + lane_off + (gi & 1u) * kBlk, pk);
          tc::tmem_st_wait();
          tc::tc_fence_before();
          tc::mbar_arrive(&s.p_full[gi & 1u]);
          continue;
        }
        {
          const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m, -m);
#pragma unroll
          for (int c = 0; c < kBlk; c += 2) {
            const float2 a2 = ffma2(make_float2(x[c], x[c + 1]), sc2, nm2);
            if (SWATTN_FA_POLY > 0 && (c / 2) % (SWATTN_FA_POLY > 0 ? SWATTN_FA_POLY : 1) ==
                                          (SWATTN_FA_POLY > 0 ? SWATTN_FA_POLY - 1 : 0)) {
              const float2 e2 = poly_exp2x2(a2);
              x[c] = e2.x;
              x[c + 1] = e2.y;
            } else {
              x[c] = fast_exp2(a2.x);
              x[c + 1] = fast_exp2(a2.y);
            }
            pk[c / 2] = tc::pack_bf16(x[c], x[c + 1]);
          }
        }
        tc::tmem_st32(tmem + lane_off + (gi & 1u) * kBlk, pk);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s.p_full[gi & 1u]);
        {
          float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < kBlk; c += 4) {
            s0 = fadd2(s0, make_float2(x[c], x[c + 1]));
            s1 = fadd2(s1, make_float2(x[c + 2], x[c + 3]));
          }
          l += (s0.x + s0.y) + (s1.x + s1.y);
        }
      }
      // epilogue: PV_{nblk-2} and PV_{nblk-1} may both be in flight here, which a
      // parity wait on one V stage cannot tell apart -> dedicated per-item barrier
      tc::mbar_wait(&s.o_final, (uint32_t)(it & 1));
      tc::tc_fence_after();
      const bool valid = tok < p.n;
      const int hq = g * kG + (r % kG);
      const int64_t idx = tok * p.h_q + hq;
      float inv_l = 1.f / l;
      // mode 3: merge with part A (O_A normalised in O, m_A / l_A in m_out /
      // l_out): O = (O_A l_A 2^(m_A-M) + O_U 2^(m-M)) / (l_A 2^(m_A-M) + l 2^(m-M))
      float ca = 0.f;
      if (kRouted && valid) {
        const float mA = p.m_out[idx], lA = p.l_out[idx];
        const float M = fmaxf(mA, m);
        const float wa = lA * fast_exp2(mA - M);
        const float wu = m == -INFINITY ? 0.f : fast_exp2(m - M);
        const float den = wa + l * wu;
        ca = wa / den;
        inv_l = wu / den;
        m = M;
        l = den;
      }
      __nv_bfloat16 *orow = p.O + idx * kD;
#pragma unroll
      for (int c0 = 0; c0 < kD; c0 += 32) {
        uint32_t o[32];
        tc::tmem_ld32(tmem_o + lane_off + c0, o);
        tc::tmem_ld_wait();
        if (valid) {
          uint4 *dst = reinterpret_cast<uint4 *>(orow + c0);
          if (kRouted) {
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              const uint4 a = dst[e / 8];
              const uint32_t aw[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&aw[q]));
                o[e + 2 * q] = __float_as_uint(fmaf(f.x, ca, __uint_as_float(o[e + 2 * q]) * inv_l));
                o[e + 2 * q + 1] =
                    __float_as_uint(fmaf(f.y, ca, __uint_as_float(o[e + 2 * q + 1]) * inv_l));
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * inv_l);
          }
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 wv;
            wv.x = tc::pack_bf16(__uint_as_float(o[e]), __uint_as_float(o[e + 1]));
            wv.y = tc::pack_bf16(__uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
            wv.z = tc::pack_bf16(__uint_as_float(o[e + 4]), __uint_as_float(o[e + 5]));
            wv.w = tc::pack_bf16(__uint_as_float(o[e + 6]), __uint_as_float(o[e + 7]));
            dst[e / 8] = wv;
          }
        }
      }
      // O is out of TMEM: the next item's first PV may overwrite it
      tc::tc_fence_before();
      tc::mbar_arrive(&s.o_empty);
      if (valid) {
        p.lse[idx] = (m + __log2f(l)) * 0.6931471805599453f;
        if (p.m_out != nullptr && !kRouted) {
          p.m_out[idx] = m;
          p.l_out[idx] = l;
        }
      }
      gi0 += (uint32_t)nblk;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<kTmemCols>(tmem);
  if (kRouted) pdl_wait();
}

}  // namespace

bool attention_tc_available() { return true; }

static int32_t launch_fa(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int64_t r0, int64_t r1, int mode, void *O, float *lse,
                         float *m_out, float *l_out, cudaStream_t stream,
                         const TileRoutes *routes = nullptr) {
  if (r1 <= r0) return SWATTN_OK;
  FaParams p;
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
  const GroupRange gr = group_range(cfg);
  p.g0 = gr.g0;
  p.gc = gr.gc;
  // row ranges are multiples of the 8-token tile (the last one may end at n)
  p.tile_end = (int)cdiv(r1, kTokTile);
  p.n_tiles = p.tile_end - (int)(r0 / kTokTile);
  p.mode = mode;
  p.N_init = cfg->N_init;
  p.N_local = cfg->N_local;
  p.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  p.O = static_cast<__nv_bfloat16 *>(O);
  p.lse = lse;
  p.m_out = m_out;
  p.l_out = l_out;
  if (routes != nullptr) p.routes = *routes;
  const size_t smem = sizeof(FaSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fa_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fa_tile_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fa_tile_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  // persistent: two CTAs per SM walk the (tile, group) items
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // Up to kPersistItems items the CTAs are persistent (two per SM; the
  // per-CTA prologue and the last partial wave dominate short sequences:
  // 4K dense 0.205 -> 0.146 ms, 32K 11.0 -> 8.1 ms); above it one CTA per
  // item lets the block scheduler balance the long causal rows (128K dense:
  // 119 ms one-per-item vs 145 ms persistent).
  const int64_t items = mode == 3 ? 2 * (int64_t)sms : (int64_t)p.n_tiles * gr.gc;
#ifndef SWATTN_FA_PERSIST_ITEMS
#define SWATTN_FA_PERSIST_ITEMS 8192
#endif
  constexpr int64_t kPersistItems = SWATTN_FA_PERSIST_ITEMS;
  if (mode == 3) {
    // programmatic launch behind part B (sparse_warp.cu releases it at once)
    const cudaError_t e =
        launch_pdl(fa_tile_kernel<true, true>, dim3((unsigned)items), dim3(kThreads), smem, stream, p);
    if (e != cudaSuccess) {
      set_error("fa_tile_kernel (routed) launch: %s", cudaGetErrorString(e));
      return SWATTN_ECUDA;
    }
  } else if (items > kPersistItems) {
    fa_tile_kernel<false><<<(unsigned)items, kThreads, smem, stream>>>(p);
  } else {
    const int64_t grid = items < 2 * (int64_t)sms ? items : 2 * (int64_t)sms;
    fa_tile_kernel<true><<<(unsigned)grid, kThreads, smem, stream>>>(p);
  }
  SWATTN_LAUNCH_CHECK("fa_tile_kernel");
  return SWATTN_OK;
}

int32_t launch_dense_tc2(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int causal, void *O, float *lse, cudaStream_t stream, int step);

int32_t launch_dense_tc(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                        int64_t n, int causal, void *O, float *lse, cudaStream_t stream) {
  // Causal: the two-tile kernel (attention_tc2.cu) -- 0.82-0.97x the one-tile
  // time from 2K to 128K (equal at 16K), profiles/r02bn_fa2_ab.txt.
  // SWATTN_FA2 (per call): 0 one-tile, 1 two-tile, 2 two-tile with 128-key
  // steps (measurement; slower: its single S buffer serialises each tile).
  const char *e = getenv("SWATTN_FA2");
  const int v = e ? atoi(e) : (causal ? 1 : 0);
  if (v == 1 || v == 2)
    return launch_dense_tc2(cfg, Q, K, V, n, causal, O, lse, stream, v == 2 ? 128 : 64);
  return launch_fa(cfg, Q, K, V, n, 0, n, causal ? 0 : 1, O, lse, nullptr, nullptr, stream);
}

// Routed tiles (route.cuh): the union of each routed tile's top-k blocks, merged
// with part A's (O_A, m_A, l_A) into the final O / lse.  The routed count is
// read on the device: a persistent grid of two CTAs per SM walks the slots.
int32_t launch_routed_tiles(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                            int64_t n, void *O, float *lse, float *m_a, float *l_a,
                            const TileRoutes &routes, cudaStream_t stream) {
  return launch_fa(cfg, Q, K, V, n, 0, n, 3, O, lse, m_a, l_a, stream, &routes);
}

int32_t launch_part_a_tc2(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, int64_t r0, int64_t r1, void *O, float *lse, float *m_out,
                          float *l_out, cudaStream_t stream);

int32_t launch_sparse_part_a(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                             int64_t n, int64_t r0, int64_t r1, void *O, float *lse, float *m_out,
                             float *l_out, cudaStream_t stream) {
  // SWATTN_FA2_PARTA=1 (measurement): part A on the two-tile kernel
  const char *e = getenv("SWATTN_FA2_PARTA");
  if (e && atoi(e) == 1 && r0 % 16 == 0)
    return launch_part_a_tc2(cfg, Q, K, V, n, r0, r1, O, lse, m_out, l_out, stream);
  return launch_fa(cfg, Q, K, V, n, r0, r1, 2, O, lse, m_out, l_out, stream);
}

}  // namespace swattn
