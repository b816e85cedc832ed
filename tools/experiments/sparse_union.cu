// EXPERIMENT (not built into the library) -- measured and rejected, r02g:
// bit-identical to sparse_warp.cu and the gathered bytes drop as predicted
// (ncu l1tex__m_xbar2l1tex_read_bytes 526 -> 335 GB at 128K), but part B
// slows from 28.7 to 48.3 ms: a stage stays resident until its slowest
// picker consumes it, so most of the 26-slot ring holds data waiting for
// lagging warps and too little is in flight to cover the ~1 us L2 latency
// at the chip-wide gather limit (~130 KB per SM needed).  Kept for the
// record and for correlated (real-model) selections, where the union ratio
// is far lower than on the bench's random inputs.
// K4 part B, union-staged form -- per-token top-k block attention where the
// T = 12 tokens of a CTA share one ring of K/V stages (sm_100a).
//
// Same arithmetic as sparse_warp.cu (one warp owns one (token, group): its 16
// query heads are the M = 16 of mma.sync.m16n8k16, Q_t in registers, P built
// in registers, O accumulated in registers, fixed softmax offset m_A, merge
// with part A at the end -- sparse.py:70-91), but the data movement is
// shared: the tile's 12 consecutive tokens (one KV group) select 12 x <= 63
// blocks, and on the bench's random inputs 20-60 % of those picks are blocks
// another token of the tile also picked.  The CTA builds the sorted union of
// the tile's picks (a 16-bit token mask per block, smem atomics + a block
// scan), streams every union block ONCE through a shared ring of 16-key K/V
// stages, and each warp consumes the stages of the blocks its token selected
// -- in ascending block order, so every token's float32 accumulation order is
// the one sparse_warp.cu uses (bitwise identical outputs).
//
// Why it pays: part B is bound by the L2 -> SMEM gather, which saturates at
// ~19.6 TB/s for the chip with all 148 SMs pulling (tools/mcast_bench.cu:
// 212 GB/s per SM at 37-74 SMs, 133 GB/s per SM at 148), i.e. by the TOTAL
// bytes gathered; sharing the tile's picks cuts them by the union ratio.
//
// No producer thread: a stage is released by an acq_rel counter; the last of
// its consumers (the popcount of the block's token mask) re-arms the slot with
// the sub-stage kSlots ahead (fence.proxy.async, then TMA) and tags the slot
// with that sub-stage's index, which a consumer checks before its parity wait.
// Warps that did not pick a block never touch its stages, so a warp runs
// ahead to its next picked block; the ring depth (26 x 8 KB) absorbs the per-warp imbalance
// (event simulation: 12 tokens, 26 slots -> ~0.8 of the gather time per
// (token, block) of the per-warp-ring design at 128K).
#include <string.h>

#include "common.cuh"
#include "tc.cuh"
#include "tma_host.cuh"

namespace swattn {

namespace {

#ifndef SWATTN_PU_SLOTS
#define SWATTN_PU_SLOTS 26
#endif
constexpr int kWarps = 12;  // tokens per tile
constexpr int kThreads = kWarps * 32;
constexpr int kSlots = SWATTN_PU_SLOTS;
constexpr int kStageKeys = 16;
constexpr int kBlk = 64;
constexpr int kSubs = kBlk / kStageKeys;  // 4 sub-stages per block
constexpr uint32_t kTileBytes = kStageKeys * kD * 2;  // 4 KB (K or V of one sub-stage)
constexpr int kMaxBlocks = 4096;                       // n <= 262144 tokens
constexpr int kMaxEntries = kWarps * 64;               // union of <= 12 x k_top (<= 64) picks
constexpr float kOverflowSum = 1.8446744073709552e19f;  // 2^64

struct PuParams {
  CUtensorMap k_map;  // K as (d lo/hi 64, token, half, group): box {64, 16, 2, 1}
  CUtensorMap v_map;
  int64_t n;
  int h_q, h_kv, k_top, g0;
  int64_t tok0, tok1;  // tokens [tok0, tok1) of this launch
  int64_t tiles_per_group, n_tiles;
  const int32_t *topk, *topk_cnt;
  const float *m_a, *l_a;
  const __nv_bfloat16 *Q;
  __nv_bfloat16 *O;  // in: O_A (normalised), out: final
  float *lse;
  float scale_log2;
  int32_t *slow_count, *slow_list;
};

struct __align__(1024) PuSmem {
  uint8_t k[kSlots][kTileBytes];
  uint8_t v[kSlots][kTileBytes];
  uint16_t mask[kMaxBlocks];     // token mask per block id (zero between tiles)
  uint32_t list[kMaxEntries];    // union entries: block << 16 | token mask, ascending
  uint64_t full[kSlots];
  uint32_t done[kSlots];         // consumers finished with the slot's current sub-stage
  uint32_t tag[kSlots];          // global sub-stage index the slot was last armed with
  int warp_tot[kWarps];
  int n_entries, nb_tile;
};

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
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(tc::smem_u32(p)), "r"(v)
               : "memory");
  return old;
}

// issue sub-stage E (global counter) of the tile whose first sub-stage is e_base
__device__ __forceinline__ void issue_stage(const PuParams &p, PuSmem &sm, uint32_t E, uint32_t e_base,
                                            int g) {
  const uint32_t rel = E - e_base;
  const int blk = (int)(sm.list[rel / kSubs] >> 16);
  const int slot = (int)(E % kSlots);
  const int row0 = blk * kBlk + (int)(rel % kSubs) * kStageKeys;
  tc::mbar_arrive_expect_tx(&sm.full[slot], 2 * kTileBytes);
  tc::tma_load_4d(&p.k_map, &sm.full[slot], sm.k[slot], 0, row0, 0, g);
  tc::tma_load_4d(&p.v_map, &sm.full[slot], sm.v[slot], 0, row0, 0, g);
  // publish which sub-stage the slot now holds (see the consumer's wait)
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(tc::smem_u32(&sm.tag[slot])), "r"(E) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(tc::smem_u32(p)) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads, 1) sparse_union_kernel(const __grid_constant__ PuParams p) {
  extern __shared__ uint8_t smem_raw[];
  PuSmem &sm = *reinterpret_cast<PuSmem *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kMaxBlocks / 2; i += kThreads) reinterpret_cast<uint32_t *>(sm.mask)[i] = 0u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      tc::mbar_init(&sm.full[i], 1);
      sm.done[i] = 0u;
      sm.tag[i] = 0xffffffffu;
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&p.k_map);
    tc::tma_prefetch(&p.v_map);
  }
  __syncthreads();

  const uint32_t kbase = tc::smem_u32(sm.k[0]), vbase = tc::smem_u32(sm.v[0]);
  const int h0 = lane >> 2;
  const int lm = lane >> 3, lr = lane & 7;
  uint32_t e_base = 0;  // global sub-stage counter at the tile's start

  for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int g = p.g0 + (int)(tile / p.tiles_per_group);
    const int64_t t = p.tok0 + (tile % p.tiles_per_group) * kWarps + warp;
    const int64_t row = (int64_t)g * p.n + t;
    const int cnt = t < p.tok1 ? p.topk_cnt[row] : 0;
    // ---- 1. token masks of the tile's picks
    if (threadIdx.x == 0) sm.nb_tile = 0;
    __syncthreads();
    int id0 = -1, id1 = -1;
    if (cnt > 0) {
      const int32_t *b = p.topk + row * p.k_top;
      if (lane < cnt) id0 = b[lane];
      if (lane + 32 < cnt) id1 = b[lane + 32];
      uint32_t *m32 = reinterpret_cast<uint32_t *>(sm.mask);
      const uint32_t bit = 1u << warp;
      if (id0 >= 0) atomicOr(&m32[id0 >> 1], bit << ((id0 & 1) * 16));
      if (id1 >= 0) atomicOr(&m32[id1 >> 1], bit << ((id1 & 1) * 16));
      const int mx = __reduce_max_sync(0xffffffffu, max(id0, id1));  // ids ascending: last pick
      if (lane == 0) atomicMax(&sm.nb_tile, mx + 1);
    }
    __syncthreads();
    // ---- 2. ascending compaction of the union: thread i scans blocks [i c, i c + c)
    {
      const int nb = sm.nb_tile;
      const int c = (nb + kThreads - 1) / kThreads;
      const int lo = threadIdx.x * c, hi = min(nb, lo + c);
      int mine = 0;
      for (int j = lo; j < hi; ++j) mine += sm.mask[j] != 0;
      int inc = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) sm.warp_tot[warp] = inc;
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const int x = sm.warp_tot[w];
        before += w < warp ? x : 0;
        total += x;
      }
      int pos = before + inc - mine;
      for (int j = lo; j < hi; ++j) {
        const uint32_t m = sm.mask[j];
        if (m) {
          sm.list[pos++] = ((uint32_t)j << 16) | m;
          sm.mask[j] = 0;
        }
      }
      if (threadIdx.x == 0) sm.n_entries = total;
    }
    __syncthreads();
    const int U = sm.n_entries;
    const uint32_t n_sub = (uint32_t)U * kSubs;
    // ---- 3. prime the ring (every slot's previous occupant was consumed before the barrier)
    if (threadIdx.x == 0) {
      const uint32_t np = n_sub < (uint32_t)kSlots ? n_sub : (uint32_t)kSlots;
      if (np) tc::fence_proxy_async();
      for (uint32_t i = 0; i < np; ++i) issue_stage(p, sm, e_base + i, e_base, g);
    }
    // ---- 4. each warp: its token's picked blocks, in union (= ascending) order
    if (cnt > 0) {
      const int64_t ridx = t * p.h_q + g * kG;
      uint32_t qa[8][4];
      {
        const uint32_t *qg = reinterpret_cast<const uint32_t *>(p.Q + ridx * kD);
        const int dw = lane & 3;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          qa[ks][0] = __ldg(qg + h0 * (kD / 2) + ks * 8 + dw);
          qa[ks][1] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + dw);
          qa[ks][2] = __ldg(qg + h0 * (kD / 2) + ks * 8 + 4 + dw);
          qa[ks][3] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + 4 + dw);
        }
      }
      const float mA0 = p.m_a[ridx + h0], mA1 = p.m_a[ridx + h0 + 8];
      float lp0 = 0.f, lp1 = 0.f;
      float o[16][4];
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

      for (int e0 = 0; e0 < U; e0 += 32) {
        const uint32_t ent = e0 + lane < U ? sm.list[e0 + lane] : 0u;
        uint32_t picked = __ballot_sync(0xffffffffu, (ent >> warp) & 1u);
        while (picked) {
          const int src = __ffs(picked) - 1;
          picked &= picked - 1;
          const uint32_t ment = __shfl_sync(0xffffffffu, ent, src);
          const uint32_t users = (uint32_t)__popc(ment & 0xffffu);
          const int e = e0 + src;
#pragma unroll 1
          for (int sub = 0; sub < kSubs; ++sub) {
            const uint32_t E = e_base + (uint32_t)(e * kSubs + sub);
            const int st = (int)(E % kSlots);
            // A warp skips the stages of blocks it did not pick, so the slot
            // may still hold (or await) an older sub-stage E - j kSlots; a
            // parity wait alone cannot tell phase j from j - 2, so first wait
            // until the slot is armed with E, then for its data.
            while (ld_acquire(&sm.tag[st]) != E) __nanosleep(32);
            tc::mbar_wait(&sm.full[st], (E / kSlots) & 1u);
            const uint32_t kst = kbase + st * kTileBytes, vst = vbase + st * kTileBytes;
            float sc[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              uint32_t b00, b01, b10, b11;
              ldsm_x4(kst + swz<kStageKeys>((lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), b00, b01, b10, b11);
              mma16816(sc[0], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b00, b01);
              mma16816(sc[1], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b10, b11);
            }
            float x[2][4];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              x[j][0] = fmaf(sc[j][0], p.scale_log2, -mA0);
              x[j][1] = fmaf(sc[j][1], p.scale_log2, -mA0);
              x[j][2] = fmaf(sc[j][2], p.scale_log2, -mA1);
              x[j][3] = fmaf(sc[j][3], p.scale_log2, -mA1);
#pragma unroll
              for (int q = 0; q < 4; ++q) x[j][q] = fast_exp2(x[j][q]);
              lp0 += x[j][0] + x[j][1];
              lp1 += x[j][2] + x[j][3];
            }
            const uint32_t pa0 = tc::pack_bf16(x[0][0], x[0][1]), pa1 = tc::pack_bf16(x[0][2], x[0][3]);
            const uint32_t pa2 = tc::pack_bf16(x[1][0], x[1][1]), pa3 = tc::pack_bf16(x[1][2], x[1][3]);
#pragma unroll
            for (int dp = 0; dp < 8; ++dp) {
              uint32_t v00, v01, v10, v11;
              ldsm_x4_t(vst + swz<kStageKeys>((lm & 1) * 8 + lr, dp * 2 + (lm >> 1)), v00, v01, v10, v11);
              mma16816(o[2 * dp], pa0, pa1, pa2, pa3, v00, v01);
              mma16816(o[2 * dp + 1], pa0, pa1, pa2, pa3, v10, v11);
            }
            // ---- release the stage; its last consumer re-arms the slot kSlots ahead
            __syncwarp();
            if (lane == 0) {
              const uint32_t old = atom_add_acq_rel(&sm.done[st], 1u);
              if (old + 1u == users) {
                sm.done[st] = 0u;
                const uint32_t En = E + kSlots;
                if (En - e_base < n_sub) {
                  tc::fence_proxy_async();
                  issue_stage(p, sm, En, e_base, g);
                }
              }
            }
          }
        }
      }

      // ---- per-token epilogue: merge with part A (as sparse_warp.cu)
      lp0 += __shfl_xor_sync(0xffffffffu, lp0, 1);
      lp0 += __shfl_xor_sync(0xffffffffu, lp0, 2);
      lp1 += __shfl_xor_sync(0xffffffffu, lp1, 1);
      lp1 += __shfl_xor_sync(0xffffffffu, lp1, 2);
      const bool big = !(lp0 <= kOverflowSum) || !(lp1 <= kOverflowSum);
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
    }
    e_base += n_sub;
    __syncthreads();  // the tile's list and every slot are free again
  }
}

}  // namespace

bool sparse_union_supported(const swattn_config *cfg, int64_t n) {
  return cfg->k_top <= 64 && cdiv(n, kBlk) <= kMaxBlocks && cfg->B == kBlk;
}

int32_t launch_sparse_part_b_union(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                                   int64_t n, int64_t r0, int64_t r1, const int32_t *topk,
                                   const int32_t *topk_cnt, const float *m_a, const float *l_a, void *O,
                                   float *lse, int32_t *slow_count, int32_t *slow_list, int num_sms,
                                   cudaStream_t stream) {
  PuParams p;
  memset(&p, 0, sizeof(p));
  {
    const uint64_t dims[4] = {64, (uint64_t)n, 2, (uint64_t)cfg->h_kv};
    const uint64_t str[3] = {(uint64_t)cfg->h_kv * kD * 2, 128, (uint64_t)kD * 2};
    const uint32_t box[4] = {64, (uint32_t)kStageKeys, 2, 1};
    if (!make_tmap_bf16(&p.k_map, K, 4, dims, str, box) || !make_tmap_bf16(&p.v_map, V, 4, dims, str, box)) {
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
  p.tiles_per_group = cdiv(r1 - p.tok0, kWarps);
  p.n_tiles = (int64_t)gr.gc * p.tiles_per_group;
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
  const size_t smem = sizeof(PuSmem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sparse_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int64_t grid = p.n_tiles < num_sms ? p.n_tiles : num_sms;
  sparse_union_kernel<<<(unsigned)grid, kThreads, smem, stream>>>(p);
  SWATTN_LAUNCH_CHECK("sparse_union_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
