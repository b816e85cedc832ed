// Tile routing for K4 (see route.cuh): one warp per (group, 8-token tile)
// builds the union of the tile's top-k lists in a shared-memory bitmap,
// ranks it (popcount prefix over the bitmap words), and routes the tile to
// the tensor-core FA tile when
//     |union| * 100 < (sum of the 8 list lengths) * ratio_pct
// i.e. when streaming the union once through the 128-row tile (cost ~ one FA
// block step per union block) beats 8 per-token gathers (cost ~ one part-B
// block gather per pick); part A + part B cost constants measured at 128K:
// 3.6 ns per FA block step, 1.75 ns per part-B pick (profiles/r02ah_bench.json
// stages) -> break-even near 45 %.  Routed tiles get a slot with the
// ascending union list and, per token, a bit mask over the union positions.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "route.cuh"

namespace swattn {

namespace {

constexpr int kRW = 4;  // warps (tiles) per CTA

struct RouteSmem {
  uint32_t bm[256];   // union bitmap over block ids (ids < 8192)
  uint32_t pre[256];  // exclusive popcount prefix of bm
  uint32_t tb[kRouteTok][kUWords];
};

__global__ void __launch_bounds__(kRW * 32) route_tiles_kernel(const int32_t *topk,
                                                               const int32_t *topk_cnt, int64_t n,
                                                               int k_top, int g0, int gc,
                                                               int64_t tile0, int64_t ntr,
                                                               TileRoutes R, int ratio_pct) {
  __shared__ RouteSmem sm_all[kRW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kRW + warp;
  if (item >= (int64_t)gc * ntr) return;
  RouteSmem &sm = sm_all[warp];
  const int g = g0 + (int)(item / ntr);
  const int64_t tile = tile0 + item % ntr;
  const int64_t t0 = tile * kRouteTok;
  uint8_t *flag = R.routed + (int64_t)g * R.ntiles + tile;
  int cnt_l = 0;
  if (lane < kRouteTok && t0 + lane < n) cnt_l = topk_cnt[(int64_t)g * n + t0 + lane];
  int sum = cnt_l;
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (sum == 0) {
    if (lane == 0) *flag = 0;
    return;
  }
  const int b = (int)(t0 / kB);
  const int W = b / 32 + 1;  // top-k ids are < b
  for (int w = lane; w < W; w += 32) sm.bm[w] = 0;
  __syncwarp();
  for (int k = 0; k < kRouteTok; ++k) {
    const int ck = __shfl_sync(0xffffffffu, cnt_l, k);
    const int32_t *lst = topk + ((int64_t)g * n + t0 + k) * k_top;
    for (int j = lane; j < ck; j += 32) {
      const int id = lst[j];
      atomicOr(&sm.bm[id >> 5], 1u << (id & 31));
    }
  }
  __syncwarp();
  int run = 0;
  for (int w0 = 0; w0 < W; w0 += 32) {
    const int w = w0 + lane;
    const int c = w < W ? __popc(sm.bm[w]) : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (w < W) sm.pre[w] = (uint32_t)(run + inc - c);
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  const int U = run;
  const bool route = U <= kUCap && (int64_t)U * 100 < (int64_t)sum * ratio_pct;
  if (!route) {
    if (lane == 0) {
      *flag = 0;
      atomicAdd(&R.sums[1], (unsigned long long)sum);
    }
    return;
  }
  int slot = 0;
  if (lane == 0) {
    slot = atomicAdd(R.count, 1);
    *flag = 1;
    R.items[slot] = (int32_t)(g * R.ntiles + tile);
    R.ucount[slot] = U;
    atomicAdd(&R.sums[0], (unsigned long long)U);
  }
  slot = __shfl_sync(0xffffffffu, slot, 0);
  int16_t *ul = R.ulist + (int64_t)slot * kUCap;
  for (int w = lane; w < W; w += 32) {
    uint32_t m = sm.bm[w];
    int pos = (int)sm.pre[w];
    while (m) {
      ul[pos++] = (int16_t)(w * 32 + __ffs(m) - 1);
      m &= m - 1;
    }
  }
  uint32_t *tbs = &sm.tb[0][0];
  for (int i = lane; i < kRouteTok * kUWords; i += 32) tbs[i] = 0;
  __syncwarp();
  for (int k = 0; k < kRouteTok; ++k) {
    const int ck = __shfl_sync(0xffffffffu, cnt_l, k);
    const int32_t *lst = topk + ((int64_t)g * n + t0 + k) * k_top;
    for (int j = lane; j < ck; j += 32) {
      const int id = lst[j];
      const int pos = (int)sm.pre[id >> 5] + __popc(sm.bm[id >> 5] & ((1u << (id & 31)) - 1u));
      atomicOr(&sm.tb[k][pos >> 5], 1u << (pos & 31));
    }
  }
  __syncwarp();
  uint32_t *tb = R.tbits + (int64_t)slot * kRouteTok * kUWords;
  for (int i = lane; i < kRouteTok * kUWords; i += 32) tb[i] = tbs[i];
}

// Split of the SMs between the routed FA tiles and part B, which run side by
// side (part B on P = num_sms - S CTAs, the FA tile on 2 CTAs on each of the
// other S SMs): S minimises max(T_fa(S), T_pb(P)) with the costs fitted to
// tools/route_ab.py decompositions (profiles/r02av_route_split.txt):
//   T_fa(S) = 0.39 ms + union blocks x 0.385 us.SM / S   (16.2 ms on 12 SMs,
//             3.45 ms on 62, 1.83 ms on 148 for ~492K union blocks)
//   T_pb(P) = max(picks x c_g(n), picks x 1.73 ns x 148 / P)
// Part B scales with its SMs while its gathers hit L2 (32K: 3.17 ms on 148,
// 5.3 ms on 86 CTAs, 1.73 ns per pick) and flattens where HBM misses set the
// pace (128K: 1.93 ns per pick on 148 or 136 CTAs, c_g growing with n).
__global__ void route_plan_kernel(TileRoutes R, int64_t n, int num_sms, int pb_max, int fa_sms,
                                  int pb_force, int debug) {
  // thread s - 1 evaluates S = s FA SMs; one block-wide argmin
  __shared__ float best_t[256];
  __shared__ int best_s[256];
  const int s = threadIdx.x + 1;
  const float U = (float)R.sums[0], picks = (float)R.sums[1];
  const float lg = log2f(fmaxf((float)n, 1.f) / 32768.f) * 0.5f;
  const float c_g = 1.73e-9f + 0.20e-9f * fminf(1.f, fmaxf(0.f, lg));
  // per-pick costs were measured chip-wide on 148 SMs: scale to this GPU's count
  const float chip = 148.f / (float)num_sms;
  const float tb_act = picks * c_g * chip, tb_sm = picks * 1.73e-9f * 148.f;
  float t = 1e30f;
  if (s <= num_sms) {
    const int pb = min(num_sms - s, pb_max);
    const float t_fa = 0.39e-3f + U * 0.385e-6f / (float)s;
    const float t_pb = picks == 0.f ? 0.f : (pb <= 0 ? 1e30f : fmaxf(tb_act, tb_sm / (float)pb));
    t = fmaxf(t_fa, t_pb);
  }
  best_t[threadIdx.x] = t;
  best_s[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      const float o = best_t[threadIdx.x + w];
      const int os = best_s[threadIdx.x + w];
      if (o < best_t[threadIdx.x] || (o == best_t[threadIdx.x] && os < best_s[threadIdx.x])) {
        best_t[threadIdx.x] = o;
        best_s[threadIdx.x] = os;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  int S = U > 0.f ? best_s[0] : 0;
  if (fa_sms >= 0 && U > 0.f) S = min(fa_sms, num_sms);
  R.plan[0] = 2 * S;
  R.plan[1] = min(num_sms - S, pb_max);
  if (pb_force >= 0) R.plan[1] = min(pb_force, pb_max);
  if (debug)
    printf("route plan: %d tiles, union blocks %llu, part-B picks %llu -> FA SMs %d, part-B CTAs %d\n",
           *R.count, R.sums[0], R.sums[1], S, R.plan[1]);
}

}  // namespace

int32_t launch_route_plan(const TileRoutes &R, int64_t n, int num_sms, int pb_max,
                          cudaStream_t stream) {
  // measurement knobs: SWATTN_ROUTE_FA_SMS forces the FA share, SWATTN_ROUTE_DEBUG prints the plan
  const char *f = getenv("SWATTN_ROUTE_FA_SMS");
  const char *d = getenv("SWATTN_ROUTE_DEBUG");
  const char *pf = getenv("SWATTN_ROUTE_PB_FORCE");
  route_plan_kernel<<<1, 256, 0, stream>>>(R, n, num_sms < 256 ? num_sms : 256, pb_max, f ? atoi(f) : -1,
                                          pf ? atoi(pf) : -1, d ? atoi(d) : 0);
  SWATTN_LAUNCH_CHECK("route_plan_kernel");
  return SWATTN_OK;
}

// Routes the tiles of rows [r0, r1) that have top-k blocks; resets the
// routed-slot count first (stream-ordered).  ratio_pct <= 0: nothing routed.
int32_t launch_route_tiles(const swattn_config *cfg, int64_t n, int64_t r0, int64_t r1,
                           const int32_t *topk, const int32_t *topk_cnt, const TileRoutes &R,
                           int ratio_pct, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(R.count, 0, 64, stream);  // count, plan, sums
  if (e != cudaSuccess) {
    set_error("memset(route count): %s", cudaGetErrorString(e));
    return SWATTN_ECUDA;
  }
  int64_t tok0 = (int64_t)(cfg->N_init + cfg->N_local) * cfg->B;
  if (tok0 < r0) tok0 = r0;
  if (ratio_pct <= 0 || tok0 >= r1 || cfg->k_top == 0) return SWATTN_OK;
  const int64_t tile0 = tok0 / kRouteTok, ntr = cdiv(r1, kRouteTok) - tile0;
  const GroupRange gr = group_range(cfg);
  const int64_t items = (int64_t)gr.gc * ntr;
  route_tiles_kernel<<<(unsigned)cdiv(items, kRW), kRW * 32, 0, stream>>>(
      topk, topk_cnt, n, cfg->k_top, gr.g0, gr.gc, tile0, ntr, R, ratio_pct);
  SWATTN_LAUNCH_CHECK("route_tiles_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
