// Exact top-k of one decode row with one CTA (shared by the stand-alone
// decode top-k kernel and the fused decode scoring kernel, csrc/decode.cu).
//
// A decode step has only batch x h_kv rows (32 at batch 16), so a warp per
// row left 4 SMs doing long serial chains (22.8 us, profiles/r02i); here the
// kThr threads of a CTA hold up to kTopkMaxCand / kThr candidates each in
// registers and an MSB-first 8-bit radix select finds the k-th key T in 4
// rounds of shared-memory histograms.  The selection (keys > T, then keys
// == T by ascending block index -- the stable argsort of
// selection.py:123-126) is emitted ascending from a candidate bitmap, and the
// k / k+1 boundary gets the same float32 error-bound test as K3's warp path
// (structural ties via the argmax flags, then the nearest distinct keys).
#pragma once

#include "common.cuh"

namespace swattn {

constexpr int kTopkMaxCand = 8192;  // per-row candidate bound (block ids < 8192 + N_init: n <= 524K)

// Outputs of K2 when it selects the top-k in its pass-2 epilogue (row f1):
// rows whose candidate set overflowed (massive exact ties) are listed for
// launch_topk_tail, which selects them from S^cmp.
struct FusedTopk {
  int32_t *topk, *topk_cnt;
  int32_t *amb_count, *amb_rows;
  int32_t amb_cap;
  int32_t *ovf_count, *ovf_rows;
};

// A proven structural tie straddling the k-th boundary still needs the
// float32 error-bound check against the nearest distinct keys on both sides
// (the pair as a whole may belong above the next key up or below the next
// key down in float64).
__device__ __forceinline__ bool tie_neighbours_close(uint32_t T, uint32_t below, uint32_t above) {
  const float vt = key2f(T);
  const bool lo = below != 0u && (vt - key2f(below)) <= 3.0f * kScoreRelErr * fabsf(vt);
  const bool hi = above != 0xffffffffu && (key2f(above) - vt) <= 3.0f * kScoreRelErr * fabsf(vt);
  return lo || hi;
}

struct AmbList {
  int32_t *count;         // device counter
  int32_t *rows;          // [cap] row ids, then [cap] k-th keys (the re-rank's T)
  int32_t cap;
  const uint64_t *flags;  // [rows, ld_f] or null
  int64_t ld_f;
};


template <int kThr>
__device__ __forceinline__ void topk_row_cta(const float *__restrict__ s_cmp, int64_t ld, int64_t row, int L,
                                             int B, int N_init, int N_local, int k_top, int l_C1,
                                             int s_C1, int pool_s, int32_t *__restrict__ topk,
                                             int32_t *__restrict__ topk_cnt, const AmbList &amb) {
  constexpr int kPer = kTopkMaxCand / kThr;
  __shared__ int hist[256];
  __shared__ uint32_t sel_bits[kTopkMaxCand / 32];
  __shared__ uint32_t eq_bits[kTopkMaxCand / 32];
  __shared__ int s_digit, s_above, s_gt, s_eq, s_first, s_second;
  __shared__ uint32_t s_below, s_abv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i = L - 1;
  const int64_t m1 = num_pooled(L, l_C1, s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, pool_s) : 0);
  const int hi = cand_hi((int)(i / B), N_local, n_cols);
  const int ncand = hi > N_init ? hi - N_init : 0;
  const int k = (L < 1 || (i + 1) < l_C1) ? 0 : min(ncand, k_top);
  int32_t *out = topk + row * k_top;
  if (tid == 0) topk_cnt[row] = k;
  if (k == ncand) {  // every candidate (or none): no ranking
    for (int t = tid; t < k_top; t += kThr) out[t] = t < k ? N_init + t : -1;
    return;
  }
  const float *src = s_cmp + row * ld + N_init;
  uint32_t key[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int t = e * kThr + tid;
    key[e] = t < ncand ? f2key(src[t]) : 0u;  // 0 = below every real key
  }
  for (int w = tid; w < kTopkMaxCand / 32; w += kThr) sel_bits[w] = eq_bits[w] = 0u;
  // ---- radix select of the k-th largest key
  uint32_t prefix = 0, pmask = 0;
  int kk = k;
#pragma unroll 1
  for (int sh = 24; sh >= 0; sh -= 8) {
    for (int t = tid; t < 256; t += kThr) hist[t] = 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int t = e * kThr + tid;
      if (t < ncand && (key[e] & pmask) == prefix) atomicAdd(&hist[(key[e] >> sh) & 255u], 1);
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns digits 255 - 8 l .. 248 - 8 l (descending); suffix counts
      int cnt[8], tot = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cnt[e] = hist[255 - 8 * lane - e];
        tot += cnt[e];
      }
      int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const int exc = inc - tot;
      if (exc < kk && kk <= inc) {
        int acc = exc;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (acc + cnt[e] >= kk) {
            s_digit = 255 - 8 * lane - e;
            s_above = acc;
            break;
          }
          acc += cnt[e];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_digit << sh;
    pmask |= 255u << sh;
    kk -= s_above;
  }
  const uint32_t T = prefix;
  // ---- counts, neighbours of T, selection bitmap (keys > T)
  if (tid == 0) {
    s_gt = 0;
    s_eq = 0;
    s_below = 0u;
    s_abv = 0xffffffffu;
    s_first = 1 << 30;
    s_second = 1 << 30;
  }
  __syncthreads();
  int gt = 0, eq = 0;
  uint32_t below = 0u, abv = 0xffffffffu;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int t = e * kThr + tid;
    if (t >= ncand) continue;
    const uint32_t v = key[e];
    if (v > T) {
      ++gt;
      atomicOr(&sel_bits[t >> 5], 1u << (t & 31));
      abv = min(abv, v);
    } else if (v == T) {
      ++eq;
      atomicOr(&eq_bits[t >> 5], 1u << (t & 31));
    } else {
      below = max(below, v);
    }
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  below = __reduce_max_sync(0xffffffffu, below);
  abv = __reduce_min_sync(0xffffffffu, abv);
  if (lane == 0) {
    atomicAdd(&s_gt, gt);
    atomicAdd(&s_eq, eq);
    atomicMax(&s_below, below);
    atomicMin(&s_abv, abv);
  }
  __syncthreads();
  gt = s_gt;
  eq = s_eq;
  const int need_eq = k - gt;  // keys == T taken, lowest block index first
  // ---- warp 0: add the first need_eq tied candidates, then emit ascending
  if (warp == 0) {
    const int nw = (ncand + 31) >> 5;
    int seen = 0;
    for (int w0 = 0; w0 < nw && seen < need_eq; w0 += 32) {
      const int w = w0 + lane;
      uint32_t e = w < nw ? eq_bits[w] : 0u;
      const int c = __popc(e);
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int r = seen + inc - c;  // tied keys of lower index
      uint32_t take = 0u;
      while (e && r < need_eq) {
        const uint32_t b = e & (0u - e);
        take |= b;
        e ^= b;
        ++r;
      }
      if (w < nw) sel_bits[w] |= take;
      seen += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncwarp();
    int written = 0;
    for (int w0 = 0; w0 < nw; w0 += 32) {
      const int w = w0 + lane;
      uint32_t x = w < nw ? sel_bits[w] : 0u;
      const int c = __popc(x);
      int inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int pos = written + inc - c;
      while (x) {
        out[pos++] = N_init + 32 * w + __ffs(x) - 1;
        x &= x - 1;
      }
      written += __shfl_sync(0xffffffffu, inc, 31);
    }
    for (int t = written + lane; t < k_top; t += 32) out[t] = -1;
    if (amb.count == nullptr) return;
    // ---- ambiguity of the k / k+1 boundary (as warp_topk_row)
    bool ambiguous;
    if (gt + eq > k) {
      ambiguous = true;
      if (eq == 2 && amb.flags != nullptr) {
        int first = -1, second = -1;
        for (int w0 = 0; w0 < nw && second < 0; w0 += 32) {
          const int w = w0 + lane;
          const uint32_t e = w < nw ? eq_bits[w] : 0u;
          unsigned has = __ballot_sync(0xffffffffu, e != 0u);
          while (has && second < 0) {
            const int src_l = __ffs(has) - 1;
            has &= has - 1;
            uint32_t x = __shfl_sync(0xffffffffu, e, src_l);
            while (x && second < 0) {
              const int pos = 32 * (w0 + src_l) + __ffs(x) - 1;
              x &= x - 1;
              if (first < 0) first = pos; else second = pos;
            }
          }
        }
        if (second == first + 1) {
          const int j = N_init + first;
          const uint64_t *fr = amb.flags + row * amb.ld_f;
          const int tj = j / 31, qj = j % 31, tj1 = (j + 1) / 31, qj1 = (j + 1) % 31;
          const bool R_j = (fr[tj] >> (2 * qj + 1)) & 1ull;
          const bool L_j1 = (fr[tj1] >> (2 * qj1)) & 1ull;
          ambiguous = !(R_j && L_j1) || tie_neighbours_close(T, s_below, s_abv);
        }
      }
    } else {
      const float vk = key2f(T);
      const float vb = s_below ? key2f(s_below) : -INFINITY;
      ambiguous = (vk - vb) <= 3.0f * kScoreRelErr * fabsf(vk);
    }
    if (ambiguous && lane == 0) {
      const int slot = atomicAdd(amb.count, 1);
      if (slot < amb.cap) {
        amb.rows[slot] = (int32_t)row;
        amb.rows[amb.cap + slot] = (int32_t)T;
      }
    }
  }
}

}  // namespace swattn
