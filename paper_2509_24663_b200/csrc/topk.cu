// K3 -- per-row top-k block selection (build_block_sets, selection.py:93-136).
//
// One warp per (group, query row).  The candidate pool of row i in query
// block b is [N_init, min(b - N_local + 1, n_cols)); k = min(k_top, #cand)
// (0 for rows with no visible pooled entry, :129).  Ranking is score
// descending with ties to the lower block index -- exactly the stable
// argsort of :125 -- realised as an 8-bit radix select of the k-th largest
// order-preserving uint32 image of the fp32 score, followed by an
// index-ordered compaction (so the output is already ascending, like
// np.unique at :133).
//
// When an ambiguity list is given (select path), rows whose k-th / (k+1)-th
// boundary is within the float32 error bound of S^cmp are appended for the
// float64 re-rank (rerank.cu); exact structural ties (adjacent blocks whose
// max-pool windows share the argmax column, see scores_tc.cu flags) are not
// ambiguous and resolve by index exactly as in float64.
//
// Roofline: HBM-bound; bytes = candidate S^cmp fp32 read + topk int32 write.
#include <algorithm>

#include "common.cuh"
#include "topk_cta.cuh"

namespace swattn {

namespace {

constexpr int kWarps = 8;
constexpr int kMaxCand = kTopkMaxCand;  // per-row candidate bound (8192 blocks: n <= 524K)
constexpr int kStageCap = 4096;         // candidates a warp stages in shared memory

// Select the k best of ncand candidate scores src[0..ncand) (block ids
// N_init + t) into out[0..k_top) ascending (-1 padded).  Warp-cooperative.
// Returns through the ambiguity list when requested.
// Key sources of the generic path: staged in shared memory, or read straight
// from S^cmp (the register path's rare fallback, no staging buffer).
struct SmemKeys {
  const uint32_t *ks;
  __device__ uint32_t operator[](int t) const { return ks[t]; }
};
struct GlobalKeys {
  const float *src;
  __device__ uint32_t operator[](int t) const { return f2key(src[t]); }
};

template <class Keys>
__device__ void warp_topk_generic(const Keys ks, int ncand, int k, int N_init, int k_top,
                                  int32_t *__restrict__ out, int *hist, const AmbList &amb,
                                  int64_t row) {
  const int lane = threadIdx.x & 31;

  // k-th largest key T: rounds of 8-bit radix select (warp-private 256-bin
  // histogram, descending scan across lanes).  The leading bits every key
  // shares (scores live in a narrow positive range) are skipped, so the
  // first histogram already spreads over many bins (low atomic contention).
  uint32_t kmin = 0xffffffffu, kmax = 0;
  for (int t = lane; t < ncand; t += 32) {
    kmin = min(kmin, ks[t]);
    kmax = max(kmax, ks[t]);
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  const int common = (kmin == kmax) ? 32 : __clz(kmin ^ kmax);  // shared leading bits
  uint32_t pmask = common >= 32 ? 0xffffffffu : ~(0xffffffffu >> common);
  uint32_t prefix = kmin & pmask;
  int kk = k;  // rank of T among the keys matching the current prefix
#pragma unroll 1
  for (int shift = 32 - common - 8; shift > -8; shift -= 8) {
    const int sh = shift < 0 ? 0 : shift;  // last round may overlap matched bits
#pragma unroll
    for (int e = 0; e < 8; ++e) hist[lane * 8 + e] = 0;
    __syncwarp();
    for (int t = lane; t < ncand; t += 32) {
      const uint32_t v = ks[t];
      if ((v & pmask) == prefix) atomicAdd(&hist[(v >> sh) & 255u], 1);
    }
    __syncwarp();
    int cnt[8], tot = 0;  // lane owns bins 255-8*lane .. 248-8*lane (descending)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      cnt[e] = hist[255 - 8 * lane - e];
      tot += cnt[e];
    }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - tot;
    const bool mine = excl < kk && kk <= incl;
    const int src_lane = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
    int digit = 0, above = 0;
    if (mine) {
      int acc = excl;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (acc + cnt[e] >= kk) {
          digit = 255 - 8 * lane - e;
          above = acc;
          break;
        }
        acc += cnt[e];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src_lane);
    above = __shfl_sync(0xffffffffu, above, src_lane);
    prefix |= (uint32_t)digit << sh;
    pmask |= 255u << sh;
    kk -= above;
    __syncwarp();
  }
  const uint32_t T = prefix;
  int gt = 0, eq = 0;
  uint32_t below = 0;             // largest key < T
  uint32_t above = 0xffffffffu;   // smallest key > T
  for (int t = lane; t < ncand; t += 32) {
    const uint32_t v = ks[t];
    gt += v > T;
    eq += v == T;
    if (v < T && v > below) below = v;
    if (v > T && v < above) above = v;
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  below = __reduce_max_sync(0xffffffffu, below);
  above = __reduce_min_sync(0xffffffffu, above);
  const int need_eq = k - gt;

  // index-ordered compaction: key > T, or key == T among the first need_eq
  int written = 0, eq_seen = 0;
  for (int base = 0; base < ncand; base += 32) {
    const int t = base + lane;
    const uint32_t v = t < ncand ? ks[t] : 0u;
    const bool is_eq = t < ncand && v == T;
    const unsigned eq_mask = __ballot_sync(0xffffffffu, is_eq);
    const int eq_rank = eq_seen + __popc(eq_mask & ((1u << lane) - 1u));
    const bool take = t < ncand && (v > T || (is_eq && eq_rank < need_eq));
    const unsigned take_mask = __ballot_sync(0xffffffffu, take);
    if (take) out[written + __popc(take_mask & ((1u << lane) - 1u))] = N_init + t;
    written += __popc(take_mask);
    eq_seen += __popc(eq_mask);
  }
  for (int t = written + lane; t < k_top; t += 32) out[t] = -1;

  if (amb.count == nullptr) return;
  // ---- ambiguity of the k / k+1 boundary under the float32 error bound
  const float vk = key2f(T);
  bool ambiguous;
  if (gt + eq > k) {
    // an exact float32 tie straddles the boundary: safe only if it is the
    // structural tie of two adjacent blocks whose max-pool windows both take
    // their maximum from the shared column (flags R_j and L_{j+1}).
    ambiguous = true;
    if (eq == 2 && amb.flags != nullptr) {
      int first = -1, second = -1;
      for (int base = 0; base < ncand; base += 32) {
        const int t = base + lane;
        unsigned mm = __ballot_sync(0xffffffffu, t < ncand && ks[t] == T);
        while (mm) {
          const int pos = base + __ffs(mm) - 1;
          mm &= mm - 1;
          if (first < 0) first = pos; else if (second < 0) second = pos;
        }
      }
      if (second == first + 1) {
        const int j = N_init + first;  // global block index
        const uint64_t *fr = amb.flags + row * amb.ld_f;
        const int tj = j / 31, qj = j % 31, tj1 = (j + 1) / 31, qj1 = (j + 1) % 31;
        const bool R_j = (fr[tj] >> (2 * qj + 1)) & 1ull;
        const bool L_j1 = (fr[tj1] >> (2 * qj1)) & 1ull;
        // the pair's own order is exact (equal float64 scores, lower index
        // first); its order against the nearest other keys is not
        ambiguous = !(R_j && L_j1) || tie_neighbours_close(T, below, above);
      }
    }
  } else {
    const float vb = below ? key2f(below) : -INFINITY;
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

__device__ void warp_topk_row(const float *__restrict__ src, int ncand, int k, int N_init,
                              int k_top, int32_t *__restrict__ out, uint32_t *ks, int *hist,
                              const AmbList &amb, int64_t row) {
  const int lane = threadIdx.x & 31;
  if (k == ncand) {  // every candidate is selected (or none)
    for (int t = lane; t < k_top; t += 32) out[t] = t < k ? N_init + t : -1;
    return;
  }
  if (ncand > kStageCap) {  // long rows (> 256K tokens): radix select straight from S^cmp
    warp_topk_generic(GlobalKeys{src}, ncand, k, N_init, k_top, out, hist, amb, row);
    return;
  }
  for (int t = lane; t < ncand; t += 32) ks[t] = f2key(src[t]);
  __syncwarp();
  warp_topk_generic(SmemKeys{ks}, ncand, k, N_init, k_top, out, hist, amb, row);
}

// ---------------------------------------------------------------------------
// Filtered path (block ids < 2048, i.e. n_cols <= 2048: the paper profile up
// to 128K; k <= 64): no per-row staging of all candidates.
//   1. stream the row (16 float4 loads per lane) keeping the lane's top-2;
//      tau = the smallest lane runner-up: every lane holds 2 keys >= tau, so
//      >= 64 >= k keys survive, and on score data only ~2-4 k do;
//   2. re-read the row (L1-resident) and compact the survivors (key >= tau,
//      with their block ids) into shared memory (<= kSurvCap, else the
//      generic path re-reads the row);
//   3. radix select of the exact k-th key T among the survivors;
//   4. selected = key > T, plus the lowest-index keys == T up to k, emitted
//      ascending from a 2048-bit block bitmap -- the stable argsort of
//      selection.py:125 followed by np.unique (:133).
constexpr int kRegChunks = 16;              // float4 chunks per lane
constexpr int kRegSpan = kRegChunks * 128;  // 2048 block ids
constexpr int kSurvCap = 512;

struct RegScratch {
  uint32_t key[kSurvCap];
  int32_t idx[kSurvCap];
  uint32_t gt_bits[kRegSpan / 32];
  uint32_t eq_bits[kRegSpan / 32];
};

// keys of chunk j of this lane (block ids 128 j + 4 lane + e), 0 outside [lo, hi)
__device__ __forceinline__ void load_chunk(const float *__restrict__ row_src, int ld, int lo, int hi,
                                           int j, int lane, uint32_t (&x)[4]) {
  const int c0 = 128 * j + 4 * lane;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c0 < ld && c0 < hi && c0 + 4 > lo) v = __ldg(reinterpret_cast<const float4 *>(row_src + c0));
  const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = (c0 + e >= lo && c0 + e < hi) ? f2key(f[e]) : 0u;
}

__device__ __forceinline__ void top2_insert(uint32_t &t1, uint32_t &t2, uint32_t x) {
  t2 = max(t2, min(t1, x));
  t1 = max(t1, x);
}

__device__ void warp_topk_row_reg(const float *__restrict__ row_src, int ld, int ncand, int k,
                                  int N_init, int k_top, int32_t *__restrict__ out,
                                  RegScratch &sc, int *hist, const AmbList &amb, int64_t row) {
  const int lane = threadIdx.x & 31;
  if (k == ncand) {
    for (int t = lane; t < k_top; t += 32) out[t] = t < k ? N_init + t : -1;
    return;
  }
  const int lo = N_init, hi = N_init + ncand;  // candidate block ids [lo, hi)
  // chunks of 128 ids that hold candidates (the rest would only load zeros)
  const int nch = min(kRegChunks, (hi + 127) / 128);
  // ---- 1. per-lane top-2 (two independent chains over even / odd chunks)
  uint32_t a1 = 0, a2 = 0, b1 = 0, b2 = 0;
#pragma unroll 2
  for (int j = 0; j < nch; j += 2) {
    uint32_t x[4], y[4];
    load_chunk(row_src, ld, lo, hi, j, lane, x);
    load_chunk(row_src, ld, lo, hi, j + 1, lane, y);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      top2_insert(a1, a2, x[e]);
      top2_insert(b1, b2, y[e]);
    }
  }
  top2_insert(a1, a2, b1);
  top2_insert(a1, a2, b2);
  // >= 1 so unused slots (key 0) never survive (short rows: every valid key does)
  const uint32_t tau = max(__reduce_min_sync(0xffffffffu, a2), 1u);
  // ---- 2. survivors
  int mine = 0;
#pragma unroll 1
  for (int j = 0; j < nch; ++j) {
    uint32_t x[4];
    load_chunk(row_src, ld, lo, hi, j, lane, x);
#pragma unroll
    for (int e = 0; e < 4; ++e) mine += x[e] >= tau;
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total > kSurvCap) {  // massive ties: generic path straight from S^cmp
    warp_topk_generic(GlobalKeys{row_src + N_init}, ncand, k, N_init, k_top, out, hist, amb, row);
    return;
  }
  int pos = incl - mine;
#pragma unroll 1
  for (int j = 0; j < nch; ++j) {
    uint32_t x[4];
    load_chunk(row_src, ld, lo, hi, j, lane, x);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (x[e] >= tau) {
        sc.key[pos] = x[e];
        sc.idx[pos] = 128 * j + 4 * lane + e;
        ++pos;
      }
  }
  for (int w = lane; w < kRegSpan / 32; w += 32) sc.gt_bits[w] = sc.eq_bits[w] = 0u;
  __syncwarp();
  // ---- 3. exact k-th key among the survivors: 8-bit radix select
  uint32_t kmin = 0xffffffffu, kmax = 0;
  for (int t = lane; t < total; t += 32) {
    kmin = min(kmin, sc.key[t]);
    kmax = max(kmax, sc.key[t]);
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  const int common = (kmin == kmax) ? 32 : __clz(kmin ^ kmax);
  uint32_t pmask = common >= 32 ? 0xffffffffu : ~(0xffffffffu >> common);
  uint32_t prefix = kmin & pmask;
  int kk = k;
#pragma unroll 1
  for (int shift = 32 - common - 8; shift > -8; shift -= 8) {
    const int sh = shift < 0 ? 0 : shift;
#pragma unroll
    for (int e = 0; e < 8; ++e) hist[lane * 8 + e] = 0;
    __syncwarp();
    for (int t = lane; t < total; t += 32) {
      const uint32_t v = sc.key[t];
      if ((v & pmask) == prefix) atomicAdd(&hist[(v >> sh) & 255u], 1);
    }
    __syncwarp();
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
    const bool hit = exc < kk && kk <= inc;
    const int src_lane = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
    int digit = 0, above = 0;
    if (hit) {
      int acc = exc;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (acc + cnt[e] >= kk) {
          digit = 255 - 8 * lane - e;
          above = acc;
          break;
        }
        acc += cnt[e];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src_lane);
    above = __shfl_sync(0xffffffffu, above, src_lane);
    prefix |= (uint32_t)digit << sh;
    pmask |= 255u << sh;
    kk -= above;
    __syncwarp();
  }
  const uint32_t T = prefix;
  // ---- 4. selection bitmap, counts, and the next key below T
  int gt = 0, eq = 0;
  for (int t = lane; t < total; t += 32) {
    const uint32_t v = sc.key[t];
    const int c = sc.idx[t];
    if (v > T) {
      ++gt;
      atomicOr(&sc.gt_bits[c >> 5], 1u << (c & 31));
    } else if (v == T) {
      ++eq;
      atomicOr(&sc.eq_bits[c >> 5], 1u << (c & 31));
    }
  }
  uint32_t below = 0;  // largest key < T: a survivor unless T is the smallest one
  uint32_t above = 0xffffffffu;  // smallest key > T (keys > T are all survivors)
  for (int t = lane; t < total; t += 32) {
    const uint32_t v = sc.key[t];
    if (v < T && v > below) below = v;
    if (v > T && v < above) above = v;
  }
  above = __reduce_min_sync(0xffffffffu, above);
  if (__reduce_max_sync(0xffffffffu, below) == 0u) {
#pragma unroll 1
    for (int j = 0; j < nch; ++j) {
      uint32_t x[4];
      load_chunk(row_src, ld, lo, hi, j, lane, x);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (x[e] < T && x[e] > below) below = x[e];
    }
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  below = __reduce_max_sync(0xffffffffu, below);
  __syncwarp();
  const int need_eq = k - gt;
  // lane owns bitmap words 2 lane, 2 lane + 1 (block ids 64 lane .. 64 lane + 63)
  uint32_t g0 = sc.gt_bits[2 * lane], g1 = sc.gt_bits[2 * lane + 1];
  uint32_t e0 = sc.eq_bits[2 * lane], e1 = sc.eq_bits[2 * lane + 1];
  const int ecnt = __popc(e0) + __popc(e1);
  int einc = ecnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, einc, o);
    if (lane >= o) einc += y;
  }
  int erank = einc - ecnt;  // equal keys of lower block ids
  uint32_t s0 = g0, s1 = g1;
  while (e0 && erank < need_eq) {
    const uint32_t b = e0 & (0u - e0);
    s0 |= b;
    e0 ^= b;
    ++erank;
  }
  while (e1 && erank < need_eq) {
    const uint32_t b = e1 & (0u - e1);
    s1 |= b;
    e1 ^= b;
    ++erank;
  }
  const int scnt = __popc(s0) + __popc(s1);
  int sinc = scnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, sinc, o);
    if (lane >= o) sinc += y;
  }
  int w = sinc - scnt;
  while (s0) {
    out[w++] = 64 * lane + __ffs(s0) - 1;
    s0 &= s0 - 1;
  }
  while (s1) {
    out[w++] = 64 * lane + 32 + __ffs(s1) - 1;
    s1 &= s1 - 1;
  }
  const int written = __shfl_sync(0xffffffffu, sinc, 31);
  for (int t = written + lane; t < k_top; t += 32) out[t] = -1;

  if (amb.count == nullptr) return;
  const float vk = key2f(T);
  bool ambiguous;
  if (gt + eq > k) {
    ambiguous = true;
    if (eq == 2 && amb.flags != nullptr) {
      // the two equal keys: lowest set bits of the eq bitmap
      int first = -1, second = -1;
      for (int wd = 0; wd < kRegSpan / 32 && second < 0; ++wd) {
        uint32_t x = sc.eq_bits[wd];
        while (x && second < 0) {
          const int c = 32 * wd + __ffs(x) - 1;
          x &= x - 1;
          if (first < 0) first = c; else second = c;
        }
      }
      if (second == first + 1) {
        const int j = first;  // global block index
        const uint64_t *fr = amb.flags + row * amb.ld_f;
        const int tj = j / 31, qj = j % 31, tj1 = (j + 1) / 31, qj1 = (j + 1) % 31;
        const bool R_j = (fr[tj] >> (2 * qj + 1)) & 1ull;
        const bool L_j1 = (fr[tj1] >> (2 * qj1)) & 1ull;
        // the pair's own order is exact (equal float64 scores, lower index
        // first); its order against the nearest other keys is not
        ambiguous = !(R_j && L_j1) || tie_neighbours_close(T, below, above);
      }
    }
  } else {
    const float vb = below ? key2f(below) : -INFINITY;
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

// kReg: rows go through the register path (launch checked N_init + n_cols
// <= 2048, a 16-byte aligned S^cmp and ld % 4 == 0); otherwise keys are
// staged in dynamic shared memory.
template <bool kReg>
__global__ void __launch_bounds__(kWarps * 32)
topk_kernel(const float *__restrict__ s_cmp, int64_t ld, int64_t n, int64_t r0, int64_t r1, int h_kv,
            int g0, int B, int N_init, int N_local, int k_top, int n_cols, int l_C1, int cand_stride,
            int32_t *__restrict__ topk, int32_t *__restrict__ topk_cnt, AmbList amb) {
  extern __shared__ uint32_t keys_s[];  // [kWarps][cand_stride] (staged path)
  __shared__ int hist_s[kWarps * 256];
  __shared__ RegScratch reg_s[kReg ? kWarps : 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = r1 - r0;
  const int64_t local = (int64_t)blockIdx.x * kWarps + warp;  // g * per + (i - r0)
  if (local >= (int64_t)h_kv * per) return;
  const int64_t i = r0 + local % per;
  const int64_t row = (g0 + local / per) * n + i;  // g * n + i
  const int b = (int)(i / B);
  const int hi = cand_hi(b, N_local, n_cols);
  const int ncand = hi > N_init ? hi - N_init : 0;
  const bool no_visible = (i + 1) < l_C1;
  const int k = no_visible ? 0 : (ncand < k_top ? ncand : k_top);
  if (lane == 0) topk_cnt[row] = k;
  if (kReg)
    warp_topk_row_reg(s_cmp + row * ld, (int)ld, ncand, k, N_init, k_top, topk + row * k_top,
                      reg_s[kReg ? warp : 0], hist_s + warp * 256, amb, row);
  else
    warp_topk_row(s_cmp + row * ld + N_init, ncand, k, N_init, k_top, topk + row * k_top,
                  keys_s + (size_t)warp * cand_stride, hist_s + warp * 256, amb, row);
}

// After the fused K2 (scores_tc.cu selects in its epilogue): rows [r0, t1)
// without candidates get count 0 / ids -1, and the rows whose candidate set
// overflowed (ovf list, usually empty) are selected here from S^cmp by the
// staged generic path, with the same ambiguity recording as topk_kernel.
__global__ void __launch_bounds__(kWarps * 32)
topk_tail_kernel(const float *__restrict__ s_cmp, int64_t ld, int64_t n, int64_t r0, int64_t t1, int gc,
                 int g0, int B, int N_init, int N_local, int k_top, int n_cols, int l_C1, int cand_stride,
                 int32_t *__restrict__ topk, int32_t *__restrict__ topk_cnt, AmbList amb,
                 const int32_t *__restrict__ ovf_count, const int32_t *__restrict__ ovf_rows) {
  extern __shared__ uint32_t keys_s[];  // [kWarps][cand_stride]
  __shared__ int hist_s[kWarps * 256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nfill = (int64_t)gc * (t1 > r0 ? t1 - r0 : 0);
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nfill; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = (g0 + f / (t1 - r0)) * n + r0 + f % (t1 - r0);
    topk_cnt[row] = 0;
    for (int q = 0; q < k_top; ++q) topk[row * k_top + q] = -1;
  }
  const int novf = *ovf_count;
  for (int it = blockIdx.x * kWarps + warp; it < novf; it += gridDim.x * kWarps) {
    const int64_t row = ovf_rows[it];
    const int64_t i = row % n;
    const int hi = cand_hi((int)(i / B), N_local, n_cols);
    const int ncand = hi > N_init ? hi - N_init : 0;
    const int k = (i + 1) < l_C1 ? 0 : (ncand < k_top ? ncand : k_top);
    if (lane == 0) topk_cnt[row] = k;
    warp_topk_row(s_cmp + row * ld + N_init, ncand, k, N_init, k_top, topk + row * k_top,
                  keys_s + (size_t)warp * cand_stride, hist_s + warp * 256, amb, row);
  }
}

// decode: one 512-thread CTA per (sequence, group) row (topk_cta.cuh)
constexpr int kDecThreads = 512;
__global__ void __launch_bounds__(kDecThreads)
decode_topk_cta_kernel(const float *__restrict__ s_cmp, int64_t ld, const int32_t *__restrict__ seq_lens,
                       int h_kv, int B, int N_init, int N_local, int k_top, int l_C1, int s_C1,
                       int pool_s, int32_t *__restrict__ topk, int32_t *__restrict__ topk_cnt,
                       AmbList amb) {
  const int64_t row = blockIdx.x;  // seq * h_kv + g
  pdl_launch_dependents();
  pdl_wait();  // S^cmp and the tie flags from decode pass 2
  topk_row_cta<kDecThreads>(s_cmp, ld, row, seq_lens[row / h_kv], B, N_init, N_local, k_top, l_C1,
                            s_C1, pool_s, topk, topk_cnt, amb);
}

bool reg_path_ok(const float *s_cmp, int64_t ld, int k_top, int n_cols) {
  return n_cols <= kRegSpan && k_top <= 64 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(s_cmp) & 15) == 0;
}

}  // namespace

int32_t launch_topk(const swattn_config *cfg, const float *s_cmp, int64_t ld, int64_t n, int64_t r0,
                    int64_t r1, int32_t *topk, int32_t *topk_cnt, int32_t *amb_count,
                    int32_t *amb_rows, int32_t amb_cap, const uint64_t *flags, int64_t ld_f,
                    cudaStream_t stream) {
  const int64_t m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, cfg->s) : 0);
  if (n_cols - cfg->N_init > kMaxCand) {
    set_error("unsupported: %d top-k candidates exceed the compiled bound %d", n_cols, kMaxCand);
    return SWATTN_EUNSUPPORTED;
  }
  if (cfg->k_top <= 0) return SWATTN_OK;
  if (r1 <= r0) return SWATTN_OK;
  const GroupRange gr = group_range(cfg);
  const int64_t rows = (int64_t)gr.gc * (r1 - r0);
  AmbList amb{amb_count, amb_rows, amb_cap, flags, ld_f};
  const int cand_stride = std::min(n_cols > cfg->N_init ? n_cols - cfg->N_init : 1, kStageCap);
  const unsigned grid = (unsigned)cdiv(rows, kWarps);
  if (reg_path_ok(s_cmp, ld, cfg->k_top, n_cols)) {
    topk_kernel<true><<<grid, kWarps * 32, 0, stream>>>(
        s_cmp, ld, n, r0, r1, gr.gc, gr.g0, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top, n_cols,
        cfg->l_C1, cand_stride, topk, topk_cnt, amb);
  } else {
    const size_t smem = (size_t)kWarps * cand_stride * sizeof(uint32_t);
    if (smem > 40 * 1024)
      cudaFuncSetAttribute(topk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    topk_kernel<false><<<grid, kWarps * 32, smem, stream>>>(
        s_cmp, ld, n, r0, r1, gr.gc, gr.g0, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top, n_cols,
        cfg->l_C1, cand_stride, topk, topk_cnt, amb);
  }
  SWATTN_LAUNCH_CHECK("topk_kernel");
  return SWATTN_OK;
}

int32_t launch_topk_tail(const swattn_config *cfg, const float *s_cmp, int64_t ld, int64_t n, int64_t r0,
                         int64_t r1, int32_t *topk, int32_t *topk_cnt, int32_t *amb_count,
                         int32_t *amb_rows, int32_t amb_cap, const uint64_t *flags, int64_t ld_f,
                         const int32_t *ovf_count, const int32_t *ovf_rows, cudaStream_t stream) {
  const int64_t m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, cfg->s) : 0);
  if (cfg->k_top <= 0 || r1 <= r0) return SWATTN_OK;
  const GroupRange gr = group_range(cfg);
  const int64_t tok0 = (int64_t)(cfg->N_init + cfg->N_local) * cfg->B;
  const int64_t t1 = std::min(r1, std::max(tok0, r0));
  AmbList amb{amb_count, amb_rows, amb_cap, flags, ld_f};
  const int cand_stride = std::min(n_cols > cfg->N_init ? n_cols - cfg->N_init : 1, kStageCap);
  const size_t smem = (size_t)kWarps * cand_stride * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(topk_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kWarps * kStageCap * sizeof(uint32_t)));
    attr = true;
  }
  topk_tail_kernel<<<148, kWarps * 32, smem, stream>>>(
      s_cmp, ld, n, r0, t1, gr.gc, gr.g0, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top, n_cols,
      cfg->l_C1, cand_stride, topk, topk_cnt, amb, ovf_count, ovf_rows);
  SWATTN_LAUNCH_CHECK("topk_tail_kernel");
  return SWATTN_OK;
}

int32_t launch_decode_topk(const swattn_config *cfg, const float *s_cmp, int64_t ld,
                           const int32_t *seq_lens, int batch, int max_ctx, int32_t *topk,
                           int32_t *topk_cnt, int32_t *amb_count, int32_t *amb_rows,
                           int32_t amb_cap, const uint64_t *flags, int64_t ld_f, cudaStream_t stream) {
  const int64_t m1 = num_pooled(max_ctx, cfg->l_C1, cfg->s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, cfg->s) : 0);
  if (n_cols - cfg->N_init > kMaxCand) {
    set_error("unsupported: %d top-k candidates exceed the compiled bound %d", n_cols, kMaxCand);
    return SWATTN_EUNSUPPORTED;
  }
  if (cfg->k_top <= 0) return SWATTN_OK;
  const int64_t rows = (int64_t)cfg->h_kv * batch;
  AmbList amb{amb_count, amb_rows, amb_cap, flags, ld_f};
  launch_pdl(decode_topk_cta_kernel, dim3((unsigned)rows), dim3(kDecThreads), 0, stream, s_cmp, ld,
             seq_lens, cfg->h_kv, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top, cfg->l_C1, cfg->s_C1,
             cfg->s, topk, topk_cnt, amb);
  SWATTN_LAUNCH_CHECK("decode_topk_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
