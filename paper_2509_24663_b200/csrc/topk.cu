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
#include "common.cuh"

namespace swattn {

namespace {

constexpr int kWarps = 8;
constexpr int kMaxCand = 4096;  // per-row candidate bound held in smem

struct AmbList {
  int32_t *count;         // device counter
  int32_t *rows;          // [cap] row ids
  int32_t cap;
  const uint64_t *flags;  // [rows, ld_f] or null
  int64_t ld_f;
};

// Select the k best of ncand candidate scores src[0..ncand) (block ids
// N_init + t) into out[0..k_top) ascending (-1 padded).  Warp-cooperative.
// Returns through the ambiguity list when requested.
__device__ void warp_topk_row(const float *__restrict__ src, int ncand, int k, int N_init,
                              int k_top, int32_t *__restrict__ out, uint32_t *ks, int *hist,
                              const AmbList &amb, int64_t row) {
  const int lane = threadIdx.x & 31;
  if (k == ncand) {  // every candidate is selected (or none)
    for (int t = lane; t < k_top; t += 32) out[t] = t < k ? N_init + t : -1;
    return;
  }
  for (int t = lane; t < ncand; t += 32) ks[t] = f2key(src[t]);
  __syncwarp();

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
  uint32_t below = 0;  // largest key < T
  for (int t = lane; t < ncand; t += 32) {
    const uint32_t v = ks[t];
    gt += v > T;
    eq += v == T;
    if (v < T && v > below) below = v;
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  below = __reduce_max_sync(0xffffffffu, below);
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
        ambiguous = !(R_j && L_j1);
      }
    }
  } else {
    const float vb = below ? key2f(below) : -INFINITY;
    ambiguous = (vk - vb) <= 3.0f * kScoreRelErr * fabsf(vk);
  }
  if (ambiguous && lane == 0) {
    const int slot = atomicAdd(amb.count, 1);
    if (slot < amb.cap) amb.rows[slot] = (int32_t)row;
  }
}

__global__ void __launch_bounds__(kWarps * 32)
topk_kernel(const float *__restrict__ s_cmp, int64_t ld, int64_t n, int64_t r0, int64_t r1, int h_kv,
            int B, int N_init, int N_local, int k_top, int n_cols, int l_C1, int cand_stride,
            int32_t *__restrict__ topk, int32_t *__restrict__ topk_cnt, AmbList amb) {
  extern __shared__ uint32_t keys_s[];  // [kWarps][cand_stride]
  __shared__ int hist_s[kWarps * 256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = r1 - r0;
  const int64_t local = (int64_t)blockIdx.x * kWarps + warp;  // g * per + (i - r0)
  if (local >= (int64_t)h_kv * per) return;
  const int64_t i = r0 + local % per;
  const int64_t row = (local / per) * n + i;  // g * n + i
  const int b = (int)(i / B);
  const int hi = cand_hi(b, N_local, n_cols);
  const int ncand = hi > N_init ? hi - N_init : 0;
  const bool no_visible = (i + 1) < l_C1;
  const int k = no_visible ? 0 : (ncand < k_top ? ncand : k_top);
  if (lane == 0) topk_cnt[row] = k;
  warp_topk_row(s_cmp + row * ld + N_init, ncand, k, N_init, k_top, topk + row * k_top,
                keys_s + (size_t)warp * cand_stride, hist_s + warp * 256, amb, row);
}

// decode: row = (seq b, group g); the query position is seq_lens[b]-1
__global__ void __launch_bounds__(kWarps * 32)
decode_topk_kernel(const float *__restrict__ s_cmp, int64_t ld, const int32_t *__restrict__ seq_lens,
                   int batch, int h_kv, int B, int N_init, int N_local, int k_top, int l_C1, int s_C1,
                   int pool_s, int cand_stride, int32_t *__restrict__ topk,
                   int32_t *__restrict__ topk_cnt, AmbList amb) {
  extern __shared__ uint32_t keys_s[];
  __shared__ int hist_s[kWarps * 256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + warp;  // seq * h_kv + g
  if (row >= (int64_t)batch * h_kv) return;
  const int L = seq_lens[row / h_kv];
  const int64_t i = L - 1;
  const int64_t m1 = num_pooled(L, l_C1, s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, pool_s) : 0);
  const int hi = cand_hi((int)(i / B), N_local, n_cols);
  const int ncand = hi > N_init ? hi - N_init : 0;
  const int k = (i + 1) < l_C1 ? 0 : min(ncand, k_top);
  if (lane == 0) topk_cnt[row] = k;
  warp_topk_row(s_cmp + row * ld + N_init, ncand, k, N_init, k_top, topk + row * k_top,
                keys_s + (size_t)warp * cand_stride, hist_s + warp * 256, amb, row);
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
  const int64_t rows = (int64_t)cfg->h_kv * (r1 - r0);
  AmbList amb{amb_count, amb_rows, amb_cap, flags, ld_f};
  const int cand_stride = n_cols > cfg->N_init ? n_cols - cfg->N_init : 1;
  const size_t smem = (size_t)kWarps * cand_stride * sizeof(uint32_t);
  if (smem > 40 * 1024)
    cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  topk_kernel<<<(unsigned)cdiv(rows, kWarps), kWarps * 32, smem, stream>>>(
      s_cmp, ld, n, r0, r1, cfg->h_kv, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top, n_cols,
      cfg->l_C1, cand_stride, topk, topk_cnt, amb);
  SWATTN_LAUNCH_CHECK("topk_kernel");
  return SWATTN_OK;
}

int32_t launch_decode_topk(const swattn_config *cfg, const float *s_cmp, int64_t ld,
                           const int32_t *seq_lens, int batch, int max_ctx, int32_t *topk,
                           int32_t *topk_cnt, int32_t *amb_count, int32_t *amb_rows,
                           int32_t amb_cap, cudaStream_t stream) {
  const int64_t m1 = num_pooled(max_ctx, cfg->l_C1, cfg->s_C1);
  const int n_cols = (int)(m1 ? cdiv(m1, cfg->s) : 0);
  if (n_cols - cfg->N_init > kMaxCand) {
    set_error("unsupported: %d top-k candidates exceed the compiled bound %d", n_cols, kMaxCand);
    return SWATTN_EUNSUPPORTED;
  }
  if (cfg->k_top <= 0) return SWATTN_OK;
  const int64_t rows = (int64_t)cfg->h_kv * batch;
  AmbList amb{amb_count, amb_rows, amb_cap, nullptr, 0};
  const int cand_stride = n_cols > cfg->N_init ? n_cols - cfg->N_init : 1;
  const size_t smem = (size_t)kWarps * cand_stride * sizeof(uint32_t);
  if (smem > 40 * 1024)
    cudaFuncSetAttribute(decode_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  decode_topk_kernel<<<(unsigned)cdiv(rows, kWarps), kWarps * 32, smem, stream>>>(
      s_cmp, ld, seq_lens, batch, cfg->h_kv, cfg->B, cfg->N_init, cfg->N_local, cfg->k_top,
      cfg->l_C1, cfg->s_C1, cfg->s, cand_stride, topk, topk_cnt, amb);
  SWATTN_LAUNCH_CHECK("decode_topk_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
