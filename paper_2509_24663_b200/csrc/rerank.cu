// Float64 boundary re-rank for selection exactness.
//
// K2 produces S^cmp in float32 with a bounded relative error (kScoreRelErr).
// K3 flags rows whose k-th / (k+1)-th boundary lies inside that bound; this
// kernel recomputes, for each flagged row, the pass-1 log-sum-exp of all 16
// heads and the max-pooled scores of the boundary cluster in float64 -- the
// reference's own arithmetic (selection.py:165-222, :336-348,
// compression.py:160-173) -- and settles the cluster with the reference's
// ordering (score desc, index asc; selection.py:125).  Blocks clearly above
// the cluster stay selected, blocks clearly below stay out.
#include <string.h>

#include "common.cuh"
#include "topk_cta.cuh"

namespace swattn {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxCluster = 256;
constexpr int kChunk = 128;  // normaliser columns staged per step

struct RerankArgs {
  const __nv_bfloat16 *Q, *kc1, *kc2;
  const float *s_cmp;
  int64_t ld, n, m1, m2;
  int h_kv, h_q, B, N_init, N_local, k_top, n_cols;
  int l_C1, s_C1, l_C2, s_C2, pl, ps;
  int approx;
  double scale;
  const int32_t *count;
  const int32_t *rows;
  int cap;
  int32_t *topk;
  // decode rows (seq * h_kv + g): per-sequence Q row, key slabs and length
  int decode;
  const int32_t *seq_lens;
  int64_t max_m1, max_m2;
  // pass-1 partials of the row-split path (few flagged rows: decode, small
  // chunks): [kSplitRows][kP1Split][kG] (max, sum), or nullptr
  double2 *partials;
};

// When at most kSplitRows rows are flagged, pass 1 of each row is split over
// kP1Split CTAs (rerank_p1_kernel) so a handful of rows -- the decode case --
// is not serialised on one SM each; larger counts keep one CTA per row.
constexpr int kSplitRows = 256;
constexpr int kP1Split = 64;
constexpr int kNarrow = 32;  // split path: columns per sub-chunk (thread = (head, column pair))

struct RowInfo {
  int g;
  int64_t i, qrow, n_cols, m1;
  const __nv_bfloat16 *kc1, *kc2;
};

__device__ __forceinline__ RowInfo row_info(const RerankArgs &a, int row) {
  RowInfo r;
  r.n_cols = a.n_cols;
  r.m1 = a.m1;
  r.kc1 = a.kc1;
  r.kc2 = a.kc2;
  if (a.decode) {
    const int seq = row / a.h_kv;
    r.g = row % a.h_kv;
    r.i = a.seq_lens[seq] - 1;
    r.qrow = seq;
    r.m1 = num_pooled(r.i + 1, a.l_C1, a.s_C1);
    r.n_cols = r.m1 ? cdiv(r.m1, a.ps) : 0;
    r.kc1 += (int64_t)seq * a.max_m1 * a.h_kv * kD;
    r.kc2 += (int64_t)seq * a.max_m2 * a.h_kv * kD;
  } else {
    r.g = row / (int)a.n;
    r.i = row % a.n;
    r.qrow = r.i;
  }
  return r;
}

// Normaliser keys of pass 1 (selection.py:165-196, :336-348).
__device__ __forceinline__ void pass1_keys(const RerankArgs &a, const RowInfo &r,
                                           const __nv_bfloat16 *&kc, int64_t &vis) {
  const int64_t vis1 = vis_count(r.i, a.l_C1, a.s_C1);
  const int64_t vis2 = a.approx ? vis_count(r.i, a.l_C2, a.s_C2) : 0;
  const bool use_c2 = a.approx && vis2 > 0;
  kc = use_c2 ? r.kc2 : r.kc1;
  vis = use_c2 ? vis2 : vis1;
}

// q_s is [d][head]: the 16 heads of one d are 128 contiguous bytes, so a
// thread's 4-head register tile is two 16-byte broadcasts and the 16 lanes
// of a member-scoring half-warp read 16 different heads conflict-free.
__device__ void load_q(const RerankArgs &a, const RowInfo &r, double (*q_s)[kG]) {
  for (int t = threadIdx.x; t < kG * kD; t += kThreads) {
    const int h = t / kD, d = t % kD;
    q_s[d][h] = (double)bf2f(a.Q[(r.qrow * a.h_q + r.g * kG + h) * kD + d]);
  }
}

// float64 (max, sum) of the 16 heads over normaliser columns [c_lo, c_hi),
// 128-column chunks staged as bf16 [d][c] (32 KB, so two CTAs fit an SM);
// thread = 4 heads x 2 columns register tile (8 DFMA per 3 shared loads).
// Result in mh[h], lh[h].
__device__ void pass1_range(const RerankArgs &a, const __nv_bfloat16 *kc, int g, int64_t c_lo,
                            int64_t c_hi, const double (*q_s)[kG], __nv_bfloat16 *kc_s,
                            double (*wm)[4], double (*wl)[4], double *mh, double *lh) {
  const int hg = threadIdx.x / 64, cg = threadIdx.x % 64;
  double mloc[4], lloc[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) { mloc[e] = -INFINITY; lloc[e] = 0.0; }
  for (int64_t c0 = c_lo; c0 < c_hi; c0 += kChunk) {
    __syncthreads();
    for (int v = threadIdx.x; v < kChunk * (kD / 8); v += kThreads) {
      const int c = v % kChunk, d0 = (v / kChunk) * 8;
      uint4 raw = make_uint4(0, 0, 0, 0);
      if (c0 + c < c_hi) raw = __ldg(reinterpret_cast<const uint4 *>(kc + ((c0 + c) * a.h_kv + g) * kD + d0));
      const __nv_bfloat16 *kv = reinterpret_cast<const __nv_bfloat16 *>(&raw);
#pragma unroll
      for (int e = 0; e < 8; ++e) kc_s[(d0 + e) * kChunk + c] = kv[e];
    }
    __syncthreads();
    double acc[4][2];
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e][0] = acc[e][1] = 0.0;
#pragma unroll 4
    for (int d = 0; d < kD; ++d) {
      const uint32_t kk2 = *reinterpret_cast<const uint32_t *>(&kc_s[d * kChunk + 2 * cg]);
      const double kx = (double)__uint_as_float(kk2 << 16), ky = (double)__uint_as_float(kk2 & 0xffff0000u);
      const double2 q01 = *reinterpret_cast<const double2 *>(&q_s[d][4 * hg]);
      const double2 q23 = *reinterpret_cast<const double2 *>(&q_s[d][4 * hg + 2]);
      const double qv[4] = {q01.x, q01.y, q23.x, q23.y};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[e][0] = fma(qv[e], kx, acc[e][0]);
        acc[e][1] = fma(qv[e], ky, acc[e][1]);
      }
    }
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      if (c0 + 2 * cg + cc >= c_hi) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double sv = acc[e][cc] * a.scale;
        if (sv > mloc[e]) { lloc[e] = lloc[e] * exp(mloc[e] - sv) + 1.0; mloc[e] = sv; }
        else lloc[e] += exp(sv - mloc[e]);
      }
    }
  }
  // reduce (m, l) over the 64 threads (2 warps) sharing a head group
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    double M = mloc[e];
    for (int o = 16; o; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    double part = (mloc[e] == -INFINITY) ? 0.0 : lloc[e] * exp(mloc[e] - M);
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) {
      wm[threadIdx.x >> 5][e] = M;
      wl[threadIdx.x >> 5][e] = part;
    }
  }
  __syncthreads();
  if (threadIdx.x < kG) {
    const int h = threadIdx.x, w0 = (h / 4) * 2, e = h % 4;
    const double M = fmax(wm[w0][e], wm[w0 + 1][e]);
    double L = 0.0;
    for (int w = w0; w < w0 + 2; ++w)
      if (wm[w][e] != -INFINITY) L += wl[w][e] * exp(wm[w][e] - M);
    mh[h] = M;
    lh[h] = L;
  }
  __syncthreads();
}

// float64 (max, sum) of the 16 heads over columns [c_lo, c_hi) for the split
// path: sub-chunks of 32 columns staged row-major [c][d] (8 KB), thread =
// (head t / 16, columns 2 (t % 16), +1), two accumulators per column (even /
// odd d), then a 16-lane shuffle merge per head.  A quarter of pass1_range's
// per-thread DFMA chain per 32 columns, so a flagged decode row's pass 1 is
// spread over 64 short CTAs.  Result in mh[h], lh[h] (log-sum of the slice).
__device__ void pass1_narrow(const RerankArgs &a, const __nv_bfloat16 *kc, int g, int64_t c_lo,
                             int64_t c_hi, const double (*q_s)[kG], __nv_bfloat16 *kn,
                             double *mh, double *lh) {
  const int h = threadIdx.x >> 4, cp = threadIdx.x & 15;
  double M = -INFINITY, S = 0.0;
  for (int64_t c0 = c_lo; c0 < c_hi; c0 += kNarrow) {
    __syncthreads();
    for (int v = threadIdx.x; v < kNarrow * (kD / 8); v += kThreads) {
      const int c = v / (kD / 8), d8 = (v % (kD / 8)) * 8;
      uint4 raw = make_uint4(0, 0, 0, 0);
      if (c0 + c < c_hi) raw = __ldg(reinterpret_cast<const uint4 *>(kc + ((c0 + c) * a.h_kv + g) * kD + d8));
      *reinterpret_cast<uint4 *>(&kn[c * kD + d8]) = raw;
    }
    __syncthreads();
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const uint32_t *k0 = reinterpret_cast<const uint32_t *>(&kn[(2 * cp) * kD]);
    const uint32_t *k1 = reinterpret_cast<const uint32_t *>(&kn[(2 * cp + 1) * kD]);
#pragma unroll 8
    for (int d2 = 0; d2 < kD / 2; ++d2) {
      const double q0 = q_s[2 * d2][h], q1 = q_s[2 * d2 + 1][h];
      const uint32_t x = k0[d2], y = k1[d2];
      a0 = fma(q0, (double)__uint_as_float(x << 16), a0);
      a1 = fma(q1, (double)__uint_as_float(x & 0xffff0000u), a1);
      b0 = fma(q0, (double)__uint_as_float(y << 16), b0);
      b1 = fma(q1, (double)__uint_as_float(y & 0xffff0000u), b1);
    }
    const bool v0 = c0 + 2 * cp < c_hi, v1 = c0 + 2 * cp + 1 < c_hi;
    const double s0 = v0 ? (a0 + a1) * a.scale : -INFINITY, s1 = v1 ? (b0 + b1) * a.scale : -INFINITY;
    const double m = fmax(fmax(s0, s1), M);
    if (m != -INFINITY) {
      S = (M == -INFINITY ? 0.0 : S * exp(M - m)) + (v0 ? exp(s0 - m) : 0.0) + (v1 ? exp(s1 - m) : 0.0);
      M = m;
    }
  }
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const double oM = __shfl_xor_sync(0xffffffffu, M, o), oS = __shfl_xor_sync(0xffffffffu, S, o);
    const double m = fmax(M, oM);
    if (m != -INFINITY) {
      S = (M == -INFINITY ? 0.0 : S * exp(M - m)) + (oM == -INFINITY ? 0.0 : oS * exp(oM - m));
      M = m;
    }
  }
  if (cp == 0) {
    mh[h] = M;
    lh[h] = S;
  }
  __syncthreads();
}

// pass-1 partials for the row-split path: work item = (flagged row, column slice)
__global__ void __launch_bounds__(kThreads, 2) rerank_p1_kernel(RerankArgs a) {
  __shared__ __align__(16) double q_s[kD][kG];
  __shared__ double wm[kThreads / 32][4], wl[kThreads / 32][4];
  __shared__ double mh[kG], lh[kG];
  extern __shared__ __nv_bfloat16 kc_s[];  // [kD][kChunk]
  pdl_wait();  // flagged rows come from the top-k kernel
  // dependents (the re-rank kernel) are released only now, so they may read
  // the top-k outputs before their own wait (which then covers the partials)
  pdl_launch_dependents();
  const int total = min(*a.count, a.cap);
  if (total > kSplitRows || a.partials == nullptr) return;
  for (int w = blockIdx.x; w < total * kP1Split; w += gridDim.x) {
    const int item = w / kP1Split, part = w % kP1Split;
    const RowInfo r = row_info(a, a.rows[item]);
    const __nv_bfloat16 *kc;
    int64_t vis;
    pass1_keys(a, r, kc, vis);
    const int64_t len = cdiv(cdiv(vis, (int64_t)kP1Split), (int64_t)kNarrow) * kNarrow;
    const int64_t lo = min((int64_t)part * len, vis), hi = min(lo + len, vis);
    __syncthreads();
    load_q(a, r, q_s);
    __syncthreads();
    (void)wm;
    (void)wl;
    pass1_narrow(a, kc, r.g, lo, hi, q_s, kc_s, mh, lh);
    if (threadIdx.x < kG)
      a.partials[((int64_t)item * kP1Split + part) * kG + threadIdx.x] =
          make_double2(mh[threadIdx.x], lh[threadIdx.x]);
  }
}

__global__ void __launch_bounds__(kThreads, 2) rerank_kernel(RerankArgs a) {
  __shared__ __align__(16) double q_s[kD][kG];
  __shared__ double lse_s[kG];
  __shared__ double wm[kThreads / 32][4], wl[kThreads / 32][4];
  extern __shared__ __nv_bfloat16 kc_s[];  // [kD][kChunk]
  __shared__ int members[kMaxCluster];
  __shared__ double mscore[kMaxCluster];
  __shared__ int n_members, n_above;
  __shared__ uint32_t abits[kTopkMaxCand / 32];  // candidates above the band

  __shared__ double mh[kG], lh[kG];
  pdl_launch_dependents();
  // The predecessor (rerank_p1_kernel) releases this grid only after its own
  // wait, so the top-k outputs (count, rows, S^cmp) are complete here; only
  // the pass-1 partials need the wait, placed right before they are read --
  // q staging, the cluster scan and the members' dot products overlap pass 1.
  const int total = min(*a.count, a.cap);
  const bool split = total <= kSplitRows && a.partials != nullptr;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int row = a.rows[item];
    const RowInfo ri = row_info(a, row);
    const int g = ri.g;
    const int64_t i = ri.i, n_cols = ri.n_cols, m1 = ri.m1;
    const __nv_bfloat16 *kc1 = ri.kc1;
    const int b = (int)(i / a.B);
    const int hi = cand_hi(b, a.N_local, (int)n_cols);
    const int ncand = hi - a.N_init;
    const int k = min(a.k_top, ncand);
    __syncthreads();
    load_q(a, ri, q_s);
    const int64_t vis1 = vis_count(i, a.l_C1, a.s_C1);

    // ---- the boundary cluster from the float32 scores (complete here, see
    // above); blocks above the band are marked for the settle step
    const float *src = a.s_cmp + (int64_t)row * a.ld;
    // k-th largest float32 score key, recorded by K3 next to the row id
    const uint32_t T = (uint32_t)a.rows[a.cap + item];
    const float vk = key2f(T);
    const float band = 3.0f * kScoreRelErr * fabsf(vk);
    const int nwords = (ncand + 31) >> 5;
    if (threadIdx.x == 0) { n_members = 0; n_above = 0; }
    for (int w = threadIdx.x; w < nwords; w += kThreads) abits[w] = 0u;
    __syncthreads();
    for (int t = threadIdx.x; t < ncand; t += kThreads) {
      const float v = src[a.N_init + t];
      if (v > vk + band) {
        atomicAdd(&n_above, 1);
        atomicOr(&abits[t >> 5], 1u << (t & 31));
      } else if (v >= vk - band) {
        const int slot = atomicAdd(&n_members, 1);
        if (slot < kMaxCluster) members[slot] = a.N_init + t;
      }
    }
    __syncthreads();
    const int nm = min(n_members, kMaxCluster);

    // ---- float64 max-pooled scores of the cluster members: warp = member,
    // lane = (head lane & 15, window columns lane >> 4, +2, +4).  The dot
    // products need no pass-1 statistics, so each warp's first member is
    // scored before the pass-1 wait; its <= 6 window rows are staged in the
    // idle staging buffer (one coalesced 16-byte load per lane and row), then
    // two-accumulator dot products from shared memory
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hh = lane & 15, c_half = lane >> 4;
    __nv_bfloat16 *wrows = kc_s + warp * 6 * kD;
    auto member_dots = [&](int j, double (&dot)[3], bool (&inwin)[3]) {
      for (int v = lane; v < 6 * (kD / 8); v += 32) {
        const int e = v / (kD / 8), d8 = (v % (kD / 8)) * 8;
        const int64_t c = (int64_t)j * a.ps + e;
        uint4 raw = make_uint4(0, 0, 0, 0);
        if (e < a.pl && c < m1 && c < vis1)
          raw = __ldg(reinterpret_cast<const uint4 *>(kc1 + (c * a.h_kv + g) * kD + d8));
        *reinterpret_cast<uint4 *>(&wrows[e * kD + d8]) = raw;
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int e = c_half + 2 * q;
        const int64_t c = (int64_t)j * a.ps + e;
        inwin[q] = e < a.pl && c < m1;   // window columns past m1 do not exist
        dot[q] = -INFINITY;              // not visible: contributes nothing (selection.py:212-222)
        if (inwin[q] && c < vis1) {
          const uint32_t *kr = reinterpret_cast<const uint32_t *>(&wrows[e * kD]);
          double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
          for (int d2 = 0; d2 < kD / 2; ++d2) {
            const uint32_t kk2 = kr[d2];
            d0 = fma(q_s[2 * d2][hh], (double)__uint_as_float(kk2 << 16), d0);
            d1 = fma(q_s[2 * d2 + 1][hh], (double)__uint_as_float(kk2 & 0xffff0000u), d1);
          }
          dot[q] = (d0 + d1) * a.scale;
        }
      }
      __syncwarp();
    };
    double dot0[3];
    bool inw0[3];
    if (warp < nm) member_dots(members[warp], dot0, inw0);

    // ---- pass 1 in float64: lse over the visible normaliser columns
    pdl_wait();  // decode: the pass-1 partials of rerank_p1_kernel
    if (split) {
      // thread = (head t / 16, partials t % 16 + 16 q): four loads each, then
      // a 16-lane max / sum (the 64 partials of a flagged row in parallel)
      {
        const int h = threadIdx.x >> 4, j = threadIdx.x & 15;
        double2 v[kP1Split / 16];
        double M = -INFINITY;
#pragma unroll
        for (int q = 0; q < kP1Split / 16; ++q) {
          v[q] = a.partials[((int64_t)item * kP1Split + j + 16 * q) * kG + h];
          M = fmax(M, v[q].x);
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
        double L = 0.0;
#pragma unroll
        for (int q = 0; q < kP1Split / 16; ++q)
          if (v[q].x != -INFINITY) L += v[q].y * exp(v[q].x - M);
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        if (j == 0) lse_s[h] = (M == -INFINITY) ? 0.0 : M + log(L);  // lse_safe (selection.py:204)
      }
    } else {
      const __nv_bfloat16 *kc;
      int64_t vis;
      pass1_keys(a, ri, kc, vis);
      pass1_range(a, kc, g, 0, vis, q_s, kc_s, wm, wl, mh, lh);
      if (threadIdx.x < kG)
        lse_s[threadIdx.x] = (mh[threadIdx.x] == -INFINITY) ? 0.0 : mh[threadIdx.x] + log(lh[threadIdx.x]);
    }
    __syncthreads();

    for (int mi = warp; mi < nm; mi += kThreads / 32) {
      double dot[3];
      bool inwin[3];
      if (mi == warp) {
#pragma unroll
        for (int q = 0; q < 3; ++q) { dot[q] = dot0[q]; inwin[q] = inw0[q]; }
      } else {
        member_dots(members[mi], dot, inwin);  // clusters wider than the CTA's warps
      }
      double val[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) val[q] = dot[q] == -INFINITY ? 0.0 : exp(dot[q] - lse_s[hh]);
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) val[q] += __shfl_xor_sync(0xffffffffu, val[q], o);
      double best = -INFINITY;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (inwin[q]) best = fmax(best, val[q]);
      best = fmax(best, __shfl_xor_sync(0xffffffffu, best, 16));
      if (lane == 0) mscore[mi] = best;
    }
    __syncthreads();

    // ---- settle: slots = k - above; rank members by (score desc, index asc).
    // The row's selection is then a bitmap over the candidates (above-cluster
    // blocks + chosen members) in the now idle staging buffer, emitted in
    // ascending order by a block-wide scan of per-thread word counts.
    uint32_t *bits = abits;  // above-band blocks from the cluster scan
    int *wsum = reinterpret_cast<int *>(kc_s) + (kChunk * kD / 2 - kThreads);  // tail of kc_s
    if (threadIdx.x == 0) {
      const int slots = k - n_above;
      // selection sort over the (small) cluster
      for (int s = 0; s < slots && s < nm; ++s) {
        int best = -1;
        for (int mi = 0; mi < nm; ++mi) {
          if (members[mi] < 0) continue;
          if (best < 0 || mscore[mi] > mscore[best] ||
              (mscore[mi] == mscore[best] && members[mi] < members[best]))
            best = mi;
        }
        const int t = members[best] - a.N_init;
        atomicOr(&bits[t >> 5], 1u << (t & 31));
        members[best] = -1 - members[best];  // mark taken
      }
    }
    __syncthreads();
    // thread = contiguous run of words; exclusive scan of the run popcounts
    const int per = (nwords + kThreads - 1) / kThreads;
    const int w0 = threadIdx.x * per, w1 = min(w0 + per, nwords);
    int mine = 0;
    for (int w = w0; w < w1; ++w) mine += __popc(bits[w]);
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int base = incl - mine;
    for (int w = 0; w < warp; ++w) base += wsum[w];
    int total_sel = 0;
    for (int w = 0; w < kThreads / 32; ++w) total_sel += wsum[w];
    int32_t *out = a.topk + (int64_t)row * a.k_top;
    for (int w = w0; w < w1; ++w) {
      uint32_t x = bits[w];
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1;
        out[base++] = a.N_init + (w << 5) + bit;
      }
    }
    for (int t = total_sel + threadIdx.x; t < a.k_top; t += kThreads) out[t] = -1;
    __syncthreads();
  }
}

int32_t run_rerank(const RerankArgs &a, int num_sms, cudaStream_t stream) {
  const size_t smem = (size_t)kD * kChunk * sizeof(__nv_bfloat16);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(rerank_p1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // decode: programmatic dependent launches (see launch_pdl, common.cuh)
  if (a.partials != nullptr) {
    // no-op unless at most kSplitRows rows were flagged (decided on the device)
    if (a.decode)
      launch_pdl(rerank_p1_kernel, dim3(num_sms * 2), dim3(kThreads), smem, stream, a);
    else
      rerank_p1_kernel<<<num_sms * 2, kThreads, smem, stream>>>(a);
    SWATTN_LAUNCH_CHECK("rerank_p1_kernel");
  }
  if (a.decode)
    launch_pdl(rerank_kernel, dim3(num_sms * 2), dim3(kThreads), smem, stream, a);
  else
    rerank_kernel<<<num_sms * 2, kThreads, smem, stream>>>(a);  // 2 CTAs per SM (launch bounds)
  SWATTN_LAUNCH_CHECK("rerank_kernel");
  return SWATTN_OK;
}

}  // namespace

size_t rerank_partials_bytes() { return (size_t)kSplitRows * kP1Split * kG * sizeof(double2); }

int32_t launch_rerank(const swattn_config *cfg, const void *Q, const void *kc1, const void *kc2,
                      int64_t n, int32_t mode, const float *s_cmp, int64_t ld,
                      const int32_t *count, const int32_t *rows, int32_t cap, int32_t *topk,
                      void *partials, int num_sms, cudaStream_t stream) {
  if (cfg->k_top > kTopMax) {
    set_error("unsupported: k_top=%d exceeds the compiled bound %d", cfg->k_top, kTopMax);
    return SWATTN_EUNSUPPORTED;
  }
  RerankArgs a;
  a.Q = static_cast<const __nv_bfloat16 *>(Q);
  a.kc1 = static_cast<const __nv_bfloat16 *>(kc1);
  a.kc2 = static_cast<const __nv_bfloat16 *>(kc2);
  a.s_cmp = s_cmp;
  a.ld = ld;
  a.n = n;
  a.m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  a.m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  a.h_kv = cfg->h_kv;
  a.h_q = cfg->h_q;
  a.B = cfg->B;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.k_top = cfg->k_top;
  a.n_cols = (int)(a.m1 ? cdiv(a.m1, cfg->s) : 0);
  a.l_C1 = cfg->l_C1; a.s_C1 = cfg->s_C1; a.l_C2 = cfg->l_C2; a.s_C2 = cfg->s_C2;
  a.pl = cfg->l; a.ps = cfg->s;
  a.approx = mode == SWATTN_SELECT_APPROX;
  a.scale = cfg->scale_compressed_logits ? 1.0 / sqrt((double)cfg->d_h) : 1.0;
  a.count = count;
  a.rows = rows;
  a.cap = cap;
  a.topk = topk;
  a.decode = 0;
  a.seq_lens = nullptr;
  a.max_m1 = a.max_m2 = 0;
  a.partials = static_cast<double2 *>(partials);
  return run_rerank(a, num_sms, stream);
}

int32_t launch_rerank_decode(const swattn_config *cfg, const void *q, const void *kc1,
                             const void *kc2, int max_m1, int max_m2, const int32_t *seq_lens,
                             int batch, const float *s_cmp, int64_t ld, const int32_t *count,
                             const int32_t *rows, int32_t cap, int32_t *topk, void *partials,
                             int num_sms, cudaStream_t stream) {
  RerankArgs a;
  memset(&a, 0, sizeof(a));
  a.Q = static_cast<const __nv_bfloat16 *>(q);
  a.kc1 = static_cast<const __nv_bfloat16 *>(kc1);
  a.kc2 = static_cast<const __nv_bfloat16 *>(kc2);
  a.s_cmp = s_cmp;
  a.ld = ld;
  a.n = 1;
  a.h_kv = cfg->h_kv;
  a.h_q = cfg->h_q;
  a.B = cfg->B;
  a.N_init = cfg->N_init;
  a.N_local = cfg->N_local;
  a.k_top = cfg->k_top;
  a.l_C1 = cfg->l_C1; a.s_C1 = cfg->s_C1; a.l_C2 = cfg->l_C2; a.s_C2 = cfg->s_C2;
  a.pl = cfg->l; a.ps = cfg->s;
  a.approx = 1;
  a.scale = cfg->scale_compressed_logits ? 1.0 / sqrt((double)cfg->d_h) : 1.0;
  a.count = count;
  a.rows = rows;
  a.cap = cap;
  a.topk = topk;
  a.decode = 1;
  a.seq_lens = seq_lens;
  a.max_m1 = max_m1;
  a.max_m2 = max_m2;
  a.partials = static_cast<double2 *>(partials);
  return run_rerank(a, num_sms, stream);
}

}  // namespace swattn
