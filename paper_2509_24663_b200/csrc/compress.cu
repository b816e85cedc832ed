// K1 -- key compression (mean_pool_keys, compression.py:64-86).
//
// Paper profile (l_C1 = 2 s_C1, s_C2 = 4 s_C1, l_C2 = 2 s_C2): one coalesced
// HBM pass over K.  A CTA owns 64 chunks of s_C1 tokens of one KV group,
// sums every chunk exactly in float64 (bf16 inputs: <= 30 significant bits,
// so the sum is exact in any order and equals the reference's float64 mean
// numerator), keeps the chunk sums in shared memory and emits
//   C1[j] = (c_j + c_{j+1}) / l_C1,   C2[i] = (c_{4i} + ... + c_{4i+7}) / l_C2
// rounded exactly like the reference's cast back to storage dtype
// (`.astype(K.dtype)`, compression.py:85): float64 -> float32 -> bf16, RNE.
//
// Roofline: HBM-bound; algorithmic bytes = n*h_kv*d*2 (read K once)
// + (m1+m2)*h_kv*d*2 (write pooled keys).
#include "common.cuh"

namespace swattn {

namespace {

constexpr int kChunksPerCta = 32;  // 512 CTAs at 128K (64: 256 CTAs, 35 us = 0.29 of HBM)
constexpr int kHalo = 4;  // C2 windows reach 4 chunks past the tile
constexpr int kThreads = 256;

__device__ __forceinline__ __nv_bfloat16 round_like_numpy(double mean) {
  // ml_dtypes/numpy cast float64 -> bfloat16 goes through float32 (RNE twice)
  return __float2bfloat16_rn(__double2float_rn(mean));
}

__global__ void __launch_bounds__(kThreads)
compress_fused_kernel(const __nv_bfloat16 *__restrict__ K, int64_t n, int h_kv,
                      int chunk, int l1, int l2, __nv_bfloat16 *__restrict__ kc1,
                      int64_t m1, __nv_bfloat16 *__restrict__ kc2, int64_t m2) {
  // chunk sums in float64, [kChunksPerCta + kHalo][128]
  extern __shared__ double csum[];
  const int g = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kChunksPerCta;
  const int64_t full_chunks = n / chunk;
  const int vec = threadIdx.x & 15;   // 8 dims each
  const int lane_c = threadIdx.x >> 4;  // 16 chunk lanes
  const int64_t row_stride = (int64_t)h_kv * kD;

  for (int cc = lane_c; cc < kChunksPerCta + kHalo; cc += 16) {
    const int64_t c = c0 + cc;
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    if (c < full_chunks) {
      const __nv_bfloat16 *src = K + (c * chunk) * row_stride + (int64_t)g * kD + vec * 8;
      // all of a chunk's row loads in flight at once (paper profile: 16 rows)
#pragma unroll 16
      for (int r = 0; r < chunk; ++r) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4 *>(src + r * row_stride));
        const __nv_bfloat16 *v = reinterpret_cast<const __nv_bfloat16 *>(&raw);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += (double)__bfloat162float(v[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) csum[cc * kD + vec * 8 + e] = acc[e];
  }
  __syncthreads();

  const double inv1 = 1.0 / (double)l1;  // power of two in the paper profile
  for (int jj = lane_c; jj < kChunksPerCta; jj += 16) {
    const int64_t j = c0 + jj;
    if (j >= m1) break;
    __align__(16) __nv_bfloat16 out[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int d = vec * 8 + e;
      out[e] = round_like_numpy((csum[jj * kD + d] + csum[(jj + 1) * kD + d]) / (double)l1);
    }
    (void)inv1;
    *reinterpret_cast<uint4 *>(kc1 + (j * h_kv + g) * kD + vec * 8) =
        *reinterpret_cast<const uint4 *>(out);
  }
  if (kc2 != nullptr) {
    const int per = l2 / chunk;           // 8 chunks per C2 window
    const int step = per / 2;             // 4 chunks stride
    const int64_t i0 = c0 / step;
    for (int ii = lane_c; ii < kChunksPerCta / step; ii += 16) {
      const int64_t i = i0 + ii;
      if (i >= m2) break;
      __align__(16) __nv_bfloat16 out[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int d = vec * 8 + e;
        double s = 0.0;
        for (int q = 0; q < per; ++q) s += csum[(ii * step + q) * kD + d];
        out[e] = round_like_numpy(s / (double)l2);
      }
      *reinterpret_cast<uint4 *>(kc2 + (i * h_kv + g) * kD + vec * 8) =
          *reinterpret_cast<const uint4 *>(out);
    }
  }
}

// Any pooling profile / head dim: one thread per (window, group, dim).
__global__ void compress_generic_kernel(const __nv_bfloat16 *__restrict__ K, int64_t n,
                                        int h_kv, int d, int length, int stride,
                                        __nv_bfloat16 *__restrict__ out, int64_t m) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = m * h_kv * d;
  if (t >= total) return;
  const int dd = (int)(t % d);
  const int g = (int)((t / d) % h_kv);
  const int64_t j = t / ((int64_t)d * h_kv);
  double s = 0.0;
  const __nv_bfloat16 *src = K + (j * stride) * (int64_t)h_kv * d + (int64_t)g * d + dd;
  for (int r = 0; r < length; ++r) s += (double)__bfloat162float(src[(int64_t)r * h_kv * d]);
  out[t] = round_like_numpy(s / (double)length);
}

}  // namespace

int32_t launch_compress(const swattn_config *cfg, const void *K, int64_t n, void *kc1,
                        void *kc2, cudaStream_t stream) {
  const int64_t m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  const int64_t m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  const bool fused = cfg->d_h == kD && cfg->l_C1 == 2 * cfg->s_C1 &&
                     cfg->s_C2 == 4 * cfg->s_C1 && cfg->l_C2 == 2 * cfg->s_C2;
  auto Kp = static_cast<const __nv_bfloat16 *>(K);
  if (fused) {
    if (m1 == 0) return SWATTN_OK;
    const int64_t chunks = n / cfg->s_C1;
    dim3 grid((unsigned)cdiv(chunks, kChunksPerCta), (unsigned)cfg->h_kv);
    const size_t smem = (size_t)(kChunksPerCta + kHalo) * kD * sizeof(double);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(compress_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      attr_set = true;
    }
    compress_fused_kernel<<<grid, kThreads, smem, stream>>>(
        Kp, n, cfg->h_kv, cfg->s_C1, cfg->l_C1, cfg->l_C2,
        static_cast<__nv_bfloat16 *>(kc1), m1,
        m2 > 0 ? static_cast<__nv_bfloat16 *>(kc2) : nullptr, m2);
    SWATTN_LAUNCH_CHECK("compress_fused_kernel");
    return SWATTN_OK;
  }
  const int64_t t1 = m1 * cfg->h_kv * cfg->d_h;
  if (t1 > 0) {
    compress_generic_kernel<<<(unsigned)cdiv(t1, 256), 256, 0, stream>>>(
        Kp, n, cfg->h_kv, cfg->d_h, cfg->l_C1, cfg->s_C1, static_cast<__nv_bfloat16 *>(kc1),
        m1);
    SWATTN_LAUNCH_CHECK("compress_generic_kernel(C1)");
  }
  const int64_t t2 = m2 * cfg->h_kv * cfg->d_h;
  if (kc2 != nullptr && t2 > 0) {
    compress_generic_kernel<<<(unsigned)cdiv(t2, 256), 256, 0, stream>>>(
        Kp, n, cfg->h_kv, cfg->d_h, cfg->l_C2, cfg->s_C2, static_cast<__nv_bfloat16 *>(kc2),
        m2);
    SWATTN_LAUNCH_CHECK("compress_generic_kernel(C2)");
  }
  return SWATTN_OK;
}

}  // namespace swattn
