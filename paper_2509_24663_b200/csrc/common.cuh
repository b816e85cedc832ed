// Shared device/host helpers for the swattn_b200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/swattn_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "swattn_b200 is written for sm_100a only"
#endif

namespace swattn {

// ---------------------------------------------------------------- error state
void set_error(const char *fmt, ...);
int32_t cuda_check(cudaError_t e, const char *what);
#define SWATTN_LAUNCH_CHECK(what)                                            \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) return ::swattn::cuda_check(_e, what);            \
  } while (0)

// ---------------------------------------------------------------- the compiled profile
constexpr int kG = 16;      // query heads per KV group
constexpr int kD = 128;     // head dim
constexpr int kB = 64;      // selection block (tokens)
constexpr int kPoolL = 5;   // max-pool window (C1 columns)
constexpr int kPoolS = 4;   // max-pool stride
constexpr int kTopMax = 128;  // compiled bound on k_top

struct Dims {
  int64_t n;
  int h_q, h_kv, d;
};

// ---------------------------------------------------------------- small device helpers
__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// #pooled entries with span_end <= i (compression.py:89-91)
__host__ __device__ __forceinline__ int64_t vis_count(int64_t i, int length, int stride) {
  return (i + 1 >= length) ? (i + 1 - length) / stride + 1 : 0;
}

__host__ __device__ __forceinline__ int64_t num_pooled(int64_t n, int length, int stride) {
  return n < length ? 0 : (n - length) / stride + 1;
}

__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Candidate block range [N_init, hi) for a row in query block b
// (selection.py:115-120).
__host__ __device__ __forceinline__ int cand_hi(int b, int N_local, int n_cols) {
  int lo = b - N_local + 1;
  if (lo < 0) lo = 0;
  return lo < n_cols ? lo : n_cols;
}

// Order-preserving float -> uint32 key (larger float -> larger key).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// Relative error bound of a float32 S^cmp entry vs the float64 reference.
// Measured max on B200 (tcgen05 K2): 3.1e-7 at 128K (tools/diag_scores.py,
// profiles/r01_gpu_run3.log); the bound keeps a >3x margin.  Boundary gaps
// below 3*kScoreRelErr are resolved in float64 (rerank.cu).
constexpr float kScoreRelErr = 1.0e-6f;

}  // namespace swattn
