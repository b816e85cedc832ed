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

// KV-group range of the current C-ABI call (batch x KV-group sharding: a rank
// computes groups [g0, g0 + gc) only -- query heads [G g0, G (g0 + gc)) and
// K/V heads [g0, g0 + gc) -- with no collective, selection.py:111-135 and
// sparse.py:70-91 being independent per group).  {0, h_kv} unless a
// swattn_*_groups entry point narrowed it for the duration of its call
// (thread-local, set and restored by GroupScope).
struct GroupRange {
  int g0, gc;
};
GroupRange group_range(const swattn_config *cfg);
struct GroupScope {
  GroupScope(int g0, int g1);
  ~GroupScope();
  int prev_g0, prev_g1;
};

struct Dims {
  int64_t n;
  int h_q, h_kv, d;
};

// ---------------------------------------------------------------- programmatic dependent launch
// Chains of small dependent kernels (the decode step) launch each kernel
// with cudaLaunchAttributeProgrammaticStreamSerialization: it is scheduled
// while its predecessor drains, runs its prologue (smem / barrier setup,
// loads of step inputs), and blocks in pdl_wait() -- griddepcontrol.wait:
// the predecessor grid has completed and its writes are visible -- before
// it reads the predecessor's outputs.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- small device helpers
__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

// three-input max (one FMNMX3 on sm_100; NaN-ignoring like fmaxf)
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// max of 64 values in 32 FMNMX3 (two independent chains)
__device__ __forceinline__ float max64(const float (&x)[64]) {
  float m0 = x[0], m1 = x[1];
#pragma unroll
  for (int c = 2; c < 62; c += 4) {
    m0 = fmax3f(m0, x[c], x[c + 1]);
    m1 = fmax3f(m1, x[c + 2], x[c + 3]);
  }
  return fmax3f(m0, m1, fmaxf(x[62], x[63]));
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe (offloads the MUFU in exp-bound epilogues): round to
// the nearest integer n with the 1.5*2^23 trick, 2^f on f in [-0.5, 0.5] by a
// degree-6 Taylor polynomial (relative error <= 1.3e-7, the same class as
// ex2.approx's 2 ulp), then add n to the exponent field.  x is clamped to
// [-126, 127]: results below 2^-126 are returned as 2^-126 instead of 0,
// which only matters for sums in which every term is below 1e-38.
// Packed fp32 pairs (sm_100a FFMA2 / FADD2: two IEEE fp32 fma / add in one
// instruction -- bit-identical to two scalar ones, half the issue slots)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

__device__ __forceinline__ float poly_exp2(float x) {
  x = fminf(fmaxf(x, -126.f), 127.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = 1.5403530393381608e-4f;
  p = fmaf(p, f, 1.3333558146428443e-3f);
  p = fmaf(p, f, 9.6181291076284772e-3f);
  p = fmaf(p, f, 5.5504108664821580e-2f);
  p = fmaf(p, f, 2.4022650695910071e-1f);
  p = fmaf(p, f, 6.9314718055994531e-1f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
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
