// Throughput of ex2.approx.f32 vs ex2.approx.ftz.bf16x2 vs ex2.approx.f16x2
// (elements per clock per SM), 8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
__global__ void k_f32(float *out, int iters, float seed) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + i) * -1e-6f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += v[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void k_bf16x2(float *out, int iters, float seed) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(seed * -1e-6f * i, seed * -2e-6f); v[i] = *reinterpret_cast<uint32_t*>(&h); }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= v[i];
  if (s == 12345u) out[0] = s;
}
__global__ void k_f16x2(float *out, int iters, float seed) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(seed * -1e-6f * i, seed * -2e-6f); v[i] = *reinterpret_cast<uint32_t*>(&h); }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= v[i];
  if (s == 12345u) out[0] = s;
}
int main() {
  float *o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = sms * 4, threads = 512;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 3; ++which) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (which == 0) k_f32<<<blocks, threads>>>(o, iters, 1.f);
      else if (which == 1) k_bf16x2<<<blocks, threads>>>(o, iters, 1.f);
      else k_f16x2<<<blocks, threads>>>(o, iters, 1.f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double instr = (double)blocks * threads * iters * 8;
      const double elems = instr * (which ? 2 : 1);
      if (rep) printf("%s: %.2f ms, %.1f instr/clk/SM, %.1f elems/clk/SM (at %d MHz nominal)\n",
                      which == 0 ? "ex2.f32" : which == 1 ? "ex2.bf16x2" : "ex2.f16x2", ms,
                      instr / (ms * 1e-3) / sms / (clk * 1e3), elems / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
