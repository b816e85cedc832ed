// Micro-benchmark: warp-level mma.sync.m16n8k16 bf16 (fp32 accumulate)
// throughput on sm_100a, registers only, as a function of warps per SM --
// the alternative to tcgen05 for K4 part B's N = 16 per-token products.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mmasync_bench mmasync_bench.cu
#include <stdio.h>
#include <stdint.h>

__global__ void mmasync_kernel(int iters, float *out, unsigned long long *cyc) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float *out;
  unsigned long long *cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    const int iters = 2000;
    mmasync_kernel<<<148, warps * 32>>>(iters, out, cyc);
    mmasync_kernel<<<148, warps * 32>>>(iters, out, cyc);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double macs = (double)warps * iters * 8 * 16 * 8 * 16;
    printf("warps/SM %2d: %.0f MAC/clk/SM (%.1f cycles per mma per warp)\n", warps, macs / mx,
           (double)mx / (iters * 8));
  }
  return 0;
}
