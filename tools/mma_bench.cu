// Micro-benchmark: tcgen05.mma (kind::f16, M = 128, cta_group::1) issue
// throughput and dependent-chain latency as a function of N and of the number
// of independent accumulators interleaved by the issuing thread -- the
// question behind K4 part B's swap-AB N = 16 design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cuda.h>
#include <stdio.h>

#include "../paper_2509_24663_b200/csrc/tc.cuh"

using namespace swattn::tc;

__global__ void __launch_bounds__(128) mma_kernel(int n, int chains, int rounds, int wait_each,
                                                 unsigned long long *out, int ncommit = 0,
                                                 int distinct_a = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar, extra[8];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 8; ++i) mbar_init(&extra[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  // zero operands (values are irrelevant for timing, but keep them finite)
  for (int i = threadIdx.x; i < (32768 + 65536) / 16; i += 128)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  // distinct_a: chain c reads A tile c (tiles 1..3 alias the B region + beyond; values are zero)
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 131072);
    const uint32_t id = idesc_bf16(128, n, false, false);
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      if (elect_one()) {
        for (int kk = 0; kk < 8; ++kk) {
          const int h = kk >> 2, j = kk & 3;
          for (int c = 0; c < chains; ++c)
            mma_ss(tmem + (uint32_t)(c * n) % 512u,
                   desc_kmajor(a + (distinct_a ? (c & 3) * 32768 : 0) + h * 16384 + j * 32),
                   desc_kmajor(b + h * (n * 128) + j * 32), id, kk > 0);
        }
        for (int c = 0; c < ncommit; ++c) mma_commit(&extra[c & 7]);
        if (wait_each) mma_commit(&bar);
      }
      __syncwarp();
      if (wait_each) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    if (!wait_each) {
      if (elect_one()) mma_commit(&bar);
      __syncwarp();
      mbar_wait(&bar, ph);
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// Handoff round trip: the MMA warp issues one 4-chain x 2-step S group and
// commits s_full[i]; a consumer warpgroup waits, loads the tile from TMEM and
// arrives on back[i]; the MMA warp may run `depth` groups ahead.
__global__ void __launch_bounds__(160) pingpong_kernel(int rounds, int depth, int extra_commits,
                                                     unsigned long long *out, int mode = 0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[8], back[8], junk[8];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&back[i], 128);
      mbar_init(&junk[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < (32768 + 8192) / 16; i += 160)
    reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const unsigned long long t0 = clock64();
  if (warp == 4) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    const uint32_t id = idesc_bf16(128, 16, false, false);
    for (int r = 0; r < rounds; ++r) {
      const int sl = r % depth;
      if (r >= depth && mode != 2) mbar_wait(&back[sl], ((r / depth) - 1) & 1);
      tc_fence_after();
      if (elect_one()) {
        for (int i = 0; i < 8; ++i) {
          const int c = i & 3, kk = 2 * c + (i >> 2);
          mma_ss(tmem + (sl * 4 + c) * 16, desc_kmajor(a + (kk >> 2) * 16384 + (kk & 3) * 32),
                 desc_kmajor(b + (kk >> 2) * 2048 + (kk & 3) * 32), id, i >> 2);
        }
        mma_commit(&full[sl]);
        for (int e = 0; e < extra_commits; ++e) mma_commit(&junk[e]);
      }
      __syncwarp();
    }
  } else if (mode != 2) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float acc = 0.f;
    for (int r = 0; r < rounds; ++r) {
      const int sl = r % depth;
      if (mode == 3) {
        if ((threadIdx.x & 31) == 0)
          while (!mbar_try_wait(&full[sl], (r / depth) & 1)) __nanosleep(32);
        __syncwarp();
      } else if (mode == 4) {
        uint32_t ok = 0;
        while (!ok) {
          asm volatile(
              "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
              "selp.b32 %0, 1, 0, P;\n\t}"
              : "=r"(ok)
              : "r"(smem_u32(&full[sl])), "r"((uint32_t)((r / depth) & 1)), "r"(1000000u)
              : "memory");
        }
      } else {
        mbar_wait(&full[sl], (r / depth) & 1);
      }
      tc_fence_after();
      if (mode == 0) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + sl * 64, v);
        tmem_ld_wait();
        acc += __uint_as_float(v[0]);
      }
      tc_fence_before();
      mbar_arrive(&back[sl]);
    }
    if (acc == 123.f) out[200] = 1;
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 128) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long *d_out;
  cudaMalloc(&d_out, 256 * sizeof(unsigned long long));
  const int smem = 4 * 32768 + 65536 + 2048;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("N chains wait_each  cycles/MMA  (rounds x 8 k-steps x chains MMAs; 148 CTAs)\n");
  const int Ns[] = {16, 32, 64, 128, 256};
  for (int wait_each = 0; wait_each < 2; ++wait_each)
    for (int ni = 0; ni < 5; ++ni)
      for (int chains = 1; chains <= 8; chains *= 2) {
        const int n = Ns[ni];
        if (chains * n > 512) continue;
        const int rounds = 200;
        mma_kernel<<<148, 128, smem>>>(n, chains, rounds, wait_each, d_out);
        mma_kernel<<<148, 128, smem>>>(n, chains, rounds, wait_each, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const double per = (double)mx / (rounds * 8.0 * chains);
        const double flop_clk = 2.0 * 128 * n * 16 / per;
        printf("%3d %2d %d  %8.1f  (%.0f flop/clk/SM)\n", n, chains, wait_each, per, flop_clk);
      }
  printf("distinct A per chain (4 tiles of 32 KB), wait_each 0\n");
  for (int n : {16, 64, 128})
    for (int chains : {1, 2, 4}) {
      const int rounds = 200;
      mma_kernel<<<148, 128, smem>>>(n, chains, rounds, 0, d_out, 0, 1);
      mma_kernel<<<148, 128, smem>>>(n, chains, rounds, 0, d_out, 0, 1);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("N %3d chains %d distinct A: %.1f cycles/MMA\n", n, chains, (double)mx / (rounds * 8.0 * chains));
    }
  printf("commit cost: N=16, 4 chains, no wait, extra commits per round of 32 MMAs\n");
  for (int nc = 0; nc <= 8; nc += 2) {
    const int rounds = 200;
    mma_kernel<<<148, 128, smem>>>(16, 4, rounds, 0, d_out, nc);
    mma_kernel<<<148, 128, smem>>>(16, 4, rounds, 0, d_out, nc);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("commits/round %d: %.1f cycles per round (32 MMAs)\n", nc, (double)mx / rounds);
  }
  cudaFuncSetAttribute(pingpong_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  printf("handoff round trip (8 MMAs + commit -> consumer ld -> arrive), per round\n");
  for (int mode : {0, 3, 4})
  for (int depth : {1, 2, 4, 8})
    for (int ec : {0}) {
      const int rounds = 400;
      pingpong_kernel<<<148, 160, smem>>>(rounds, depth, ec, d_out, mode);
      pingpong_kernel<<<148, 160, smem>>>(rounds, depth, ec, d_out, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("mode %d (0 ld, 1 no ld, 2 no consumer) depth %d: %.1f cycles per round\n", mode, depth, (double)mx / rounds);
    }
  return 0;
}
