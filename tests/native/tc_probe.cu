// Test-only probe of the tcgen05 / TMEM / TMA encodings in csrc/tc.cuh:
// D[128 x N] = A[128 x 128] . B[N x 128]^T in four operand configurations.
//   mode 0: A, B K-major SW128, staged by threads (manual swizzle)
//   mode 1: A, B K-major SW128, staged by TMA
//   mode 2: A K-major (TMA), B MN-major SW128 from Bt [128 x N] (TMA)
//   mode 3: A from TMEM (tcgen05.st), B K-major (TMA)
//   mode 4: A MN-major SW128 from At [128 x 128] (TMA), B K-major (TMA)
// Built into tests/native/libtcprobe.so by __graft_entry__.build().
#include <cuda_bf16.h>
#include <stdio.h>

#include "../../paper_2509_24663_b200/csrc/tc.cuh"
#include "../../paper_2509_24663_b200/csrc/tma_host.cuh"

using namespace swattn;
using namespace swattn::tc;

struct Maps {
  CUtensorMap a, b, bt, at;
};

__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ Maps maps,
                                                    const __nv_bfloat16 *A, const __nv_bfloat16 *B,
                                                    float *D, int N, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;                 // 2 halves x 128 rows x 128 B = 32 KB
  uint8_t *sB = smem + 32768;         // 2 halves x N rows x 128 B (or MN-major 2 x 128 x 128 B)
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  if (mode == 0) {
    for (int idx = threadIdx.x; idx < 128 * 128; idx += 128) {
      const int r = idx / 128, k = idx % 128, h = k / 64, kk = k % 64;
      const uint32_t off = h * 128 * 128 + r * 128 + ((((kk * 2) / 16) ^ (r % 8)) * 16) + (kk * 2) % 16;
      *reinterpret_cast<__nv_bfloat16 *>(sA + off) = A[idx];
    }
    for (int idx = threadIdx.x; idx < N * 128; idx += 128) {
      const int r = idx / 128, k = idx % 128, h = k / 64, kk = k % 64;
      const uint32_t off = h * N * 128 + r * 128 + ((((kk * 2) / 16) ^ (r % 8)) * 16) + (kk * 2) % 16;
      *reinterpret_cast<__nv_bfloat16 *>(sB + off) = B[idx];
    }
    fence_proxy_async();
    __syncthreads();
  } else {
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      if (mode == 4) {
        tma_load_2d(&maps.at, &bar_load, sA, 0, 0);
        tma_load_2d(&maps.at, &bar_load, sA + 128 * 128, 64, 0);
        bytes += 32768;
      } else if (mode != 3) {
        tma_load_2d(&maps.a, &bar_load, sA, 0, 0);
        tma_load_2d(&maps.a, &bar_load, sA + 128 * 128, 64, 0);
        bytes += 32768;
      }
      if (mode == 2) {
        tma_load_2d(&maps.bt, &bar_load, sB, 0, 0);
        if (N > 64) tma_load_2d(&maps.bt, &bar_load, sB + 128 * 128, 64, 0);
        bytes += 128 * 128 * (N > 64 ? 2 : 1);
      } else {
        tma_load_2d(&maps.b, &bar_load, sB, 0, 0);
        tma_load_2d(&maps.b, &bar_load, sB + N * 128, 64, 0);
        bytes += N * 256;
      }
      mbar_arrive_expect_tx(&bar_load, bytes);
    }
    if (mode == 3) {
      // A row r = 32*warp + lane into TMEM columns [256, 320): 2 bf16 per column
      const int r = 32 * warp + lane;
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t v[16];
        for (int e = 0; e < 16; ++e) {
          const int k = 2 * (c0 + e);
          v[e] = pack_bf16(__bfloat162float(A[r * 128 + k]), __bfloat162float(A[r * 128 + k + 1]));
        }
        tmem_st16(tmem + ((uint32_t)(32 * warp) << 16) + 256 + c0, v);
      }
      tmem_st_wait();
    }
    mbar_wait(&bar_load, 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp == 0) {
    if (elect_one()) {
      const uint32_t id = idesc_bf16(128, N, mode == 4, mode == 2);
      for (int kk = 0; kk < 8; ++kk) {
        const int h = kk / 4, j = kk % 4;
        uint64_t bdesc;
        if (mode == 2) bdesc = desc_mnmajor(smem_u32(sB) + kk * 16 * 128, 128 * 128);
        else bdesc = desc_kmajor(smem_u32(sB) + h * N * 128 + j * 32);
        if (mode == 3) {
          mma_ts(tmem, tmem + 256 + kk * 8, bdesc, id, kk > 0);
        } else {
          const uint64_t adesc = (mode == 4) ? desc_mnmajor(smem_u32(sA) + kk * 16 * 128, 128 * 128)
                                             : desc_kmajor(smem_u32(sA) + h * 128 * 128 + j * 32);
          mma_ss(tmem, adesc, bdesc, id, kk > 0);
        }
      }
      mma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int r = 32 * warp + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    tmem_ld_wait();
    for (int e = 0; e < 16; ++e) D[r * N + c0 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

extern "C" int tc_probe(const void *A, const void *B, const void *Bt, const void *At, float *D,
                        int N, int mode) {
  Maps maps;
  uint64_t dimsA[2] = {128, 128}, strA[1] = {256};
  uint32_t boxA[2] = {64, 128};
  if (!make_tmap_bf16(&maps.a, A, 2, dimsA, strA, boxA)) return -1;
  uint64_t dimsB[2] = {128, (uint64_t)N}, strB[1] = {256};
  uint32_t boxB[2] = {64, (uint32_t)N};
  if (!make_tmap_bf16(&maps.b, B, 2, dimsB, strB, boxB)) return -2;
  uint64_t dimsBt[2] = {(uint64_t)N, 128}, strBt[1] = {(uint64_t)N * 2};
  uint32_t boxBt[2] = {64, 128};
  if (!make_tmap_bf16(&maps.bt, Bt, 2, dimsBt, strBt, boxBt)) return -3;
  if (!make_tmap_bf16(&maps.at, At, 2, dimsA, strA, boxA)) return -4;
  const int smem = 32768 + 65536 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(maps, (const __nv_bfloat16 *)A, (const __nv_bfloat16 *)B, D, N, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("probe error: %s\n", cudaGetErrorString(e));
    return -10;
  }
  return 0;
}
