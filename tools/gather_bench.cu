// Micro-benchmark: L2 -> SMEM gather bandwidth of random 8 KB tiles (the
// K4 part-B access pattern: selected 64-key blocks of one KV group), by
// copy mechanism and pipeline depth.  No compute; one elected producer and
// an immediate consumer release.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2509_24663_b200/csrc/tc.cuh"
#include "../paper_2509_24663_b200/csrc/tma_host.cuh"

using namespace swattn;
using namespace swattn::tc;

constexpr int kTile = 8192;

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int kMode>
__global__ void __launch_bounds__(128) gather_kernel(const __grid_constant__ CUtensorMap map,
                                                     const uint8_t *base, const int *ids,
                                                     int iters, int stages, unsigned long long *sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[32];
  __shared__ int ids_s[2048];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < iters && i < 2048; i += blockDim.x)
    ids_s[i] = ids[(blockIdx.x * iters + i) & 0xFFFFF];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (kMode == 2) {
    // LDGSTS: all threads copy, ring of stages, wait group
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
      const int st = it % stages;
      const int id = ids_s[it & 2047];
      const uint8_t *src = base + (size_t)id * kTile;
      for (int v = threadIdx.x; v < kTile / 16; v += 128) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem + st * kTile + v * 16)),
                     "l"(src + v * 16));
      }
      asm volatile("cp.async.commit_group;");
      if (it >= stages - 1) {
        asm volatile("cp.async.wait_group %0;" ::"n"(6));
      }
    }
    asm volatile("cp.async.wait_all;");
    __syncthreads();
    acc += smem[threadIdx.x];
    if (threadIdx.x == 0) atomicAdd(sink, acc);
    return;
  }
  if (kMode == 3 || kMode == 4) {
    // 4 issuers, each with its own ring of stages/4 slots: mode 3 = one
    // elected lane in each of 4 warps, mode 4 = lanes 0..3 of warp 0
    const int ring = stages / 4;
    const int who = kMode == 3 ? warp : (threadIdx.x & 31);
    uint8_t *mine = smem + who * ring * kTile;
    uint64_t *bars = full + who * 8;
    const bool issuer = kMode == 3 ? elect_one() : (warp == 0 && who < 4);
    if (issuer) {
      const int warp = who;
      const int per = iters / 4;
      for (int it = 0; it < per + ring; ++it) {
        if (it >= ring) {
          const int c = it - ring;
          mbar_wait(&bars[c % ring], (c / ring) & 1);
        }
        if (it < per) {
          const int st = it % ring;
          const int id = ids_s[(warp * per + it) & 2047];
          mbar_arrive_expect_tx(&bars[st], kTile);
          tma_load_2d(&map, &bars[st], mine + st * kTile, (id & 1) * 128 + ((id >> 1) & 1) * 64,
                      (id >> 2) * 64);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)smem[5]);
    return;
  }
  if (warp == 0 && elect_one()) {
    for (int it = 0; it < iters + stages; ++it) {
      if (it >= stages) {  // consume (wait) tile it - stages, then reuse the slot
        const int c = it - stages;
        mbar_wait(&full[c % stages], (c / stages) & 1);
      }
      if (it < iters) {
        const int st = it % stages;
        const int id = ids_s[it & 2047];
        mbar_arrive_expect_tx(&full[st], kTile);
        if (kMode == 0) {
          // 2D TMA box {64 elems, 64 rows} from a [rows][256 elems] tensor (row stride 512 B)
          tma_load_2d(&map, &full[st], smem + st * kTile, (id & 1) * 128 + ((id >> 1) & 1) * 64,
                      (id >> 2) * 64);
        } else {
          bulk_load(smem + st * kTile, base + (size_t)id * kTile, kTile, &full[st]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)smem[5]);
}

int main() {
  const size_t region = 64ull << 20;  // one KV group's K+V at 128K = 64 MB (L2-resident)
  uint8_t *base;
  cudaMalloc(&base, region);
  cudaMemset(base, 1, region);
  const int ntiles = (int)(region / kTile);
  int *ids;
  const int nid = 1 << 20;
  int *h = (int *)malloc(nid * sizeof(int));
  srand(1);
  for (int i = 0; i < nid; ++i) h[i] = rand() % ntiles;
  cudaMalloc(&ids, nid * sizeof(int));
  cudaMemcpy(ids, h, nid * sizeof(int), cudaMemcpyHostToDevice);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  CUtensorMap map;
  // view: rows of 256 bf16 (512 B) -> region/512 rows
  uint64_t dims[2] = {256, region / 512}, str[1] = {512};
  uint32_t box[2] = {64, 64};
  if (!make_tmap_bf16(&map, base, 2, dims, str, box)) {
    printf("tmap fail\n");
    return 1;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048;
  const char *names[5] = {"TMA 2D box 64x128B (strided rows)", "cp.async.bulk 8 KB contiguous",
                          "LDGSTS 16 B x 512 per tile", "TMA, 4 producer warps",
                          "TMA, 4 producer lanes of 1 warp"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int stages : {4, 8, 16, 24}) {
      for (int cpsm : {1, 2, 3, 4}) {
        const int smem = stages * kTile + 1024;
        if (smem * cpsm > 220 * 1024) continue;
        if (mode == 2 && stages < 8) continue;
        if (mode >= 3 && stages < 8) continue;
        if (mode < 3 && stages > 8) continue;
        void (*k)(CUtensorMap, const uint8_t *, const int *, int, int, unsigned long long *) =
            mode == 0 ? gather_kernel<0> : mode == 1 ? gather_kernel<1> : mode == 2 ? gather_kernel<2> : mode == 3 ? gather_kernel<3> : gather_kernel<4>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = sms * cpsm;
        k<<<grid, 128, smem>>>(map, base, ids, 64, stages, sink);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<grid, 128, smem>>>(map, base, ids, iters, stages, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("%-36s stages=%2d ctas/sm=%d : %7.0f GB/s %s\n", names[mode], stages, cpsm,
               (double)grid * iters * kTile / (ms * 1e6), e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  // SM-count sweep: is the gather bound per SM (ingress) or chip-level (L2)?
  // one CTA per SM (smem forces occupancy 1), 4 issuer warps, 24 stages
  for (int stages : {16, 24}) {
    const int smem = stages * kTile + 1024;
    cudaFuncSetAttribute(gather_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {sms / 4, sms / 2, (3 * sms) / 4, sms}) {
      gather_kernel<3><<<grid, 128, smem>>>(map, base, ids, 64, stages, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      gather_kernel<3><<<grid, 128, smem>>>(map, base, ids, iters, stages, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gbs = (double)grid * iters * kTile / (ms * 1e6);
      printf("SM sweep: TMA 4 issuers stages=%2d sms=%3d : %7.0f GB/s chip, %6.1f GB/s per SM\n", stages, grid,
             gbs, gbs / grid);
    }
  }
  return 0;
}
