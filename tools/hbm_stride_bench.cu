// Micro-benchmark: HBM gather rate of 16-row K/V stages for the decode cache
// layouts.  Random 16-row tiles (one KV group, d = 128 bf16) of a 4 GB pool
// (well beyond L2), TMA 4-D boxes {64, 16, 2, 1} as in csrc/decode.cu:
//   layout 0: token-major pages [page][64 rows][h_kv = 2][128]  (256 B per row
//             at a 512 B stride -- the other group's half is skipped)
//   layout 1: group-major pages [page][h_kv][64 rows][128]  (4 KB contiguous)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o hbm_stride_bench hbm_stride_bench.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2509_24663_b200/csrc/tc.cuh"
#include "../paper_2509_24663_b200/csrc/tma_host.cuh"

using namespace swattn;
using namespace swattn::tc;

constexpr int kWarps = 8, kRing = 3, kTile = 4096;

__global__ void __launch_bounds__(kWarps * 32) gather(const __grid_constant__ CUtensorMap map, int layout,
                                                       int pages, int iters, unsigned long long *sink) {
  extern __shared__ uint8_t raw[];
  uint8_t *sm = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  __shared__ uint64_t full[kWarps][kRing];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *ring = sm + warp * kRing * kTile;
  if (lane == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&full[warp][i], 1);
    fence_barrier_init();
  }
  __syncwarp();
  unsigned s = (blockIdx.x * kWarps + warp) * 2654435761u + 12345u;
  auto issue = [&](int slot) {
    s = s * 1664525u + 1013904223u;
    const int page = (int)((s >> 8) % (unsigned)pages), sub = (s >> 4) & 3, g = s & 1;
    mbar_arrive_expect_tx(&full[warp][slot], kTile);
    if (layout == 0)
      tma_load_4d(&map, &full[warp][slot], ring + slot * kTile, 0, page * 64 + sub * 16, 0, g);
    else
      tma_load_4d(&map, &full[warp][slot], ring + slot * kTile, 0, (page * 2 + g) * 64 + sub * 16, 0, 0);
  };
  if (lane == 0)
    for (int i = 0; i < kRing; ++i) issue(i);
  for (int it = 0; it < iters; ++it) {
    const int slot = it % kRing;
    mbar_wait(&full[warp][slot], (it / kRing) & 1);
    if (lane == 0 && it + kRing < iters) issue(slot);
  }
  if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)ring[7]);
}

int main() {
  const size_t bytes = 4ull << 30;
  const int pages = (int)(bytes / (64 * 2 * 256));
  uint8_t *base;
  cudaMalloc(&base, bytes);
  cudaMemset(base, 1, bytes);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kWarps * kRing * kTile + 1024;
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int layout = 0; layout < 2; ++layout) {
    CUtensorMap map;
    if (layout == 0) {  // (d 64, row, half, group): strides row 512 B, half 128 B, group 256 B
      const uint64_t dims[4] = {64, (uint64_t)pages * 64, 2, 2}, str[3] = {512, 128, 256};
      const uint32_t box[4] = {64, 16, 2, 1};
      make_tmap_bf16(&map, base, 4, dims, str, box);
    } else {  // (d 64, row, half, 1): rows of 256 B contiguous
      const uint64_t dims[4] = {64, (uint64_t)pages * 128, 2, 1}, str[3] = {256, 128, bytes};
      const uint32_t box[4] = {64, 16, 2, 1};
      make_tmap_bf16(&map, base, 4, dims, str, box);
    }
    for (int ctas_per_sm : {1, 2, 4}) {
      const int grid = sms * ctas_per_sm, iters = 256;
      gather<<<grid, kWarps * 32, smem>>>(map, layout, pages, 16, sink);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      gather<<<grid, kWarps * 32, smem>>>(map, layout, pages, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double gb = (double)grid * kWarps * iters * kTile / 1e9;
      printf("layout %d (%s) ctas/sm %d: %.0f GB/s %s\n", layout,
             layout ? "group-major 4 KB contiguous" : "token-major 256 B @ 512 B", ctas_per_sm, gb / ms * 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
