// Micro-benchmark: can a thread-block cluster beat the per-SM L2 -> SMEM
// gather ceiling (~133 GB/s per SM, profiles/r01c_gather_sm_sweep.txt) that
// bounds K4 part B?  Random 8 KB tiles of one KV group (64 MB, L2-resident):
//   mode 0: no cluster, 4 issuer warps per CTA, each its own ring (baseline)
//   mode 1: cluster of C CTAs, TMA .multicast::cluster -- every tile issued
//           once (round robin over the cluster) and delivered to all C CTAs;
//           reports bytes DELIVERED per SM (= what each SM ingests)
//   mode 2: DSMEM: each warp streams 16-byte ld.shared::cluster from the peer
//           CTA's shared memory (no L2 traffic) -- per-SM remote read rate
//   mode 3: mode 0 (L2 gather by 4 warps) and mode 2 (DSMEM reads by 4 other
//           warps) at the same time: are the two ingress paths additive?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mcast_bench mcast_bench.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2509_24663_b200/csrc/tc.cuh"
#include "../paper_2509_24663_b200/csrc/tma_host.cuh"

using namespace swattn;
using namespace swattn::tc;

constexpr int kTile = 8192;
constexpr int kRing = 4;  // slots per issuer warp

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap *map, uint64_t *bar, void *dst, int32_t c0,
                                               int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

struct Smem {
  uint8_t tiles[4][kRing][kTile];  // 128 KB
  uint64_t full[4][kRing];
  uint64_t empty[4][kRing];
};

// mode 0 / 1 (kC = cluster size; 1 => plain TMA)
template <int kC>
__global__ void __launch_bounds__(128) gather_mc(const __grid_constant__ CUtensorMap map, const int *ids,
                                                 int iters, unsigned long long *sink) {
  extern __shared__ uint8_t raw[];
  Smem &s = *reinterpret_cast<Smem *>(raw + ((1024 - (smem_u32(raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = kC > 1 ? cluster_rank() : 0;
  const int cluster = blockIdx.x / kC;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; ++w)
      for (int i = 0; i < kRing; ++i) {
        mbar_init(&s.full[w][i], 1);
        mbar_init(&s.empty[w][i], kC);
      }
    fence_barrier_init();
  }
  if (kC > 1) cluster_sync(); else __syncthreads();
  if (elect_one()) {
    const int w = warp;
    for (int it = 0; it < iters + kRing; ++it) {
      if (it >= kRing) {  // consume tile it - kRing, release its slot to its issuer
        const int c = it - kRing;
        const int st = c % kRing;
        mbar_wait(&s.full[w][st], (c / kRing) & 1);
        if (kC > 1) arrive_remote(mapa(smem_u32(&s.empty[w][st]), c % kC));
      }
      if (it < iters) {
        const int st = it % kRing;
        mbar_arrive_expect_tx(&s.full[w][st], kTile);
        if ((uint32_t)(it % kC) == rank) {
          const int id = ids[((cluster * 4 + w) * iters + it) & 0xFFFFF];
          if (kC > 1) {
            if (it >= kRing) while (!try_wait_cluster(&s.empty[w][st], ((it / kRing) - 1) & 1)) {}
            tma_load_2d_mc(&map, &s.full[w][st], s.tiles[w][st], (id & 1) * 128 + ((id >> 1) & 1) * 64,
                           (id >> 2) * 64, (uint16_t)((1u << kC) - 1));
          } else {
            tma_load_2d(&map, &s.full[w][st], s.tiles[w][st], (id & 1) * 128 + ((id >> 1) & 1) * 64,
                        (id >> 2) * 64);
          }
        }
      }
    }
  }
  if (kC > 1) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)s.tiles[0][0][5]);
}

// mode 2 / 3: cluster of 2.  Warps 0-3 (mode 3 only) gather from L2 as in
// mode 0; warps 4-7 read the peer's 128 KB tile area with 16-byte DSMEM loads.
template <bool kWithL2>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256)
    dsmem_read(const __grid_constant__ CUtensorMap map, const int *ids, int iters, int reps,
               unsigned long long *sink) {
  extern __shared__ uint8_t raw[];
  Smem &s = *reinterpret_cast<Smem *>(raw + ((1024 - (smem_u32(raw) & 1023)) & 1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; ++w)
      for (int i = 0; i < kRing; ++i) mbar_init(&s.full[w][i], 1);
    fence_barrier_init();
  }
  cluster_sync();
  if (warp < 4) {
    if (kWithL2 && elect_one()) {
      const int w = warp;
      // separate L2 landing zone would be cleaner; the tiles area is overwritten
      // while the peer reads it (values are irrelevant here)
      for (int it = 0; it < iters + kRing; ++it) {
        if (it >= kRing) {
          const int c = it - kRing;
          mbar_wait(&s.full[w][c % kRing], (c / kRing) & 1);
        }
        if (it < iters) {
          const int st = it % kRing;
          const int id = ids[((blockIdx.x * 4 + w) * iters + it) & 0xFFFFF];
          mbar_arrive_expect_tx(&s.full[w][st], kTile);
          tma_load_2d(&map, &s.full[w][st], s.tiles[w][st], (id & 1) * 128 + ((id >> 1) & 1) * 64,
                      (id >> 2) * 64);
        }
      }
    }
  } else {
    const uint32_t base = mapa(smem_u32(&s.tiles[0][0][0]), rank ^ 1);
    uint32_t acc = 0;
    const int t = threadIdx.x - 128;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 8
      for (int off = t * 16; off < 4 * kRing * kTile; off += 128 * 16) {
        uint32_t a, b, c, d;
        asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                     : "r"(base + off));
        acc ^= a ^ b ^ c ^ d;
      }
    }
    if (lane == 0) atomicAdd(sink, (unsigned long long)acc);
  }
  cluster_sync();
}

template <int kC>
static float run_mc(const CUtensorMap &map, const int *ids, int grid, int iters, unsigned long long *sink) {
  const int smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(gather_mc<kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gather_mc<kC>, map, ids, 64, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, gather_mc<kC>, map, ids, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error C=%d: %s\n", kC, cudaGetErrorString(e));
  return ms;
}

int main() {
  const size_t region = 64ull << 20;
  uint8_t *base;
  cudaMalloc(&base, region);
  cudaMemset(base, 1, region);
  const int ntiles = (int)(region / kTile);
  const int nid = 1 << 20;
  int *h = (int *)malloc(nid * sizeof(int));
  srand(1);
  for (int i = 0; i < nid; ++i) h[i] = rand() % ntiles;
  int *ids;
  cudaMalloc(&ids, nid * sizeof(int));
  cudaMemcpy(ids, h, nid * sizeof(int), cudaMemcpyHostToDevice);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  CUtensorMap map;
  uint64_t dims[2] = {256, region / 512}, str[1] = {512};
  uint32_t box[2] = {64, 64};
  if (!make_tmap_bf16(&map, base, 2, dims, str, box)) {
    printf("tmap fail\n");
    return 1;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2048;
  // each CTA receives 4 warps x iters tiles; L2 reads = that / C per CTA
  {
    for (int grid : {sms / 4, sms / 2, sms}) {
      float ms = run_mc<1>(map, ids, grid, iters, sink);
      double gb = (double)grid * 4 * iters * kTile / 1e9;
      printf("mode0 plain TMA      C=1 ctas=%3d : delivered %7.1f GB/s per SM (%7.0f chip), L2 read %7.0f GB/s\n",
             grid, gb / ms * 1e3 / grid, gb / ms * 1e3, gb / ms * 1e3);
    }
    for (int grid : {sms / 2 / 2 * 2, (sms / 2) * 2}) {
      float ms = run_mc<2>(map, ids, grid, iters, sink);
      double gb = (double)grid * 4 * iters * kTile / 1e9;
      printf("mode1 multicast      C=2 ctas=%3d : delivered %7.1f GB/s per SM (%7.0f chip), L2 read %7.0f GB/s\n",
             grid, gb / ms * 1e3 / grid, gb / ms * 1e3, gb / ms * 1e3 / 2);
    }
    for (int grid : {(sms / 4) * 4}) {
      float ms = run_mc<4>(map, ids, grid, iters, sink);
      double gb = (double)grid * 4 * iters * kTile / 1e9;
      printf("mode1 multicast      C=4 ctas=%3d : delivered %7.1f GB/s per SM (%7.0f chip), L2 read %7.0f GB/s\n",
             grid, gb / ms * 1e3 / grid, gb / ms * 1e3, gb / ms * 1e3 / 4);
    }
  }
  {
    const int smem = sizeof(Smem) + 1024;
    const int grid = (sms / 2) * 2;
    // L2-only time of 1024 iterations (mode 0 at this grid) to size the DSMEM side
    const float l2ms = run_mc<1>(map, ids, grid, 1024, sink);
    float dsm_ms = 0.f;
    int reps = 64;
    for (int with = 0; with < 2; ++with) {
      auto k = with ? dsmem_read<true> : dsmem_read<false>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<grid, 256, smem>>>(map, ids, 64, 2, sink);
      if (with) reps = (int)(64 * l2ms / dsm_ms) + 1;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<grid, 256, smem>>>(map, ids, with ? 1024 : 0, reps, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (!with) dsm_ms = ms;
      cudaError_t e = cudaGetLastError();
      double dsm = (double)grid * reps * 4 * kRing * kTile / 1e9;
      double l2 = with ? (double)grid * 4 * 1024 * kTile / 1e9 : 0;
      printf("mode%d DSMEM%s ctas=%3d reps=%d: %.3f ms (L2 alone %.3f); DSMEM %7.1f GB/s per SM, L2 %7.1f GB/s per SM %s\n",
             2 + with, with ? "+L2 gather" : "          ", grid, reps, ms, l2ms, dsm / ms * 1e3 / grid,
             l2 / ms * 1e3 / grid, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
