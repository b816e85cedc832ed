// Tile routing for K4 (sparse attention) -- shared by route.cu, the FA tile
// (attention_tc.cu, mode 3), part B (sparse_warp.cu) and the C ABI.
//
// A tile = 8 consecutive tokens of one KV group (the FA tile's 128 rows).
// Part B gathers every token's top-k blocks separately; when the union of the
// tile's 8 top-k lists is small against the sum of the lists (early query
// blocks, where a token's candidates are few and every token picks most of
// them), streaming that union ONCE through the tensor-core FA tile with a
// per-row block mask is cheaper than 8 per-token gathers.  route.cu decides
// per tile; routed tiles are finished by the FA tile (mode 3, merged with
// part A's O_A / m_A / l_A exactly like part B merges) and skipped by part B.
// The attention each row computes is unchanged: init U local U its own top-k
// (sparse.py:70-91).
#pragma once

#include <stdint.h>
#include <stddef.h>

namespace swattn {

constexpr int kRouteTok = 8;      // tokens per tile (FA tile rows / G)
constexpr int kUCap = 256;        // union blocks per routed tile
constexpr int kUWords = kUCap / 32;

struct TileRoutes {
  uint8_t *routed;   // [h_kv][ntiles] 1 = finished by the FA tile
  int32_t *count;    // routed tiles of the current call
  int32_t *plan;     // [0] FA-tile CTAs, [1] part-B CTAs (plan_kernel)
  unsigned long long *sums;  // [0] union blocks of routed tiles, [1] part-B picks
  int32_t *items;    // [slot] g * ntiles + tile
  int32_t *ucount;   // [slot] union size
  int16_t *ulist;    // [slot][kUCap] ascending block ids
  uint32_t *tbits;   // [slot][kRouteTok][kUWords] bit i of token k: block ulist[i] is k's
  int64_t ntiles;    // cdiv(n, 8)
};

inline size_t route_align(size_t x) { return (x + 255) & ~(size_t)255; }

inline size_t route_workspace_bytes(int h_kv, int64_t n) {
  const int64_t nt = (n + kRouteTok - 1) / kRouteTok, slots = (int64_t)h_kv * nt;
  return route_align((size_t)slots) + route_align(64) + 2 * route_align((size_t)slots * 4) +
         route_align((size_t)slots * kUCap * 2) + route_align((size_t)slots * kRouteTok * kUWords * 4);
}

inline TileRoutes carve_routes(char *base, int h_kv, int64_t n) {
  TileRoutes r;
  r.ntiles = (n + kRouteTok - 1) / kRouteTok;
  const int64_t slots = (int64_t)h_kv * r.ntiles;
  r.routed = reinterpret_cast<uint8_t *>(base);
  base += route_align((size_t)slots);
  r.count = reinterpret_cast<int32_t *>(base);
  r.plan = r.count + 1;
  r.sums = reinterpret_cast<unsigned long long *>(base + 16);
  base += route_align(64);
  r.items = reinterpret_cast<int32_t *>(base);
  base += route_align((size_t)slots * 4);
  r.ucount = reinterpret_cast<int32_t *>(base);
  base += route_align((size_t)slots * 4);
  r.ulist = reinterpret_cast<int16_t *>(base);
  base += route_align((size_t)slots * kUCap * 2);
  r.tbits = reinterpret_cast<uint32_t *>(base);
  return r;
}

}  // namespace swattn
