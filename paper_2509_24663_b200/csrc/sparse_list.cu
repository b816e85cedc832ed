// K4, general form -- sparse_forward over an ARBITRARY block selection
// (sparse.py:43-98 with any BlockSelection, selection.py:51-90: e.g. a
// fixture from load_selection, or every causal block as in the reference's
// _all_blocks_selection, bench.py:207-210).  The hot path (init U local U
// top-k, selection.py:113-126) goes through part A + part B instead; this
// kernel serves selections without that structure.
//
// Row (group g, token i) visits its listed blocks in list order (ascending in
// a BlockSelection); block j covers keys [j B, min(j B + B, n, i + 1))
// (selection.py:73-87: causal clip, empty spans skipped).  One warp per row:
// the 16 query heads of the group are the M = 16 of mma.sync.m16n8k16 (as in
// part B, sparse_warp.cu), Q in registers, S -> P in registers, O in
// registers with the online max / sum recurrence of sparse.py:78-88 (running
// max + rescale, since no part-A offset exists here).  Keys stream in 16-row
// stages through a per-warp 2-stage cp.async ring ([d half][row][64], 16-byte
// chunks XOR-swizzled by row: conflict-free ldmatrix); rows outside the span
// are zero-filled and masked.  Any block size B >= 1.  A row with an empty
// visible set gets O = 0, lse = -inf (the Python layer raises the
// reference's RuntimeError before launching, sparse.py:75-76).
#include <string.h>

#include "common.cuh"
#include "tc.cuh"

namespace swattn {

namespace {

constexpr int kLW = 4;                          // warps per CTA
constexpr int kLK = 16;                         // keys per stage
constexpr uint32_t kLTile = kLK * kD * 2;       // 4 KB

struct ListArgs {
  const __nv_bfloat16 *Q, *K, *V;
  const int32_t *blocks, *cnt;  // [h_kv][n][ld], [h_kv][n]
  int64_t ld, n;
  int h_q, h_kv, B;
  float scale_log2;
  __nv_bfloat16 *O;
  float *lse;
};

__device__ __forceinline__ uint32_t lswz(int row, int c) {
  const int line = (c >> 3) * kLK + row;
  return (uint32_t)(line * 128 + (((c & 7) ^ (line & 7)) << 4));
}
__device__ __forceinline__ void lmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void lldsm(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                      uint32_t &r3, bool trans) {
  if (trans)
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
  else
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// Cursor over the 16-key stages of one row's visible spans (warp-uniform).
struct SpanCursor {
  const int32_t *list;
  int cnt, idx;          // list position
  int64_t k0, end;       // current stage start, current span end
  __device__ bool next_span(const ListArgs &a, int64_t i) {
    while (idx < cnt) {
      const int j = list[idx++];
      if (j < 0) continue;
      const int64_t s = (int64_t)j * a.B;
      int64_t e = s + a.B;
      if (e > a.n) e = a.n;
      if (e > i + 1) e = i + 1;
      if (e > s) {
        k0 = s;
        end = e;
        return true;
      }
    }
    return false;
  }
  // advance to the next stage; false when the row is exhausted
  __device__ bool advance(const ListArgs &a, int64_t i) {
    k0 += kLK;
    if (k0 < end) return true;
    return next_span(a, i);
  }
};

__global__ void __launch_bounds__(kLW * 32) sparse_list_kernel(const ListArgs a) {
  extern __shared__ uint8_t lsm_raw[];
  uint8_t *lsm = lsm_raw + ((1024u - (tc::smem_u32(lsm_raw) & 1023u)) & 1023u);
  auto ring = reinterpret_cast<uint8_t(*)[2][2][kLTile]>(lsm);  // [warp][slot][K|V]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h0 = lane >> 2, dw = lane & 3;
  const int lm = lane >> 3, lr = lane & 7;
  const int64_t rows = a.n * a.h_kv;
  for (int64_t item = (int64_t)blockIdx.x * kLW + warp; item < rows;
       item += (int64_t)gridDim.x * kLW) {
    // token-major items: neighbouring warps share K/V rows in L2
    const int64_t i = item / a.h_kv;
    const int g = (int)(item % a.h_kv);
    const int64_t row = (int64_t)g * a.n + i;
    const int64_t ridx = i * a.h_q + (int64_t)g * kG;  // [n][h_q] row of head 0
    SpanCursor cur{a.blocks + row * a.ld, a.cnt[row], 0, 0, 0};
    const bool any = cur.next_span(a, i);
    if (!any) {
      // empty visible set: defined outputs
      __nv_bfloat16 *o0 = a.O + ridx * kD;
      for (int e = lane; e < kG * kD; e += 32) o0[e] = __float2bfloat16_rn(0.f);
      if (lane < kG) a.lse[ridx + lane] = -INFINITY;
      continue;
    }
    uint32_t qa[8][4];
    {
      const uint32_t *qg = reinterpret_cast<const uint32_t *>(a.Q + ridx * kD);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qa[ks][0] = __ldg(qg + h0 * (kD / 2) + ks * 8 + dw);
        qa[ks][1] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + dw);
        qa[ks][2] = __ldg(qg + h0 * (kD / 2) + ks * 8 + 4 + dw);
        qa[ks][3] = __ldg(qg + (h0 + 8) * (kD / 2) + ks * 8 + 4 + dw);
      }
    }
    // producer: copy stage (k0, end) into ring slot
    auto issue = [&](int64_t k0, int64_t end, int slot) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int idx = e * 32 + lane, rr = idx >> 4, c = idx & 15;
        const uint32_t dk = tc::smem_u32(ring[warp][slot][0]) + lswz(rr, c);
        const uint32_t dv = tc::smem_u32(ring[warp][slot][1]) + lswz(rr, c);
        const int64_t key = k0 + rr;
        if (key < end) {
          const int64_t off = (key * a.h_kv + g) * kD + c * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dk), "l"(a.K + off));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dv), "l"(a.V + off));
        } else {
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dk), "r"(0u));
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(dv), "r"(0u));
        }
      }
      asm volatile("cp.async.commit_group;");
    };
    SpanCursor prod = cur;
    bool prod_ok = true;
    issue(prod.k0, prod.end, 0);
    prod_ok = prod.advance(a, i);
    if (prod_ok) issue(prod.k0, prod.end, 1);
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float o[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    int slot = 0;
    bool cons_ok = true;
    while (cons_ok) {
      if (prod_ok) asm volatile("cp.async.wait_group 1;");
      else asm volatile("cp.async.wait_group 0;");
      __syncwarp();
      const uint32_t kst = tc::smem_u32(ring[warp][slot][0]), vst = tc::smem_u32(ring[warp][slot][1]);
      float sc[2][4] = {};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t b00, b01, b10, b11;
        lldsm(kst + lswz((lm >> 1) * 8 + lr, ks * 2 + (lm & 1)), b00, b01, b10, b11, false);
        lmma(sc[0], qa[ks], b00, b01);
        lmma(sc[1], qa[ks], b10, b11);
      }
      float x[2][4];
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int jt = 0; jt < 2; ++jt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t key = cur.k0 + jt * 8 + dw * 2 + (e & 1);
          const float v = key < cur.end ? sc[jt][e] * a.scale_log2 : -INFINITY;
          x[jt][e] = v;
          if (e < 2) mx0 = fmaxf(mx0, v); else mx1 = fmaxf(mx1, v);
        }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float al0 = (m0 == -INFINITY) ? 0.f : fast_exp2(m0 - mn0);
      const float al1 = (m1 == -INFINITY) ? 0.f : fast_exp2(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int jt = 0; jt < 2; ++jt) {
        x[jt][0] = fast_exp2(x[jt][0] - mn0);
        x[jt][1] = fast_exp2(x[jt][1] - mn0);
        x[jt][2] = fast_exp2(x[jt][2] - mn1);
        x[jt][3] = fast_exp2(x[jt][3] - mn1);
        ps0 += x[jt][0] + x[jt][1];
        ps1 += x[jt][2] + x[jt][3];
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int jt = 0; jt < 16; ++jt) {
        o[jt][0] *= al0;
        o[jt][1] *= al0;
        o[jt][2] *= al1;
        o[jt][3] *= al1;
      }
      const uint32_t pa[4] = {tc::pack_bf16(x[0][0], x[0][1]), tc::pack_bf16(x[0][2], x[0][3]),
                              tc::pack_bf16(x[1][0], x[1][1]), tc::pack_bf16(x[1][2], x[1][3])};
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        uint32_t v00, v01, v10, v11;
        lldsm(vst + lswz((lm & 1) * 8 + lr, dp * 2 + (lm >> 1)), v00, v01, v10, v11, true);
        lmma(o[2 * dp], pa, v00, v01);
        lmma(o[2 * dp + 1], pa, v10, v11);
      }
      __syncwarp();
      if (prod_ok) {
        prod_ok = prod.advance(a, i);
        if (prod_ok) issue(prod.k0, prod.end, slot);
      }
      cons_ok = cur.advance(a, i);
      slot ^= 1;
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float i0 = 1.f / l0, i1 = 1.f / l1;
    __nv_bfloat16 *o0 = a.O + (ridx + h0) * kD, *o1 = a.O + (ridx + h0 + 8) * kD;
    const int dc = dw * 2;
#pragma unroll
    for (int jt = 0; jt < 16; ++jt) {
      *reinterpret_cast<__nv_bfloat162 *>(o0 + jt * 8 + dc) =
          __floats2bfloat162_rn(o[jt][0] * i0, o[jt][1] * i0);
      *reinterpret_cast<__nv_bfloat162 *>(o1 + jt * 8 + dc) =
          __floats2bfloat162_rn(o[jt][2] * i1, o[jt][3] * i1);
    }
    if (dw == 0) {
      a.lse[ridx + h0] = (m0 + __log2f(l0)) * 0.6931471805599453f;
      a.lse[ridx + h0 + 8] = (m1 + __log2f(l1)) * 0.6931471805599453f;
    }
    __syncwarp();  // ring slots are reused by the warp's next row
  }
}

}  // namespace

int32_t launch_sparse_list(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                           int64_t n, const int32_t *blocks, int64_t ld, const int32_t *cnt,
                           void *O, float *lse, int num_sms, cudaStream_t stream) {
  ListArgs a;
  memset(&a, 0, sizeof(a));
  a.Q = static_cast<const __nv_bfloat16 *>(Q);
  a.K = static_cast<const __nv_bfloat16 *>(K);
  a.V = static_cast<const __nv_bfloat16 *>(V);
  a.blocks = blocks;
  a.cnt = cnt;
  a.ld = ld;
  a.n = n;
  a.h_q = cfg->h_q;
  a.h_kv = cfg->h_kv;
  a.B = cfg->B;
  a.scale_log2 = (1.f / sqrtf((float)cfg->d_h)) * 1.4426950408889634f;
  a.O = static_cast<__nv_bfloat16 *>(O);
  a.lse = lse;
  const int smem = kLW * 4 * (int)kLTile + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sparse_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int64_t rows = n * cfg->h_kv;
  int64_t grid = cdiv(rows, kLW);
  const int64_t cap = (int64_t)num_sms * 12;  // 3 CTAs of 64 KB per SM, a few waves deep
  if (grid > cap) grid = cap;
  sparse_list_kernel<<<(unsigned)grid, kLW * 32, smem, stream>>>(a);
  SWATTN_LAUNCH_CHECK("sparse_list_kernel");
  return SWATTN_OK;
}

}  // namespace swattn
