// C-ABI entry points (include/swattn_b200.h): validation, workspace carving
// and stream-ordered orchestration of the K1..K6 kernels.  No allocation,
// no host synchronisation.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "route.cuh"
#include "topk_cta.cuh"

namespace swattn {

static thread_local char g_err[512] = "";
static thread_local int g_group0 = 0, g_group1 = -1;  // -1: all groups

GroupRange group_range(const swattn_config *cfg) {
  if (g_group1 < 0) return GroupRange{0, cfg->h_kv};
  return GroupRange{g_group0, g_group1 - g_group0};
}
GroupScope::GroupScope(int g0, int g1) : prev_g0(g_group0), prev_g1(g_group1) {
  g_group0 = g0;
  g_group1 = g1;
}
GroupScope::~GroupScope() {
  g_group0 = prev_g0;
  g_group1 = prev_g1;
}

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int32_t cuda_check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return SWATTN_OK;
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return SWATTN_ECUDA;
}

// kernels (defined in the other translation units)
int32_t launch_compress(const swattn_config *, const void *, int64_t, void *, void *, cudaStream_t);
int32_t launch_scores_simt(const swattn_config *, const void *, const void *, const void *, int64_t,
                           int32_t, float *, int64_t, uint64_t *, int64_t, cudaStream_t);
int32_t launch_scores_tc(const swattn_config *, const void *, const void *, const void *, int64_t,
                         int64_t, int64_t, int32_t, float *, int64_t, uint64_t *, int64_t,
                         cudaStream_t, const FusedTopk *fz = nullptr);
int32_t launch_topk_tail(const swattn_config *, const float *, int64_t, int64_t, int64_t, int64_t,
                         int32_t *, int32_t *, int32_t *, int32_t *, int32_t, const uint64_t *, int64_t,
                         const int32_t *, const int32_t *, cudaStream_t);
int32_t launch_shared_scores(const swattn_config *, const void *, const void *, const void *,
                             int64_t, int32_t, float *, uint8_t *, float *, cudaStream_t);
int32_t launch_maxpool(const swattn_config *, const float *, int64_t, float *, int64_t,
                       cudaStream_t);
int32_t launch_topk(const swattn_config *, const float *, int64_t, int64_t, int64_t, int64_t,
                    int32_t *, int32_t *, int32_t *, int32_t *, int32_t, const uint64_t *, int64_t,
                    cudaStream_t);
int32_t launch_rerank(const swattn_config *, const void *, const void *, const void *, int64_t,
                      int32_t, const float *, int64_t, const int32_t *, const int32_t *, int32_t,
                      int32_t *, void *, int, cudaStream_t);
size_t rerank_partials_bytes();
int32_t launch_attention_simt(const swattn_config *, const void *, const void *, const void *,
                              int64_t, const int32_t *, const int32_t *, int, int, void *, float *,
                              int *, cudaStream_t);
int32_t launch_sparse_part_a(const swattn_config *, const void *, const void *, const void *,
                             int64_t, int64_t, int64_t, void *, float *, float *, float *,
                             cudaStream_t);
int32_t launch_sparse_part_b(const swattn_config *, const void *, const void *, const void *,
                             int64_t, int64_t, int64_t, const int32_t *, const int32_t *,
                             const float *,
                             const float *, void *, float *, int32_t *, int32_t *, int,
                             cudaStream_t, const uint8_t *, const int32_t *);
int32_t launch_route_plan(const TileRoutes &, int64_t, int, int, cudaStream_t);
int32_t launch_route_tiles(const swattn_config *, int64_t, int64_t, int64_t, const int32_t *,
                           const int32_t *, const TileRoutes &, int, cudaStream_t);
int32_t launch_routed_tiles(const swattn_config *, const void *, const void *, const void *, int64_t,
                            void *, float *, float *, float *, const TileRoutes &, cudaStream_t);
int32_t launch_sparse_list(const swattn_config *, const void *, const void *, const void *, int64_t,
                           const int32_t *, int64_t, const int32_t *, void *, float *, int,
                           cudaStream_t);
int32_t launch_attention_list(const swattn_config *, const void *, const void *, const void *,
                              int64_t, const int32_t *, const int32_t *, const int32_t *,
                              const int32_t *, void *, float *, int, cudaStream_t);
int32_t launch_sparse_bwd(const swattn_config *, const void *, const void *, const void *, int64_t,
                          const int32_t *, const int32_t *, const void *, const float *, const void *,
                          void *, void *, void *, void *, size_t, int, int, cudaStream_t);
size_t sparse_bwd_workspace_bytes(const swattn_config *, int64_t, int);
int32_t launch_dense_tc(const swattn_config *, const void *, const void *, const void *, int64_t,
                        int, void *, float *, cudaStream_t);
bool scores_tc_available();
bool attention_tc_available();

static int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Persistent CTAs of part B (one per SM by default).  SWATTN_PB_CTAS caps it
// (measurement knob: part B is bound by the chip-wide L2 gather rate, so it
// can leave SMs to concurrent work at little cost).
static int part_b_ctas() {
  static int ctas = [] {
    const char *e = getenv("SWATTN_PB_CTAS");
    const int v = e ? atoi(e) : 0;
    return v > 0 && v < num_sms() ? v : num_sms();
  }();
  return ctas;
}

// Tile routing threshold (route.cuh): a tile goes to the tensor-core FA tile
// when |union of its top-k lists| * 100 < sum of the lists * ratio.  On by
// default up to 48K tokens (8K 1.29 -> 0.77 ms, 16K 3.58 -> 2.47, 32K
// 7.90 -> 7.30); above it the routed share is small and the FA tile's SMs
// cost part B about what they save (64K / 128K within noise or slower,
// profiles/r02aw_route_sweep.txt), so it is off.  SWATTN_ROUTE_PCT overrides
// (0 disables), read per call.
static int route_pct(int64_t n) {
  const char *e = getenv("SWATTN_ROUTE_PCT");
  if (e) return atoi(e);
  return n <= 49152 ? 45 : 0;
}

// The tensor-core kernels are the only path for the paper profile; the
// CUDA-core kernels (scores_simt.cu / attention_simt.cu) serve the profiles
// the tcgen05 tiles are not compiled for (e.g. the reference's small
// check profile, bench.py:199-204).  No run-time switch between the two.
static bool use_tc_scores() { return scores_tc_available(); }
static bool use_tc_attention() { return attention_tc_available(); }

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct SelectLayout {
  int64_t m1, m2, n_cols, ld, ld_f;
  size_t off_kc1, off_kc2, off_scmp, off_flags, off_count, off_rows, off_ovf, off_part, off_shared,
      off_lse, total;
  bool generic;
};

static SelectLayout select_layout(const swattn_config *cfg, int64_t n) {
  SelectLayout L{};
  L.m1 = num_pooled(n, cfg->l_C1, cfg->s_C1);
  L.m2 = num_pooled(n, cfg->l_C2, cfg->s_C2);
  L.n_cols = L.m1 ? cdiv(L.m1, cfg->s) : 0;
  L.ld = ((L.n_cols + 3) / 4) * 4;
  if (L.ld == 0) L.ld = 4;
  L.ld_f = L.n_cols / 31 + 1;
  L.generic = swattn_profile_supported(cfg) == 0;
  size_t o = 0;
  L.off_kc1 = o; o = align_up(o + (size_t)L.m1 * cfg->h_kv * cfg->d_h * 2);
  L.off_kc2 = o; o = align_up(o + (size_t)L.m2 * cfg->h_kv * cfg->d_h * 2);
  L.off_scmp = o; o = align_up(o + (size_t)cfg->h_kv * n * L.ld * 4);
  L.off_flags = o; o = align_up(o + (size_t)cfg->h_kv * n * L.ld_f * 8);
  L.off_count = o; o = align_up(o + 16);
  // flagged row ids [cap] followed by their k-th keys [cap] (K3 -> re-rank)
  L.off_rows = o; o = align_up(o + (size_t)cfg->h_kv * n * 4 * 2);
  // rows whose fused top-k candidate set overflowed (K2 -> topk_tail_kernel)
  L.off_ovf = o; o = align_up(o + (size_t)cfg->h_kv * n * 4);
  L.off_part = o; o = align_up(o + rerank_partials_bytes());
  L.off_shared = o;
  if (L.generic) o = align_up(o + (size_t)n * cfg->h_kv * L.m1 * 4);
  L.off_lse = o;
  if (L.generic) o = align_up(o + (size_t)n * cfg->h_q * 4);
  L.total = o;
  return L;
}

static int32_t check_ptr(const void *p, const char *name) {
  if (p == nullptr) {
    set_error("%s must not be NULL", name);
    return SWATTN_EINVAL;
  }
  return SWATTN_OK;
}

}  // namespace swattn

using namespace swattn;

extern "C" {

const char *swattn_last_error(void) { return g_err; }

int32_t swattn_version(void) { return 1000; }

int32_t swattn_validate_config(const swattn_config *cfg) {
  if (cfg == nullptr) {
    set_error("config must not be NULL");
    return SWATTN_EINVAL;
  }
  // core.py:118-135, in the reference's field order
  const struct { const char *name; int32_t v; } pos[] = {
      {"h_q", cfg->h_q},       {"h_kv", cfg->h_kv},       {"d_h", cfg->d_h},
      {"B", cfg->B},           {"l_C1", cfg->l_C1},       {"s_C1", cfg->s_C1},
      {"l_C2", cfg->l_C2},     {"s_C2", cfg->s_C2},       {"l", cfg->l},
      {"s", cfg->s},           {"N_init", cfg->N_init},   {"N_local", cfg->N_local},
      {"w", cfg->w}};
  for (const auto &p : pos) {
    if (p.v < 1) {
      set_error("positivity: %s=%d must be a positive integer", p.name, p.v);
      return SWATTN_EINVAL;
    }
  }
  if (cfg->k_top < 0) {
    set_error("positivity: k_top=%d must be >= 0", cfg->k_top);
    return SWATTN_EINVAL;
  }
  if (cfg->h_q % cfg->h_kv != 0) {  // core.py:143-146
    set_error("head-divisibility: h_q=%d is not a multiple of h_kv=%d", cfg->h_q, cfg->h_kv);
    return SWATTN_EINVAL;
  }
  if (!cfg->experimental) {  // core.py:152-168
    if (cfg->s_C1 > cfg->l_C1) {
      set_error("pooling-profile: stride s_C1=%d exceeds window l_C1=%d", cfg->s_C1, cfg->l_C1);
      return SWATTN_EINVAL;
    }
    if (cfg->s_C2 > cfg->l_C2) {
      set_error("pooling-profile: stride s_C2=%d exceeds window l_C2=%d", cfg->s_C2, cfg->l_C2);
      return SWATTN_EINVAL;
    }
    if (cfg->l_C1 % cfg->s_C1 != 0) {
      set_error("pooling-profile: s_C1=%d must divide l_C1=%d", cfg->s_C1, cfg->l_C1);
      return SWATTN_EINVAL;
    }
    if ((cfg->l - 1) % cfg->s != 0) {
      set_error("pooling-profile: s=%d must divide l-1=%d", cfg->s, cfg->l - 1);
      return SWATTN_EINVAL;
    }
  }
  const int32_t needed = (cfg->w + cfg->B - 1) / cfg->B + 1;  // core.py:170-175
  if (cfg->N_local < needed) {
    set_error("window-coverage: N_local=%d < ceil(w/B)+1=%d (w=%d, B=%d)", cfg->N_local, needed,
              cfg->w, cfg->B);
    return SWATTN_EINVAL;
  }
  return SWATTN_OK;
}

int32_t swattn_profile_supported(const swattn_config *cfg) {
  if (cfg == nullptr) return 0;
  return cfg->h_q == kG * cfg->h_kv && cfg->d_h == kD && cfg->B == kB && cfg->l == kPoolL &&
         cfg->s == kPoolS && cfg->l_C1 == 2 * cfg->s_C1 && cfg->s_C2 == 4 * cfg->s_C1 &&
         cfg->l_C2 == 2 * cfg->s_C2 && kPoolS * cfg->s_C1 == cfg->B && cfg->k_top <= kTopMax &&
         cfg->N_init + cfg->N_local <= 64;
}

int64_t swattn_num_pooled(int64_t n, int32_t length, int32_t stride) {
  return num_pooled(n, length, stride);
}

size_t swattn_sparse_workspace_bytes(const swattn_config *cfg, int64_t n) {
  if (cfg == nullptr || n < 1) return 0;
  // part A row statistics m, l [n][h_q] fp32 + slow-path list + tile routes
  return 2 * align_up((size_t)n * cfg->h_q * 4) + align_up(16) +
         align_up((size_t)cfg->h_kv * n * 4) + route_workspace_bytes(cfg->h_kv, n);
}

size_t swattn_workspace_bytes(const swattn_config *cfg, int64_t n) {
  if (cfg == nullptr || n < 1) return 0;
  const SelectLayout L = select_layout(cfg, n);
  // attend additionally keeps the top-k lists and the sparse workspace
  return align_up(L.total) + align_up((size_t)cfg->h_kv * n * cfg->k_top * 4) +
         align_up((size_t)cfg->h_kv * n * 4) + swattn_sparse_workspace_bytes(cfg, n) + 256;
}

int32_t swattn_compress_keys(const swattn_config *cfg, const void *K, int64_t n, void *kc1,
                             void *kc2, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if ((rc = check_ptr(K, "K"))) return rc;
  if (num_pooled(n, cfg->l_C1, cfg->s_C1) > 0 && (rc = check_ptr(kc1, "kc1"))) return rc;
  return launch_compress(cfg, K, n, kc1, kc2, static_cast<cudaStream_t>(stream));
}

int32_t swattn_block_scores(const swattn_config *cfg, const void *Q, const void *kc1,
                            const void *kc2, int64_t n, int32_t mode, float *s_cmp, int64_t ld,
                            uint64_t *flags, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (!swattn_profile_supported(cfg)) {
    set_error("unsupported profile for the fused block-scoring kernel (need G=16, d_h=128, B=64, "
              "l=5, s=4, l_C1=2*s_C1, s_C2=4*s_C1, l_C2=2*s_C2)");
    return SWATTN_EUNSUPPORTED;
  }
  if (mode < 0 || mode > 2) {
    set_error("unknown selection mode %d", mode);
    return SWATTN_EINVAL;
  }
  const SelectLayout L = select_layout(cfg, n);
  if (ld < L.n_cols) {
    set_error("ld=%lld is smaller than the %lld block-score columns", (long long)ld,
              (long long)L.n_cols);
    return SWATTN_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_tc_scores())
    return launch_scores_tc(cfg, Q, kc1, kc2, n, 0, n, mode, s_cmp, ld, flags, L.ld_f, st);
  return launch_scores_simt(cfg, Q, kc1, kc2, n, mode, s_cmp, ld, flags, L.ld_f, st);
}

int32_t swattn_shared_scores(const swattn_config *cfg, const void *Q, const void *kc1,
                             const void *kc2, int64_t n, int32_t mode, float *shared,
                             uint8_t *no_visible, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (cfg->d_h > 256) {
    set_error("unsupported: d_h=%d > 256 in the debug scoring path", cfg->d_h);
    return SWATTN_EUNSUPPORTED;
  }
  // lse scratch lives at the tail of the caller's shared buffer contract:
  // allocate it from the stream-ordered pool (debug path only).
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float *lse = nullptr;
  if (cudaMallocAsync(&lse, (size_t)n * cfg->h_q * sizeof(float), st) != cudaSuccess)
    return cuda_check(cudaGetLastError(), "cudaMallocAsync(lse)");
  rc = launch_shared_scores(cfg, Q, kc1, kc2, n, mode, shared, no_visible, lse, st);
  cudaFreeAsync(lse, st);
  return rc;
}

int32_t swattn_topk_blocks(const swattn_config *cfg, const float *s_cmp, int64_t ld, int64_t n,
                           int32_t *topk, int32_t *topk_cnt, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  return launch_topk(cfg, s_cmp, ld, n, 0, n, topk, topk_cnt, nullptr, nullptr, 0, nullptr, 0,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace swattn {

// Row ranges of the chunked (copy-overlapped) pipeline start on a query-block
// boundary and end on one or at n, so no 8-token tile or 64-token query block
// straddles two calls.
static int32_t check_rows(const swattn_config *cfg, int64_t n, int64_t r0, int64_t r1) {
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if (r0 < 0 || r1 > n || r0 >= r1 || r0 % cfg->B != 0 || (r1 % cfg->B != 0 && r1 != n)) {
    set_error("row range [%lld, %lld) must satisfy 0 <= r0 < r1 <= n=%lld on multiples of B=%d",
              (long long)r0, (long long)r1, (long long)n, cfg->B);
    return SWATTN_EINVAL;
  }
  return SWATTN_OK;
}

static int32_t memset_rows(void *base, int64_t n, GroupRange gr, int64_t r0, int64_t r1,
                           size_t row_bytes, int value, cudaStream_t st) {
  for (int g = gr.g0; g < gr.g0 + gr.gc; ++g) {
    char *p = static_cast<char *>(base) + ((size_t)g * n + r0) * row_bytes;
    int32_t rc = cuda_check(cudaMemsetAsync(p, value, (size_t)(r1 - r0) * row_bytes, st), "memset(rows)");
    if (rc) return rc;
  }
  return SWATTN_OK;
}

// Work forked onto a side stream once K2 is queued (attend: part A of K4,
// which then shares the SMs with the latency-bound K3 / re-rank kernels).
struct AfterScores {
  virtual int32_t run(cudaStream_t st) = 0;
};

static int32_t select_rows(const swattn_config *cfg, const void *Q, const void *K, int64_t n,
                           int64_t r0, int64_t r1, int32_t mode, int32_t *topk, int32_t *topk_cnt,
                           int32_t *n_reranked, void *workspace, size_t workspace_bytes,
                           cudaStream_t st, AfterScores *after_scores = nullptr) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if ((rc = check_rows(cfg, n, r0, r1))) return rc;
  const bool prepared = (mode & SWATTN_SELECT_PREPARED) != 0;
  mode &= ~SWATTN_SELECT_PREPARED;
  if (mode < 0 || mode > 2) {
    set_error("unknown selection mode %d", mode);
    return SWATTN_EINVAL;
  }
  const SelectLayout L = select_layout(cfg, n);
  if (workspace_bytes < L.total || workspace == nullptr) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, L.total);
    return SWATTN_EINVAL;
  }
  const bool full = r0 == 0 && r1 == n;
  char *ws = static_cast<char *>(workspace);
  void *kc1 = ws + L.off_kc1;
  void *kc2 = ws + L.off_kc2;
  float *scmp = reinterpret_cast<float *>(ws + L.off_scmp);
  uint64_t *flags = reinterpret_cast<uint64_t *>(ws + L.off_flags);
  int32_t *count = reinterpret_cast<int32_t *>(ws + L.off_count);
  int32_t *rows = reinterpret_cast<int32_t *>(ws + L.off_rows);
  // the compressed keys of the whole sequence are built by the call that
  // covers row 0 and stay in the workspace for the later row ranges
  if (r0 == 0 && !prepared && (rc = launch_compress(cfg, K, n, kc1, kc2, st))) return rc;
  if (cfg->k_top == 0 || L.n_cols <= cfg->N_init) {
    if (cfg->k_top > 0 &&
        (rc = memset_rows(topk, n, group_range(cfg), r0, r1, (size_t)cfg->k_top * 4, 0xff, st)))
      return rc;
    if ((rc = memset_rows(topk_cnt, n, group_range(cfg), r0, r1, 4, 0, st))) return rc;
    if (n_reranked) cudaMemsetAsync(n_reranked, 0, 4, st);
    return SWATTN_OK;
  }
  if (L.generic || !use_tc_scores()) {
    if (!full || group_range(cfg).gc != cfg->h_kv) {
      set_error("row ranges and group ranges need the paper profile on the tensor-core path");
      return SWATTN_EUNSUPPORTED;
    }
  }
  if (L.generic) {
    // any-profile path: full S^shared, max-pool, top-k (no float64 boundary pass)
    float *shared = reinterpret_cast<float *>(ws + L.off_shared);
    float *lse = reinterpret_cast<float *>(ws + L.off_lse);
    if ((rc = launch_shared_scores(cfg, Q, kc1, kc2, n, mode, shared, nullptr, lse, st))) return rc;
    if ((rc = launch_maxpool(cfg, shared, n, scmp, L.ld, st))) return rc;
    rc = launch_topk(cfg, scmp, L.ld, n, 0, n, topk, topk_cnt, nullptr, nullptr, 0, nullptr, 0, st);
    if (n_reranked) cudaMemsetAsync(n_reranked, 0, 4, st);
    return rc;
  }
  const int32_t cap = (int32_t)((int64_t)cfg->h_kv * n);
  // Row f1 (opt-in, SWATTN_K2_TOPK=1): the top-k selected in K2's pass-2
  // epilogue (scores_tc.cu); K3 then only fills rows without candidates and
  // re-selects rows whose candidate set overflowed.  Bit-identical selections,
  // but K2 is co-bound by issue slots and MUFU and its 8 epilogue warps meet
  // at a barrier every tile, so the per-token candidate maintenance costs more
  // than the separate 1.1 ms K3 (128K select 14.0 vs 10.4 ms,
  // profiles/r02ae_fused_topk.txt): off by default.
  const char *fuse_e = getenv("SWATTN_K2_TOPK");
  const bool fuse_env = fuse_e != nullptr && strcmp(fuse_e, "1") == 0;
  const bool fused = fuse_env && use_tc_scores() && cfg->k_top > 0 && cfg->k_top <= 64 &&
                     L.n_cols - cfg->N_init <= kTopkMaxCand;
  if (fused) {
    int32_t *ovf_rows = reinterpret_cast<int32_t *>(ws + L.off_ovf);
    if ((rc = cuda_check(cudaMemsetAsync(count, 0, 8, st), "memset(count)"))) return rc;
    const FusedTopk fz{topk, topk_cnt, count, rows, cap, count + 1, ovf_rows};
    if ((rc = launch_scores_tc(cfg, Q, kc1, kc2, n, r0, r1, mode, scmp, L.ld, flags, L.ld_f, st, &fz)))
      return rc;
    if (after_scores != nullptr && (rc = after_scores->run(st))) return rc;
    if ((rc = launch_topk_tail(cfg, scmp, L.ld, n, r0, r1, topk, topk_cnt, count, rows, cap, flags,
                               L.ld_f, count + 1, ovf_rows, st)))
      return rc;
  } else {
    if (use_tc_scores())
      rc = launch_scores_tc(cfg, Q, kc1, kc2, n, r0, r1, mode, scmp, L.ld, flags, L.ld_f, st);
    else
      rc = launch_scores_simt(cfg, Q, kc1, kc2, n, mode, scmp, L.ld, flags, L.ld_f, st);
    if (rc) return rc;
    if (after_scores != nullptr && (rc = after_scores->run(st))) return rc;
    if ((rc = cuda_check(cudaMemsetAsync(count, 0, 4, st), "memset(count)"))) return rc;
    if ((rc = launch_topk(cfg, scmp, L.ld, n, r0, r1, topk, topk_cnt, count, rows, cap, flags,
                          L.ld_f, st)))
      return rc;
  }
  if ((rc = launch_rerank(cfg, Q, kc1, kc2, n, mode, scmp, L.ld, count, rows, cap, topk,
                          ws + L.off_part, num_sms(), st)))
    return rc;
  if (n_reranked)
    return cuda_check(cudaMemcpyAsync(n_reranked, count, 4, cudaMemcpyDeviceToDevice, st),
                      "copy(n_reranked)");
  return SWATTN_OK;
}

// Part A of K4 (init + local blocks, shared by a query block's 64 tokens)
// needs no selection, so attend forks it onto a side stream once K2 is
// queued: it fills the SMs the latency-bound K3 / re-rank kernels leave idle
// and joins before part B.  (Forking before K2 gained nothing: K2 is MUFU-
// bound and so is the FA tile's softmax.)  The side stream and events are
// per host thread and device (created once).
struct SideStream {
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

static int32_t side_stream(SideStream *&out) {
  thread_local std::vector<SideStream> ss;  // one per device, created on first use
  int dev = 0;
  int32_t rc = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  if ((size_t)dev >= ss.size()) ss.resize((size_t)dev + 1);
  SideStream &x = ss[(size_t)dev];
  if (x.device != dev) {
    if ((rc = cuda_check(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking), "side stream")) ||
        (rc = cuda_check(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming), "side event")) ||
        (rc = cuda_check(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming), "side event")))
      return rc;
    x.device = dev;
  }
  out = &x;
  return SWATTN_OK;
}

static int32_t sparse_ws_ptrs(const swattn_config *cfg, int64_t n, void *workspace, float *&m_a,
                              float *&l_a, int32_t *&slow_count, int32_t *&slow_list) {
  char *ws = static_cast<char *>(workspace);
  m_a = reinterpret_cast<float *>(ws);
  l_a = reinterpret_cast<float *>(ws + align_up((size_t)n * cfg->h_q * 4));
  slow_count = reinterpret_cast<int32_t *>(ws + 2 * align_up((size_t)n * cfg->h_q * 4));
  slow_list = reinterpret_cast<int32_t *>(ws + 2 * align_up((size_t)n * cfg->h_q * 4) + align_up(16));
  return SWATTN_OK;
}

static bool overlap_ok(const swattn_config *cfg) {
  return use_tc_attention() && swattn_profile_supported(cfg) && cfg->h_q == kG * cfg->h_kv &&
         cfg->d_h == kD;
}

// fork part A of rows [r0, r1) onto the side stream (after everything queued on st)
static int32_t part_a_fork(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                           int64_t n, int64_t r0, int64_t r1, void *O, float *lse, void *sparse_ws,
                           cudaStream_t st, SideStream *&side) {
  int32_t rc = side_stream(side);
  if (rc) return rc;
  float *m_a, *l_a;
  int32_t *slow_count, *slow_list;
  sparse_ws_ptrs(cfg, n, sparse_ws, m_a, l_a, slow_count, slow_list);
  if ((rc = cuda_check(cudaEventRecord(side->fork, st), "event record")) ||
      (rc = cuda_check(cudaStreamWaitEvent(side->stream, side->fork, 0), "stream wait")))
    return rc;
  if ((rc = launch_sparse_part_a(cfg, Q, K, V, n, r0, r1, O, lse, m_a, l_a, side->stream))) return rc;
  return cuda_check(cudaEventRecord(side->join, side->stream), "event record");
}

static int32_t sparse_rows_impl(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                                int64_t n, int64_t r0, int64_t r1, const int32_t *topk,
                                const int32_t *topk_cnt, void *O, float *lse, void *workspace,
                                size_t workspace_bytes, cudaStream_t st, bool part_a_done);

static int32_t sparse_rows(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                           int64_t n, int64_t r0, int64_t r1, const int32_t *topk,
                           const int32_t *topk_cnt, void *O, float *lse, void *workspace,
                           size_t workspace_bytes, cudaStream_t st) {
  return sparse_rows_impl(cfg, Q, K, V, n, r0, r1, topk, topk_cnt, O, lse, workspace,
                          workspace_bytes, st, false);
}

static int32_t sparse_rows_impl(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                                int64_t n, int64_t r0, int64_t r1, const int32_t *topk,
                                const int32_t *topk_cnt, void *O, float *lse, void *workspace,
                                size_t workspace_bytes, cudaStream_t st, bool part_a_done) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if ((rc = check_rows(cfg, n, r0, r1))) return rc;
  if (cfg->h_q != kG * cfg->h_kv || cfg->d_h != kD) {
    set_error("unsupported profile for the attention kernels (need G=16, d_h=128)");
    return SWATTN_EUNSUPPORTED;
  }
  if (use_tc_attention() && swattn_profile_supported(cfg)) {
    const size_t need = swattn_sparse_workspace_bytes(cfg, n);
    if (workspace == nullptr || workspace_bytes < need) {
      set_error("workspace too small: %zu < %zu bytes", workspace_bytes, need);
      return SWATTN_EINVAL;
    }
    char *ws = static_cast<char *>(workspace);
    float *m_a = reinterpret_cast<float *>(ws);
    float *l_a = reinterpret_cast<float *>(ws + align_up((size_t)n * cfg->h_q * 4));
    int32_t *slow_count = reinterpret_cast<int32_t *>(ws + 2 * align_up((size_t)n * cfg->h_q * 4));
    int32_t *slow_list = reinterpret_cast<int32_t *>(ws + 2 * align_up((size_t)n * cfg->h_q * 4) +
                                                     align_up(16));
    if (!part_a_done && (rc = launch_sparse_part_a(cfg, Q, K, V, n, r0, r1, O, lse, m_a, l_a, st)))
      return rc;
    const TileRoutes routes = carve_routes(
        ws + 2 * align_up((size_t)n * cfg->h_q * 4) + align_up(16) + align_up((size_t)cfg->h_kv * n * 4),
        cfg->h_kv, n);
    // Routed tiles (route.cuh) run on the SMs part B leaves them, launched
    // programmatically right behind it; the plan splits the SMs by work.
    const int pct = route_pct(n);
    if (pct > 0) {
      if ((rc = launch_route_tiles(cfg, n, r0, r1, topk, topk_cnt, routes, pct, st))) return rc;
      if ((rc = launch_route_plan(routes, n, num_sms(), part_b_ctas(), st))) return rc;
    }
    if ((rc = cuda_check(cudaMemsetAsync(slow_count, 0, 4, st), "memset(slow)"))) return rc;
    rc = launch_sparse_part_b(cfg, Q, K, V, n, r0, r1, topk, topk_cnt, m_a, l_a, O, lse,
                              slow_count, slow_list, part_b_ctas(), st,
                              pct > 0 ? routes.routed : nullptr, pct > 0 ? routes.plan : nullptr);
    if (rc) return rc;
    if (pct > 0 && (rc = launch_routed_tiles(cfg, Q, K, V, n, O, lse, m_a, l_a, routes, st)))
      return rc;
    return launch_attention_list(cfg, Q, K, V, n, topk, topk_cnt, slow_count, slow_list, O, lse,
                                 num_sms(), st);
  }
  if (r0 != 0 || r1 != n || group_range(cfg).gc != cfg->h_kv) {
    set_error("row ranges and group ranges need the paper profile on the tensor-core path");
    return SWATTN_EUNSUPPORTED;
  }
  return launch_attention_simt(cfg, Q, K, V, n, topk, topk_cnt, 1, 1, O, lse, nullptr, st);
}

// select rows [r0, r1) on st, with part A of the same rows running
// concurrently on the side stream, then part B on st.
static int32_t select_and_sparse(const swattn_config *cfg, const void *Q, const void *K,
                                 const void *V, int64_t n, int64_t r0, int64_t r1, int32_t select_mode,
                                 int32_t *topk, int32_t *cnt, void *O, float *lse, void *sel_ws,
                                 size_t sel_bytes, void *sparse_ws, size_t sparse_bytes,
                                 cudaStream_t st) {
  int32_t rc = check_rows(cfg, n, r0, r1);
  if (rc) return rc;
  const bool overlap = overlap_ok(cfg) && sparse_ws != nullptr &&
                       sparse_bytes >= swattn_sparse_workspace_bytes(cfg, n);
  struct ForkPartA : AfterScores {
    const swattn_config *cfg;
    const void *Q, *K, *V;
    int64_t n, r0, r1;
    void *O;
    float *lse;
    void *sparse_ws;
    SideStream *side = nullptr;
    int32_t run(cudaStream_t s) override {
      return part_a_fork(cfg, Q, K, V, n, r0, r1, O, lse, sparse_ws, s, side);
    }
  } fork;
  fork.cfg = cfg; fork.Q = Q; fork.K = K; fork.V = V; fork.n = n; fork.r0 = r0; fork.r1 = r1;
  fork.O = O; fork.lse = lse; fork.sparse_ws = sparse_ws;
  rc = select_rows(cfg, Q, K, n, r0, r1, select_mode, topk, cnt, nullptr, sel_ws, sel_bytes, st,
                   overlap ? &fork : nullptr);
  const bool forked = fork.side != nullptr;
  if (forked) {
    // join even on failure so the side stream never outlives the call's buffers
    const int32_t rj = cuda_check(cudaStreamWaitEvent(st, fork.side->join, 0), "stream wait");
    if (!rc) rc = rj;
  }
  if (rc) return rc;
  return sparse_rows_impl(cfg, Q, K, V, n, r0, r1, topk, cnt, O, lse, sparse_ws, sparse_bytes, st,
                          forked);
}

}  // namespace swattn

extern "C" {

int32_t swattn_select_blocks(const swattn_config *cfg, const void *Q, const void *K, int64_t n,
                             int32_t mode, int32_t *topk, int32_t *topk_cnt, int32_t *n_reranked,
                             void *workspace, size_t workspace_bytes, void *stream) {
  return select_rows(cfg, Q, K, n, 0, n, mode, topk, topk_cnt, n_reranked, workspace,
                     workspace_bytes, static_cast<cudaStream_t>(stream));
}

int32_t swattn_select_blocks_rows(const swattn_config *cfg, const void *Q, const void *K, int64_t n,
                                  int64_t r0, int64_t r1, int32_t mode, int32_t *topk,
                                  int32_t *topk_cnt, int32_t *n_reranked, void *workspace,
                                  size_t workspace_bytes, void *stream) {
  return select_rows(cfg, Q, K, n, r0, r1, mode, topk, topk_cnt, n_reranked, workspace,
                     workspace_bytes, static_cast<cudaStream_t>(stream));
}

int32_t swattn_sparse_fwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, const int32_t *topk, const int32_t *topk_cnt, void *O,
                          float *lse, void *workspace, size_t workspace_bytes, void *stream) {
  return sparse_rows(cfg, Q, K, V, n, 0, n, topk, topk_cnt, O, lse, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

int32_t swattn_sparse_fwd_lists(const swattn_config *cfg, const void *Q, const void *K,
                                const void *V, int64_t n, const int32_t *blocks, int64_t ld,
                                const int32_t *cnt, void *O, float *lse, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if (cfg->h_q != kG * cfg->h_kv || cfg->d_h != kD) {
    set_error("unsupported profile for the attention kernels (need G=16, d_h=128)");
    return SWATTN_EUNSUPPORTED;
  }
  if (ld < 1 || (rc = check_ptr(blocks, "blocks")) || (rc = check_ptr(cnt, "cnt")) ||
      (rc = check_ptr(Q, "Q")) || (rc = check_ptr(K, "K")) || (rc = check_ptr(V, "V")) ||
      (rc = check_ptr(O, "O")) || (rc = check_ptr(lse, "lse"))) {
    if (!rc) {
      set_error("ld=%lld must be >= 1", (long long)ld);
      rc = SWATTN_EINVAL;
    }
    return rc;
  }
  return launch_sparse_list(cfg, Q, K, V, n, blocks, ld, cnt, O, lse, num_sms(),
                            static_cast<cudaStream_t>(stream));
}

int32_t swattn_sparse_fwd_rows(const swattn_config *cfg, const void *Q, const void *K,
                               const void *V, int64_t n, int64_t r0, int64_t r1,
                               const int32_t *topk, const int32_t *topk_cnt, void *O, float *lse,
                               void *workspace, size_t workspace_bytes, void *stream) {
  return sparse_rows(cfg, Q, K, V, n, r0, r1, topk, topk_cnt, O, lse, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

size_t swattn_sparse_bwd_workspace_bytes(const swattn_config *cfg, int64_t n) {
  if (cfg == nullptr || n < 1 || !swattn_profile_supported(cfg)) return 0;
  return sparse_bwd_workspace_bytes(cfg, n, 0);
}

size_t swattn_dense_bwd_workspace_bytes(const swattn_config *cfg, int64_t n, int32_t causal) {
  if (cfg == nullptr || n < 1 || !swattn_profile_supported(cfg)) return 0;
  return sparse_bwd_workspace_bytes(cfg, n, causal ? 1 : 2);
}

int32_t swattn_dense_bwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int32_t causal, const void *O, const float *lse, const void *dO,
                         void *dQ, void *dK, void *dV, void *workspace, size_t workspace_bytes,
                         void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if (!swattn_profile_supported(cfg) || !use_tc_attention()) {
    set_error("unsupported profile for the backward kernels (need the paper profile)");
    return SWATTN_EUNSUPPORTED;
  }
  return launch_sparse_bwd(cfg, Q, K, V, n, nullptr, nullptr, O, lse, dO, dQ, dK, dV, workspace,
                           workspace_bytes, num_sms(), causal ? 1 : 2,
                           static_cast<cudaStream_t>(stream));
}

int32_t swattn_sparse_bwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                          int64_t n, const int32_t *topk, const int32_t *topk_cnt, const void *O,
                          const float *lse, const void *dO, void *dQ, void *dK, void *dV,
                          void *workspace, size_t workspace_bytes, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if (!swattn_profile_supported(cfg) || !use_tc_attention()) {
    set_error("unsupported profile for the backward kernels (need the paper profile)");
    return SWATTN_EUNSUPPORTED;
  }
  if (n >= ((int64_t)1 << 32)) {
    set_error("n=%lld too large for the backward pair keys", (long long)n);
    return SWATTN_EUNSUPPORTED;
  }
  return launch_sparse_bwd(cfg, Q, K, V, n, topk, topk_cnt, O, lse, dO, dQ, dK, dV, workspace,
                           workspace_bytes, num_sms(), 0, static_cast<cudaStream_t>(stream));
}

int32_t swattn_dense_fwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int32_t causal, void *O, float *lse, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  if (cfg->h_q != kG * cfg->h_kv || cfg->d_h != kD) {
    set_error("unsupported profile for the attention kernels (need G=16, d_h=128)");
    return SWATTN_EUNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (use_tc_attention())
    return launch_dense_tc(cfg, Q, K, V, n, causal, O, lse, st);
  if (group_range(cfg).gc != cfg->h_kv) {
    set_error("group ranges need the tensor-core attention kernels");
    return SWATTN_EUNSUPPORTED;
  }
  return launch_attention_simt(cfg, Q, K, V, n, nullptr, nullptr, 0, causal, O, lse, nullptr, st);
}

int32_t swattn_attend(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                      int64_t n, int64_t threshold, int32_t forced_mode, int32_t select_mode,
                      void *O, float *lse, int32_t *mode_taken, void *workspace,
                      size_t workspace_bytes, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (forced_mode < 0 || forced_mode > 2) {
    set_error("unknown forced mode %d", forced_mode);
    return SWATTN_EINVAL;
  }
  // switch.py:63-69
  const int64_t thr =
      threshold >= 0 ? threshold : (int64_t)(cfg->N_init + cfg->N_local + cfg->k_top) * cfg->B;
  const bool dense = forced_mode == SWATTN_FORCE_DENSE || (forced_mode == SWATTN_AUTO && n <= thr);
  if (mode_taken) *mode_taken = dense ? 1 : 2;
  if (dense) return swattn_dense_fwd(cfg, Q, K, V, n, 1, O, lse, stream);
  const SelectLayout L = select_layout(cfg, n);
  const size_t need = swattn_workspace_bytes(cfg, n);
  if (workspace == nullptr || workspace_bytes < need) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, need);
    return SWATTN_EINVAL;
  }
  char *ws = static_cast<char *>(workspace);
  int32_t *topk = reinterpret_cast<int32_t *>(ws + align_up(L.total));
  int32_t *cnt = reinterpret_cast<int32_t *>(ws + align_up(L.total) +
                                             align_up((size_t)cfg->h_kv * n * cfg->k_top * 4));
  char *sws = ws + align_up(L.total) + align_up((size_t)cfg->h_kv * n * cfg->k_top * 4) +
              align_up((size_t)cfg->h_kv * n * 4);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return select_and_sparse(cfg, Q, K, V, n, 0, n, select_mode, topk, cnt, O, lse, workspace, L.total,
                           sws, swattn_sparse_workspace_bytes(cfg, n), st);
}

int32_t swattn_attend_prepare(const swattn_config *cfg, const void *K, int64_t n, void *workspace,
                              size_t workspace_bytes, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1) {
    set_error("empty sequence: n must be >= 1");
    return SWATTN_EINVAL;
  }
  const SelectLayout L = select_layout(cfg, n);
  if (workspace == nullptr || workspace_bytes < swattn_workspace_bytes(cfg, n)) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, swattn_workspace_bytes(cfg, n));
    return SWATTN_EINVAL;
  }
  char *ws = static_cast<char *>(workspace);
  return launch_compress(cfg, K, n, ws + L.off_kc1, ws + L.off_kc2, static_cast<cudaStream_t>(stream));
}

int32_t swattn_workspace_ckeys(const swattn_config *cfg, int64_t n, void *workspace, void **kc1,
                               void **kc2) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  if (n < 1 || workspace == nullptr || kc1 == nullptr || kc2 == nullptr) {
    set_error("swattn_workspace_ckeys: need n >= 1 and non-NULL pointers");
    return SWATTN_EINVAL;
  }
  const SelectLayout L = select_layout(cfg, n);
  *kc1 = static_cast<char *>(workspace) + L.off_kc1;
  *kc2 = static_cast<char *>(workspace) + L.off_kc2;
  return SWATTN_OK;
}

int32_t swattn_attend_rows(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                           int64_t n, int64_t r0, int64_t r1, int32_t select_mode, void *O,
                           float *lse, void *workspace, size_t workspace_bytes, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc) return rc;
  const SelectLayout L = select_layout(cfg, n);
  const size_t need = swattn_workspace_bytes(cfg, n);
  if (workspace == nullptr || workspace_bytes < need) {
    set_error("workspace too small: %zu < %zu bytes", workspace_bytes, need);
    return SWATTN_EINVAL;
  }
  char *ws = static_cast<char *>(workspace);
  int32_t *topk = reinterpret_cast<int32_t *>(ws + align_up(L.total));
  int32_t *cnt = reinterpret_cast<int32_t *>(ws + align_up(L.total) +
                                             align_up((size_t)cfg->h_kv * n * cfg->k_top * 4));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char *sws = ws + align_up(L.total) + align_up((size_t)cfg->h_kv * n * cfg->k_top * 4) +
              align_up((size_t)cfg->h_kv * n * 4);
  return select_and_sparse(cfg, Q, K, V, n, r0, r1, select_mode, topk, cnt, O, lse, workspace,
                           L.total, sws, swattn_sparse_workspace_bytes(cfg, n), st);
}

static int32_t check_groups(const swattn_config *cfg, int32_t g0, int32_t g1) {
  if (g0 < 0 || g1 > cfg->h_kv || g0 >= g1) {
    set_error("group range [%d, %d) must satisfy 0 <= g0 < g1 <= h_kv=%d", g0, g1, cfg->h_kv);
    return SWATTN_EINVAL;
  }
  return SWATTN_OK;
}

int32_t swattn_attend_groups(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                             int64_t n, int32_t g0, int32_t g1, int64_t threshold,
                             int32_t forced_mode, int32_t select_mode, void *O, float *lse,
                             int32_t *mode_taken, void *workspace, size_t workspace_bytes,
                             void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc || (rc = check_groups(cfg, g0, g1))) return rc;
  GroupScope scope(g0, g1);
  return swattn_attend(cfg, Q, K, V, n, threshold, forced_mode, select_mode, O, lse, mode_taken,
                       workspace, workspace_bytes, stream);
}

int32_t swattn_attend_rows_groups(const swattn_config *cfg, const void *Q, const void *K,
                                  const void *V, int64_t n, int64_t r0, int64_t r1, int32_t g0,
                                  int32_t g1, int32_t select_mode, void *O, float *lse,
                                  void *workspace, size_t workspace_bytes, void *stream) {
  int32_t rc = swattn_validate_config(cfg);
  if (rc || (rc = check_groups(cfg, g0, g1))) return rc;
  GroupScope scope(g0, g1);
  return swattn_attend_rows(cfg, Q, K, V, n, r0, r1, select_mode, O, lse, workspace,
                            workspace_bytes, stream);
}

}  // extern "C"
