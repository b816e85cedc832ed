/*
 * swattn_b200 -- C ABI of the B200-native (sm_100a) InfLLM-V2 switchable
 * attention hot path.  Plain pointers, sizes and an opaque stream handle:
 * no torch / CUDA types in any signature.
 *
 * The reference (`swattn` 0.1.0, /root/reference/pkg/src/swattn) is a pure
 * numpy library with no FFI; each entry point below names the reference
 * function whose semantics it implements (file:line), and INTEGRATION.md
 * shows the ctypes binding a maintainer would add on the reference side.
 *
 * Conventions (all entry points):
 *  - tensors are device pointers, C-contiguous, token axis outermost:
 *      Q [n, h_q, d_h], K/V [n, h_kv, d_h], bf16 (core.py:6-7)
 *    query head h reads KV head h / (h_q/h_kv) (dense.py:11-13);
 *  - outputs and the workspace are allocated by the caller; the library
 *    allocates no device memory and keeps no global state except the
 *    thread-local error message and, per host thread and device, one side
 *    stream with two events (swattn_attend / swattn_attend_rows run K4 part A
 *    on it beside the selection kernels, joined back into `stream` before
 *    the call's last kernel);
 *  - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default stream); no implicit device synchronisation (exception: the
 *    backward entry points read the data-dependent pair count back once);
 *  - return value: SWATTN_OK or an error code; swattn_last_error() holds the
 *    message (same invariant-prefixed wording as the reference's ConfigError
 *    / ValueError / RuntimeError, core.py:118-175, dense.py:36-56).
 *  - results are bitwise deterministic run to run.
 */
#ifndef SWATTN_B200_H
#define SWATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* AttentionConfig (core.py:48-108), field for field. */
typedef struct swattn_config {
  int32_t h_q, h_kv, d_h, B;
  int32_t l_C1, s_C1, l_C2, s_C2;
  int32_t l, s;
  int32_t N_init, N_local, k_top, w;
  int32_t scale_compressed_logits; /* core.py:96 */
  int32_t experimental;            /* core.py:97 */
} swattn_config;

enum swattn_status {
  SWATTN_OK = 0,
  SWATTN_EINVAL = 1,       /* ValueError / ConfigError in the reference     */
  SWATTN_EUNSUPPORTED = 2, /* valid config, but not the compiled profile    */
  SWATTN_ECUDA = 3,        /* CUDA launch / runtime failure                 */
  SWATTN_EEMPTY = 4        /* RuntimeError: empty visible set (sparse.py:75) */
};

/* select_blocks modes (selection.py:351) */
enum swattn_select_mode {
  SWATTN_SELECT_EXACT = 0,
  SWATTN_SELECT_FUSED_EXACT = 1,
  SWATTN_SELECT_APPROX = 2
};
/* OR'ed into a select mode of the row-range entry points: the compressed keys
 * of the whole sequence are already in the workspace (written through
 * swattn_workspace_ckeys, e.g. after an all-gather of per-rank shards), so
 * K1 is never run, not even for a range starting at row 0. */
#define SWATTN_SELECT_PREPARED 0x100

/* attend forced modes (switch.py:27-34) */
enum swattn_forced_mode { SWATTN_AUTO = 0, SWATTN_FORCE_DENSE = 1, SWATTN_FORCE_SPARSE = 2 };

/* Message of the last failing call on this thread ("" if none). */
const char *swattn_last_error(void);
int32_t swattn_version(void);

/* validate_config (core.py:111-176): 0 if every invariant holds. */
int32_t swattn_validate_config(const swattn_config *cfg);

/* 1 if the hot-path kernels are compiled for this profile (G=16, d_h=128,
 * B=64, l=5, s=4, l_C1=2 s_C1, s_C2=4 s_C1, l_C2=2 s_C2, 4 s_C1 = B). */
int32_t swattn_profile_supported(const swattn_config *cfg);

/* Compressed-key counts m = floor((n-l)/s)+1 (compression.py:64-78). */
int64_t swattn_num_pooled(int64_t n, int32_t length, int32_t stride);

/* Workspace bytes needed by swattn_select_blocks / swattn_attend for n
 * tokens (pooled keys, S^cmp candidate region, tie-resolution lists). */
size_t swattn_workspace_bytes(const swattn_config *cfg, int64_t n);

/* K1 -- mean_pool_keys (compression.py:64-86) for both pooling profiles in
 * one HBM pass: kc1 [m1, h_kv, d_h], kc2 [m2, h_kv, d_h] bf16 (kc2 may be
 * NULL).  Windows are summed exactly (float64) and rounded like the
 * reference's cast back to storage dtype. */
int32_t swattn_compress_keys(const swattn_config *cfg, const void *K, int64_t n,
                             void *kc1, void *kc2, void *stream);

/* K2 -- fused two-pass block scoring + max-pool (selection.py:238-348,
 * compression.py:160-173) restricted to the top-k candidate region of every
 * row: s_cmp [h_kv, n, ld] fp32, entry (g, i, j) for candidate blocks
 * N_init <= j < min(i/B - N_local + 1, n_cols).  mode: APPROX (pass 1 over
 * C2) or FUSED_EXACT/EXACT (pass 1 over C1).  flags [h_kv, n, ld/31+1]
 * uint64 (may be NULL): per-block argmax-at-shared-column bits used for exact
 * tie classification. */
int32_t swattn_block_scores(const swattn_config *cfg, const void *Q, const void *kc1,
                            const void *kc2, int64_t n, int32_t mode, float *s_cmp,
                            int64_t ld, uint64_t *flags, void *stream);

/* Debug / parity path: full S^shared [n, h_kv, m1] fp32 (selection.py:238-348
 * incl. fallback rows) and no_visible [n] uint8.  Any profile; small n. */
int32_t swattn_shared_scores(const swattn_config *cfg, const void *Q, const void *kc1,
                             const void *kc2, int64_t n, int32_t mode, float *shared,
                             uint8_t *no_visible, void *stream);

/* K3 -- build_block_sets top-k part (selection.py:93-136): topk [h_kv, n,
 * k_top] int32 ascending, -1 padded; topk_cnt [h_kv, n] int32.  Ranking is
 * score descending, ties to the lower block index (stable argsort, :125). */
int32_t swattn_topk_blocks(const swattn_config *cfg, const float *s_cmp, int64_t ld,
                           int64_t n, int32_t *topk, int32_t *topk_cnt, void *stream);

/* K1 -> K2 -> K3 (+ float64 re-rank of near-tied rows) on one stream:
 * select_blocks(Q, K, cfg, mode) (selection.py:354-383).  Outputs as
 * swattn_topk_blocks.  n_reranked (device int32, may be NULL) receives the
 * number of rows whose boundary was resolved in float64. */
int32_t swattn_select_blocks(const swattn_config *cfg, const void *Q, const void *K,
                             int64_t n, int32_t mode, int32_t *topk, int32_t *topk_cnt,
                             int32_t *n_reranked, void *workspace, size_t workspace_bytes,
                             void *stream);

/* K4 -- sparse_forward (sparse.py:43-98): O [n, h_q, d_h] bf16, lse [n, h_q]
 * fp32 (natural log).  Visible set of row i per group = init U local U
 * topk[g, i] clipped causally (selection.py:73-87).  Part A (init + local,
 * shared per query block) and part B (per-token top-k) run as two tcgen05
 * kernels; the workspace holds part A's row statistics. */
int32_t swattn_sparse_fwd(const swattn_config *cfg, const void *Q, const void *K,
                          const void *V, int64_t n, const int32_t *topk,
                          const int32_t *topk_cnt, void *O, float *lse, void *workspace,
                          size_t workspace_bytes, void *stream);
size_t swattn_sparse_workspace_bytes(const swattn_config *cfg, int64_t n);

/* K4, general form -- sparse_forward (sparse.py:43-98) over an ARBITRARY
 * BlockSelection (selection.py:51-66: any sorted block ids per (group, row),
 * e.g. load_selection(path) fixtures, selection.py:403-430, or every causal
 * block, bench.py:207-210).  blocks [h_kv, n, ld] int32, row (g, i) lists
 * cnt[g, i] block ids in visiting order (ascending in a BlockSelection);
 * negative ids are ignored.  Block j covers keys [j B, min(j B + B, n, i + 1))
 * (selection.py:73-87).  A row with no visible key gets O = 0, lse = -inf
 * (the reference raises RuntimeError, sparse.py:75-76: callers check first).
 * Needs G = 16, d_h = 128; any B. */
int32_t swattn_sparse_fwd_lists(const swattn_config *cfg, const void *Q, const void *K,
                                const void *V, int64_t n, const int32_t *blocks, int64_t ld,
                                const int32_t *cnt, void *O, float *lse, void *stream);

/* K5 -- tiled_gqa_forward (dense.py:112-170): causal (or full) GQA flash
 * attention, O bf16, lse fp32. */
int32_t swattn_dense_fwd(const swattn_config *cfg, const void *Q, const void *K,
                         const void *V, int64_t n, int32_t causal, void *O, float *lse,
                         void *stream);

/* attend (switch.py:42-82): threshold < 0 -> cfg default
 * (N_init+N_local+k_top)*B; n <= threshold -> dense.  *mode_taken = 1 dense,
 * 2 sparse (host value, set before any kernel runs). */
int32_t swattn_attend(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                      int64_t n, int64_t threshold, int32_t forced_mode, int32_t select_mode,
                      void *O, float *lse, int32_t *mode_taken, void *workspace,
                      size_t workspace_bytes, void *stream);

/* sparse_backward (sparse.py:130-185): dQ [n,h_q,d_h], dK / dV [n,h_kv,d_h]
 * bf16 of sum(O * dO) through the masked softmax over each row's init U local
 * U top-k blocks, given the forward's O (bf16) and lse (fp32, natural log) --
 * e.g. from swattn_sparse_fwd -- and dO (bf16).  Deterministic: every
 * reduction has a fixed order.  One host synchronisation (the data-dependent
 * pair count).  Paper profile only (SWATTN_EUNSUPPORTED otherwise). */
int32_t swattn_sparse_bwd(const swattn_config *cfg, const void *Q, const void *K,
                          const void *V, int64_t n, const int32_t *topk,
                          const int32_t *topk_cnt, const void *O, const float *lse,
                          const void *dO, void *dQ, void *dK, void *dV, void *workspace,
                          size_t workspace_bytes, void *stream);
size_t swattn_sparse_bwd_workspace_bytes(const swattn_config *cfg, int64_t n);
/* naive_gqa_backward (dense.py:173-221): the same kernels with every causal
 * block (causal = 1) or every block (causal = 0) visible; O / lse from
 * swattn_dense_fwd with the same causal flag. */
int32_t swattn_dense_bwd(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                         int64_t n, int32_t causal, const void *O, const float *lse,
                         const void *dO, void *dQ, void *dK, void *dV, void *workspace,
                         size_t workspace_bytes, void *stream);
size_t swattn_dense_bwd_workspace_bytes(const swattn_config *cfg, int64_t n, int32_t causal);

/* ---- row ranges (copy-overlapped chunked prefill) ----
 * The same computations restricted to query rows [r0, r1) of an n-token
 * sequence: r0 and r1 are multiples of B (r1 may equal n).  Rows only read
 * their own Q rows and K/V rows < r1, so a caller can stream Q in chunks
 * and overlap host<->device copies with compute.  The call covering r0 == 0
 * also builds the compressed keys of all n tokens into the workspace (K must
 * be complete then); later ranges of the same sequence reuse them.  No
 * reference counterpart: the reference processes whole arrays
 * (selection.py:354-383, sparse.py:43-98); outputs are identical to the
 * whole-sequence calls row for row. */
int32_t swattn_select_blocks_rows(const swattn_config *cfg, const void *Q, const void *K,
                                  int64_t n, int64_t r0, int64_t r1, int32_t mode,
                                  int32_t *topk, int32_t *topk_cnt, int32_t *n_reranked,
                                  void *workspace, size_t workspace_bytes, void *stream);
int32_t swattn_sparse_fwd_rows(const swattn_config *cfg, const void *Q, const void *K,
                               const void *V, int64_t n, int64_t r0, int64_t r1,
                               const int32_t *topk, const int32_t *topk_cnt, void *O,
                               float *lse, void *workspace, size_t workspace_bytes,
                               void *stream);
/* Build the compressed keys of all n tokens into an attend workspace, for a
 * caller whose first row range does not start at 0 (context parallelism:
 * each rank computes its own rows of one sequence). */
int32_t swattn_attend_prepare(const swattn_config *cfg, const void *K, int64_t n,
                              void *workspace, size_t workspace_bytes, void *stream);
/* Device pointers of the compressed-key slots K_C1 [m1, h_kv, d_h] and
 * K_C2 [m2, h_kv, d_h] (bf16) inside an attend workspace for n tokens. */
int32_t swattn_workspace_ckeys(const swattn_config *cfg, int64_t n, void *workspace,
                               void **kc1, void **kc2);
/* sparse branch of attend over rows [r0, r1) (workspace as swattn_attend) */
int32_t swattn_attend_rows(const swattn_config *cfg, const void *Q, const void *K,
                           const void *V, int64_t n, int64_t r0, int64_t r1,
                           int32_t select_mode, void *O, float *lse, void *workspace,
                           size_t workspace_bytes, void *stream);

/* ---- batch x KV-group sharding ----
 * The same calls restricted to KV groups [g0, g1): query heads
 * [g0 G, g1 G) and K/V heads [g0, g1) of the full tensors (G = h_q / h_kv);
 * only those heads' O / lse rows are written.  Groups are independent end to
 * end (selection.py:111-135, sparse.py:70-91), so rank r of a group-sharded
 * job calls these with its own groups and needs no collective.  The
 * workspace is sized as for the full call (swattn_workspace_bytes). */
int32_t swattn_attend_groups(const swattn_config *cfg, const void *Q, const void *K, const void *V,
                             int64_t n, int32_t g0, int32_t g1, int64_t threshold,
                             int32_t forced_mode, int32_t select_mode, void *O, float *lse,
                             int32_t *mode_taken, void *workspace, size_t workspace_bytes,
                             void *stream);
int32_t swattn_attend_rows_groups(const swattn_config *cfg, const void *Q, const void *K,
                                  const void *V, int64_t n, int64_t r0, int64_t r1, int32_t g0,
                                  int32_t g1, int32_t select_mode, void *O, float *lse,
                                  void *workspace, size_t workspace_bytes, void *stream);

/* ---- decode over a paged KV cache (K6; semantics = last row of attend) ----
 * Paged layout: page = B tokens; k_pages/v_pages [num_pages, B, h_kv, d_h]
 * bf16; block_table [batch, max_pages] int32; seq_lens [batch] int32 = tokens
 * already in the cache INCLUDING the current one.  Compressed keys live in
 * per-sequence slabs kc1 [batch, max_m1, h_kv, d_h], kc2 [batch, max_m2, ...]
 * maintained by swattn_kcache_append. */
typedef struct swattn_paged_kv {
  const void *k_pages;
  const void *v_pages;
  const int32_t *block_table;
  const int32_t *seq_lens;
  int32_t max_pages;
  void *kc1;
  void *kc2;
  int32_t max_m1;
  int32_t max_m2;
  int32_t num_pages; /* pages in the k_pages / v_pages pools (bounds the TMA
                        descriptors of the attention stage); 0 = batch * max_pages */
} swattn_paged_kv;

/* Recompute the compressed-key entries that became complete when the
 * sequences grew from prev_lens[b] to seq_lens[b] tokens. */
int32_t swattn_kcache_append(const swattn_config *cfg, const swattn_paged_kv *kv,
                             const int32_t *prev_lens, int32_t batch, void *stream);

/* Serving-loop append of ONE token per sequence, entirely on the device:
 * K, V [batch, h_kv, d_h] bf16 are written at position seq_lens[b] (the
 * block table must already map page seq_lens[b] / B), the compressed keys
 * are extended, and seq_lens[b] is advanced by one (kv->seq_lens is written
 * through).  active [batch] int32 (NULL = all): sequences with active[b] == 0
 * are left untouched.  One launch, no host synchronisation; capturable in a
 * CUDA graph together with swattn_decode_step. */
int32_t swattn_kcache_append_tokens(const swattn_config *cfg, const swattn_paged_kv *kv,
                                    const void *K, const void *V, const int32_t *active,
                                    int32_t batch, void *stream);

/* One decode step: q [batch, h_q, d_h] bf16 for token seq_lens[b]-1 ->
 * o [batch, h_q, d_h] bf16, lse [batch, h_q] fp32; topk [batch, h_kv, k_top]
 * int32 (optional, may be NULL). */
int32_t swattn_decode_step(const swattn_config *cfg, const swattn_paged_kv *kv,
                           const void *q, int32_t batch, void *o, float *lse,
                           int32_t *topk, void *workspace, size_t workspace_bytes,
                           void *stream);
size_t swattn_decode_workspace_bytes(const swattn_config *cfg, int32_t batch,
                                     int32_t max_pages);
/* Diagnostics: byte offset in the decode workspace of the int32 count of
 * (sequence, group) rows the last swattn_decode_step settled by the float64
 * boundary re-rank (valid after the step completes; -1 on bad arguments). */
int64_t swattn_decode_reranked_offset(const swattn_config *cfg, int32_t batch,
                                      int32_t max_pages);

#ifdef __cplusplus
}
#endif
#endif /* SWATTN_B200_H */
