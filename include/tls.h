/*
 * tls.h -- C ABI of the B200-native AsyncTLS two-level sparse decode attention
 * operator (arXiv 2604.07815).  Implemented by libtls.so
 * (paper_2604_07815_b200/csrc/*.cu, sm_100a).
 *
 * Citation key: P:n = line n of PAPER.md (the paper's LaTeX source).
 *
 * Conventions shared by every call
 * --------------------------------
 * - Every pointer is a caller-owned DEVICE pointer unless noted otherwise.
 *   The library allocates no device memory.  Host-side state: a thread-local
 *   error string and, only when TLS_NSPLIT > 1 pipelines a call over
 *   sub-batches, per-thread internal CUDA streams and events.
 * - Every call validates its host-visible arguments synchronously, then
 *   enqueues its kernels on `stream` and returns; outputs are valid once the
 *   stream reaches that point.  No call synchronises the host.
 * - Results are bitwise deterministic for fixed inputs and configuration
 *   (no order-nondeterministic float atomics).
 * - Return value: TLS_OK, or a tls_status describing the first problem found;
 *   tls_last_error() then returns a human-readable detail string.  Nothing is
 *   enqueued when a call returns an error detected before launch.
 * - Pairs: a *pair* (b, g) is one batch element b and one KV head g; every
 *   pair is an independent unit of work ("for each key-value group").
 *   Query head h belongs to KV head g = h / G, G = num_q_heads / num_kv_heads.
 *   MLA: one shared latent KV head (num_kv_heads = 1), G = num_q_heads.
 *
 * Tensor layouts (row-major, innermost last; element type = cfg.dtype):
 *   q        [batch, num_q_heads, d_k]
 *   k_cache  GQA: [batch, num_kv_heads, max_seq_len, d_k]
 *            MLA: [batch, max_seq_len, d_k]      (latent ++ rope, d_k = 576)
 *   v_cache  GQA: [batch, num_kv_heads, max_seq_len, d_v]
 *            MLA: NULL -- V is the first d_v dims of each k_cache row
 *   seq_lens [batch] int32, 1 <= seq_lens[b] <= max_seq_len (device memory)
 */
#ifndef TLS_H_
#define TLS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without the CUDA headers (same underlying type). */
typedef struct CUstream_st* tls_stream_t;

typedef enum {
  TLS_OK = 0,
  TLS_ERR_DIM = 1,         /* inconsistent shapes / widths                       */
  TLS_ERR_CONFIG = 2,      /* invalid hyper-parameter (B, d_c, k_b, k_t, ...)    */
  TLS_ERR_INPUT = 3,       /* NULL required pointer, empty batch / selection     */
  TLS_ERR_WORKSPACE = 4,   /* workspace missing or too small                     */
  TLS_ERR_UNSUPPORTED = 5, /* valid request outside what the kernels implement   */
  TLS_ERR_CUDA = 6         /* a CUDA launch failed                               */
} tls_status;

typedef enum { TLS_BF16 = 0, TLS_FP32 = 1 } tls_dtype;

typedef enum {
  TLS_GQA = 0, /* grouped-query attention; MHA is G = 1, MQA is num_kv_heads = 1 */
  TLS_MLA = 1  /* absorbed multi-head latent attention: one shared KV head */
} tls_layout;

typedef struct {
  int32_t batch;        /* number of sequences                                   */
  int32_t num_q_heads;  /* H_q                                                    */
  int32_t num_kv_heads; /* H_kv (1 for MLA)                                       */
  int32_t d_k;          /* key / query width (GQA: head dim; MLA: 576)            */
  int32_t d_v;          /* value width (GQA: = d_k; MLA: 512)                     */
  int32_t max_seq_len;  /* capacity S of the caches (tokens)                      */
  int32_t block_size;   /* B, tokens per block (64 in P:397)                */
  int32_t d_c;          /* token-index channels (32 GQA / 128 MLA)  */
  int32_t top_blocks;   /* k_b (128 in P:397)                              */
  int32_t top_tokens;   /* k_t (512 / 1024 / 2048 in P:397)                */
  float sm_scale;       /* 1/sqrt(d): alpha-tilde logits AND final attention       */
                        /*                                           */
  int32_t dtype;        /* tls_dtype of q / caches / block summaries / outputs    */
  int32_t layout;       /* tls_layout                                             */
} tls_config;

/*
 * The hierarchical index of one KV cache (Fig. 2 "construct hierarchical
 * indices"; built by tls_build_index).  All buffers are caller-owned device
 * memory; M = ceil(max_seq_len / block_size), Hkv = num_kv_heads.
 */
typedef struct {
  void* block_minmax;      /* [batch, Hkv, M, 2, d_k] dtype: [..,0,:] = k^max_i,
                              [..,1,:] = k^min_i                        */
  uint8_t* codes;          /* [batch, Hkv, max_seq_len, d_c/2] INT4 codes of the
                              channel-projected keys; channel 2i in the
                              low nibble, 2i+1 in the high nibble of byte i      */
  float* scale_zero;       /* [batch, Hkv, max_seq_len, 2] fp32 (scale, zero):
                              k~ = zero + scale * code                            */
  const int32_t* channels; /* [Hkv, d_c] ascending channel ids C; an
                              input, produced by tls_calibrate_channels or the
                              caller's own calibration                            */
} tls_index;

/*
 * Channel calibration:
 *   s_i = (1/G) sum_h max_{D_cal} |q_h[i]| * max_{D_cal} |k[i]|,  C = top-d_c(s)
 * per KV head, ties -> lower channel id; C is written ascending.
 *   q_cal          [n_q, num_q_heads, d_k] calibration queries
 *   k_cal          base of the calibration keys of KV head 0: n_k rows of d_k
 *                  contiguous elements; KV head g starts k_head_stride
 *                  ELEMENTS after head g-1 (for a GQA cache slice
 *                  k_cache[b] pass k_head_stride = max_seq_len * d_k).
 *   channels_out   [Hkv, d_c] int32 (output)
 *   channel_scores [Hkv, d_k] fp32, nullable (output; the s_i above)
 * Errors: TLS_ERR_CONFIG if d_c > d_k; TLS_ERR_INPUT if n_q < 1 or n_k < 1.
 */
tls_status tls_calibrate_channels(const tls_config* cfg, const void* q_cal, int32_t n_q,
                                  const void* k_cal, int32_t n_k, int64_t k_head_stride,
                                  int32_t* channels_out, float* channel_scores,
                                  tls_stream_t stream);

/*
 * Index construction: for every pair and every
 * block i with i*B < seq_lens[b], and i >= start_token / B:
 *   k^max_i / k^min_i = channelwise max / min of the block's valid keys;
 * for every valid token j of those blocks, the INT4 token index:
 *   x = fp32(k_j[C]); zero = min x; scale = fp32(fp32(max x - zero) / 15);
 *   code_c = scale > 0 ? clamp(rint(fp32(fp32(x_c - zero) / scale)), 0, 15) : 0
 * (IEEE fp32, round-to-nearest-even; bit-identical to the oracle).
 * start_token = 0 builds everything (prefill); start_token > 0 rebuilds only
 * from block start_token / B on (incremental append of decode tokens).
 * Entries of blocks / tokens at or beyond seq_lens[b] are left untouched.
 */
tls_status tls_build_index(const tls_config* cfg, const void* k_cache, const int32_t* seq_lens,
                           int32_t start_token, const tls_index* idx, tls_stream_t stream);

/*
 * Block scores alone (step a1, P:99 via the P:104-118 GEMM identity; the
 * scoring phase of select_kernel, mode 0):
 *   scores[b, g, i] = sum_h sum_c max(q_hc k^max_ic, q_hc k^min_ic)   (fp32)
 * for every block i < ceil(seq_lens[b] / B); entries at or beyond that are
 * left untouched.  scores: [batch, Hkv, ceil(max_seq_len / B)] fp32 device
 * memory.  This is phase a1 of tls_select (also usable on its own, e.g. for
 * block-only Quest-style selection).
 */
tls_status tls_block_scores(const tls_config* cfg, const void* q, const int32_t* seq_lens,
                            const void* block_minmax, float* scores, tls_stream_t stream);

/*
 * Two-level selection for one decode step:
 *   s_i   = sum_h sum_k max(q_hk k^max_ik, q_hk k^min_ik)
 *         (computed as Q+ . k^max_i + Q- . k^min_i, Q+- = sum_h max/min(q_h,0),
 *          the P:110 identity plus linearity of sum_h)
 *   M_t   = top-k_b blocks (ties -> lower id)
 *   alpha~_j = (1/G) sum_h softmax_{j in J}(q~_h . k~_j * sm_scale)
 *          over the candidate tokens J of M_t (or of guide_block_ids)
 *   S_t   = top-k_t tokens of J by alpha~ (ties -> lower token id)
 * Outputs (all ascending ids, -1 padded):
 *   block_ids    [batch, Hkv, top_blocks]  M_t
 *   token_ids    [batch, Hkv, top_tokens]  S_t
 *   num_tokens   [batch, Hkv]              |S_t| = min(k_t, |J|)
 *   token_scores [batch, Hkv, top_tokens]  nullable; ln(alpha~_j) of S_t
 * guide_block_ids: NULL -> candidates are this step's M_t (synchronous form,
 *   P:137); else [batch, Hkv, top_blocks] ascending, -1 padded: candidates are
 *   those blocks (one-step-lag form S_t = TokenSelect(q_t, M_{t-1})).
 * workspace: >= tls_workspace_bytes(cfg, 0) bytes of device memory, 256-B
 *   aligned, not shared with a concurrently running call.
 * Kernels (fused.cu, select.cu, attend.cu): select_kernel scores every
 * pair's blocks tile by tile; the pair's last tile CTA waits for the others'
 * completion flags and runs the pair's top-k_b (a2) while other pairs' tiles
 * still stream; token_cluster_kernel (a3, one thread-block cluster per pair)
 * and the attention kernel's selection prologue (a4) follow.
 */
tls_status tls_select(const tls_config* cfg, const void* q, const int32_t* seq_lens,
                      const tls_index* idx, const int32_t* guide_block_ids, int32_t* block_ids,
                      int32_t* token_ids, int32_t* num_tokens, float* token_scores,
                      void* workspace, size_t workspace_bytes, tls_stream_t stream);

/*
 * Sparse attention over the selected tokens:
 *   o^(h) = softmax_{j in S}(q^(h) . k_j * sm_scale) V_S,  lse^(h) = ln sum_j exp(.)
 * with full-dimensional K, V.  token_ids / num_tokens as written by tls_select
 * (ids must lie in [0, seq_lens[b]); entries past num_tokens are ignored).
 *   out [batch, num_q_heads, d_v] dtype;  lse [batch, num_q_heads] fp32, nullable.
 * Errors: TLS_ERR_INPUT if top_tokens < 1.  A pair with num_tokens == 0 gets
 * out = 0 and lse = -inf.
 */
tls_status tls_sparse_attend(const tls_config* cfg, const void* q, const void* k_cache,
                             const void* v_cache, const int32_t* token_ids,
                             const int32_t* num_tokens, void* out, float* lse, void* workspace,
                             size_t workspace_bytes, tls_stream_t stream);

/* tls_select followed by tls_sparse_attend on the same stream (one decode step
 * of the operator).  workspace >= tls_workspace_bytes(cfg, 2).
 * TLS_NSPLIT=n (environment, tuning) cuts the batch into n sub-batches whose
 * launch chains run on internal streams (results identical up to the
 * attention's split-K rounding). */
tls_status tls_decode(const tls_config* cfg, const void* q, const void* k_cache,
                      const void* v_cache, const int32_t* seq_lens, const tls_index* idx,
                      const int32_t* guide_block_ids, int32_t* block_ids, int32_t* token_ids,
                      int32_t* num_tokens, float* token_scores, void* out, float* lse,
                      void* workspace, size_t workspace_bytes, tls_stream_t stream);

/*
 * KV offload (AsyncTLS §4.2): the full K/V caches live in pinned,
 * device-mapped host memory (cudaHostAlloc(..., cudaHostAllocMapped), layouts
 * of k_cache / v_cache above); every pair owns a GPU token cache of
 * `capacity` slots.  tls_cache_fetch makes a selection S_t (token_ids /
 * num_tokens from tls_select) resident: tokens already cached are hits (the
 * step-to-step locality of the selection), slots of tokens that
 * left the selection are evicted (the cache keeps the current selection, the
 * token-granular form of C_{t+1} = M_t), and every miss is copied from
 * host memory by a zero-copy gather kernel.  slot_ids [batch, Hkv, top_tokens]
 * receives the cache row of each selected token in selection order, so
 * tls_sparse_attend over (k_slots, v_slots, slot_ids) with max_seq_len =
 * capacity computes exactly the attention over S_t.  miss_count [batch, Hkv]
 * (nullable) receives the number of rows fetched.  One launch (one CTA per
 * pair); the cache state is deterministic.
 * Errors: TLS_ERR_CONFIG if capacity < top_tokens; TLS_ERR_INPUT for NULL
 * buffers or host caches that are not device-mapped.
 */
typedef struct {
  int32_t capacity;       /* slots per pair, >= top_tokens                          */
  void* k_slots;          /* [batch, Hkv, capacity, d_k] dtype, device              */
  void* v_slots;          /* [batch, Hkv, capacity, d_v] dtype, device (NULL: MLA)  */
  int32_t* slot_of_token; /* [batch, Hkv, max_seq_len], -1 = not resident; init -1  */
  int32_t* token_of_slot; /* [batch, Hkv, capacity], -1 = free; init -1             */
} tls_token_cache;

tls_status tls_cache_fetch(const tls_config* cfg, const void* k_host, const void* v_host,
                           const int32_t* token_ids, const int32_t* num_tokens,
                           const tls_token_cache* cache, int32_t* slot_ids, int32_t* miss_count,
                           tls_stream_t stream);

/*
 * Block-granular, asynchronous form of the offload engine (AsyncTLS §4.2,
 * P:373-383).  The GPU keeps whole B-token blocks: every
 * pair owns `capacity` block slots (>= 2 * top_blocks).  With the one-step
 * lag S_t = TokenSelect(q_t, M_{t-1}) (tls_select / tls_decode with
 * guide_block_ids = M_{t-1}) the token selection of step t only reads
 * blocks of M_{t-1}, so the blocks of M_t can be transferred while step t's
 * attention runs and the next layer computes:
 *   step t (main stream):  tls_select(q_t, guide = M_{t-1}) -> M_t, S_t
 *                          wait for the update of step t-1 (event)
 *                          tls_block_cache_rows(S_t) -> slot_rows
 *                          tls_sparse_attend over (k_slots, v_slots, slot_rows)
 *   step t (side stream):  after the select: tls_block_cache_update(keep =
 *                          M_{t-1}, block_ids = M_t), record an event
 * tls_block_cache_update frees the slots whose block is in neither M_{t-1}
 * (still read by step t's attention) nor M_t, assigns free slots to the blocks
 * of M_t that are not resident (in M_t order: the cache state is
 * deterministic), copies their B rows of K (and V) from pinned, device-mapped
 * host memory with a zero-copy gather, and writes the number of blocks fetched
 * per pair to miss_count (nullable): the transfer T_t = M_t \ C_t of P:378,
 * where the resident set before the update is C_t = M_{t-2} u M_{t-1} (the
 * previous update kept M_{t-2} and added M_{t-1}), a superset of the paper's
 * C_t = M_{t-1} -- so |T_t| <= |M_t \ M_{t-1}| (tests/test_gpu_decode_loop.py
 * checks the exact ledger on stationary, alternating and drifting queries).
 * keep_block_ids may be NULL (nothing pinned).  tls_block_cache_rows writes
 * the cache row slot_of_block[t / B] * B + t % B of every selected token
 * (0 past num_tokens or when the token's block is not resident, counted in
 * absent [batch, Hkv], nullable), so tls_sparse_attend with max_seq_len =
 * capacity * B over the slot arrays computes exactly the attention over S_t.
 * One launch each (one CTA per pair).
 * Errors: TLS_ERR_CONFIG if capacity < 2 * top_blocks; TLS_ERR_INPUT for NULL
 * buffers or host caches that are not device-mapped.
 */
typedef struct {
  int32_t capacity;       /* block slots per pair, >= 2 * top_blocks                          */
  void* k_slots;          /* [batch, Hkv, capacity * block_size, d_k] dtype, device           */
  void* v_slots;          /* [batch, Hkv, capacity * block_size, d_v] dtype (NULL: MLA)       */
  int32_t* slot_of_block; /* [batch, Hkv, ceil(max_seq_len / block_size)], -1 = not resident  */
  int32_t* block_of_slot; /* [batch, Hkv, capacity], -1 = free; both initialised to -1        */
} tls_block_cache;

tls_status tls_block_cache_update(const tls_config* cfg, const void* k_host, const void* v_host,
                                  const int32_t* keep_block_ids, const int32_t* block_ids,
                                  const tls_block_cache* cache, int32_t* miss_count, tls_stream_t stream);
tls_status tls_block_cache_rows(const tls_config* cfg, const int32_t* token_ids, const int32_t* num_tokens,
                                const tls_block_cache* cache, int32_t* slot_rows, int32_t* absent,
                                tls_stream_t stream);

/* tls_decode with the K/V rows read from a block cache: the attention of token
 * t reads row slot_of_block[t / B] * B + t % B of (k_slots, v_slots), so every
 * block of the candidate set (M_t, or guide_block_ids = M_{t-1} in lag mode)
 * must be resident (tls_block_cache_update).  Same outputs and workspace as
 * tls_decode (which = 2); one fused launch chain.  guide_block_ids (M_{t-1},
 * the lag mode of P:373) is required: TLS_ERR_INPUT when NULL, because the
 * blocks of this step's M_t are not resident yet.  A selected token whose
 * block is nevertheless not resident reads cache row 0 (no out-of-bounds
 * access; use tls_block_cache_rows' `absent` count to detect it). */
tls_status tls_decode_block_cache(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                                  const int32_t* guide_block_ids, const tls_block_cache* cache, int32_t* block_ids,
                                  int32_t* token_ids, int32_t* num_tokens, float* token_scores, void* out,
                                  float* lse, void* workspace, size_t workspace_bytes, tls_stream_t stream);

/*
 * ---- Sequence-split decode: one long sequence whose KV
 * cache and index are split along the sequence over P ranks (rank r holds the
 * block-aligned token range [t0_r, t0_r + n_r) of every sequence, its index
 * built over that range).  The step stays exact: every global decision is
 * taken from gathered local pieces that contain it (orchestrated, with the
 * all_gathers, by paper_2604_07815_b200/seqsplit.py):
 *   1. tls_block_scores on the local range; tls_block_topk -> local top-k_b
 *      (score, global block id); all_gather; tls_topk_rows -> global M_t
 *      (the global top-k_b is among the union of local top-k_b);
 *   2. tls_select_range -> the local blocks of M_t; tls_token_stats -> this
 *      rank's per-head softmax statistics over its candidates; all_gather;
 *   3. tls_token_keys (merges the P statistics: alpha~ is a softmax over ALL
 *      candidates J) -> ln alpha~ + global token id per local
 *      candidate; tls_topk_rows -> local top-k_t; all_gather; tls_topk_rows ->
 *      global S_t;
 *   4. tls_select_range -> the local tokens of S_t; tls_sparse_attend_f32 ->
 *      partial (out, lse); all_gather; tls_attn_merge (LSE identity) -> out
 *      (P:142).
 * All pointers are device memory; calls are asynchronous on `stream`.
 */

/* Exact top-k of each of `rows` rows of n (key, id) pairs (ids ascending per
 * row, -1 = empty entry): the k largest keys, equal keys -> lower id (U2).
 * keys/ids: [rows, n]; out_keys/out_ids: [rows, k] in ascending id order,
 * padded with -inf / -1; out_count: [rows] (nullable) = min(k, #entries).
 * TLS_ERR_INPUT for rows < 1, n < 1, k < 1 or a NULL pointer. */
tls_status tls_topk_rows(int32_t rows, int32_t n, const float* keys, const int32_t* ids, int32_t k,
                         float* out_keys, int32_t* out_ids, int32_t* out_count, tls_stream_t stream);

/* A rank's local top-k_b with GLOBAL block ids: scores [batch, Hkv,
 * ceil(max_seq_len / B)] from tls_block_scores on the local range; block i of
 * pair (b, g) exists iff i < ceil(seq_lens[b] / B).  out_scores / out_block_ids
 * [batch, Hkv, top_blocks]: the top_blocks largest scores (ties -> lower id),
 * ids = i + block_offset in ascending order, -inf / -1 padded. */
tls_status tls_block_topk(const tls_config* cfg, const float* scores, const int32_t* seq_lens, int32_t block_offset,
                          float* out_scores, int32_t* out_block_ids, tls_stream_t stream);

/* The ids of each row (ascending, -1 padded, k per row) that lie in [lo, hi),
 * shifted by -lo, compacted in order and -1 padded: out_ids [rows, k];
 * out_count [rows] (nullable).  TLS_ERR_INPUT for rows/k < 1, lo > hi, NULL. */
tls_status tls_select_range(int32_t rows, int32_t k, const int32_t* ids, int32_t lo, int32_t hi,
                            int32_t* out_ids, int32_t* out_count, tls_stream_t stream);

/* This rank's part of a3's softmax normaliser over its candidate
 * tokens: the tokens of block_ids [batch, Hkv, top_blocks] (local ids,
 * ascending, -1 padded) below seq_lens[b].  For every pair and head h of the
 * group, with L_hj = sm_scale log2(e) q~_h . k~_j (log2 units, q~_h = q_h[C]):
 *   stats [batch, Hkv, G, 2] = (M_h = max_j L_hj, Z_h = sum_j 2^(L_hj - M_h)),
 * (-inf, 0) when the rank has no candidate.  cfg describes the local range
 * (max_seq_len = the local cache length).  GQA and MLA, bf16 and fp32. */
tls_status tls_token_stats(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                           const int32_t* block_ids, float* stats, tls_stream_t stream);

/* Ranking keys of this rank's candidates under the GLOBAL normaliser:
 * stats_parts [n_parts, batch, Hkv, G, 2] are every rank's tls_token_stats
 * (rank order); lz_h = M_h + log2 Z_h of their LSE merge.  For candidate slot
 * s = k * B + r (block k of block_ids, row r):
 *   keys [batch, Hkv, top_blocks * B] = ln alpha~_j = ln((1/G) sum_h 2^(L_hj - lz_h)),
 *   token_ids (same shape) = j + token_offset (the global token id),
 * (-inf, -1) for slots past the candidates or the sequence. */
tls_status tls_token_keys(const tls_config* cfg, const void* q, const int32_t* seq_lens, const tls_index* idx,
                          const int32_t* block_ids, int32_t n_parts, const float* stats_parts,
                          int32_t token_offset, float* keys, int32_t* token_ids, tls_stream_t stream);

/* tls_sparse_attend with an fp32 output [batch, Hq, d_v] whatever the cache
 * dtype (the partial results of the sequence split: rounded once, by the merge). */
tls_status tls_sparse_attend_f32(const tls_config* cfg, const void* q, const void* k_cache, const void* v_cache,
                                 const int32_t* token_ids, const int32_t* num_tokens, float* out, float* lse,
                                 void* workspace, size_t workspace_bytes, tls_stream_t stream);

/* LSE merge of n_parts partial attention results (split-K identity):
 * parts_out [n_parts, batch, Hq, d_v] fp32 (tls_sparse_attend_f32), parts_lse [n_parts, batch,
 * Hq] (natural log, -inf = no token in that part):
 *   lse = log sum_p exp(lse_p);  out = sum_p exp(lse_p - lse) parts_out_p.
 * out [batch, Hq, d_v] (cfg dtype); lse [batch, Hq] nullable. */
tls_status tls_attn_merge(const tls_config* cfg, int32_t n_parts, const float* parts_out, const float* parts_lse,
                          void* out, float* lse, tls_stream_t stream);

/*
 * ---- The paper's comparison operators,
 * built from the calls above:
 *   Quest (block level only): tls_block_scores -> tls_block_topk (offset 0) ->
 *     tls_expand_blocks -> tls_sparse_attend over every token of M_t;
 *   DS (token level only, every block a candidate): tls_block_iota ->
 *     tls_token_stats -> tls_token_keys (one part) -> tls_topk_rows(k_t) ->
 *     tls_sparse_attend;
 * (paper_2604_07815_b200/ops.py quest_decode, ds_decode).
 *
 * tls_expand_blocks: token_ids [batch, Hkv, k_out] = the tokens below
 * seq_lens[b] of block_ids [batch, Hkv, top_blocks] (ascending, -1 padded),
 * ascending, truncated to k_out, -1 padded; num_tokens [batch, Hkv].
 * TLS_ERR_UNSUPPORTED for top_blocks > 1024.
 * tls_block_iota: block_ids [batch, Hkv, top_blocks] = 0 .. m-1 (m =
 * ceil(seq_lens[b] / B)), -1 padded (top_blocks >= m selects every block).
 */
tls_status tls_expand_blocks(const tls_config* cfg, const int32_t* block_ids, const int32_t* seq_lens,
                             int32_t k_out, int32_t* token_ids, int32_t* num_tokens, tls_stream_t stream);
tls_status tls_block_iota(const tls_config* cfg, const int32_t* seq_lens, int32_t* block_ids, tls_stream_t stream);

/* Workspace bytes needed by: which = 0 tls_select, 1 tls_sparse_attend,
 * 2 tls_decode.  The select part holds the fp32 block scores of every pair,
 * per-chunk softmax statistics, the ranking key of every candidate token and a
 * per-pair key histogram; the attention part the
 * per-CTA partial (max, sum, o) of the split-K attention, plus the pair
 * completion words of the selection kernels (tile flags and a call
 * generation per pair; per-pair hand-off flags between the kernels).  Sizes
 * are rounded up to 256 B.  Contract: initialise the workspace once with
 * tls_workspace_init (every call leaves it ready for the next one), do not
 * write it from outside between calls -- reuse one buffer per configuration
 * (and per TLS_NSPLIT, which changes the layout) -- and do not share it
 * between calls that may run concurrently.
 * (size_t)-1 for an invalid configuration or `which`.  A NULL / too small /
 * misaligned workspace -> TLS_ERR_WORKSPACE. */
size_t tls_workspace_bytes(const tls_config* cfg, int32_t which);

/* Initialise a workspace before its first use (and after any outside write
 * to it): zero-fills it and sets every block-score word to the completion
 * sentinel 0xffffffff (a NaN no arithmetic produces).  select_kernel's pair
 * worker waits until the pair's scores differ from the sentinel -- the
 * scores themselves signal completion, so the tile CTAs need no fences or
 * flags -- and writes the sentinel back after use, so every call leaves the
 * workspace ready for the next.  Enqueued on `stream`.  Errors:
 * TLS_ERR_WORKSPACE if the buffer is smaller than
 * tls_workspace_bytes(cfg, which). */
tls_status tls_workspace_init(const tls_config* cfg, int32_t which, void* workspace, size_t workspace_bytes,
                              tls_stream_t stream);

/* Number of kernel launches one call enqueues (which as above; 3 =
 * tls_build_index, 4 = tls_calibrate_channels), for launch accounting:
 * tls_select and tls_decode 4 each (qq_kernel, select_kernel,
 * token_cluster_kernel, attend_kernel), times TLS_NSPLIT sub-batches;
 * tls_sparse_attend 1.
 * -1 for an invalid configuration. */
int32_t tls_launch_count(const tls_config* cfg, int32_t which);

/* Selection mode of tls_select / tls_decode: 1 = select_kernel a1-a2,
 * token_cluster_kernel a3, the attention kernel's prologue a4 (the only mode
 * of this build).  -1 for an invalid configuration. */
int32_t tls_select_mode(const tls_config* cfg);

/* CTAs per (batch, KV-head) pair -- the thread-block cluster size -- of the
 * token-select kernel (which = 0 or 2) or of the attention kernel (which = 1);
 * which = 3: the tokens per staged chunk of the MLA attention plan of
 * tls_sparse_attend (64, or 32 when the selected-token list leaves no room for
 * 64-token double buffering; 0 for GQA); which = 4: that plan's engine (3 =
 * tcgen05 tensor cores with TMEM accumulators, 2 = mma.sync, 1 = CUDA cores);
 * which = 5: the token-scoring (a3) kernel's form (1 = one 1024-thread CTA per
 * pair holding the pair's whole candidate index in shared memory, 4 = a cluster
 * of two 512-thread CTAs holding half each, 2 = a cluster of chunk CTAs with the
 * logits in registers, 3 = a cluster of chunk CTAs with two passes over shared
 * memory; TLS_K2_FORM=cluster excludes forms 1 and 4, TLS_K2_FORM=1 / 2 forces
 * form 1 / 4 where it fits).
 * -1 for an invalid configuration.
 * The environment variable TLS_CLUSTER overrides the heuristic for both
 * cluster sizes (1, 2, 4, 8 or 16). */
int32_t tls_cluster_size(const tls_config* cfg, int32_t which);

/* Live per-kernel device timing (diagnostics; used by bench.py for the
 * roofline of the dominant kernel).  While enabled, every tls_select /
 * tls_decode call records library-owned CUDA events on its stream before and
 * after each of its launches (no extra synchronisation; events sit between
 * launches that are already stream-ordered).  Slots: 0 = qq_kernel +
 * select_kernel (a1-a2), 1 = token_cluster_kernel (a3), 2 = attend kernel
 * (a4 prologue + a5).  With TLS_NSPLIT > 1
 * the whole overlapped step is recorded in slot 2.
 *   tls_timing_enable(n): n > 0 enables and pre-creates events for n calls
 *     (more are created on demand), clearing previous records; n == 0
 *     disables and frees the events.
 *   tls_timing_read(ms_sum[3], calls): synchronises the recorded events,
 *     writes the summed milliseconds per slot and the number of calls
 *     recorded, and clears the records (enable state unchanged).
 * Process-global, not thread-safe: enable/read from one host thread. */
tls_status tls_timing_enable(int32_t n_calls);
tls_status tls_timing_read(double* ms_sum, int64_t* calls);

const char* tls_status_string(tls_status status);
const char* tls_last_error(void); /* thread-local detail of the last error */
const char* tls_version(void);


#ifdef __cplusplus
}
#endif

#endif /* TLS_H_ */
