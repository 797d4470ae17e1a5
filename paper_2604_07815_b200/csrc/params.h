// params.h -- host/device parameter blocks and shared-memory plans of the
// decode-step kernels:
//   qq_kernel, select_kernel (fused.cu)          a1: block scores; a2: top-k_b
//   token_pair_kernel / token_pair_nt_kernel / token_reg_kernel / token_cluster_kernel (select.cu)  a3: ranking keys
//   attend_kernel / attend_mla_kernel (attend.cu)        a4: top-k_t; a5: attention
//   pstep_kernel (pstep.cu, opt-in)              a1-a5 in one persistent launch
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace tls {

constexpr int kAttnChunk = 64;     // tokens per K/V staging stage of the GQA mma attention (8 warps x 8)
constexpr int kAttnStages = 3;     // cp.async pipeline depth of the GQA mma attention
// MLA attention staging: 64-token chunks, double-buffered (default), or 32-token chunks, 3 stages (when the
// selected-token list of a CTA leaves no room for the larger buffers)
constexpr int mla_stages(int tc) { return tc == 64 ? 2 : 3; }
constexpr int kScoreTileBytes = 32 * 1024;  // K1: bytes of block summaries per CTA (TMA tile)

struct Dims {
  int batch, Hq, Hkv, G, d_k, d_v, S, B, d_c, Kb, Kt;
  int M;  // ceil(S / B): block-index rows per pair
  float sm_scale;
  int mla;
  int bf16;
  int log2B;  // block_size is a power of two
  int Ms;     // score row stride (floats): M rounded up to a multiple of 4 (16-byte rows)
};

constexpr int kBracketWords = 2048;  // fast_topk's bracket scratch (fasttopk.cuh kBracketCap)
constexpr int kPairGroups = 8;      // token_pair_kernel: staging groups (one mbarrier each)
constexpr int kPairSmemMax = 219 * 1024;  // token_pair_kernel: dynamic shared-memory budget (api.cu kMaxSmem)
constexpr int kPairSmemHalf = 104 * 1024; // ... of its two-CTA form (two CTAs per SM with their static blocks)
constexpr int kPairSmemQuarter = 50 * 1024;  // ... of its four-CTA form (four CTAs per SM)
constexpr int kKeyBins = 1024;      // fixed binning of the ranking keys: 1/16 log2 unit below kKeyTop
constexpr float kKeyTop = 6.0f;     // > log2(32) >= every key (key = log2 alpha~ + log2 G <= log2 G)

// Selection kernel (fused.cu): every CTA scores one tile of a pair's blocks
// (a1); the pair's last tile CTA then runs the pair's top-k_b (a2) and
// prepares the token kernel's inputs.  Mode 0 = scores only.
struct FusedParams {
  Dims d;
  int mode;     // 0: scores only (tls_block_scores); 1: + top-k_b worker
  int tb;       // block-summary rows per CTA (<= kScoreTileBytes)
  int sstride;  // scores row stride (floats)
  int kb_eff;
  const void* q;
  const int* seq_lens;
  const void* block_minmax;
  const int* channels;
  float* scores;           // workspace [pairs, sstride] fp32; the completion sentinel between calls (fused.cu)
  float* qq;               // workspace [pairs, 2 d_k] fp32 [Q+ | Q-] from qq_kernel (NULL: computed per tile)
  int qq_local;            // 1: tile CTAs form QQ from the pair's (small) q rows themselves and never wait for
                           // qq_kernel; only the pair's worker waits for it (griddepcontrol.wait) before its hand-off
  uint32_t* khist;         // workspace [pairs, kKeyBins], zeroed by the worker for the token kernel
  uint8_t* qfrag;          // workspace [pairs, qfrag_bytes(d)]: q~ fragment blobs for the token kernel
  int* block_ids;          // [pairs, Kb] out: M_t ascending, -1 padded
  unsigned* ready;         // workspace [pairs]: set to `epoch` when the pair's a2 outputs are written
  unsigned* tcount;        // workspace [pairs]: scored tiles of the pair (stream_select_kernel; reset by a2)
  unsigned* sched;         // workspace [256]: stream_select_kernel's ticket / exit counters, per-SM streamer epoch
  unsigned epoch;          // this call's hand-off value (host call counter, never 0)
  unsigned long long* dbg; // diagnostics only (env TLS_DEBUG_BUF): worker phase stamps
  unsigned off_bkeys, off_scratch, off_fk, smem_bytes;
};


struct SelectParams {  // K2 (token_reg_kernel, or token_cluster_kernel when a chunk exceeds the registers)
  Dims d;
  int kb_eff, kt_eff;  // min(Kb, M); min(Kt, kb_eff*B, S)
  int cb;              // candidate blocks per chunk CTA
  int tpw;             // > 0: token_reg_kernel with tpw 16-token tiles per warp; 0: token_cluster_kernel
  int nch;             // chunks per pair = ceil(kb_eff / cb)
  int pairk;           // 1 / 2: token_pair_kernel with pairk CTAs per pair (cb = candidate blocks per CTA)
  int gsh;             // token_pair_kernel: staging group = 2^gsh candidate blocks (<= kPairGroups groups)
  int tmtpw, tmcols;   // token_pair_kernel: 16-token tiles per warp (even), TMEM columns allocated per CTA
  const void* q;
  const int* seq_lens;
  const float* scores;  // workspace [pairs, M] (K1)
  const uint8_t* codes;
  const float* scale_zero;
  const int* channels;
  const int* guide;
  int* block_ids;
  uint32_t* keys;  // workspace [pairs, kb_eff * B] ranking keys (0 = past the end)
  uint32_t* khist; // workspace [pairs, kKeyBins] histogram of the keys (PASS 2 adds)
  unsigned long long* dbg;  // diagnostics only (env TLS_DEBUG_BUF): per-CTA phase stamps
  int qtma;  // 1: the q rows of the pair arrive by TMA into smem (off_qrows)
  const uint8_t* qfrag;  // token_reg_kernel: K1b's q-fragment blobs [pairs, qfrag_bytes(d)]
  unsigned* ready_in;    // workspace [pairs]: select_kernel's hand-off (== epoch when a2 is done); reset here
  unsigned* ready_out;   // workspace [pairs]: +1 per chunk CTA once its keys and histogram counts are visible
  unsigned epoch;
  unsigned off_cblk, off_qb, off_qsum, off_qc, off_qrows, off_stage, smem_bytes;
};

struct AttendParams {  // K3 (attend_kernel / attend_mla_kernel), optionally with the a4 prologue
  Dims d;
  unsigned* ready_in;  // select only: the token kernel's per-pair count of finished chunk CTAs; reset here
  int ready_count;     // the count that means "done" (the token kernel's nch)
  unsigned epoch;
  int cs;
  int mma;       // 1: bf16 mma.sync GQA path (d in {64,128}, G <= 16); 2: bf16 mma.sync MLA path (576/512)
  int tloc_max;  // ceil(kt_eff / cs)
  int mla_tc;      // MLA attention chunk tokens (64 or 32; see mla_stages); 128 on the tcgen05 path (mma 3)
  int select;    // 1: first select S_t = top-k_t from the keys (a4); 0: read token_ids / num_tokens
  int attend;    // 1: attention (a5); 0: selection only (tls_select)
  int kb_eff;
  const void* q;
  const void* k_cache;
  const void* v_cache;
  long long kv_rows;          // rows per pair of k_cache / v_cache (max_seq_len; block cache: capacity * B)
  const int* slot_of_block;   // select only, nullable: block cache slot map [pairs, M]; the attention then reads
                              // row slot_of_block[t / B] * B + t % B for token t
  const int* seq_lens;  // select only
  const int* cand;      // select only: candidate blocks (block_ids, or the lag-mode guide)
  const uint32_t* keys;  // select only: workspace keys [pairs, kb_eff*B]
  const uint32_t* khist; // select only: workspace key histogram [pairs, kKeyBins]
  int* token_ids;
  int* num_tokens;
  float* token_scores;
  void* out;
  int out_f32;     // 1: out is fp32 [batch, Hq, d_v] whatever the cache dtype (tls_sparse_attend_f32)
  float* lse;
  float* part_o;   // workspace [pairs, cs, G, d_v] fp32 partial outputs
  float* part_ml;  // workspace [pairs, cs, G, 2] fp32 partial (max, sum), log2 units
  unsigned long long* dbg;  // diagnostics only (env TLS_DEBUG_BUF): per-CTA phase stamps
  unsigned off_sel, off_cblk, off_union, off_skeys, off_fk, off_slist, off_akv, off_aq, off_as, smem_bytes;
};

// Persistent decode step (pstep.cu): one kernel, resident CTAs claim work items (TILE a1(+a2), TOKEN a3,
// SEL a4, ATT a5) from a ticket counter in schedule-row order.
struct PStepParams {
  Dims d;
  int pairs, kb_eff;
  int tb, ntile;     // TILE: block rows per item, items per pair
  int cb, nch;       // TOKEN: candidate blocks per item, items per pair
  int ns;            // ATT: items (slices of S_t) per pair
  int ntiles_total;  // TILE tickets (pairs * ntile, pair-major)
  int nready;        // items that pass through the ready queue (pairs * (1 + nch + ns))
  int nstream;       // streamer CTAs (blockIdx < nstream): a1 tiles, then ready items
  int attend;        // 0: tls_select (no ATT items)
  unsigned epoch;    // this call's hand-off value (host call counter)
  const void* q;
  const int* seq_lens;
  const void* block_minmax;
  const uint8_t* codes;
  const float* scale_zero;
  const int* channels;
  const int* guide;          // lag mode: candidate blocks M_{t-1}, else NULL
  const void* k_cache;
  const void* v_cache;
  long long kv_rows;         // rows per pair of k_cache / v_cache
  const int* slot_of_block;  // block cache (offload engine), else NULL
  int* block_ids;
  int* token_ids;
  int* num_tokens;
  float* token_scores;
  void* out;
  float* lse;
  // workspace (zeroed once by tls_workspace_init; every call leaves it so)
  unsigned* sched;   // [0] next TILE ticket, [1] CTAs finished, [2] ready-queue head, [3] ready-queue tail
  unsigned long long* rq;  // [nready] ready queue: (epoch << 32) | item
  unsigned* ctr;     // [pairs][8] per-pair counters and flags
  float* scores;     // [pairs][Ms] a1 block scores
  uint32_t* keys;    // [pairs][kb_eff * B] a3 ranking keys
  uint32_t* khist;   // [pairs][kKeyBins] histogram of the keys
  float* stats;      // [pairs][nch][8][2] a3 chunk softmax statistics
  float* part_o;     // [pairs][ns][8][128] a5 partial outputs
  float* part_ml;    // [pairs][ns][8][2] a5 partial (max, sum)
  unsigned long long* dbg;  // diagnostics only (env TLS_DEBUG_BUF): per item (start, end, smid|role|sub|pair)
  unsigned off_tile, off_qq, off_bkeys, off_scratch, off_fk;            // TILE (two tile buffers from off_tile)
  unsigned off_stage, off_qb, off_cblk, off_lhist;                      // TOKEN
  unsigned off_skeys, off_sscratch, off_shist, off_sfk, off_slist, off_scblk;  // SEL
  unsigned off_kv, off_pbuf, off_sel;                                   // ATT
  unsigned smem_bytes;
};

// GPU token cache of the offload engine (offload.cu): make S_t resident.
struct CacheFetchParams {
  Dims d;
  int capacity;      // slots per pair (>= top_tokens)
  int bitmap_words;  // ceil(S / 32)
  const uint8_t* k_host;  // device-accessible pointer to the pinned host K cache (layout of k_cache)
  const uint8_t* v_host;  // ... V cache (NULL for MLA)
  const int* token_ids;   // [pairs, Kt] S_t (tls_select)
  const int* num_tokens;  // [pairs]
  uint8_t* k_slots;       // [pairs, capacity, d_k]
  uint8_t* v_slots;       // [pairs, capacity, d_v] (NULL for MLA)
  int* slot_of_token;     // [pairs, S], -1 = not resident
  int* token_of_slot;     // [pairs, capacity], -1 = free
  int* slot_ids;          // [pairs, Kt] out: the cache row of each selected token
  int* miss_count;        // [pairs] out, nullable
};

// Block-granular offload cache (the paper's form): whole B-token
// blocks of M_t, fetched asynchronously for the next step's one-step-lag
// token selection.
struct BlockCacheParams {
  Dims d;
  int capacity;           // block slots per pair (>= 2 * top_blocks: M_{t-1} in use + M_t arriving)
  int bitmap_words;       // ceil(M / 32)
  const uint8_t* k_host;  // device-accessible pointer to the pinned host K cache (layout of k_cache)
  const uint8_t* v_host;  // ... V cache (NULL for MLA)
  const int* keep_ids;    // [pairs, Kb] blocks still in use (M_{t-1}), -1 padded; nullable
  const int* block_ids;   // [pairs, Kb] blocks to make resident (M_t), -1 padded
  uint8_t* k_slots;       // [pairs, capacity * B, d_k]
  uint8_t* v_slots;       // [pairs, capacity * B, d_v] (NULL for MLA)
  int* slot_of_block;     // [pairs, M], -1 = not resident
  int* block_of_slot;     // [pairs, capacity], -1 = free
  int* miss_count;        // [pairs] out, nullable: blocks fetched
  // tls_block_cache_rows
  const int* token_ids;   // [pairs, Kt]
  const int* num_tokens;  // [pairs]
  int* slot_rows;         // [pairs, Kt] out: cache row of each selected token (0 if its block is not resident)
  int* absent;            // [pairs] out, nullable: selected tokens whose block is not resident
};

static inline unsigned align16(size_t x) { return (unsigned)((x + 15) & ~(size_t)15); }

static inline int kb_effective(const Dims& d) { return d.Kb < d.M ? d.Kb : d.M; }
static inline int kt_effective(const Dims& d) {
  const long long cand = (long long)kb_effective(d) * d.B < d.S ? (long long)kb_effective(d) * d.B : d.S;
  return d.Kt < cand ? d.Kt : (int)cand;
}

static inline void plan_select(SelectParams& p, int pair_form = 0) {
  const Dims& d = p.d;
  p.kb_eff = kb_effective(d);
  p.kt_eff = kt_effective(d);
  const int nt0 = (d.G + 7) / 8, nt = nt0 <= 1 ? 1 : (nt0 <= 2 ? 2 : 4);  // instantiated NT
  const int ks = d.d_c / 16, nsplit = d.bf16 ? 1 : 3;
  const int per_block = d.B * (d.d_c / 2 + 8);
  // one or two CTAs per pair (token_pair_kernel) when G <= 8, every block's scale/zero rows are 16-byte aligned
  // (S even) and the candidate index fits shared memory: two 512-thread CTAs (two per SM) when half of it fits
  // ~100 KB, else one 1024-thread CTA.  pair_form: 0 automatic, 1 / 2 force that many CTAs, < 0 the cluster forms
  p.pairk = 0;
  if (pair_form >= 0 && nt == 1 && (d.S & 1) == 0 && d.Kb <= 512) {
    for (int nch = (pair_form ? pair_form : 2); nch >= 1; nch = nch == 4 ? 2 : nch - 1) {
      const int cb = (p.kb_eff + nch - 1) / nch;
      size_t o = 0;
      p.off_cblk = 0;
      o = align16((size_t)p.kb_eff * 4);
      p.off_qb = (unsigned)o;
      o = align16(o + (size_t)nsplit * ks * 64 * 4);
      p.off_qsum = (unsigned)o;
      o = align16(o + 8 * 4);
      p.off_qc = p.off_qrows = (unsigned)o;
      o = (o + 127) & ~(size_t)127;
      p.off_stage = (unsigned)o;
      o = align16(o + (size_t)cb * per_block);
      // TMEM logit store: 4 columns per tile, tiles per warp rounded up to even (pass 2 reads tiles in pairs)
      const int nw = 32 / nch, tpw = (((cb << d.log2B) / 16 + nw - 1) / nw + 1) & ~1;
      int cols = 32;
      while (cols < nw * tpw) cols <<= 1;
      if (d.B >= 16 && cols <= 512 / nch &&
          o <= (size_t)(nch == 4 ? kPairSmemQuarter : (nch == 2 ? kPairSmemHalf : kPairSmemMax))) {
        p.tmtpw = tpw;
        p.tmcols = cols;
        p.pairk = nch;
        p.nch = nch;
        p.tpw = 0;
        p.cb = cb;
        p.gsh = 0;
        while (((cb + (1 << p.gsh) - 1) >> p.gsh) > kPairGroups) ++p.gsh;
        p.smem_bytes = (unsigned)o;
        return;
      }
      if (pair_form) break;
    }
  }
  // a pair's candidate blocks split over a cluster of nch <= 8 CTAs, ~24 KB (or more) of index each
  p.cb = (24 * 1024) / per_block;
  if (p.cb < 1) p.cb = 1;
  if (p.cb * 8 < p.kb_eff) p.cb = (p.kb_eff + 7) / 8;
  // G > 8 (MLA): token_pair_nt_kernel, a cluster of 16 (else 8) 256-thread CTAs per pair holding the candidate
  // index in shared memory and the logits in TMEM (bf16, d_c in {32, 128})
  if (pair_form >= 0 && nt > 1 && d.bf16 && (d.S & 1) == 0 && d.Kb <= 512 && (ks == 2 || ks == 8) && d.B >= 16) {
    for (int nch = 16; nch >= 8; nch /= 2) {
      const int cb = (p.kb_eff + nch - 1) / nch;
      size_t o = 0;
      p.off_cblk = 0;
      o = align16((size_t)p.kb_eff * 4);
      p.off_qb = (unsigned)o;
      o = align16(o + (size_t)nsplit * nt * ks * 64 * 4);
      p.off_qsum = (unsigned)o;
      o = align16(o + (size_t)nt * 8 * 4);
      p.off_qc = p.off_qrows = (unsigned)o;
      o = (o + 127) & ~(size_t)127;
      p.off_stage = (unsigned)o;
      o = align16(o + (size_t)cb * per_block);
      const size_t stat = 4096 + 8 * nt * 8 * 4 + 2 * nt * 8 * 4 + 2 * (size_t)nch * nt * 8 * 4 + 256;
      int per_sm = (int)((228 * 1024) / (o + stat + 1024));
      if (per_sm > 4) per_sm = 4;
      const int tpw = ((cb << d.log2B) / 16 + 7) / 8;
      int cols = 32;
      while (cols < 2 * 4 * nt * tpw) cols <<= 1;
      if (per_sm >= 1 && cols * per_sm <= 512 && o <= (size_t)kPairSmemMax) {
        p.tmtpw = tpw;
        p.tmcols = cols;
        p.pairk = nch;
        p.nch = nch;
        p.tpw = 0;
        p.cb = cb;
        p.gsh = 0;
        while (((cb + (1 << p.gsh) - 1) >> p.gsh) > kPairGroups) ++p.gsh;
        p.smem_bytes = (unsigned)o;
        return;
      }
    }
  }
  // register-resident K2: a CTA holds at most 8 warps x tpw tiles x 16 tokens, in a cluster of <= 16
  p.tpw = 8 / nt;
  const int cb_reg = (8 * p.tpw * 16) / d.B;  // 8 warps (kThreads = 256)
  if (cb_reg >= 1 && (p.kb_eff + cb_reg - 1) / cb_reg <= 16) {
    if (p.cb > cb_reg) p.cb = cb_reg;
  } else {
    p.tpw = 0;
  }
  if (p.cb > p.kb_eff) p.cb = p.kb_eff;
  p.nch = (p.kb_eff + p.cb - 1) / p.cb;
  size_t o = 0;
  p.off_cblk = (unsigned)o;
  o = align16(o + (size_t)p.kb_eff * 4);
  p.off_qb = (unsigned)o;
  o = align16(o + (size_t)nsplit * nt * ks * 64 * 4);
  p.off_qsum = (unsigned)o;
  o = align16(o + (size_t)nt * 8 * 4);
  p.off_qc = (unsigned)o;
  o = align16(o + (size_t)nt * 8 * d.d_c * 4);
  const size_t qbytes = (size_t)d.G * d.d_k * (d.bf16 ? 2 : 4);
  p.qtma = qbytes <= 16 * 1024;
  p.off_qrows = (unsigned)o;
  if (p.qtma) o = align16(o + qbytes + (size_t)d.d_c * 4);
  o = (o + 127) & ~(size_t)127;
  p.off_stage = (unsigned)o;  // staged candidate index
  o = align16(o + (size_t)p.cb * per_block);
  p.smem_bytes = (unsigned)o;
}

static inline void plan_attend(AttendParams& p, size_t fastctl_bytes) {
  const Dims& d = p.d;
  p.kb_eff = kb_effective(d);
  // with the a4 prologue the list is |S_t| <= min(Kt, Kb*B, S); standalone attention takes any num_tokens <= min(Kt, S)
  const int kmax = p.select ? kt_effective(d) : (d.Kt < d.S ? d.Kt : d.S);
  p.tloc_max = (kmax + p.cs - 1) / p.cs;
  size_t o = 0;
  p.off_sel = (unsigned)o;
  o = align16(o + (size_t)(p.tloc_max + 1) * 4);
  p.off_cblk = (unsigned)o;
  o = align16(o + (size_t)p.kb_eff * 4);
  o = (o + 127) & ~(size_t)127;
  p.off_union = (unsigned)o;
  size_t sel_end = o, att_end = o;
  if (p.select) {  // keys of every candidate slot + bracket scratch + top-k control block
    size_t s2 = o;
    p.off_skeys = (unsigned)s2;
    s2 = align16(s2 + (size_t)p.kb_eff * d.B * 4 + 2048 * 4 + kKeyBins * 4);
    p.off_fk = (unsigned)s2;
    s2 = align16(s2 + fastctl_bytes);
    p.off_slist = (unsigned)s2;  // compacted selected slots (hist_topk_emit)
    s2 = align16(s2 + (size_t)kt_effective(d) * 4);
    sel_end = s2;
  }
  if (p.attend) {
    size_t s2 = o;
    if (p.mma == 3) {  // MLA tcgen05 path: two 64-token chunks (core-matrix layout), Q, 2 x P hi + lo
      const int nh = d.G <= 16 ? 16 : 32;
      p.off_akv = (unsigned)s2;
      s2 = align16(s2 + (size_t)2 * 64 * d.d_k * 2 + (size_t)nh * d.d_k * 2 + (size_t)2 * 2 * 64 * nh * 2);
    } else if (p.mma == 2) {  // MLA tensor-core path: Q, 2 latent-row chunks, S, P, alpha/m/l
      const int mt16 = d.G <= 16 ? 16 : 32;
      p.off_akv = (unsigned)s2;
      const int tc = p.mla_tc == 32 ? 32 : 64;
      s2 += (size_t)mt16 * d.d_k * 2 + (size_t)mla_stages(tc) * tc * d.d_k * 2;
      s2 += (size_t)mt16 * (tc + 4) * 4 + (size_t)2 * mt16 * (tc + 8) * 2 + (size_t)3 * mt16 * 4;  // S, P_hi, P_lo
      s2 = align16(s2);
    } else if (p.mma) {
      p.off_akv = (unsigned)s2;  // 2 stages x (K chunk + V chunk); reused as the warp-partial scratch
      size_t kv = (size_t)kAttnStages * 2 * kAttnChunk * d.d_k * 2 + (size_t)8 * 256;  // + per-warp P^T buffers
      size_t scratch = (size_t)8 * d.G * (d.d_v + 4) * 4 + (size_t)8 * 16 * 2 * 4;
      s2 = align16(s2 + (kv > scratch ? kv : scratch));
    } else {
      p.off_aq = (unsigned)s2;
      s2 = align16(s2 + (size_t)d.G * d.d_k * 4);
      p.off_as = (unsigned)s2;
      s2 = align16(s2 + (size_t)d.G * p.tloc_max * 4);
    }
    att_end = s2;
  }
  p.smem_bytes = (unsigned)(sel_end > att_end ? sel_end : att_end);
}

static inline size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// Shared-memory plan of select_kernel: the worker's regions (block keys,
// bracket scratch, FastTopKCtl) alias the scoring tile of phase S (the worker
// starts after its own tile is scored).
static inline void plan_fused(FusedParams& p, size_t fastctl_bytes) {
  const Dims& d = p.d;
  p.kb_eff = kb_effective(d);
  size_t o = 0;
  p.off_bkeys = (unsigned)o;
  o = align16(o + (size_t)((d.M + 31) & ~31) * 4);
  p.off_scratch = (unsigned)o;
  o = align16(o + (size_t)kBracketWords * 4);
  p.off_fk = (unsigned)o;
  o = align16(o + fastctl_bytes);
  const size_t tile = (size_t)p.tb * 2 * d.d_k * (d.bf16 ? 2 : 4);
  p.smem_bytes = (unsigned)(o > tile ? o : tile);
}

// Workspace of tls_select: K1's fp32 block scores | chunk statistics | keys.
// Per-pair q-fragment blob (K1b -> K2): the B fragments of q~ (NSPLIT x NT x
// KS x 32 lanes x 2 words) followed by sum_c q~_h[c] for the NT*8 padded heads,
// laid out exactly as K2's shared-memory regions off_qb .. off_qsum.
static inline int qfrag_nt(const Dims& d) {
  const int nt0 = (d.G + 7) / 8;
  return nt0 <= 1 ? 1 : (nt0 <= 2 ? 2 : 4);
}
static inline int qfrag_bytes(const Dims& d) {
  const int nsplit = d.bf16 ? 1 : 3;
  return nsplit * qfrag_nt(d) * (d.d_c / 16) * 256 + qfrag_nt(d) * 8 * 4;
}

struct SelectWs {
  size_t scores, keys, khist, qfrag, ready_b, ready_t, tcount, sched, qq, total;
};
static inline SelectWs select_workspace(const Dims& d) {
  SelectWs w;
  const size_t pairs = (size_t)d.batch * d.Hkv;
  const size_t kb = (size_t)kb_effective(d);
  w.scores = 0;
  w.keys = a256(pairs * d.Ms * 4);
  w.khist = w.keys + a256(pairs * kb * d.B * 4);
  w.qfrag = w.khist + a256(pairs * kKeyBins * 4);
  w.ready_b = w.qfrag + a256(pairs * (size_t)qfrag_bytes(d));
  w.ready_t = w.ready_b + a256(pairs * 4);
  w.tcount = w.ready_t + a256(pairs * 4);
  w.sched = w.tcount + a256(pairs * 4);
  w.qq = w.sched + a256(256 * 4);
  w.total = w.qq + a256(pairs * 2 * (size_t)d.d_k * 4);
  return w;
}
static inline size_t select_workspace_bytes(const Dims& d) { return select_workspace(d).total; }
// Workspace of tls_sparse_attend with cluster size cs: the CTA partials.
static inline size_t attend_workspace_bytes(const Dims& d, int cs) {
  const size_t pairs = (size_t)d.batch * d.Hkv;
  const size_t o = (pairs * cs * d.G * d.d_v * 4 + 255) & ~(size_t)255;
  const size_t ml = (pairs * cs * d.G * 2 * 4 + 255) & ~(size_t)255;
  return o + ml;
}

}  // namespace tls
