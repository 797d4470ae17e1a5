// params.h -- host/device parameter blocks and shared-memory plans of the
// three decode-step kernels:
//   K1 block_score_kernel   (select.cu)  a1: block scores -> workspace
//   K2 token_select_kernel  (select.cu)  a2-a4: top-k_b, token scores, top-k_t
//   K3 attend_kernel        (attend.cu)  a5: sparse attention + LSE merge
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace tls {

constexpr int kAttnChunk = 64;     // tokens per K/V staging stage of the GQA mma attention (8 warps x 8)
constexpr int kMlaChunkTokens = 32;  // latent rows per staging chunk of the MLA attention (double-buffered)
constexpr int kScoreTileBytes = 32 * 1024;  // K1: bytes of block summaries per CTA (TMA tile)

struct Dims {
  int batch, Hq, Hkv, G, d_k, d_v, S, B, d_c, Kb, Kt;
  int M;  // ceil(S / B): block-index rows per pair
  float sm_scale;
  int mla;
  int bf16;
  int log2B;  // block_size is a power of two
};

struct ScoreParams {  // K1
  Dims d;
  int tb;  // block-summary rows per CTA (<= kScoreTileBytes)
  const void* q;
  const int* seq_lens;
  const void* block_minmax;
  float* scores;  // workspace [pairs, M] fp32
};

struct SelectParams {  // K2
  Dims d;
  int cs;
  int kb_eff, kt_eff;  // min(Kb, M); min(Kt, kb_eff*B, S)
  int rb;              // candidate blocks per ring stage
  int ring_stage_bytes;
  const void* q;
  const int* seq_lens;
  const float* scores;
  const uint8_t* codes;
  const float* scale_zero;
  const int* channels;
  const int* guide;
  int* block_ids;
  int* token_ids;
  int* num_tokens;
  float* token_scores;
  unsigned long long* dbg;  // diagnostics: per-CTA phase timestamps (NULL = off)
  unsigned off_bkeys, off_cblk, off_qb, off_qsum, off_qc, off_ring, off_tkeys, smem_bytes;
};

struct AttendParams {  // K3
  Dims d;
  int cs;
  int mma;       // 1: bf16 mma.sync GQA path (d in {64,128}, G <= 16); 2: bf16 mma.sync MLA path (576/512)
  int tloc_max;  // ceil(kt_eff / cs)
  const void* q;
  const void* k_cache;
  const void* v_cache;
  const int* token_ids;
  const int* num_tokens;
  void* out;
  float* lse;
  float* part_o;   // workspace [pairs, cs, G, d_v] fp32 partial outputs
  float* part_ml;  // workspace [pairs, cs, G, 2] fp32 partial (max, sum), log2 units
  unsigned off_sel, off_akv, off_aq, off_as, smem_bytes;
};

static inline unsigned align16(size_t x) { return (unsigned)((x + 15) & ~(size_t)15); }

static inline int kb_effective(const Dims& d) { return d.Kb < d.M ? d.Kb : d.M; }
static inline int kt_effective(const Dims& d) {
  const long long cand = (long long)kb_effective(d) * d.B < d.S ? (long long)kb_effective(d) * d.B : d.S;
  return d.Kt < cand ? d.Kt : (int)cand;
}

static inline void plan_select(SelectParams& p) {
  const Dims& d = p.d;
  p.kb_eff = kb_effective(d);
  p.kt_eff = kt_effective(d);
  const int nt0 = (d.G + 7) / 8, nt = nt0 <= 1 ? 1 : (nt0 <= 2 ? 2 : 4);  // instantiated NT
  const int ks = d.d_c / 16, nsplit = d.bf16 ? 1 : 3;
  const int per_block = d.B * (d.d_c / 2 + 8);
  p.rb = (16 * 1024) / per_block;  // ~16 KB per ring stage
  if (p.rb < 1) p.rb = 1;
  p.ring_stage_bytes = (int)align16((size_t)p.rb * per_block);
  size_t o = 0;
  p.off_bkeys = (unsigned)o;
  o = align16(o + (size_t)d.M * 4);
  p.off_cblk = (unsigned)o;
  o = align16(o + (size_t)p.kb_eff * 4);
  p.off_qb = (unsigned)o;
  o = align16(o + (size_t)nsplit * nt * ks * 64 * 4);
  p.off_qsum = (unsigned)o;
  o = align16(o + (size_t)nt * 8 * 4);
  p.off_qc = (unsigned)o;
  o = align16(o + (size_t)nt * 8 * d.d_c * 4);
  o = (o + 127) & ~(size_t)127;
  p.off_ring = (unsigned)o;
  o = align16(o + (size_t)3 * p.ring_stage_bytes);
  p.off_tkeys = (unsigned)o;  // keys of ALL candidate slots of the pair (rank 0 selects)
  o = align16(o + (size_t)p.kb_eff * d.B * 4);
  p.smem_bytes = (unsigned)o;
}

static inline void plan_attend(AttendParams& p) {
  const Dims& d = p.d;
  p.tloc_max = (kt_effective(d) + p.cs - 1) / p.cs;
  size_t o = 0;
  p.off_sel = (unsigned)o;
  o = align16(o + (size_t)(p.tloc_max + 1) * 4);
  if (p.mma == 2) {  // MLA tensor-core path: Q, 2 latent-row chunks, S, P, alpha/m/l
    const int mt16 = d.G <= 16 ? 16 : 32;
    o = (o + 127) & ~(size_t)127;
    p.off_akv = (unsigned)o;
    o += (size_t)mt16 * d.d_k * 2 + (size_t)2 * kMlaChunkTokens * d.d_k * 2;
    o += (size_t)mt16 * (kMlaChunkTokens + 4) * 4 + (size_t)mt16 * (kMlaChunkTokens + 8) * 2 + (size_t)3 * mt16 * 4;
    o = align16(o);
  } else if (p.mma) {
    o = (o + 127) & ~(size_t)127;
    p.off_akv = (unsigned)o;  // 2 stages x (K chunk + V chunk); reused as the warp-partial scratch
    size_t kv = (size_t)2 * 2 * kAttnChunk * d.d_k * 2;
    size_t scratch = (size_t)8 * d.G * (d.d_v + 4) * 4 + (size_t)8 * 16 * 2 * 4;
    o = align16(o + (kv > scratch ? kv : scratch));
  } else {
    p.off_aq = (unsigned)o;
    o = align16(o + (size_t)d.G * d.d_k * 4);
    p.off_as = (unsigned)o;
    o = align16(o + (size_t)d.G * p.tloc_max * 4);
  }
  p.smem_bytes = (unsigned)o;
}

// Workspace of tls_select: K1's fp32 block scores.
static inline size_t select_workspace_bytes(const Dims& d) {
  return ((size_t)d.batch * d.Hkv * d.M * 4 + 255) & ~(size_t)255;
}
// Workspace of tls_sparse_attend with cluster size cs: the CTA partials.
static inline size_t attend_workspace_bytes(const Dims& d, int cs) {
  const size_t pairs = (size_t)d.batch * d.Hkv;
  const size_t o = (pairs * cs * d.G * d.d_v * 4 + 255) & ~(size_t)255;
  const size_t ml = (pairs * cs * d.G * 2 * 4 + 255) & ~(size_t)255;
  return o + ml;
}

}  // namespace tls
