// decode.h -- host/device parameter block and shared-memory plan of the
// fused two-level selection + sparse attention kernel (decode.cu).
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace tls {

struct DecodeParams {
  // ---- problem (tls_config) ----
  int batch, Hq, Hkv, G, d_k, d_v, S, B, d_c, Kb, Kt;
  int M;  // ceil(S / B): block-index rows per pair
  float sm_scale;
  int mla;
  // ---- launch plan ----
  int cs;         // CTAs per pair = cluster size
  int do_select;  // phases A-D (tls_select)
  int do_attend;  // phase E (tls_sparse_attend)
  int attn_mma;   // 1: bf16 mma.sync attention, 0: generic CUDA-core attention
  int nt;         // ceil(G / 8): n-tiles of query heads in token scoring
  int nsplit;     // bf16 pieces per query value in token scoring (1 bf16, 3 fp32)
  int ksteps;     // d_c / 16
  int wpt;        // d_c / 32: 32-bit code words per thread and row
  int mloc_max;   // ceil(M / cs)
  int cblk_loc_max;  // ceil(Kb / cs)
  int lc_max;     // cblk_loc_max * B candidate slots per CTA
  int ls;         // logits row stride (floats)
  int tloc_max;   // ceil(Kt / cs) attended tokens per CTA
  // ---- tensors ----
  const void* q;
  const void* k_cache;
  const void* v_cache;
  const int* seq_lens;
  const void* block_minmax;
  const uint8_t* codes;
  const float* scale_zero;
  const int* channels;
  const int* guide;
  int* block_ids;
  int* token_ids;
  int* num_tokens;
  float* token_scores;
  void* out;
  float* lse;
  // ---- dynamic shared-memory plan (byte offsets) ----
  unsigned off_sel, off_cblk, off_union;
  unsigned off_qq, off_bkeys, off_qb, off_qsum, off_logits, off_tkeys;  // select
  unsigned off_aq, off_as, off_ao;                                      // attend (generic)
  unsigned smem_bytes;
};

static inline unsigned align16(size_t x) { return (unsigned)((x + 15) & ~(size_t)15); }

// Fill the shared-memory plan of `p` (dims, cs, modes already set).
static inline void plan_decode_smem(DecodeParams& p, size_t elem_bytes) {
  p.mloc_max = (p.M + p.cs - 1) / p.cs;
  p.cblk_loc_max = (p.Kb + p.cs - 1) / p.cs;
  p.lc_max = p.cblk_loc_max * p.B;
  p.ls = p.lc_max + 4;  // 4h + j bank pattern: conflict-free epilogue stores
  p.tloc_max = (p.Kt + p.cs - 1) / p.cs;
  p.nt = (p.G + 7) / 8;
  p.ksteps = p.d_c / 16;
  p.wpt = p.d_c / 32;
  size_t o = 0;
  p.off_sel = (unsigned)o;
  o = align16(o + (size_t)(p.tloc_max + 1) * 4);
  p.off_cblk = (unsigned)o;
  o = align16(o + (size_t)p.Kb * 4);
  p.off_union = (unsigned)o;
  size_t sel_end = o, att_end = o;
  if (p.do_select) {
    size_t s = o;
    p.off_qq = (unsigned)s;
    s = align16(s + (size_t)2 * p.d_k * 4);
    p.off_bkeys = (unsigned)s;
    s = align16(s + (size_t)p.mloc_max * 4);
    p.off_qb = (unsigned)s;
    s = align16(s + (size_t)p.nsplit * p.nt * p.ksteps * 64 * 4);
    p.off_qsum = (unsigned)s;
    s = align16(s + (size_t)p.nt * 8 * 4);
    p.off_logits = (unsigned)s;
    s = align16(s + (size_t)p.G * p.ls * 4);
    p.off_tkeys = (unsigned)s;
    s = align16(s + (size_t)p.lc_max * 4);
    sel_end = s;
  }
  if (p.do_attend) {
    size_t s = o;
    p.off_aq = (unsigned)s;
    s = align16(s + (size_t)p.G * p.d_k * 4);
    p.off_as = (unsigned)s;
    s = align16(s + (size_t)p.G * p.tloc_max * 4);
    p.off_ao = (unsigned)s;
    s = align16(s + (size_t)p.G * p.d_v * 4);
    att_end = s;
  }
  (void)elem_bytes;
  p.smem_bytes = (unsigned)(sel_end > att_end ? sel_end : att_end);
}

}  // namespace tls
