// token.cuh -- a3 helpers shared by the token-scoring kernels (select.cu)
// and the fused selection kernel (fused.cu): the channel-projected query q~
// as mma B fragments, the INT4-code x q~ tensor-core tile, and the
// online-softmax merge.  Citation key: P:n = line n of PAPER.md.
#pragma once

#include <math_constants.h>

#include "common.cuh"
#include "params.h"

namespace tls {

// bf16 piece `sp` of x: x ~= hi + mid + lo (sp = 0, 1, 2), each exact in bf16.
__device__ __forceinline__ float split_piece(float x, int sp) {
  float hi = __bfloat162float(__float2bfloat16_rn(x));
  if (sp == 0) return hi;
  float r1 = x - hi;
  float mid = __bfloat162float(__float2bfloat16_rn(r1));
  if (sp == 1) return mid;
  return __bfloat162float(__float2bfloat16_rn(r1 - mid));
}

// The pair's q-fragment blob (see params.h qfrag_bytes): q~_h[c] = q_h[ch_c]
// for the NT*8 padded heads, packed as K2's mma B fragments in the
// permuted channel order of token_tile_mma, then sum_c q~_h[c].  qc: >= NT*8*d_c
// floats of shared scratch.  Called by all threads of K1b.
// qrows: the pair's G query rows [G][d_k] (global or shared memory); ch: the
// pair's d_c channel ids (global or shared memory).
// [ntlo, nthi): the n-tiles (groups of 8 heads) this CTA builds (a split qq_kernel builds one per CTA).
template <int NB>  // gathers in flight per thread
__device__ inline void build_qfrag(const Dims& d, const void* qrows, const int* ch, uint8_t* qfrag, int pair,
                                   float* qc, int ntlo = 0, int nthi = 4) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt0 = (d.G + 7) / 8, NT = nt0 <= 1 ? 1 : (nt0 <= 2 ? 2 : 4);
  const int DC = d.d_c, KS = DC / 16, WPT = KS / 2, NSPLIT = d.bf16 ? 1 : 3;
  nthi = min(nthi, NT);
  const int ilo = ntlo * 8 * DC, ihi = nthi * 8 * DC;
  for (int i0 = ilo; i0 < ihi; i0 += NB * kThreads) {  // NB independent loads in flight per thread
    float v[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int i = i0 + u * kThreads + tid;
      const int h = i / DC, c = i - h * DC;
      v[u] = 0.f;
      if (i < ihi && h < d.G) {
        const size_t o = (size_t)h * d.d_k + ch[c];
        v[u] = d.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(qrows)[o])
                      : reinterpret_cast<const float*>(qrows)[o];
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int i = i0 + u * kThreads + tid;
      if (i < ihi) qc[i] = v[u];
    }
  }
  __syncthreads();
  const int qfb = NSPLIT * NT * KS * 256 + NT * 32;
  uint32_t* qb = reinterpret_cast<uint32_t*>(qfrag + (size_t)pair * qfb);
  for (int idx = tid; idx < NSPLIT * NT * KS * 32; idx += kThreads) {
    const int ln = idx & 31, rest = idx >> 5;
    const int s = rest % KS, nt = (rest / KS) % NT, sp = rest / (KS * NT);
    if (nt < ntlo || nt >= nthi) continue;
    const float* qh = qc + (nt * 8 + (ln >> 2)) * DC;
    const int cb = 8 * ((ln & 3) * WPT + (s >> 1)) + 2 * (s & 1);
    uint2 v;
    v.x = pack_bf16x2(split_piece(qh[cb], sp), split_piece(qh[cb + 4], sp));
    v.y = pack_bf16x2(split_piece(qh[cb + 1], sp), split_piece(qh[cb + 5], sp));
    reinterpret_cast<uint2*>(qb)[idx] = v;
  }
  float* qsum = reinterpret_cast<float*>(qb + 2 * NSPLIT * NT * KS * 32);
  for (int h = ntlo * 8 + warp; h < nthi * 8; h += kWarps) {
    float sum = 0.f;
    for (int c = lane; c < DC; c += 32) sum += qc[h * DC + c];
    sum = warp_sum(sum);
    if (lane == 0) qsum[h] = sum;
  }
  __syncthreads();  // qc (scratch) is reused by the caller
}

// merge two online-softmax states (m, s) in log2 units
__device__ __forceinline__ void stat_merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  if (nm == -CUDART_INF_F) return;
  s = (m == -CUDART_INF_F ? 0.f : s * fexp2(m - nm)) + (om == -CUDART_INF_F ? 0.f : os * fexp2(om - nm));
  m = nm;
}

// acc[nt][*] = codes(16-token tile at `codes`) x q-fragments, for the NT n-tiles
// of 8 heads.  A = codes (16 tokens x 16 channels per k-step), nibbles -> exact
// bf16; the channel order inside the MMA's K dimension is a permutation
// (thread q4 owns the contiguous code word(s) q4*WPT..), applied identically to
// the B fragments.
// The INT4 code words of one 16-token tile that lane (r0, q4) feeds to the
// mma: rows r0 and r0 + 8, words q4*WPT .. q4*WPT + WPT - 1 of each row.
template <int KS>
struct CodeWords {
  uint32_t w0[KS / 2], w1[KS / 2];
};

// Loads them from `codes` (the tile's first row; shared or global memory).
// Rows with !v0 / !v1 (past the end of the index) are not read and give 0.
template <int KS>
__device__ __forceinline__ void load_code_words(const uint8_t* codes, bool v0, bool v1, CodeWords<KS>& cw) {
  constexpr int WPT = KS / 2;
  constexpr int ROWB = KS * 8;  // d_c / 2
  const int lane = threadIdx.x & 31, q4 = lane & 3, r0 = lane >> 2;
  const uint8_t* p0 = codes + r0 * ROWB + q4 * WPT * 4;
  const uint8_t* p1 = p0 + 8 * ROWB;
  if constexpr (WPT == 4) {
    const uint4 x = v0 ? *reinterpret_cast<const uint4*>(p0) : make_uint4(0, 0, 0, 0);
    const uint4 y = v1 ? *reinterpret_cast<const uint4*>(p1) : make_uint4(0, 0, 0, 0);
    cw.w0[0] = x.x; cw.w0[1] = x.y; cw.w0[2] = x.z; cw.w0[3] = x.w;
    cw.w1[0] = y.x; cw.w1[1] = y.y; cw.w1[2] = y.z; cw.w1[3] = y.w;
  } else if constexpr (WPT == 2) {
    const uint2 x = v0 ? *reinterpret_cast<const uint2*>(p0) : make_uint2(0, 0);
    const uint2 y = v1 ? *reinterpret_cast<const uint2*>(p1) : make_uint2(0, 0);
    cw.w0[0] = x.x; cw.w0[1] = x.y;
    cw.w1[0] = y.x; cw.w1[1] = y.y;
  } else {
    cw.w0[0] = v0 ? *reinterpret_cast<const uint32_t*>(p0) : 0u;
    cw.w1[0] = v1 ? *reinterpret_cast<const uint32_t*>(p1) : 0u;
  }
}

// acc[nt][*] = codes(tile) x q-fragments for the NT n-tiles of 8 heads.
// A = codes (16 tokens x 16 channels per k-step), nibbles -> exact bf16; the
// channel order inside the MMA's K dimension is a permutation (thread q4 owns
// the contiguous code word(s) q4*WPT..), applied identically to the B
// fragments.
template <int KS, int NT, int NSPLIT>
__device__ __forceinline__ void token_mma_words(const CodeWords<KS>& cw, const uint2* qb2, float (&acc)[NT][4]) {
  constexpr int WPT = KS / 2;
  const int lane = threadIdx.x & 31;
  uint32_t a[KS][4];
#pragma unroll
  for (int u = 0; u < WPT; ++u) {
    uint32_t x0[4], x1[4];
    unpack_nibbles8(cw.w0[u], x0);
    unpack_nibbles8(cw.w1[u], x1);
#pragma unroll
    for (int v = 0; v < 2; ++v) {  // k-step 2u+v uses nibble pairs (2v, 2v+4) and (2v+1, 2v+5)
      a[2 * u + v][0] = x0[2 * v];
      a[2 * u + v][1] = x1[2 * v];
      a[2 * u + v][2] = x0[2 * v + 1];
      a[2 * u + v][3] = x1[2 * v + 1];
    }
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
      for (int sp = 0; sp < NSPLIT; ++sp) {
        const uint2 bb = qb2[((sp * NT + nt) * KS + s) * 32 + lane];
        mma_bf16_16816(acc[nt], a[s], bb.x, bb.y);
      }
  }
}

template <int KS, int NT, int NSPLIT>
__device__ __forceinline__ void token_tile_mma(const uint8_t* codes, const uint2* qb2, float (&acc)[NT][4]) {
  CodeWords<KS> cw;
  load_code_words<KS>(codes, true, true, cw);
  token_mma_words<KS, NT, NSPLIT>(cw, qb2, acc);
}

}  // namespace tls
