// attend.cu -- sparse attention over the selected tokens
// for sm_100a: K3 attend_kernel, one thread-block cluster of cs CTAs per
// (batch, KV-head) pair, each CTA a 1/cs slice of the pair's k_t tokens
// (split-K flash decoding); the cs partials go to an L2-resident workspace,
// one cluster barrier, then every CTA merges a slice with the LSE identity (T10).
// bf16 GQA with head dim 64/128 runs on tensor cores (mma.sync), MLA on
// attend_mla_kernel (mma.sync; tcgen05 + TMEM form opt-in, TLS_MLA_TC=1), fp32
// on the generic CUDA-core path.
#include <math_constants.h>

#include <type_traits>

#include "common.cuh"
#include "fasttopk.cuh"
#include "params.h"
#include "launch.h"
#include "topk.cuh"
#include "tokensel.cuh"

namespace tls {

// --------------------------------------------------------------------------
// a4 prologue: S_t = top-k_t tokens from the ranking keys the
// token kernels left in the workspace, ties -> lower token id (U2).  Every CTA
// of the pair's cluster selects redundantly from identical keys; rank 0
// writes token_ids / token_scores / num_tokens, and each CTA keeps its own
// slice [t0, t1) of the selected ids in `sel`.  Returns K = |S_t|.
// --------------------------------------------------------------------------
static __device__ int select_tokens_prologue(const AttendParams& p, int pair, int b, unsigned rank, uint8_t* smem, int* sel,
                                             TopKCtl& tk) {
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cs = p.cs;
  const int n = min(max(p.seq_lens[b], 0), d.S);
  const int m = (n + d.B - 1) >> d.log2B;
  int* cblk = reinterpret_cast<int*>(smem + p.off_cblk);
  uint32_t* skeys = reinterpret_cast<uint32_t*>(smem + p.off_skeys);
  uint32_t* scratch = skeys + p.kb_eff * d.B;
  uint32_t* shist = scratch + 2048;
  FastTopKCtl& fk = *reinterpret_cast<FastTopKCtl*>(smem + p.off_fk);
  __shared__ int s_kc;
  unsigned long long* dbg = (p.dbg && rank == 0) ? p.dbg + (size_t)pair * 8 : nullptr;
#define TLS_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TLS_STAMP(0)
  // keys of every candidate slot (the whole region; only the first kc blocks' slots are read) and the key
  // histogram: two TMA bulk copies, issued first so they overlap the candidate compaction below
  __shared__ __align__(8) uint64_t kbar;
  if (tid == 0) {
    const uint32_t kbytes = (uint32_t)(p.kb_eff * d.B * 4);
    mbar_init(&kbar, 1);
    mbar_fence_init();
    mbar_arrive_expect_tx(&kbar, kbytes + kKeyBins * 4);
    tma_bulk_g2s(shist, p.khist + (size_t)pair * kKeyBins, kKeyBins * 4, &kbar);
    tma_bulk_g2s(skeys, p.keys + (size_t)pair * p.kb_eff * d.B, kbytes, &kbar);
  }
  // candidate blocks in the order the token kernels used (valid entries, in order)
  const int* cand = p.cand + (size_t)pair * d.Kb;
  {
    const int per = (d.Kb + kThreads - 1) / kThreads;
    const int lo = min(tid * per, d.Kb), hi = min(lo + per, d.Kb);
    int cnt = 0;
    for (int i = lo; i < hi; ++i) cnt += (cand[i] >= 0 && cand[i] < m);
    int total;
    int pos = block_exclusive_scan(cnt, tk.scan, &total);  // (its barriers also order the mbarrier init)
    for (int i = lo; i < hi; ++i)
      if (cand[i] >= 0 && cand[i] < m && pos < p.kb_eff) cblk[pos++] = cand[i];
    if (tid == 0) s_kc = min(total, p.kb_eff);
  }
  __syncthreads();
  const int nslots = s_kc << d.log2B;
  mbar_wait(&kbar, 0);
  TLS_STAMP(1)
  TLS_STAMP(2)
  __shared__ HistSel hs;
  // every CTA selects the same S_t; CTA rank keeps positions [t0, t1) of it
  int* tout = p.token_ids + (size_t)pair * d.Kt;
  float* sout = p.token_scores ? p.token_scores + (size_t)pair * d.Kt : nullptr;
  const float lnG = logf((float)d.G);
  const int* sob = p.slot_of_block ? p.slot_of_block + (size_t)pair * d.M : nullptr;  // block cache rows
  int t0 = 0, t1 = 0;
  auto on_k = [&](int K) {
    t0 = K * (int)rank / cs;  // K <= top_tokens, cs <= 16: no overflow
    t1 = K * ((int)rank + 1) / cs;
  };
  auto put = [&](int i, int pos) {
    const int tok = (cblk[i >> d.log2B] << d.log2B) + (i & (d.B - 1));
    if (rank == 0) {
      tout[pos] = tok;
      if (sout) sout[pos] = key2f(skeys[i]) * kLn2 - lnG;
    }
    if (pos >= t0 && pos < t1) {
      // block cache: row of the token's slot (a non-resident block -- a caller error, the guide must be resident --
      // reads row 0 instead of out of bounds)
      const int sl = sob ? sob[tok >> d.log2B] : 0;
      sel[pos - t0] = sob ? (sl >= 0 ? (sl << d.log2B) + (tok & (d.B - 1)) : 0) : tok;
    }
  };
  int* slist = reinterpret_cast<int*>(smem + p.off_slist);
  int K;
  if (nslots <= kSelRunMax * kThreads) {
    K = hist_topk_select(skeys, nslots, shist, d.Kt, scratch, fk, tk, hs, slist, on_k, put, dbg);
  } else {
    const HistPlan pl = hist_topk_plan(skeys, nslots, shist, d.Kt, scratch, fk, tk, hs, dbg);
    K = pl.K;
    on_k(K);
    hist_topk_emit(skeys, nslots, pl, hs, tk, slist, put);
  }
  TLS_STAMP(3)
  if (rank == 0) {
    for (int pos = K + tid; pos < d.Kt; pos += kThreads) {
      tout[pos] = -1;
      if (sout) sout[pos] = -CUDART_INF_F;
    }
    if (tid == 0) p.num_tokens[pair] = K;
  }
  __syncthreads();
  TLS_STAMP(4)
#undef TLS_STAMP
  return K;
}

// --------------------------------------------------------------------------
// Output element idx of the pair's [G, d_v] block: the cfg dtype, or fp32 when the caller asked for fp32
// partials (tls_sparse_attend_f32: the sequence-split merge then rounds once).
template <typename T>
__device__ __forceinline__ void store_out(const AttendParams& p, T* outg, int idx, float v) {
  if (p.out_f32) {
    const size_t off = (size_t)(reinterpret_cast<const char*>(outg) - reinterpret_cast<const char*>(p.out)) / sizeof(T);
    reinterpret_cast<float*>(p.out)[off + idx] = v;
  } else {
    outg[idx] = from_f32<T>(v);
  }
}

// Phase E (generic CUDA-core path): partial attention of this CTA over its
// tokens sel[0..tloc) for the G heads of the pair, log2 domain.
// Leaves (am_h, al_h) in ctl and the unnormalised partial o in ao.
// --------------------------------------------------------------------------
template <typename T>
__device__ void phase_attend_generic(const AttendParams& p, int pair, int b, int g, const int* sel, int tloc,
                                     float* aq, float* as, float* po, float* pml) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T* qg = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * p.d.d_k;
  for (int i = tid; i < p.d.G * p.d.d_k; i += kThreads) aq[i] = to_f32<T>(qg[i]);
  __syncthreads();
  const T* kb = reinterpret_cast<const T*>(p.k_cache) + (size_t)pair * p.kv_rows * p.d.d_k;
  const T* vb = p.d.mla ? kb : reinterpret_cast<const T*>(p.v_cache) + (size_t)pair * p.kv_rows * p.d.d_v;
  const int vstride = p.d.mla ? p.d.d_k : p.d.d_v;
  const float sm2 = p.d.sm_scale * kLog2e;
  for (int t = warp; t < tloc; t += kWarps) {
    const T* krow = kb + (size_t)sel[t] * p.d.d_k;
    for (int h = 0; h < p.d.G; ++h) {
      float acc = 0.f;
      for (int e = lane; e < p.d.d_k; e += 32) acc = fmaf(aq[h * p.d.d_k + e], to_f32<T>(krow[e]), acc);
      acc = warp_sum(acc);
      if (lane == 0) as[h * p.tloc_max + t] = acc * sm2;
    }
  }
  __syncthreads();
  for (int h = warp; h < p.d.G; h += kWarps) {
    float mx = -CUDART_INF_F;
    for (int t = lane; t < tloc; t += 32) mx = fmaxf(mx, as[h * p.tloc_max + t]);
    mx = warp_max(mx);
    float l = 0.f;
    for (int t = lane; t < tloc; t += 32) {
      const float e = fexp2(as[h * p.tloc_max + t] - mx);
      as[h * p.tloc_max + t] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      pml[2 * h] = mx;
      pml[2 * h + 1] = l;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < p.d.G * p.d.d_v; idx += kThreads) {
    const int h = idx / p.d.d_v, c = idx - h * p.d.d_v;
    float acc = 0.f;
    for (int t = 0; t < tloc; ++t) acc = fmaf(as[h * p.tloc_max + t], to_f32<T>(vb[(size_t)sel[t] * vstride + c]), acc);
    po[idx] = acc;
  }
}

// --------------------------------------------------------------------------
// Phase E (tensor-core path, bf16 GQA, head dim D): FlashAttention-2 style
// split-K decode over this CTA's tokens sel[0..tloc).  Heads are the M rows of
// mma.sync m16n8k16 (G <= 16, padded), tokens the N / K dimension.  K and V
// rows of a 128-token chunk are gathered into XOR-swizzled shared memory with
// cp.async (16 B per op), read back with ldmatrix (.trans for V); each warp
// owns 16 tokens of the chunk and keeps its own online softmax state; the 8
// warp partials are merged in smem, then the cs CTA partials over DSMEM.
// --------------------------------------------------------------------------
template <int D>
__device__ void phase_attend_mma(const AttendParams& p, int pair, int b, int g, const int* sel, int tloc,
                                 uint8_t* kvbuf, float* po, float* pml) {
  constexpr int TC = kAttnChunk;  // 64 tokens per stage: 8 warps x 8 tokens
  constexpr int CPR = D / 8;      // 16-byte chunks per row
  constexpr int KS = D / 16;      // k-steps of QK^T
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, c2 = 2 * (lane & 3);
  __nv_bfloat16* sbuf = reinterpret_cast<__nv_bfloat16*>(kvbuf);  // [kAttnStages][K TC*D | V TC*D]
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * D;
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * D;
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) + (size_t)pair * p.kv_rows * D;
  const int nchunks = (tloc + TC - 1) / TC;
  // thread tid copies 16-byte chunk tid % CPR of rows tid / CPR + (kThreads / CPR) * it: a fixed column and
  // swizzle (row & 7 is the same for every it), so per row only the token id and two addresses change
  static_assert(kThreads % CPR == 0 && (kThreads / CPR) % 8 == 0, "fixed swizzle per thread");
  const int lch = tid % CPR, lrow = tid / CPR;
  const uint32_t sdst = smem_u32(sbuf) + (uint32_t)(lrow * D + ((lch ^ (lrow & 7)) << 3)) * 2u;
  const __nv_bfloat16* kcol = kb + lch * 8;
  const __nv_bfloat16* vcol = vb + lch * 8;
  auto load_chunk = [&](int c, int stage) {
    const uint32_t dK = sdst + (uint32_t)stage * (2 * TC * D * 2), dV = dK + TC * D * 2;
    const int nt = min(TC, tloc - c * TC);
    const int* sc = sel + c * TC + lrow;
#pragma unroll
    for (int it = 0; it < (TC * CPR) / kThreads; ++it) {
      const int row = lrow + it * (kThreads / CPR);
      const bool ok = row < nt;
      const size_t tok = (size_t)(ok ? sc[it * (kThreads / CPR)] : 0) * D;
      const uint32_t o = (uint32_t)(it * (kThreads / CPR) * D * 2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dK + o), "l"(kcol + tok), "r"(ok ? 16 : 0));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dV + o), "l"(vcol + tok), "r"(ok ? 16 : 0));
    }
    cp_async_commit();
  };
  // kAttnStages-deep cp.async pipeline: kAttnStages - 1 chunks in flight while one is used
#pragma unroll
  for (int c = 0; c < kAttnStages - 1; ++c) {
    if (c < nchunks) load_chunk(c, c);
    else cp_async_commit();
  }
  // Q as the A operand (rows = heads; rows >= G are zero)
  uint32_t qa[KS][4];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int col = kk * 16 + c2;
    qa[kk][0] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + col) : 0u;
    qa[kk][1] = r + 8 < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + (r + 8) * D + col) : 0u;
    qa[kk][2] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + col + 8) : 0u;
    qa[kk][3] = r + 8 < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + (r + 8) * D + col + 8) : 0u;
  }
  const float sm2 = p.d.sm_scale * kLog2e;
  float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
  float o[D / 8][4];
#pragma unroll
  for (int j = 0; j < D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

  for (int c = 0; c < nchunks; ++c) {
    if (c + kAttnStages - 1 < nchunks) load_chunk(c + kAttnStages - 1, (c + kAttnStages - 1) % kAttnStages);
    else cp_async_commit();
    cp_async_wait<kAttnStages - 1>();
    __syncthreads();  // chunk c landed for every thread's copies
    const __nv_bfloat16* sK = sbuf + (size_t)(c % kAttnStages) * 2 * TC * D;
    const __nv_bfloat16* sV = sK + TC * D;
    const int nt = min(TC, tloc - c * TC);
    const int tb = warp * 8;
    if (tb < nt) {
      // S (16 head rows x 8 tokens) = Q K^T
      float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < KS; kk += 2) {
        const int row = tb + (lane & 7);
        const int ch = kk * 2 + (lane >> 3);  // 4 matrices: k-steps kk (b0, b1) and kk+1 (b0, b1)
        uint32_t bk[4];
        ldsm_x4(bk, sK + row * D + ((ch ^ (row & 7)) << 3));
        mma_bf16_16816(s, qa[kk], bk[0], bk[1]);
        mma_bf16_16816(s, qa[kk + 1], bk[2], bk[3]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t = tb + c2 + (e & 1);
        s[e] = t < nt ? s[e] * sm2 : -CUDART_INF_F;
      }
      float x0 = fmaxf(s[0], s[1]), x1 = fmaxf(s[2], s[3]);
      x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 1));
      x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, 2));
      x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 1));
      x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, 2));
      // lazy rescaling: the running reference max moves only when a score exceeds it by more than
      // 8 (log2 units); p = 2^(s - m) <= 2^8 stays well inside fp32 / bf16 and o / l is unchanged,
      // so most chunks skip the rescale of the 64 accumulators
      const bool g0 = x0 > m0 + 8.f, g1 = x1 > m1 + 8.f;  // m = -inf at first: true (token tb is valid)
      const float n0 = g0 ? x0 : m0, n1 = g1 ? x1 : m1;
      const float a0 = g0 ? fexp2(m0 - n0) : 1.f, a1 = g1 ? fexp2(m1 - n1) : 1.f;
      const float p0 = fexp2(s[0] - n0), p1 = fexp2(s[1] - n0), p2 = fexp2(s[2] - n1), p3 = fexp2(s[3] - n1);
      float r0s = p0 + p1, r1s = p2 + p3;
      r0s += __shfl_xor_sync(0xffffffffu, r0s, 1);
      r0s += __shfl_xor_sync(0xffffffffu, r0s, 2);
      r1s += __shfl_xor_sync(0xffffffffu, r1s, 1);
      r1s += __shfl_xor_sync(0xffffffffu, r1s, 2);
      l0 = l0 * a0 + r0s;
      l1 = l1 * a1 + r1s;
      m0 = n0;
      m1 = n1;
      if (__any_sync(0xffffffffu, g0 || g1)) {
#pragma unroll
        for (int j = 0; j < D / 8; ++j) {
          o[j][0] *= a0;
          o[j][1] *= a0;
          o[j][2] *= a1;
          o[j][3] *= a1;
        }
      }
      // P (16 x 16, tokens 8..15 of the k-step zero) x V (8 tokens of this warp)
      uint32_t pa[4];
      pa[0] = pack_bf16x2(p0, p1);
      pa[1] = pack_bf16x2(p2, p3);
      pa[2] = 0u;
      pa[3] = 0u;
#pragma unroll
      for (int jj = 0; jj < D / 32; ++jj) {
        const int row = tb + (lane & 7);
        const int ch = jj * 4 + (lane >> 3);  // dims 32jj + 8*(lane>>3): 4 n-tiles
        uint32_t bv[4];
        ldsm_x4_trans(bv, sV + row * D + ((ch ^ (row & 7)) << 3));
        mma_bf16_16816(o[4 * jj + 0], pa, bv[0], 0u);
        mma_bf16_16816(o[4 * jj + 1], pa, bv[1], 0u);
        mma_bf16_16816(o[4 * jj + 2], pa, bv[2], 0u);
        mma_bf16_16816(o[4 * jj + 3], pa, bv[3], 0u);
      }
    }
    __syncthreads();  // stage c % kAttnStages consumed before it is refilled
  }
  cp_async_wait<0>();
  // ---- merge the 8 warp partials (the staging buffers become scratch) ----
  constexpr int WS = D + 4;  // padded row stride of the warp partials
  float* wo = reinterpret_cast<float*>(kvbuf);  // [warp][G][WS]
  float* wml = wo + kWarps * p.d.G * WS;        // [warp][16][2]
  if ((lane & 3) == 0) {
    wml[(warp * 16 + r) * 2] = m0;
    wml[(warp * 16 + r) * 2 + 1] = l0;
    wml[(warp * 16 + r + 8) * 2] = m1;
    wml[(warp * 16 + r + 8) * 2 + 1] = l1;
  }
#pragma unroll
  for (int j = 0; j < D / 8; ++j) {
    const int d = j * 8 + c2;
    if (r < p.d.G) *reinterpret_cast<float2*>(wo + (warp * p.d.G + r) * WS + d) = make_float2(o[j][0], o[j][1]);
    if (r + 8 < p.d.G)
      *reinterpret_cast<float2*>(wo + (warp * p.d.G + r + 8) * WS + d) = make_float2(o[j][2], o[j][3]);
  }
  __syncthreads();
  const bool direct = p.cs == 1;  // one CTA per pair: normalise and write the output here
  __nv_bfloat16* outg =
      reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * p.d.d_v;
  for (int idx = tid; idx < p.d.G * D; idx += kThreads) {
    const int h = idx / D, dcol = idx - h * D;
    float M = -CUDART_INF_F;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, wml[(w * 16 + h) * 2]);
    float L = 0.f, acc = 0.f;
    if (M != -CUDART_INF_F) {
      for (int w = 0; w < kWarps; ++w) {
        const float mw = wml[(w * 16 + h) * 2];
        const float sc = mw == -CUDART_INF_F ? 0.f : fexp2(mw - M);
        L = fmaf(wml[(w * 16 + h) * 2 + 1], sc, L);
        acc = fmaf(wo[(w * p.d.G + h) * WS + dcol], sc, acc);
      }
    }
    if (direct) {
      store_out(p, outg, idx, L > 0.f ? acc / L : 0.f);
      if (dcol == 0 && p.lse != nullptr)
        p.lse[(size_t)b * p.d.Hq + (size_t)g * p.d.G + h] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
    } else {
      po[idx] = acc;
      if (dcol == 0) {
        pml[2 * h] = M;
        pml[2 * h + 1] = L;
      }
    }
  }
}

// --------------------------------------------------------------------------
// Phase E, tokens-as-M tensor-core form (bf16 GQA, D = 128, G <= 8): the
// group's G heads fill the N = 8 side of mma.sync m16n8k16 exactly, instead of
// half of a 16-row M tile.  Warp w owns the 16 tokens 16*(w/2) .. +15 of each
// 64-token chunk and the output dims 64*(w%2) .. +63:
//   S^T (16 tokens x 8 heads) = K Q^T      8 k-steps: A = K rows (ldmatrix),
//                                          B = Q^T fragments held in registers
//   online softmax per head over the tokens (lazy rescaling as above); P^T
//   goes through a 256-byte per-warp buffer into the B layout
//   O^T (64 dims x 8 heads) += V^T P^T     4 m-tiles: A = V^T (ldmatrix.trans)
// 12 mma per warp per chunk instead of 24, 16 accumulator registers instead of
// 64.  The two warps of a token group compute the same S^T (no exchange).  At
// the end the 4 token groups' partials merge in shared memory.
// --------------------------------------------------------------------------
template <int D>
__device__ void phase_attend_mma_t(const AttendParams& p, int pair, int b, int g, const int* sel, int tloc,
                                   uint8_t* kvbuf, float* po, float* pml) {
  static_assert(D == 128, "tokens-as-M attention: D = 128");
  constexpr int TC = kAttnChunk;  // 64 tokens per stage
  constexpr int CPR = D / 8;      // 16-byte chunks per row
  constexpr int KS = D / 16;      // k-steps of K Q^T
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int tg = warp >> 1, dh = warp & 1;
  __nv_bfloat16* sbuf = reinterpret_cast<__nv_bfloat16*>(kvbuf);  // [kAttnStages][K TC*D | V TC*D]
  __nv_bfloat16* pbuf = reinterpret_cast<__nv_bfloat16*>(kvbuf + (size_t)kAttnStages * 2 * TC * D * 2) + warp * 128;
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * D;
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * D;
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(p.v_cache) + (size_t)pair * p.kv_rows * D;
  const int nchunks = (tloc + TC - 1) / TC;
  auto load_chunk = [&](int c, int stage) {
    __nv_bfloat16* sK = sbuf + (size_t)stage * 2 * TC * D;
    __nv_bfloat16* sV = sK + TC * D;
    const int nt = min(TC, tloc - c * TC);
#pragma unroll
    for (int it = 0; it < (TC * CPR) / kThreads; ++it) {
      const int i = tid + it * kThreads;
      const int row = i / CPR, ch = i - row * CPR;
      const bool ok = row < nt;
      const int tok = ok ? sel[c * TC + row] : 0;
      const int dst = row * D + ((ch ^ (row & 7)) << 3);
      cp_async16(sK + dst, kb + (size_t)tok * D + ch * 8, ok);
      cp_async16(sV + dst, vb + (size_t)tok * D + ch * 8, ok);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int c = 0; c < kAttnStages - 1; ++c) {
    if (c < nchunks) load_chunk(c, c);
    else cp_async_commit();
  }
  // Q^T as the B operand: b0 = Q[head r][16k + 2q, +1], b1 = Q[head r][16k + 2q + 8, +9] (heads >= G: 0)
  uint32_t qb[KS][2];
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    qb[k][0] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + 16 * k + 2 * q) : 0u;
    qb[k][1] = r < p.d.G ? *reinterpret_cast<const uint32_t*>(qg + r * D + 16 * k + 2 * q + 8) : 0u;
  }
  const float sm2 = p.d.sm_scale * kLog2e;
  float m[2] = {-CUDART_INF_F, -CUDART_INF_F}, l[2] = {0.f, 0.f};  // heads 2q, 2q + 1 over this warp's tokens
  float o[4][4];  // O^T: m-tile mt = dims 64*dh + 16*mt + (r, r + 8), heads (2q, 2q + 1)
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<kAttnStages - 2>();
    // one barrier per chunk: chunk c landed for every thread's copies, and every warp finished chunk c - 1, whose
    // stage the refill below overwrites
    __syncthreads();
    if (c + kAttnStages - 1 < nchunks) load_chunk(c + kAttnStages - 1, (c + kAttnStages - 1) % kAttnStages);
    else cp_async_commit();
    const __nv_bfloat16* sK = sbuf + (size_t)(c % kAttnStages) * 2 * TC * D;
    const __nv_bfloat16* sV = sK + TC * D;
    const int nt = min(TC, tloc - c * TC);
    const int t0 = tg * 16;
    if (t0 < nt) {
      // ---- S^T (16 tokens x 8 heads) = K Q^T ----
      float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const int row = t0 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int ch = 2 * k + (lane >> 4);
        uint32_t a[4];
        ldsm_x4(a, sK + row * D + ((ch ^ (row & 7)) << 3));
        mma_bf16_16816(s, a, qb[k][0], qb[k][1]);
      }
      // s = S^T[token t0 + r][heads 2q, 2q + 1], S^T[token t0 + r + 8][...]
      const bool v0 = t0 + r < nt, v1 = t0 + r + 8 < nt;
      s[0] = v0 ? s[0] * sm2 : -CUDART_INF_F;
      s[1] = v0 ? s[1] * sm2 : -CUDART_INF_F;
      s[2] = v1 ? s[2] * sm2 : -CUDART_INF_F;
      s[3] = v1 ? s[3] * sm2 : -CUDART_INF_F;
      float x0 = fmaxf(s[0], s[2]), x1 = fmaxf(s[1], s[3]);  // per head, over the lane's two tokens
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
        x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
      }
      // lazy rescaling (x is finite: token t0 is valid)
      const bool g0 = x0 > m[0] + 8.f, g1 = x1 > m[1] + 8.f;
      const float n0 = g0 ? x0 : m[0], n1 = g1 ? x1 : m[1];
      const float a0 = g0 ? fexp2(m[0] - n0) : 1.f, a1 = g1 ? fexp2(m[1] - n1) : 1.f;
      const float p0 = fexp2(s[0] - n0), p1 = fexp2(s[1] - n1), p2 = fexp2(s[2] - n0), p3 = fexp2(s[3] - n1);
      float r0s = p0 + p2, r1s = p1 + p3;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        r0s += __shfl_xor_sync(0xffffffffu, r0s, off);
        r1s += __shfl_xor_sync(0xffffffffu, r1s, off);
      }
      l[0] = l[0] * a0 + r0s;
      l[1] = l[1] * a1 + r1s;
      m[0] = n0;
      m[1] = n1;
      if (__any_sync(0xffffffffu, g0 || g1)) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          o[mt][0] *= a0;
          o[mt][1] *= a1;
          o[mt][2] *= a0;
          o[mt][3] *= a1;
        }
      }
      // ---- P^T into the B layout: P[head][token] in a per-warp buffer ----
      pbuf[(2 * q) * 16 + r] = __float2bfloat16_rn(p0);
      pbuf[(2 * q + 1) * 16 + r] = __float2bfloat16_rn(p1);
      pbuf[(2 * q) * 16 + r + 8] = __float2bfloat16_rn(p2);
      pbuf[(2 * q + 1) * 16 + r + 8] = __float2bfloat16_rn(p3);
      __syncwarp();
      const uint32_t pb0 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q);
      const uint32_t pb1 = *reinterpret_cast<const uint32_t*>(pbuf + r * 16 + 2 * q + 8);
      __syncwarp();
      // ---- O^T (64 dims x 8 heads) += V^T (dims x 16 tokens) P^T ----
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int token = t0 + (lane & 7) + ((lane >> 4) & 1) * 8;
        const int ch = (dh * 64 + 16 * mt) / 8 + ((lane >> 3) & 1);
        uint32_t a[4];
        ldsm_x4_trans(a, sV + token * D + ((ch ^ (token & 7)) << 3));
        mma_bf16_16816(o[mt], a, pb0, pb1);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp done with the last stage
  // ---- merge the 4 token groups (the staging buffers become scratch) ----
  constexpr int WS = D + 4;
  float* wo = reinterpret_cast<float*>(kvbuf);  // [tg][8 heads][WS]
  float* wml = wo + 4 * 8 * WS;                  // [tg][8 heads][2]
  if (dh == 0 && r == 0) {
    wml[(tg * 8 + 2 * q) * 2] = m[0];
    wml[(tg * 8 + 2 * q) * 2 + 1] = l[0];
    wml[(tg * 8 + 2 * q + 1) * 2] = m[1];
    wml[(tg * 8 + 2 * q + 1) * 2 + 1] = l[1];
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int d0 = dh * 64 + 16 * mt + r;
    wo[(tg * 8 + 2 * q) * WS + d0] = o[mt][0];
    wo[(tg * 8 + 2 * q + 1) * WS + d0] = o[mt][1];
    wo[(tg * 8 + 2 * q) * WS + d0 + 8] = o[mt][2];
    wo[(tg * 8 + 2 * q + 1) * WS + d0 + 8] = o[mt][3];
  }
  __syncthreads();
  const bool direct = p.cs == 1;
  __nv_bfloat16* outg =
      reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)b * p.d.Hq + (size_t)g * p.d.G) * p.d.d_v;
  const int ngroups = min(4, (min(tloc, TC) + 15) / 16);  // token groups that saw at least one token
  for (int idx = tid; idx < p.d.G * D; idx += kThreads) {
    const int h = idx / D, dcol = idx - h * D;
    float M = -CUDART_INF_F;
    for (int t = 0; t < ngroups; ++t) M = fmaxf(M, wml[(t * 8 + h) * 2]);
    float L = 0.f, acc = 0.f;
    if (M != -CUDART_INF_F) {
      for (int t = 0; t < ngroups; ++t) {
        const float mw = wml[(t * 8 + h) * 2];
        const float sc = mw == -CUDART_INF_F ? 0.f : fexp2(mw - M);
        L = fmaf(wml[(t * 8 + h) * 2 + 1], sc, L);
        acc = fmaf(wo[(t * 8 + h) * WS + dcol], sc, acc);
      }
    }
    if (direct) {
      store_out(p, outg, idx, L > 0.f ? acc / L : 0.f);
      if (dcol == 0 && p.lse != nullptr)
        p.lse[(size_t)b * p.d.Hq + (size_t)g * p.d.G + h] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
    } else {
      po[idx] = acc;
      if (dcol == 0) {
        pml[2 * h] = M;
        pml[2 * h + 1] = L;
      }
    }
  }
}

// Merge the cs CTA partials of the pair (flash-decoding LSE merge, T10) from
// the L2-resident workspace and write out / lse; CTA `rank` writes a 1/cs
// slice of the G*d_v outputs.
template <typename T, int U>
__device__ void phase_merge(const AttendParams& p, int pair, int b, int g, unsigned rank) {
  // per-head merge weights once (G <= 32 heads, cs <= 16 partials), then every
  // output element is a cs-term dot product with its loads batched ahead (U
  // elements per thread per step)
  __shared__ float s_w[16][32], s_inv[32];
  const int G = p.d.G, cs = p.cs;
  const int tot = G * p.d.d_v;
  const int lo = (int)((long long)tot * rank / cs), hi = (int)((long long)tot * (rank + 1) / cs);
  const float* po = p.part_o + (size_t)pair * cs * tot;
  const float* pml = p.part_ml + (size_t)pair * cs * G * 2;
  T* outg = reinterpret_cast<T*>(p.out) + ((size_t)b * p.d.Hq + (size_t)g * G) * p.d.d_v;
  if ((int)threadIdx.x < G) {
    const int h = threadIdx.x;
    float M = -CUDART_INF_F;
    for (int rr = 0; rr < cs; ++rr) M = fmaxf(M, __ldcg(pml + (rr * G + h) * 2));
    float L = 0.f;
    for (int rr = 0; rr < cs; ++rr) {
      const float mr = __ldcg(pml + (rr * G + h) * 2);
      const float w = (M == -CUDART_INF_F || mr == -CUDART_INF_F) ? 0.f : fexp2(mr - M);
      L = fmaf(__ldcg(pml + (rr * G + h) * 2 + 1), w, L);
      s_w[rr][h] = w;
    }
    s_inv[h] = L > 0.f ? 1.f / L : 0.f;
    if (rank == 0 && p.lse != nullptr)
      p.lse[(size_t)b * p.d.Hq + (size_t)g * G + h] = L > 0.f ? (M + flog2(L)) * kLn2 : -CUDART_INF_F;
  }
  __syncthreads();
  if constexpr (U == 1) {
    for (int idx = lo + (int)threadIdx.x; idx < hi; idx += kThreads) {
      const int h = idx / p.d.d_v;
      float o = 0.f;
#pragma unroll 4
      for (int rr = 0; rr < cs; ++rr) o = fmaf(__ldcg(po + (size_t)rr * tot + idx), s_w[rr][h], o);
      store_out(p, outg, idx, o * s_inv[h]);
    }
  } else {
    for (int i0 = lo; i0 < hi; i0 += U * kThreads) {
      float v[U][16];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * kThreads + (int)threadIdx.x;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) v[u][rr] = (rr < cs && idx < hi) ? __ldcg(po + (size_t)rr * tot + idx) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = i0 + u * kThreads + (int)threadIdx.x;
        if (idx < hi) {
          const int h = idx / p.d.d_v;
          float o = 0.f;
#pragma unroll
          for (int rr = 0; rr < 16; ++rr)
            if (rr < cs) o = fmaf(v[u][rr], s_w[rr][h], o);
          store_out(p, outg, idx, o * s_inv[h]);
        }
      }
    }
  }
}

template <typename T, bool MMA, int D>
__global__ void __launch_bounds__(kThreads, 2) attend_kernel(const __grid_constant__ AttendParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ TopKCtl tk;
  const int tid = threadIdx.x;
  const unsigned rank = blockIdx.x;
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair / p.d.Hkv, g = pair - b * p.d.Hkv;
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  if (p.ready_in != nullptr) {  // the token kernel's keys and histogram for this pair
    if (tid == 0) {
      wait_count(p.ready_in + pair, (unsigned)p.ready_count);
      if (cs == 1) p.ready_in[pair] = 0u;
    }
    __syncthreads();
  }
  int K;
  if (p.select) {
    K = select_tokens_prologue(p, pair, b, rank, smem, sel, tk);
    if (!p.attend) return;
  } else {
    K = min(min(max(p.num_tokens[pair], 0), p.d.Kt), p.tloc_max * cs);
  }
  const int t0 = (int)((long long)K * rank / cs), t1 = (int)((long long)K * (rank + 1) / cs);
  const int tloc = t1 - t0;
  if (!p.select) {
    const int* ids = p.token_ids + (size_t)pair * p.d.Kt;
    for (int i = tid; i < tloc; i += kThreads) sel[i] = ids[t0 + i];
    __syncthreads();
  }
  const int tot = p.d.G * p.d.d_v;
  float* po = p.part_o + ((size_t)pair * cs + rank) * tot;
  float* pml = p.part_ml + ((size_t)pair * cs + rank) * p.d.G * 2;
  if constexpr (MMA) {
    if constexpr (D == 128) {
      if (p.d.G <= 8) phase_attend_mma_t<D>(p, pair, b, g, sel, tloc, smem + p.off_akv, po, pml);
      else phase_attend_mma<D>(p, pair, b, g, sel, tloc, smem + p.off_akv, po, pml);
    } else {
      phase_attend_mma<D>(p, pair, b, g, sel, tloc, smem + p.off_akv, po, pml);
    }
  } else {
    phase_attend_generic<T>(p, pair, b, g, sel, tloc, reinterpret_cast<float*>(smem + p.off_aq),
                            reinterpret_cast<float*>(smem + p.off_as), po, pml);
  }
  if (p.dbg && rank == 0 && tid == 0) p.dbg[(size_t)pair * 8 + 5] = gtimer();
  if (MMA && cs == 1) return;  // the mma path wrote the output directly
  if (cs > 1) cluster_sync_all();  // release/acquire at cluster scope: partials visible in L2
  if (cs > 1 && p.ready_in != nullptr && rank == 0 && tid == 0) p.ready_in[pair] = 0u;  // all CTAs passed the wait
  __syncthreads();
  phase_merge<T, 1>(p, pair, b, g, rank);  // U = 1: within the 128-register budget
}

// --------------------------------------------------------------------------
// MLA tensor-core path (one shared latent KV head; V = the first d_v
// dims of each cached row).  Per CTA: the G <= 32 query heads (MT m-tiles of
// 16) against 32-token chunks of latent rows gathered with cp.async into
// XOR-swizzled smem, double-buffered.  S = Q K^T: warp w computes head-tile
// w/4, tokens 8*(w%4)..+8 over the DK/16 k-steps (Q and K fragments via
// ldmatrix).  Online softmax per head in smem (P stored as bf16).  O += P V:
// warp w owns output dims [64w, 64w + 64) (V^T fragments via ldmatrix.trans).
// --------------------------------------------------------------------------

template <int DK, int DV, int MT, int TC>
__global__ void __launch_bounds__(kThreads, 1) attend_mla_kernel(const __grid_constant__ AttendParams p) {
  static_assert(DV == 64 * kWarps, "each warp owns 64 output dims");
  constexpr int kMlaStages = mla_stages(TC);
  constexpr int CPR = DK / 8;       // 16-byte chunks per latent row
  constexpr int KS = DK / 16;       // k-steps of QK^T
  constexpr int PST = TC + 8;       // P row stride (bf16): 80 B, conflict-free ldmatrix
  constexpr int SST = TC + 4;       // S row stride (fp32)
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = blockIdx.x;
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair;  // MLA: one KV head
  const int G = p.d.G;
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  __shared__ TopKCtl tk;
  if (p.ready_in != nullptr) {  // the token kernel's keys and histogram for this pair
    if (tid == 0) {
      wait_count(p.ready_in + pair, (unsigned)p.ready_count);
      if (cs == 1) p.ready_in[pair] = 0u;
    }
    __syncthreads();
  }
  int K;
  if (p.select) {
    K = select_tokens_prologue(p, pair, b, rank, smem, sel, tk);
    if (!p.attend) return;
  } else {
    K = min(min(max(p.num_tokens[pair], 0), p.d.Kt), p.tloc_max * cs);
  }
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem + p.off_akv);
  __nv_bfloat16* sKV = sQ + MT * 16 * DK;           // kMlaStages buffers of TC rows
  float* sS = reinterpret_cast<float*>(sKV + kMlaStages * TC * DK);
  // P = exp2(S - m) as two bf16 pieces P_hi + P_lo (both exact sums of the fp32 value to ~2^-17): a single bf16 P
  // costs up to 2^-9 |V| per selected token, which for peaked attention over the latent (outlier channels, |V| ~ 5)
  // alone uses half the 2e-2 output tolerance; the second PV product removes it
  __nv_bfloat16* sP = reinterpret_cast<__nv_bfloat16*>(sS + MT * 16 * SST);
  __nv_bfloat16* sPl = sP + MT * 16 * PST;
  float* sAlpha = reinterpret_cast<float*>(sPl + MT * 16 * PST);
  float* sM = sAlpha + MT * 16;
  float* sL = sM + MT * 16;
  const int t0 = (int)((long long)K * rank / cs), t1 = (int)((long long)K * (rank + 1) / cs);
  const int tloc = t1 - t0;
  if (!p.select) {
    const int* ids = p.token_ids + (size_t)pair * p.d.Kt;
    for (int i = tid; i < tloc; i += kThreads) sel[i] = ids[t0 + i];
  }
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + (size_t)b * p.d.Hq * DK;
  for (int i = tid; i < MT * 16 * CPR; i += kThreads) {
    const int row = i / CPR, ch = i - row * CPR;
    cp_async16(sQ + row * DK + ((ch ^ (row & 7)) << 3), qg + (size_t)(row < G ? row : 0) * DK + ch * 8, row < G);
  }
  cp_async_commit();
  if (tid < MT * 16) {
    sM[tid] = -CUDART_INF_F;
    sL[tid] = 0.f;
  }
  __syncthreads();  // sel visible
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * DK;
  auto load_chunk = [&](int c, int buf) {
    __nv_bfloat16* dst = sKV + buf * TC * DK;
    for (int i = tid; i < TC * CPR; i += kThreads) {
      const int row = i / CPR, ch = i - row * CPR;
      const int t = c * TC + row;
      const bool ok = t < tloc;
      cp_async16(dst + row * DK + ((ch ^ (row & 7)) << 3), kb + (size_t)(ok ? sel[t] : 0) * DK + ch * 8, ok);
    }
    cp_async_commit();
  };
  const int nchunks = (tloc + TC - 1) / TC;
#pragma unroll
  for (int c = 0; c < kMlaStages - 1; ++c) {
    if (c < nchunks) load_chunk(c, c);
    else cp_async_commit();
  }
  const float sm2 = p.d.sm_scale * kLog2e;
  float o[MT][8][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int j = 0; j < 8; ++j) o[mt][j][0] = o[mt][j][1] = o[mt][j][2] = o[mt][j][3] = 0.f;
  const int r = lane >> 2, c2 = 2 * (lane & 3);
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kMlaStages;
    // refill the buffer chunk c-1 used (every warp passed the trailing barrier of c-1)
    if (c + kMlaStages - 1 < nchunks) load_chunk(c + kMlaStages - 1, (c + kMlaStages - 1) % kMlaStages);
    else cp_async_commit();
    cp_async_wait<kMlaStages - 1>();
    __syncthreads();
    const __nv_bfloat16* sK = sKV + buf * TC * DK;
    // ---- S = Q K^T (log2 units) ----
    {
      // warp: head tile mt, token n-tile(s) nb..nb+7 (and nb+32..nb+39 for 64-token chunks: one ldmatrix.x4
      // fetches both B fragments)
      const int mt = warp >> 2, nb = (warp & 3) * 8;
      static_assert(TC == 64 || TC == 32, "32- or 64-token chunks");
      if (mt < MT) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (TC == 64) {
#pragma unroll 4
          for (int kk = 0; kk < KS; ++kk) {
            uint32_t a[4], bk[4];
            const int qrow = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, qch = kk * 2 + (lane >> 4);
            ldsm_x4(a, sQ + qrow * DK + ((qch ^ (qrow & 7)) << 3));
            const int krow = nb + (lane & 7) + ((lane >> 4) & 1) * 32, kch = kk * 2 + ((lane >> 3) & 1);
            ldsm_x4(bk, sK + krow * DK + ((kch ^ (krow & 7)) << 3));
            mma_bf16_16816(acc, a, bk[0], bk[1]);
            mma_bf16_16816(acc2, a, bk[2], bk[3]);
          }
        } else {  // one n-tile on two chains (even / odd k-steps), folded into acc
          static_assert(KS % 2 == 0, "even number of k-steps");
#pragma unroll 4
          for (int kk = 0; kk < KS; kk += 2) {
            uint32_t a[4], bk[4], a2[4], bk2[4];
            const int qrow = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, qch = kk * 2 + (lane >> 4);
            ldsm_x4(a, sQ + qrow * DK + ((qch ^ (qrow & 7)) << 3));
            ldsm_x4(a2, sQ + qrow * DK + (((qch + 2) ^ (qrow & 7)) << 3));
            const int krow = nb + (lane & 7), kch = kk * 2 + ((lane >> 3) & 1);
            ldsm_x4(bk, sK + krow * DK + ((kch ^ (krow & 7)) << 3));  // lanes 16-31 duplicate 0-15
            ldsm_x4(bk2, sK + krow * DK + (((kch + 2) ^ (krow & 7)) << 3));
            mma_bf16_16816(acc, a, bk[0], bk[1]);
            mma_bf16_16816(acc2, a2, bk2[0], bk2[1]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] += acc2[i];
        }
#pragma unroll
        for (int u = 0; u < TC / 32; ++u) {
          const float* ac = u ? acc2 : acc;
          const int tk = nb + 32 * u + c2;
          const bool v0 = c * TC + tk < tloc, v1 = c * TC + tk + 1 < tloc;
          sS[(mt * 16 + r) * SST + tk] = v0 ? ac[0] * sm2 : -CUDART_INF_F;
          sS[(mt * 16 + r) * SST + tk + 1] = v1 ? ac[1] * sm2 : -CUDART_INF_F;
          sS[(mt * 16 + r + 8) * SST + tk] = v0 ? ac[2] * sm2 : -CUDART_INF_F;
          sS[(mt * 16 + r + 8) * SST + tk + 1] = v1 ? ac[3] * sm2 : -CUDART_INF_F;
        }
      }
    }
    __syncthreads();
    // ---- online softmax: 8 threads per head, TC / 8 tokens each ----
    {
      constexpr int NV = TC / 8;
      const int h = tid >> 3, tq = (tid & 7) * NV;
      if (h < MT * 16) {
        float x[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) x[i] = sS[h * SST + tq + i];
        float mx = x[0];
#pragma unroll
        for (int i = 1; i < NV; ++i) mx = fmaxf(mx, x[i]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        const float mo = sM[h];
        const float mn = fmaxf(mo, mx);  // finite: every chunk has >= 1 valid token
        float ps = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const float e = fexp2(x[i] - mn);
          ps += e;
          const __nv_bfloat16 eh = __float2bfloat16_rn(e);
          sP[h * PST + tq + i] = eh;
          sPl[h * PST + tq + i] = __float2bfloat16_rn(e - __bfloat162float(eh));
        }
        ps += __shfl_xor_sync(0xffffffffu, ps, 1);
        ps += __shfl_xor_sync(0xffffffffu, ps, 2);
        ps += __shfl_xor_sync(0xffffffffu, ps, 4);
        __syncwarp();
        if ((tid & 7) == 0) {
          const float al = fexp2(mo - mn);
          sAlpha[h] = al;
          sL[h] = sL[h] * al + ps;
          sM[h] = mn;
        }
      }
    }
    __syncthreads();
    // ---- O = O * alpha + P V  (warp owns dims [64w, 64w+64)) ----
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const float a0 = sAlpha[mt * 16 + r], a1 = sAlpha[mt * 16 + r + 8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o[mt][j][0] *= a0;
        o[mt][j][1] *= a0;
        o[mt][j][2] *= a1;
        o[mt][j][3] *= a1;
      }
    }
#pragma unroll
    for (int kk = 0; kk < TC / 16; ++kk) {
      uint32_t pa[MT][4], pl[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int prow = mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int pcol = kk * 16 + (lane >> 4) * 8;
        ldsm_x4(pa[mt], sP + prow * PST + pcol);
        ldsm_x4(pl[mt], sPl + prow * PST + pcol);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int vrow = kk * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
        const int vch = (warp * 64 + jj * 16) / 8 + (lane >> 4);
        uint32_t bv[4];
        ldsm_x4_trans(bv, sK + vrow * DK + ((vch ^ (vrow & 7)) << 3));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma_bf16_16816(o[mt][2 * jj], pa[mt], bv[0], bv[1]);
          mma_bf16_16816(o[mt][2 * jj + 1], pa[mt], bv[2], bv[3]);
          mma_bf16_16816(o[mt][2 * jj], pl[mt], bv[0], bv[1]);
          mma_bf16_16816(o[mt][2 * jj + 1], pl[mt], bv[2], bv[3]);
        }
      }
    }
    __syncthreads();  // buffer `buf` and sS / sP free for the next chunk
  }
  if (p.dbg && rank == 0 && tid == 0) p.dbg[(size_t)pair * 8 + 5] = gtimer();
  // ---- this CTA's partial (unnormalised o, max, sum) -> workspace ----
  const int tot = G * DV;
  float* po = p.part_o + ((size_t)pair * cs + rank) * tot;
  float* pml = p.part_ml + ((size_t)pair * cs + rank) * G * 2;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int dcol = warp * 64 + j * 8 + c2;
      const int h0 = mt * 16 + r, h1 = h0 + 8;
      if (h0 < G) *reinterpret_cast<float2*>(po + (size_t)h0 * DV + dcol) = make_float2(o[mt][j][0], o[mt][j][1]);
      if (h1 < G) *reinterpret_cast<float2*>(po + (size_t)h1 * DV + dcol) = make_float2(o[mt][j][2], o[mt][j][3]);
    }
  if (tid < G) {
    pml[2 * tid] = nchunks > 0 ? sM[tid] : -CUDART_INF_F;
    pml[2 * tid + 1] = nchunks > 0 ? sL[tid] : 0.f;
  }
  if (cs > 1) cluster_sync_all();
  if (cs > 1 && p.ready_in != nullptr && rank == 0 && tid == 0) p.ready_in[pair] = 0u;  // all CTAs passed the wait
  __syncthreads();
  phase_merge<__nv_bfloat16, 4>(p, pair, b, 0, rank);
}

// --------------------------------------------------------------------------
// MLA attention on the 5th-generation tensor cores (tcgen05 + TMEM), p.mma == 3.
// Per CTA: chunks of 64 selected tokens, double-buffered (the gather of chunk
// c + 2 is in flight while chunk c + 1 is computed).  A chunk's latent rows
// (576 bf16) are gathered once into shared memory in the canonical
// no-swizzle core-matrix layout (8 tokens x 16 B per 128-byte core matrix;
// token groups SBO = 9216 B apart, 8-dim groups LBO = 128 B apart), which
// serves BOTH products:
//   S^T[64 tok x NH] = K_chunk . Q^T        (A = the chunk, K-major: M = 64)
//   O^T[512 x NH]   += V^T . P^T            (A = the chunk's first 512 dims,
//        MN-major: the same core matrices with the roles of LBO / SBO swapped)
// Q (NH padded heads, K-major) and P^T (bf16 hi + lo pieces, MN-major over
// heads) are the B operands.  Accumulators in TMEM: S^T double-buffered in
// columns [0, 64), O^T in 4 M-blocks of NH columns from column 64.  One thread
// issues the MMAs; tcgen05.commit -> mbarriers hand them to the softmax warps
// (0-3: lanes 0-15 of each quarter hold one token each, the M = 64 layout)
// and to the epilogue.  P = 2^(S - m_ref) against a per-head reference max set
// by the first chunk and raised (with an O rescale through tcgen05.ld/st) only
// when a chunk exceeds it by more than 2^8, so TMEM is rarely touched between
// products.  The epilogue writes this CTA's partial (o, m_ref, l); the cluster
// merge of attend_mla_kernel (phase_merge) finishes the pair.
// P:73 (one shared latent head, V = the first d_v dims).
// --------------------------------------------------------------------------
namespace tc {
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);  // version 1, SWIZZLE_NONE
}
// kind::f16, D fp32, A/B bf16; a_mn / b_mn: MN-major operand
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
          tmem),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 columns (32-bit): thread t of the warp gets lane (32 * (warp % 4) + t), columns c0..c0+31
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
  } while (!done);
}
// transposed butterfly over the 32 lanes: on entry every lane holds 32 values (one per column); on exit lane l
// holds op over the lanes of column l (31 shuffles)
template <bool MAX>
__device__ __forceinline__ float transpose_reduce(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool up = lane & w;
#pragma unroll
    for (int j = 0; j < w; ++j) {
      const float send = up ? v[j] : v[j + w];
      const float keep = up ? v[j + w] : v[j];
      const float got = __shfl_xor_sync(0xffffffffu, send, w);
      v[j] = MAX ? fmaxf(keep, got) : keep + got;
    }
  }
  return v[0];  // lane l: column l
}
}  // namespace tc

constexpr int kTcTok = 64;            // tokens per chunk (the M of S^T; M = 64 puts row m in TMEM lane 32(m/16) + m%16)
constexpr int kTcRowGrp = 576 / 8;    // 72 core matrices per token group
constexpr uint32_t kTcSbo = kTcRowGrp * 128;  // 9216 B between token groups (and head groups of Q)
constexpr float kTcLazy = 8.f;        // rescale O only when a chunk's max exceeds the reference by > 2^8

template <int NH>
__global__ void __launch_bounds__(kThreads, 1) attend_mla_tc_kernel(const __grid_constant__ AttendParams p) {
  constexpr int DK = 576, DV = 512;
  constexpr uint32_t kChunkBytes = (uint32_t)kTcTok * DK * 2;  // 73728
  constexpr uint32_t kPBytes = (uint32_t)kTcTok * NH * 2;      // one bf16 piece of P^T
  constexpr int kOcol = 64;                                     // O^T: 4 M-blocks x NH columns from column 64
  constexpr uint32_t kTmemCols = 256;
  static_assert(kOcol + (DV / 128) * NH <= (int)kTmemCols, "TMEM plan");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_s[2], bar_o[2];
  __shared__ uint32_t s_tmem;
  __shared__ float s_red[4][NH];
  __shared__ float s_mref[NH], s_l[NH], s_scale[NH];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = blockIdx.x;
  const int cs = p.cs;
  const int pair = blockIdx.y;
  const int b = pair;  // MLA: one KV head
  const int G = p.d.G;
  int* sel = reinterpret_cast<int*>(smem + p.off_sel);
  __shared__ TopKCtl tk;
  unsigned long long* dbg = p.dbg ? p.dbg + ((size_t)pair * cs + rank) * 32 : nullptr;  // diagnostics
#define TC_STAMP(i) \
  if (dbg && tid == 0) dbg[i] = gtimer();
  TC_STAMP(0)
  if (p.ready_in != nullptr) {  // the token kernel's keys and histogram for this pair
    if (tid == 0) {
      wait_count(p.ready_in + pair, (unsigned)p.ready_count);
      if (cs == 1) p.ready_in[pair] = 0u;
    }
    __syncthreads();
  }
  int K;
  if (p.select) {
    K = select_tokens_prologue(p, pair, b, rank, smem, sel, tk);
    if (!p.attend) return;
  } else {
    K = min(min(max(p.num_tokens[pair], 0), p.d.Kt), p.tloc_max * cs);
  }
  const int t0 = (int)((long long)K * rank / cs), t1 = (int)((long long)K * (rank + 1) / cs);
  const int tloc = t1 - t0;
  TC_STAMP(1)
  if (!p.select) {
    const int* ids = p.token_ids + (size_t)pair * p.d.Kt;
    for (int i = tid; i < tloc; i += kThreads) sel[i] = ids[t0 + i];
  }
  uint8_t* sKV = smem + p.off_akv;            // 2 chunk buffers: [8 token groups][72 dim groups][128 B]
  uint8_t* sQ = sKV + 2 * kChunkBytes;        // [NH/8 head groups][72][128 B]
  uint8_t* sP = sQ + (size_t)NH * DK * 2;     // [2 buffers][hi | lo][8 token groups][NH/8][128 B]
  // warp roles: 0-3 softmax (TMEM lane quarters), 4 lane 0 MMA issue, 5-7 gather (cp.async)
  constexpr int kProd = 3 * 32;
  __shared__ __align__(8) uint64_t bar_full[2], bar_pfull[2];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&s_tmem)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_s[i], 1);       // S(c) MMAs complete (tcgen05.commit)
      mbar_init(&bar_o[i], 1);       // PV(c) MMAs complete: buffer c % 2 and P(c % 2) free (tcgen05.commit)
      mbar_init(&bar_full[i], kProd);  // the chunk's rows landed (cp.async.mbarrier.arrive per producer thread)
      mbar_init(&bar_pfull[i], 128);   // P(c) written, S(c) read, O rescaled (softmax threads)
    }
    mbar_fence_init();
  }
  if (tid < NH) s_l[tid] = 0.f;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();  // sel, barriers, the TMEM address
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = s_tmem;
  const float sm2 = p.d.sm_scale * kLog2e;
  const int nchunks = (tloc + kTcTok - 1) / kTcTok;
  const __nv_bfloat16* qg = reinterpret_cast<const __nv_bfloat16*>(p.q) + (size_t)b * p.d.Hq * DK;
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(p.k_cache) + (size_t)pair * p.kv_rows * DK;
  if (warp >= 5) {  // ======================= gather =======================
    for (int c = 0; c < nchunks; ++c) {
      const int bf = c & 1;
      if (c >= 2) tc::wait_bar(&bar_o[bf], ((c - 2) >> 1) & 1);  // PV(c - 2) read this buffer
      // 16-byte pieces, 8 rows x 4 chunks per warp instruction: each quarter-warp writes one contiguous 128-byte
      // core matrix (conflict-free) and the warp reads 64 contiguous bytes of each of its 8 rows (whole sectors)
      // (one row per lane group of 72 chunks: 128-byte-strided shared writes, a 4.5x slower gather)
      const int lr = lane & 7, lc = lane >> 3, wp = warp - 5;
      if (c == 0)  // Q: NH padded heads, K-major core matrices (head h, dims 8c..8c+7 at (h/8)*SBO + c*128 + (h%8)*16)
        for (int j = wp; j < (NH / 8) * (kTcRowGrp / 4); j += 3) {
          const int h = (j % (NH / 8)) * 8 + lr, ch = (j / (NH / 8)) * 4 + lc;
          cp_async16(sQ + (h >> 3) * kTcSbo + ch * 128 + (h & 7) * 16, qg + (size_t)(h < G ? h : 0) * DK + ch * 8, h < G);
        }
      uint8_t* dst = sKV + bf * kChunkBytes;
      for (int j = wp; j < (kTcTok / 8) * (kTcRowGrp / 4); j += 3) {
        const int row = (j % (kTcTok / 8)) * 8 + lr, ch = (j / (kTcTok / 8)) * 4 + lc;
        const int t = c * kTcTok + row;
        const bool ok = t < tloc;
        cp_async16(dst + (row >> 3) * kTcSbo + ch * 128 + (row & 7) * 16, kb + (size_t)(ok ? sel[t] : 0) * DK + ch * 8,
                   ok);
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&bar_full[bf])) : "memory");
    }
  } else if (warp == 4) {  // ======================= MMA issue =======================
    if (lane == 0) {
      constexpr uint32_t id_s = tc::idesc(64, NH, 0, 0), id_o = tc::idesc(128, NH, 1, 1);
      auto issue_s = [&](int c) {  // S^T = K Q^T: M = 64 tokens, N = NH, K = 576 (36 steps of 2 core matrices)
        const int bf = c & 1;
        tc::wait_bar(&bar_full[bf], (c >> 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the gathered rows, for the tensor cores
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t a0 = smem_u32(sKV + bf * kChunkBytes), b0 = smem_u32(sQ);
        for (int ks = 0; ks < DK / 16; ++ks)
          tc::mma(tmem + bf * 32, tc::sdesc(a0 + ks * 256, 128, kTcSbo), tc::sdesc(b0 + ks * 256, 128, kTcSbo), id_s,
                  ks > 0);
        tc::commit(&bar_s[bf]);
      };
      if (nchunks > 0) issue_s(0);
      for (int c = 0; c < nchunks; ++c) {
        const int bf = c & 1;
        if (c + 1 < nchunks) issue_s(c + 1);  // overlaps the softmax of chunk c (S is double-buffered)
        tc::wait_bar(&bar_pfull[bf], (c >> 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P, for the tensor cores
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // O^T += V^T P^T: 4 M-blocks of 128 dims, N = NH, K = 64 tokens (4 steps of 2 token groups)
        const uint32_t a0 = smem_u32(sKV + bf * kChunkBytes);
        for (int part = 0; part < 2; ++part) {  // P_hi, then P_lo
          const uint32_t pb = smem_u32(sP) + bf * 2 * kPBytes + part * kPBytes;
          for (int mb = 0; mb < DV / 128; ++mb)
            for (int ks = 0; ks < kTcTok / 16; ++ks)
              tc::mma(tmem + kOcol + mb * NH, tc::sdesc(a0 + mb * 16 * 128 + ks * 2 * kTcSbo, kTcSbo, 128),
                      tc::sdesc(pb + ks * 2 * ((NH / 8) * 128), (NH / 8) * 128, 128), id_o, c > 0 || part > 0 || ks > 0);
        }
        tc::commit(&bar_o[bf]);
      }
    }
  } else {  // ======================= softmax (warps 0-3) =======================
    for (int c = 0; c < nchunks; ++c) {
      const int bf = c & 1;
      tc::wait_bar(&bar_s[bf], (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (c < 4) TC_STAMP(3 + 4 * c)
      float v[32];
      tc::ld32(tmem + ((uint32_t)(warp * 32) << 16) + bf * 32, v);  // lanes 0-15 of warp w: tokens 16w .. 16w+15
      const int tok = warp * 16 + lane;
      const bool valid = lane < 16 && c * kTcTok + tok < tloc;
#pragma unroll
      for (int h = 0; h < 32; ++h) v[h] = (valid && h < NH) ? v[h] * sm2 : -CUDART_INF_F;
      float w[32];
#pragma unroll
      for (int h = 0; h < 32; ++h) w[h] = v[h];
      const float wm = tc::transpose_reduce<true>(w);  // lane h: this warp's max of head h
      if (lane < NH) s_red[warp][lane] = wm;
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (tid < NH) {  // the reference max: the first chunk's, raised only by more than 2^kTcLazy
        const float mc = fmaxf(fmaxf(s_red[0][tid], s_red[1][tid]), fmaxf(s_red[2][tid], s_red[3][tid]));
        const float mo = c == 0 ? -CUDART_INF_F : s_mref[tid];
        const bool up = mc > mo + kTcLazy;  // (first chunk: always)
        s_scale[tid] = up ? (mo == -CUDART_INF_F ? 0.f : fexp2(mo - mc)) : 1.f;
        if (up) s_mref[tid] = mc;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      int any = 0;
#pragma unroll
      for (int h = 0; h < NH; ++h) any |= (c > 0 && s_scale[h] != 1.f);
      float e[32];
#pragma unroll
      for (int h = 0; h < 32; ++h) {
        const float m = h < NH ? s_mref[h] : 0.f;
        e[h] = (h < NH && m != -CUDART_INF_F) ? fexp2(v[h] - m) : 0.f;
      }
      if (c >= 2) tc::wait_bar(&bar_o[bf], ((c - 2) >> 1) & 1);  // PV(c - 2) read P(bf)
      if (lane < 16) {  // P = 2^(S - m_ref) as bf16 hi + lo pieces into the MN-major B layout of buffer bf:
                        // token t, heads 8j..8j+7 at (t/8)*((NH/8)*128) + j*128 + (t%8)*16 (0 past tloc)
        uint8_t* phi = sP + bf * 2 * kPBytes + (tok >> 3) * ((NH / 8) * 128) + (tok & 7) * 16;
        uint8_t* plo = phi + kPBytes;
#pragma unroll
        for (int j = 0; j < NH / 8; ++j) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float a = valid ? e[8 * j + 2 * u] : 0.f, bb = valid ? e[8 * j + 2 * u + 1] : 0.f;
            const float ah = __bfloat162float(__float2bfloat16_rn(a)), bh = __bfloat162float(__float2bfloat16_rn(bb));
            hi[u] = pack_bf16x2(ah, bh);
            lo[u] = pack_bf16x2(a - ah, bb - bh);
          }
          *reinterpret_cast<uint4*>(phi + j * 128) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(plo + j * 128) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        }
      }
      const float ws = tc::transpose_reduce<false>(e);  // lane h: this warp's sum of head h
      asm volatile("bar.sync 1, 128;\n" ::: "memory");   // s_red (max) read by every thread before reuse
      if (lane < NH) s_red[warp][lane] = ws;
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (tid < NH) s_l[tid] = s_l[tid] * s_scale[tid] + s_red[0][tid] + s_red[1][tid] + s_red[2][tid] + s_red[3][tid];
      if (any) {  // O *= scale per head (column): PV(c - 1) must be complete
        tc::wait_bar(&bar_o[bf ^ 1], ((c - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        for (int mb = 0; mb < DV / 128; ++mb) {
          const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + kOcol + mb * NH;
          float o[32];
          tc::ld32(ta, o);
          uint32_t r[32];
#pragma unroll
          for (int h = 0; h < 32; ++h) r[h] = __float_as_uint(h < NH ? o[h] * s_scale[h] : o[h]);
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
              "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(ta),
              "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
              "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
              "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
              "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // P, for the tensor cores
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      if (c < 4) TC_STAMP(4 + 4 * c)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar_pfull[bf])) : "memory");
    }
  }
  if (nchunks > 0) {  // every thread: the last PV is complete
    tc::wait_bar(&bar_o[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  __syncthreads();  // s_l, s_mref final
  // ---- epilogue: this CTA's partial (unnormalised o, reference max, sum) ----
  const int tot = G * DV;
  float* po = p.part_o + ((size_t)pair * cs + rank) * tot;
  float* pml = p.part_ml + ((size_t)pair * cs + rank) * G * 2;
  if (tid < G) {
    pml[2 * tid] = nchunks > 0 ? s_mref[tid] : -CUDART_INF_F;
    pml[2 * tid + 1] = nchunks > 0 ? s_l[tid] : 0.f;
  }
  if (warp < 4 && nchunks > 0) {
    for (int mb = 0; mb < DV / 128; ++mb) {
      float v[32];
      tc::ld32(tmem + ((uint32_t)(warp * 32) << 16) + kOcol + mb * NH, v);
      const int dcol = mb * 128 + warp * 32 + lane;  // TMEM lane = output dim
#pragma unroll
      for (int h = 0; h < 32; ++h)
        if (h < G) po[(size_t)h * DV + dcol] = v[h];
    }
  }
  TC_STAMP(18)
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols));
  if (cs > 1) cluster_sync_all();
  if (cs > 1 && p.ready_in != nullptr && rank == 0 && tid == 0) p.ready_in[pair] = 0u;  // all CTAs passed the wait
  __syncthreads();
  TC_STAMP(19)
  phase_merge<__nv_bfloat16, 4>(p, pair, b, 0, rank);
  TC_STAMP(20)
#undef TC_STAMP
}

template <int NH>
static cudaError_t launch_mla_tc(const AttendParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = attend_mla_tc_kernel<NH>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, p.cs > 8);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3((unsigned)p.cs, (unsigned)(p.d.batch * p.d.Hkv), 1), kThreads, p.smem_bytes, st, o,
                   (unsigned)p.cs, p);
}

template <typename T, bool MMA, int D>
static cudaError_t launch_k3(const AttendParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = attend_kernel<T, MMA, D>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, p.cs > 8);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3((unsigned)p.cs, (unsigned)(p.d.batch * p.d.Hkv), 1), kThreads, p.smem_bytes, st, o,
                   (unsigned)p.cs, p);
}

template <int MT, int TC>
static cudaError_t launch_mla(const AttendParams& p, cudaStream_t st, const LaunchOpts& o) {
  auto kern = attend_mla_kernel<576, 512, MT, TC>;
  cudaError_t e = prepare_kernel(reinterpret_cast<const void*>(kern), p.smem_bytes, p.cs > 8);
  if (e != cudaSuccess) return e;
  return launch_ex(kern, dim3((unsigned)p.cs, (unsigned)(p.d.batch * p.d.Hkv), 1), kThreads, p.smem_bytes, st, o,
                   (unsigned)p.cs, p);
}

cudaError_t launch_attend(const AttendParams& p, cudaStream_t st, const LaunchOpts& o) {
  if (!p.attend) {  // selection only: any instantiation runs just the prologue
    if (p.d.bf16) return launch_k3<__nv_bfloat16, false, 0>(p, st, o);
    return launch_k3<float, false, 0>(p, st, o);
  }
  if (p.mma == 3) return p.d.G <= 16 ? launch_mla_tc<16>(p, st, o) : launch_mla_tc<32>(p, st, o);
  if (p.mma == 2) {
    if (p.mla_tc == 32) return p.d.G <= 16 ? launch_mla<1, 32>(p, st, o) : launch_mla<2, 32>(p, st, o);
    return p.d.G <= 16 ? launch_mla<1, 64>(p, st, o) : launch_mla<2, 64>(p, st, o);
  }
  if (p.d.bf16) {
    if (p.mma) return p.d.d_k == 128 ? launch_k3<__nv_bfloat16, true, 128>(p, st, o)
                                     : launch_k3<__nv_bfloat16, true, 64>(p, st, o);
    return launch_k3<__nv_bfloat16, false, 0>(p, st, o);
  }
  return launch_k3<float, false, 0>(p, st, o);
}

}  // namespace tls
